"""Hit-bearing (9,80) alpha-group goldens from the streaming CPU oracle (oracle/msp_oracle_groups.cc).

(9,80) seed 1 is beyond any full CPU run.  Its 99 hash hits (92 of them 64-bit FNV
collisions) sit in 92 of its 1911 batches.  This script pins ten of those batches -- the smallest
collision-only ones plus the two smallest that hold a solution -- with oracle.alpha_group, the
streaming restatement of validate_chunked/fastval.join_pairs (pinned in tests/test_oracle.py
against the reference's own per-batch goldens).  Every one of these batches takes the GPU's
two-level (coarse HBM + fine shared-memory) join path.

    python tests/golden/make_golden_groups.py        # ~15 min on 8 cores, ~20 GB RAM peak
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402
from paper_2507_05045_b200.instances import generate_instance  # noqa: E402

# (alpha) of hit-bearing batches, from the GPU's per-batch stats (MSP_FLAG_BATCH_STATS) of the full
# (9,80) s1 solve; 1343 and 1213 hold solutions, the others only FNV collisions
ALPHAS = [1499, 638, 665, 1343, 1309, 739, 1281, 1261, 799, 1213]

inst = generate_instance(9, 100, 1)
out = {"instance": {"a": inst.a.tolist(), "d": inst.d.tolist()},
       "source": "oracle.alpha_group (oracle/msp_oracle_groups.cc), pinned to the reference", "groups": []}
path = os.path.join(HERE, "alpha_groups_9_100_1_hits.json")
for alpha in ALPHAS:
    t0 = time.time()
    r = O.alpha_group(inst.a, inst.d, alpha)
    r["alpha"] = alpha
    r["oracle_seconds"] = round(time.time() - t0, 1)
    out["groups"].append(r)
    print(alpha, {k: r[k] for k in ("n_left", "n_right", "filtered", "hash_hits", "exact_hits", "passes", "oracle_seconds")},
          flush=True)
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
