"""Goldens beyond the reference's CPU reach, from the pinned C oracle (oracle/msp_oracle.c).

The oracle is pinned bit-exactly to the reference on every fixture make_golden.py writes
(tests/test_oracle.py), so its full-enumeration results for (8,70) are the reference's results
computed faster: same algorithm (heap stream + fused FNV join), with the 2^22 bucket cap raised
(fastval.py:111-113 -- the cap changes speed only, never results; tests/test_oracle.py
test_chunk_and_bucket_invariance).

    python tests/golden/make_golden_oracle.py 8 1      # ~15 min on 8 cores
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402
from paper_2507_05045_b200.instances import generate_instance  # noqa: E402

m, seed = int(sys.argv[1]), int(sys.argv[2])
inst = generate_instance(m, 100, seed)
t0 = time.time()
r = O.solve(inst.a, inst.d, mode="all", bucket_bits_cap=26, chunk_pairs=1 << 26, workers=6, record_batches=True)
assert r.status == 0
rec = {
    "name": f"gen_{m}_100_{seed}",
    "source": "oracle/msp_oracle.c (pinned to the reference), bucket_bits_cap=26, chunk_pairs=2^26",
    "instance": {"a": inst.a.tolist(), "d": inst.d.tolist()},
    "verdict": "feasible" if r.solutions else "infeasible",
    "solutions": ["".join(map(str, x)) for x in r.solutions],
    "stats": {k: r.stats[k] for k in ("batches", "candidates_left", "candidates_right", "hash_hits",
                                      "exact_hits", "filtered_residuals", "peak_table_entries",
                                      "peak_heap1", "peak_heap2")},
    "row1_candidate_pairs": r.stats["row1_candidate_pairs"],
    "batches": r.batch_records[:, :6].tolist(),
    "oracle_seconds": round(time.time() - t0, 1),
    "threads": r.stats["threads_used"],
}
with open(os.path.join(HERE, f"solve_{m}_100_{seed}.json"), "w") as fh:
    json.dump(rec, fh, separators=(",", ":"))
print(rec["stats"], rec["oracle_seconds"])
