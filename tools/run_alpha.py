"""Join one batch (alpha) of a generated instance through msp_join_alpha; print stats as JSON.

    python tools/run_alpha.py --m 9 --seed 1 --quantile 0.5
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2507_05045_b200 as msb  # noqa: E402
from paper_2507_05045_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, required=True)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--quantile", type=float, default=0.5, help="pick the batch at this cost quantile")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--wave-keys", type=int, default=0)
args = ap.parse_args()
inst = msb.generate_instance(args.m, 100, args.seed)
plan = _native.alpha_plan(inst.a, inst.d)
order = sorted(plan, key=lambda p: p[2] + p[3])
alpha, beta, nl, nr = order[int(args.quantile * (len(order) - 1))]
rep_ms = []
for rep in range(args.reps):
    t0 = time.perf_counter()
    rc, xb, st = _native.solve_raw(inst.a, inst.d, _native.make_options(mode="all", wave_keys=args.wave_keys), alpha=alpha)
    dt = time.perf_counter() - t0
    assert rc == 0, _native.last_error()
    rep_ms.append(round(st["dev_ms_join"], 2))
print(json.dumps({"alpha": alpha, "n_left": nl, "n_right": nr, "wall_s": dt, "rep_dev_ms_join": rep_ms,
                  "pairs_per_s": (nl + nr) / dt, "stats": st}))
