"""Solve one generated instance through the public API and print a JSON record (stats + timing).

    python tools/run_solve.py --m 9 --seed 1 [--mode all] [--device 0] [--profile]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2507_05045_b200 as msb  # noqa: E402
from paper_2507_05045_b200 import _native  # noqa: E402
from paper_2507_05045_b200.solver import native_solve  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, required=True)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--K", type=int, default=100)
    ap.add_argument("--mode", default="all")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--planted", action="store_true")
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--wave-keys", type=int, default=0)
    ap.add_argument("--batch-stats", action="store_true", help="record per-batch (alpha, nl, nr, filtered, hash_hits)")
    args = ap.parse_args()
    if args.planted:
        inst, x = msb.plant_instance(args.m, args.K, args.seed)
    else:
        inst, x = msb.generate_instance(args.m, args.K, args.seed), None
    t0 = time.perf_counter()
    sols, st = native_solve(inst, args.mode, None, device=args.device, wave_keys=args.wave_keys,
                            flags=(_native.MSP_FLAG_PROFILE if args.profile else 0)
                            | (_native.MSP_FLAG_BATCH_STATS if args.batch_stats else 0))
    wall = time.perf_counter() - t0
    for s in sols:
        assert msb.verify_solution(inst, s)
    sols = sorted(sols, key=msb.solution_encoding)
    rec = {"instance": f"({args.m},{inst.n}) K={args.K} seed={args.seed}" + (" planted" if args.planted else ""),
           "mode": args.mode, "wall_s": round(wall, 3), "solutions": [msb.solution_to_string(s) for s in sols],
           "planted_found": (tuple(x) in sols) if x is not None else None,
           "pairs_per_s": (st["candidates_left"] + st["candidates_right"]) / wall,
           "stats": {k: v for k, v in st.items() if k != "batch_stats"}}
    if args.batch_stats:
        rec["hit_batches"] = [b for b in st.get("batch_stats", []) if b[4] > 0]
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
