"""Every hit-bearing (9,80) alpha-group, pinned by the CPU oracle's filter join (TEST INFRASTRUCTURE).

(9,80) seed 1 has 99 hash hits in 92 of its 1911 batches (the GPU's per-batch stats of the full
solve, MSP_FLAG_BATCH_STATS, `tools/run_solve.py --m 9 --batch-stats`).  make_golden_groups.py pins
ten of them with the sort-merge restatement (oracle.alpha_group); this script pins the other 82 with
oracle.AlphaGroups.run(method=1), the filter join of msp_oracle_groups.cc, which computes the same
per-batch counters (checked against the sort-merge method and the reference-pinned goldens in
tests/test_oracle.py).  Together the two files hold every batch whose hash_hits is nonzero, so the
GPU's 99 hash hits and 7 solutions are checked batch by batch (tests/test_gpu_parity.py).

The batches of 1.3e9 - 4.8e9 keys take 30-90 s each on 8 cores (~2 h in all, ~12 GB RAM); the output
is rewritten after every batch, in ascending batch size, so a partial run is a valid (smaller) golden.

    python tests/golden/make_golden_groups_all.py [--threads N]
"""
import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402
from paper_2507_05045_b200.instances import generate_instance  # noqa: E402

# alpha of the 92 hit-bearing batches in ascending batch size (GPU per-batch stats of the full solve)
HIT_ALPHAS = [1499, 638, 665, 1343, 1309, 739, 1281, 1261, 799, 1226, 1220, 823, 1219, 1213, 1210, 1208,
              1207, 1203, 1189, 861, 1181, 1179, 871, 1170, 1164, 880, 1158, 886, 1155, 888, 1154, 1150,
              893, 1147, 899, 1142, 903, 904, 1138, 1131, 1127, 917, 1123, 1121, 925, 1117, 926, 927,
              1115, 936, 937, 941, 1101, 1098, 1095, 948, 1093, 951, 952, 1090, 953, 954, 955, 1083,
              1082, 1081, 1079, 967, 1075, 968, 969, 972, 1068, 1062, 1061, 983, 985, 1053, 991, 992,
              996, 1046, 998, 999, 1001, 1041, 1039, 1035, 1011, 1029, 1024, 1022]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--alphas", default="", help="comma-separated subset, in the order given (default: all)")
    ap.add_argument("--out", default="", help="output path (default: alpha_groups_9_100_1_hits_all.json)")
    args = ap.parse_args()
    done = {g["alpha"] for g in json.load(open(os.path.join(HERE, "alpha_groups_9_100_1_hits.json")))["groups"]}
    inst = generate_instance(9, 100, 1)
    path = args.out or os.path.join(HERE, "alpha_groups_9_100_1_hits_all.json")
    todo = [int(x) for x in args.alphas.split(",") if x] or HIT_ALPHAS
    out = {"source": "oracle.AlphaGroups.run(method=1) (filter join, oracle/msp_oracle_groups.cc), pinned to the "
                     "reference; instance generate_instance(9, 100, 1)",
           "hit_alphas": HIT_ALPHAS, "groups": []}
    with O.AlphaGroups(inst.a, inst.d) as G:
        for alpha in todo:
            if alpha in done:
                continue
            t0 = time.time()
            r = G.run(alpha, method=1, threads=args.threads)
            r["alpha"] = alpha
            r["oracle_seconds"] = round(time.time() - t0, 1)
            out["groups"].append(r)
            print(alpha, {k: r[k] for k in ("n_left", "n_right", "filtered", "hash_hits", "exact_hits", "oracle_seconds")},
                  flush=True)
            with open(path + ".tmp", "w") as fh:
                json.dump(out, fh, separators=(",", ":"))
            os.replace(path + ".tmp", path)


if __name__ == "__main__":
    main()
