"""Per-batch counters of EVERY (9,80) s1 batch from the CPU oracle (TEST INFRASTRUCTURE).

The batch list is the reference's own stream (stream_9_100_1.json from make_golden_stream_9_80.py: the
heap enumeration of fastenum restated in oracle/msp_oracle.c, pinned to the reference's streams); each batch is
joined by oracle.AlphaGroups.run(method=1), the filter join (tests/test_oracle.py pins it to the
reference's per-batch goldens).  The 92 hit-bearing batches are already in alpha_groups_9_100_1_hits*.json
and are skipped.  Batches run in ascending size and the output is rewritten every few batches, so a
time-boxed run is a valid golden for the batches it holds (`complete` says whether it holds all).

2.2e12 keys in all: hours on 8 cores, ~2 h on the GPU box's host.

    python tests/golden/make_golden_batches_9_80.py [--out PATH] [--deadline SECONDS]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(HERE, "batches_9_100_1.json"))
    ap.add_argument("--deadline", type=float, default=0.0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--descending", action="store_true", help="largest batches first (a second worker)")
    ap.add_argument("--skip-done", default="", help="a previous output: its batches are skipped")
    args = ap.parse_args()
    t_start = time.time()
    inst = generate_instance(9, 100, 1)
    hdrs = [tuple(h) for h in json.load(open(os.path.join(HERE, "stream_9_100_1.json")))["headers"]]
    pinned = {g["alpha"] for f in ("alpha_groups_9_100_1_hits.json", "alpha_groups_9_100_1_hits_all.json")
              for g in json.load(open(os.path.join(HERE, f)))["groups"]}
    if args.skip_done:
        pinned |= {r[0] for r in json.load(open(args.skip_done))["records"]}
    todo = sorted((h for h in hdrs if h[0] not in pinned), key=lambda h: h[2] + h[3], reverse=args.descending)
    out = {"source": "oracle.stream_headers (reference batch stream) + oracle.AlphaGroups.run(method=1) per batch; "
                     "instance generate_instance(9, 100, 1); the 92 hit-bearing batches are in "
                     "alpha_groups_9_100_1_hits*.json",
           "n_batches": len(hdrs), "n_skipped_hit_batches": len(hdrs) - len(todo),
           "columns": ["alpha", "n_left", "n_right", "filtered", "hash_hits", "exact_hits"],
           "records": [], "complete": False}

    def save():
        with open(args.out + ".tmp", "w") as fh:
            json.dump(out, fh, separators=(",", ":"))
        os.replace(args.out + ".tmp", args.out)

    keys = 0
    with O.AlphaGroups(inst.a, inst.d) as G:
        for i, (alpha, beta, nl, nr) in enumerate(todo):
            if args.deadline and time.time() - t_start > args.deadline:
                break
            r = G.run(alpha, method=1, threads=args.threads)
            assert (r["n_left"], r["n_right"]) == (nl, nr), alpha
            out["records"].append([alpha, nl, nr, r["filtered"], r["hash_hits"], r["exact_hits"]])
            keys += nl + nr
            if i % 20 == 19 or i + 1 == len(todo):
                out["complete"] = len(out["records"]) == len(todo)
                out["keys"] = keys
                save()
                print(i + 1, len(todo), alpha, nl + nr, keys, round(time.time() - t_start), flush=True)
    out["complete"] = len(out["records"]) == len(todo)
    out["keys"] = keys
    save()


if __name__ == "__main__":
    main()
