"""Generate golden fixtures by running the UNMODIFIED reference in this container.

Usage (from the repo root, in the build container where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py [--big]

Nothing here runs on the GPU box; the JSON files it writes are committed and are what the
tests read.  Every number comes from the reference's own public API:
``build_quarter_tables`` (enumerate1d.py:86-135), ``JitPairSumEnumerator`` (fastenum.py:161-218),
``validate_chunked`` + ``ParallelBackend`` fused join (validate.py:316-379, fastval.py:116-139),
``solve`` (solver.py:170-245), ``SplitMix64``/``encode_vector`` KATs.

--big additionally writes the (7,60) s1 per-batch golden (~4 min on 8 cores) and the sampled
alpha-group goldens for (8,70) s1 and (9,80) s1 (SURVEY.md §8(c) pinning route (ii)).
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

import marketsplit as ms
from marketsplit import fastenum
from marketsplit.enumerate1d import CandidateBatch, build_quarter_tables, permuted_rhs
from marketsplit.validate import ParallelBackend, ValidationStats, validate_chunked, encode_vector

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2507_05045_b200.instances import plant_instance  # noqa: E402  (new generator, not reference)

HERE = os.path.dirname(os.path.abspath(__file__))


def seeded_instance(seed, m, n, k, d_mode="half"):
    """Same construction as the reference tests' helper (pkg/tests/conftest.py:10-26)."""
    rng = ms.instances.SplitMix64(seed)
    rows = [[rng.below(k) for _ in range(n)] for _ in range(m)]
    if d_mode == "half":
        d = [sum(r) // 2 for r in rows]
    else:
        d = [rng.below(sum(r) + 1) for r in rows]
    return ms.MspInstance(rows, d, k_bound=k)


def inst_json(inst):
    return {"a": inst.a.tolist(), "d": inst.d.tolist()}


STAT_KEYS = ("batches", "candidates_left", "candidates_right", "hash_hits",
             "exact_hits", "filtered_residuals", "peak_table_entries", "peak_heap1", "peak_heap2")


def solve_record(name, inst, per_batch=False):
    t0 = time.time()
    res = ms.solve(inst, ms.SolverConfig(mode="all"))
    rec = {
        "name": name,
        "instance": inst_json(inst),
        "verdict": res.verdict,
        "solutions": [ms.solution_to_string(x) for x in res.solutions],
        "stats": {k: getattr(res.stats, k) for k in STAT_KEYS},
        "fallback": res.stats.fallback,
        "ref_seconds": round(time.time() - t0, 3),
    }
    if per_batch and res.stats.fallback == "none":
        rec["batches"] = per_batch_stats(inst)
        assert len(rec["batches"]) == res.stats.batches
    return rec


def _validate_one(args):
    alpha, beta, lp, rp = args
    tables, inst, d = _G["tables"], _G["inst"], _G["d"]
    batch = CandidateBatch(alpha=alpha, beta=beta, left_pairs=lp, right_pairs=rp)
    st = ValidationStats()
    sols = validate_chunked(batch, tables, inst, 1 << 40, ParallelBackend(), d, st)
    return [alpha, batch.n_left, batch.n_right, st.filtered_residuals, st.hash_hits,
            st.exact_hits, sorted(ms.solution_to_string(x) for x in sols)]


_G: dict = {}


def _init_worker(inst_a, inst_d):
    inst = ms.MspInstance(inst_a, inst_d)
    tables = build_quarter_tables(inst, 0)
    _G.update(inst=inst, tables=tables, d=permuted_rhs(inst, tables))


def _batch_stream(inst):
    tables = build_quarter_tables(inst, 0)
    enum = fastenum.JitPairSumEnumerator(tables, int(inst.d[0]))
    while (b := enum.next_batch()) is not None:
        yield (b.alpha, b.beta, b.left_pairs, b.right_pairs)


def per_batch_stats(inst, procs=None):
    """[alpha, n_left, n_right, filtered, hash_hits, exact_hits, solutions] per reference batch."""
    with mp.Pool(procs or os.cpu_count(), initializer=_init_worker,
                 initargs=(inst.a.tolist(), inst.d.tolist())) as pool:
        return list(pool.imap(_validate_one, _batch_stream(inst), chunksize=4))


def kats():
    rng = ms.instances.SplitMix64(0)
    sm0 = [rng.next_u64() for _ in range(8)]
    rng = ms.instances.SplitMix64(0xFEED)
    corpus = [[rng.next_u64() for _ in range(6)] for _ in range(64)]
    small = [[int(v) for v in np.random.default_rng(s).integers(0, 4000, size=1 + s % 12)]
             for s in range(64)]
    below = []
    rng = ms.instances.SplitMix64(12345)
    for k in (2, 3, 7, 100, 1000, (1 << 63) + 5):
        below.append([k, [rng.below(k) for _ in range(6)]])
    return {
        "splitmix64_seed0": sm0,
        "splitmix64_below_seed12345": below,
        "fnv_offset": ms.validate.FNV_OFFSET,
        "fnv_prime": ms.validate.FNV_PRIME,
        "fnv_corpus_u64": [[v, encode_vector(v)] for v in corpus],
        "fnv_corpus_small": [[v, encode_vector(v)] for v in small],
        "generate": {f"{m},{k},{s}": inst_json(ms.generate_instance(m, k, s))
                     for (m, k, s) in ((2, 10, 0), (3, 100, 27), (4, 100, 11))},
    }


def tables_golden():
    out = []
    cases = [
        ("seeded5_m2_n8", seeded_instance(5, m=2, n=8, k=7)),
        ("seeded6_m3_n10", seeded_instance(6, m=3, n=10, k=9)),
        ("ties", ms.MspInstance([[0, 0, 0, 0, 1, 2, 3, 4]], [5])),
        ("ties_desc", ms.MspInstance([[1, 2, 3, 4, 0, 0, 0, 0]], [5])),
        ("gen_4_100_11", ms.generate_instance(4, 100, 11)),
        ("seeded9_m2_n13_k3", seeded_instance(9, m=2, n=13, k=3)),
    ]
    for name, inst in cases:
        tabs = build_quarter_tables(inst, 0)
        out.append({
            "name": name,
            "instance": inst_json(inst),
            "tables": [{
                "var_indices": list(t.var_indices),
                "ascending": t.ascending,
                "weights": t.weights.tolist(),
                "masks": t.masks.tolist(),
                "contribs": t.contribs.tolist(),
                "run_end": t.run_end.tolist(),
            } for t in tabs],
        })
    return out


def streams_golden():
    out = []
    for seed in range(12):
        inst = seeded_instance(seed, m=2, n=4 + seed % 11, k=11)
        tabs = build_quarter_tables(inst, 0)
        enum = fastenum.JitPairSumEnumerator(tabs, int(inst.d[0]))
        batches = []
        while (b := enum.next_batch()) is not None:
            batches.append([b.alpha, b.beta, b.left_pairs.tolist(), b.right_pairs.tolist()])
        out.append({"name": f"seeded{seed}", "instance": inst_json(inst), "batches": batches})
    return out


def solves_small():
    recs = []
    for seed in range(40):
        inst = seeded_instance(seed, m=1 + seed % 3, n=13 + seed % 8,
                               k=10 if seed % 2 else 5,
                               d_mode="half" if seed % 3 else "random")
        recs.append(solve_record(f"seeded{seed}", inst))
    for seed in range(8):
        inst = seeded_instance(500 + seed, m=4 + seed % 3, n=16 + seed, k=20)
        recs.append(solve_record(f"seeded_wide{seed}", inst))
    for seed in range(6):  # tiny n: reference brute-force fallback (solver.py:197-211)
        inst = seeded_instance(900 + seed, m=1 + seed % 2, n=4 + seed, k=6, d_mode="random")
        recs.append(solve_record(f"bf{seed}", inst))
    recs.append(solve_record("allzero_n13", ms.MspInstance([[0] * 13], [0])))
    recs.append(solve_record("zero_cols", ms.MspInstance([[0, 1, 2, 3, 4, 0, 5, 6, 0, 7, 8, 9, 1, 1]], [10])))
    recs.append(solve_record("m1_n16_k3", seeded_instance(77, m=1, n=16, k=3)))
    recs.append(solve_record("parity_infeasible", ms.MspInstance([[2] * 14, [1] * 14], [7, 7])))
    return recs


def solves_medium():
    recs = []
    for (m, s) in ((3, 27), (3, 98), (4, 11), (4, 1), (4, 12), (5, 1), (5, 3), (6, 1), (6, 4)):
        recs.append(solve_record(f"gen_{m}_100_{s}", ms.generate_instance(m, 100, s), per_batch=(m >= 4)))
    for (m, s) in ((4, 1), (5, 2), (6, 1)):
        inst, x = plant_instance(m, 100, s)
        rec = solve_record(f"plant_{m}_100_{s}", inst, per_batch=(m >= 4))
        rec["planted"] = ms.solution_to_string(x)
        assert rec["planted"] in rec["solutions"]
        recs.append(rec)
    return recs


def plan_counts(inst):
    """Plan counters by histogram convolution (SURVEY.md App. A restatement)."""
    tabs = build_quarter_tables(inst, 0)
    w = [t.weights.astype(np.int64) for t in tabs]
    hl = np.convolve(np.bincount(w[0]).astype(object), np.bincount(w[1]).astype(object))
    hr = np.convolve(np.bincount(w[2]).astype(object), np.bincount(w[3]).astype(object))
    t = int(inst.d[0])
    batches = sl = sr = prod = 0
    for a in range(len(hl)):
        b = t - a
        if hl[a] > 0 and 0 <= b < len(hr) and hr[b] > 0:
            batches += 1
            sl += int(hl[a]); sr += int(hr[b]); prod += int(hl[a]) * int(hr[b])
    return {"batches": batches, "candidates_left": sl, "candidates_right": sr,
            "row1_candidate_pairs": prod}


def alpha_group_golden(inst, max_pairs=6_000_000, picks=8):
    """Per-alpha reference join on groups built by the verified restatement."""
    tabs = build_quarter_tables(inst, 0)
    d = permuted_rhs(inst, tabs)
    wa, wb, wc, wd = (t.weights.astype(np.int64) for t in tabs)
    t = int(inst.d[0])
    hl = np.convolve(np.bincount(wa), np.bincount(wb))
    hr = np.convolve(np.bincount(wc), np.bincount(wd))
    cands = [(a, int(hl[a]), int(hr[t - a])) for a in range(len(hl))
             if hl[a] > 0 and 0 <= t - a < len(hr) and hr[t - a] > 0]
    cands = [c for c in cands if c[1] + c[2] <= max_pairs]
    # spread picks over sizes: smallest, largest-allowed, and quantiles in between
    cands.sort(key=lambda c: c[1] + c[2])
    idx = sorted({int(round(q * (len(cands) - 1))) for q in np.linspace(0, 1, picks)})
    out = []
    for i in idx:
        alpha, nl, nr = cands[i]
        beta = t - alpha
        left = _pairs_vec(wa, wb, alpha)
        right = _pairs_vec(wc, wd, beta)
        assert len(left) == nl and len(right) == nr
        batch = CandidateBatch(alpha=alpha, beta=beta, left_pairs=left, right_pairs=right)
        st = ValidationStats()
        t0 = time.time()
        sols = validate_chunked(batch, tabs, inst, 1 << 40, ParallelBackend(), d, st)
        out.append({"alpha": alpha, "n_left": nl, "n_right": nr,
                    "filtered": st.filtered_residuals, "hash_hits": st.hash_hits,
                    "exact_hits": st.exact_hits,
                    "solutions": sorted(ms.solution_to_string(x) for x in sols),
                    "ref_seconds": round(time.time() - t0, 2)})
        print("  alpha", alpha, nl, nr, out[-1]["hash_hits"], out[-1]["ref_seconds"], flush=True)
    return out


def _pairs_vec(wx, wy, total):
    """All (x, y) with wx[x] + wy[y] == total, ordered (y asc, x asc).

    wx is a sorted table (asc or desc), so each weight occupies one contiguous index run.
    """
    vals, first, counts = np.unique(wx, return_index=True, return_counts=True)
    need = total - wy
    pos = np.searchsorted(vals, need)
    ok = (pos < len(vals)) & (vals[np.minimum(pos, len(vals) - 1)] == need)
    ys = np.flatnonzero(ok)
    starts = first[pos[ys]]
    lens = counts[pos[ys]]
    tot = int(lens.sum())
    offs = np.cumsum(lens) - lens
    xs = np.repeat(starts - offs, lens) + np.arange(tot)
    return np.stack([xs, np.repeat(ys, lens)], axis=1).astype(np.int64)


def solves_generic():
    """Generic u64 weights: K = 10^6 instances (companion sums past 16 bits,
    row-0 block sums far past any dense histogram) and surrogate-reduced instances (reduce_rows 2, 3:
    the merged row 0 is (nD)-based, instances.py:266-319), solved by the reference in all mode."""
    out = []
    for (m, s) in ((4, 1), (4, 2), (4, 3), (4, 7), (5, 1), (5, 2)):
        inst = ms.generate_instance(m, 10**6, s)
        rec = solve_record(f"gen_{m}_1e6_{s}", inst, per_batch=(m == 4))
        rec["reduce_rows"] = 1
        out.append(rec)
    for (m, s) in ((4, 1), (5, 1)):
        inst, _ = plant_instance(m, 10**6, s)
        rec = solve_record(f"plant_{m}_1e6_{s}", inst)
        rec["reduce_rows"] = 1
        out.append(rec)
    for (m, K, s, r) in ((4, 100, 11, 2), (4, 100, 11, 3), (4, 100, 1, 2), (4, 100, 12, 3), (5, 100, 1, 2),
                         (5, 100, 3, 2), (5, 100, 3, 3), (5, 1000, 2, 2)):
        inst = ms.generate_instance(m, K, s)
        t0 = time.time()
        res = ms.solve(inst, ms.SolverConfig(mode="all", reduce_rows=r))
        out.append({"name": f"gen_{m}_{K}_{s}_reduce{r}", "instance": inst_json(inst), "reduce_rows": r,
                    "verdict": res.verdict, "solutions": [ms.solution_to_string(x) for x in res.solutions],
                    "stats": {k: getattr(res.stats, k) for k in STAT_KEYS}, "fallback": res.stats.fallback,
                    "ref_seconds": round(time.time() - t0, 3)})
    return out


def dump(name, obj):
    path = os.path.join(HERE, name)
    with open(path, "w") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    jobs = {
        "kats.json": kats,
        "tables.json": tables_golden,
        "streams.json": streams_golden,
        "solves_small.json": solves_small,
        "solves_medium.json": solves_medium,
        "solves_generic.json": solves_generic,
        "plan_counts.json": lambda: {f"{m},{s}": plan_counts(ms.generate_instance(m, 100, s))
                                     for (m, s) in ((4, 1), (4, 11), (6, 1), (6, 4), (7, 1),
                                                    (8, 1), (9, 1))},
    }
    if args.big:
        jobs["solve_7_100_1.json"] = lambda: solve_record("gen_7_100_1", ms.generate_instance(7, 100, 1), per_batch=True)
        jobs["alpha_groups_8_100_1.json"] = lambda: {"instance": inst_json(ms.generate_instance(8, 100, 1)),
                                                     "groups": alpha_group_golden(ms.generate_instance(8, 100, 1), max_pairs=60_000_000, picks=10)}
        jobs["alpha_groups_9_100_1.json"] = lambda: {"instance": inst_json(ms.generate_instance(9, 100, 1)),
                                                     "groups": alpha_group_golden(ms.generate_instance(9, 100, 1), max_pairs=30_000_000, picks=8)}
    for name, fn in jobs.items():
        if args.only and args.only not in name:
            continue
        t0 = time.time()
        dump(name, fn())
        print(f"  {name}: {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
