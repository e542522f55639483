"""GPU parity: the CUDA path through the C-ABI against reference-generated goldens and the oracle.

Bit-exact bar (integer work): identical quarter tables, batch headers, solution sets and every
deterministic SolveStats counter (batches, candidates_left/right, filtered_residuals, hash_hits,
exact_hits, peak_*), plus the row-1 candidate pair count.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import STAT_KEYS, inst_from, load_golden, seeded_instance

pytestmark = pytest.mark.gpu

import paper_2507_05045_b200 as msb  # noqa: E402
from paper_2507_05045_b200 import _native  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker only)


def _solve_all(inst, **kw):
    return msb.solve(inst, msb.SolverConfig(mode="all", **kw))


def _strings(sols):
    return [msb.solution_to_string(x) for x in sols]


def test_tables_match_reference():
    for rec in load_golden("tables.json"):
        inst = inst_from(rec["instance"])
        got = _native.build_tables(inst.a, inst.d)  # every golden is inside the packed-16 mode
        for mine, ref in zip(got, rec["tables"]):
            assert mine["weights"].tolist() == ref["weights"], rec["name"]
            assert mine["masks"].tolist() == ref["masks"], rec["name"]
            assert mine["contribs"].tolist() == ref["contribs"], rec["name"]
            assert mine["run_end"].tolist() == ref["run_end"], rec["name"]


def test_tables_match_oracle_large():
    for (m, s) in ((6, 4), (7, 1), (8, 1)):
        inst = msb.generate_instance(m, 100, s)
        got = _native.build_tables(inst.a, inst.d)
        ref = O.build_tables(inst.a)
        for mine, r in zip(got, ref):
            assert np.array_equal(mine["weights"], r["weights"])
            assert np.array_equal(mine["masks"].astype(np.uint64), r["masks"])
            assert np.array_equal(mine["contribs"], r["contribs"])
            assert np.array_equal(mine["run_end"], r["run_end"])


def test_plan_matches_reference_streams():
    for rec in load_golden("streams.json"):
        inst = inst_from(rec["instance"])
        if inst.n < 4:
            continue
        plan = _native.alpha_plan(inst.a, inst.d)
        ref = [(b[0], b[1], len(b[2]), len(b[3])) for b in rec["batches"]]
        assert plan == ref, rec["name"]


def test_plan_counts_all_configs():
    counts = load_golden("plan_counts.json")
    for key, ref in counts.items():
        m, s = map(int, key.split(","))
        inst = msb.generate_instance(m, 100, s)
        plan = _native.alpha_plan(inst.a, inst.d)
        assert len(plan) == ref["batches"], key
        assert sum(p[2] for p in plan) == ref["candidates_left"], key
        assert sum(p[3] for p in plan) == ref["candidates_right"], key
        assert sum(p[2] * p[3] for p in plan) == ref["row1_candidate_pairs"], key


@pytest.mark.parametrize("fixture", ["solves_small.json", "solves_medium.json"])
def test_full_solves_match_reference(fixture):
    for rec in load_golden(fixture):
        inst = inst_from(rec["instance"])
        res = _solve_all(inst)
        assert _strings(res.solutions) == rec["solutions"], rec["name"]
        assert res.verdict == rec["verdict"], rec["name"]
        assert res.stats.fallback == rec["fallback"], rec["name"]
        if rec["fallback"] == "none":
            for k in STAT_KEYS:
                assert getattr(res.stats, k) == rec["stats"][k], (rec["name"], k)
            assert res.stats.engine == "cuda"


def test_per_batch_join_matches_reference():
    """msp_join_alpha on single batches vs the reference's per-batch validate_chunked stats."""
    for rec in load_golden("solves_medium.json"):
        if "batches" not in rec:
            continue
        inst = inst_from(rec["instance"])
        batches = rec["batches"]
        picks = batches[:: max(1, len(batches) // 25)] + [max(batches, key=lambda b: b[1] + b[2])]
        picks += [b for b in batches if b[5] > 0]
        for alpha, nl, nr, filt, hh, eh, sols in picks:
            opts = _native.make_options(mode="all")
            rc, xb, st = _native.solve_raw(inst.a, inst.d, opts, alpha=alpha)
            assert rc == 0, _native.last_error()
            assert (st["batches"], st["candidates_left"], st["candidates_right"]) == (1, nl, nr)
            assert (st["filtered_residuals"], st["hash_hits"], st["exact_hits"]) == (filt, hh, eh), (rec["name"], alpha)
            got = sorted("".join(map(str, r)) for r in xb.tolist())
            assert got == sols


@pytest.mark.parametrize("fixture", ["alpha_groups_8_100_1.json", "alpha_groups_9_100_1.json"])
def test_alpha_groups_large_configs(fixture):
    g = load_golden(fixture)
    inst = inst_from(g["instance"])
    for grp in g["groups"]:
        opts = _native.make_options(mode="all")
        rc, xb, st = _native.solve_raw(inst.a, inst.d, opts, alpha=grp["alpha"])
        assert rc == 0, _native.last_error()
        assert st["candidates_left"] == grp["n_left"] and st["candidates_right"] == grp["n_right"]
        assert st["filtered_residuals"] == grp["filtered"], grp["alpha"]
        assert st["hash_hits"] == grp["hash_hits"] and st["exact_hits"] == grp["exact_hits"]
        assert sorted("".join(map(str, r)) for r in xb.tolist()) == grp["solutions"]


def test_random_instances_match_oracle():
    for seed in range(30):
        m = 2 + seed % 5
        inst = seeded_instance(3000 + seed, m=m, n=13 + seed % 12, k=3 + seed % 40,
                               d_mode="half" if seed % 3 else "random")
        res = _solve_all(inst)
        ref = O.solve(inst.a, inst.d, mode="all")
        assert res.solutions == ref.solutions, seed
        for k in STAT_KEYS:
            assert getattr(res.stats, k) == ref.stats[k], (seed, k)


def test_stress_duplicates_and_tiny_waves():
    """Duplicate-heavy instances (m = 1, tiny K: many equal keys in a bucket -> stage overflow,
    spills, join stash and the global-table fallback) and tiny wave budgets (many pipeline waves,
    two-level batches), each against the oracle."""
    from paper_2507_05045_b200.solver import native_solve

    for seed in range(12):
        m = 1 + seed % 3
        n = 14 + seed % 5
        inst = seeded_instance(9100 + seed, m=m, n=n, k=3 + seed % 6, d_mode="half")
        ref = O.solve(inst.a, inst.d, mode="all")
        for wk in (0, 4096, 50000):
            sols, st = native_solve(inst, "all", None, brute_force_max_n=0, wave_keys=wk,
                                    flags=_native.MSP_FLAG_FORCE_TABLE_PATH)
            assert sorted(sols, key=msb.solution_encoding) == ref.solutions, (seed, wk)
            for k in STAT_KEYS:
                assert st[k] == ref.stats[k], (seed, wk, k)


def test_many_rows_match_oracle():
    """m = 10, 12, 16 (8-word companion vectors: the largest stage + loop-buffer layout) vs the oracle."""
    from paper_2507_05045_b200.solver import native_solve

    for seed, m in ((1, 10), (2, 12), (3, 16), (4, 10), (5, 14)):
        inst = seeded_instance(500 + seed, m=m, n=26, k=20)
        if seed >= 4:  # planted: d = A x* for a fixed x*, so the instance is feasible
            x = [(j * 7 + seed) % 3 == 0 for j in range(inst.n)]
            rows = inst.a.tolist()
            inst = msb.MspInstance(rows, [sum(r[j] for j in range(inst.n) if x[j]) for r in rows], k_bound=20)
        ref = O.solve(inst.a, inst.d, mode="all")
        assert seed < 4 or ref.solutions
        sols, st = native_solve(inst, "all", None, brute_force_max_n=0, flags=_native.MSP_FLAG_FORCE_TABLE_PATH)
        assert sorted(sols, key=msb.solution_encoding) == ref.solutions, m
        for k in STAT_KEYS:
            assert st[k] == ref.stats[k], (m, k)


def test_small_waves_force_multi_pass_join():
    """A tiny wave budget forces batches to split into hash-range passes: results unchanged."""
    inst = msb.generate_instance(6, 100, 4)
    ref = _solve_all(inst)
    tiny = _solve_all(inst, wave_keys=4096)
    assert tiny.solutions == ref.solutions
    for k in STAT_KEYS:
        assert getattr(tiny.stats, k) == getattr(ref.stats, k), k
    assert tiny.stats.waves > ref.stats.waves


@pytest.mark.parametrize("m,s,wave_keys", [(6, 4, 20000), (6, 1, 60000), (7, 1, 400000)])
def test_two_level_huge_batch_path(m, s, wave_keys):
    """A small wave budget routes the big batches through the two-level (coarse HBM + fine L2) join."""
    inst = msb.generate_instance(m, 100, s)
    ref = _solve_all(inst)
    got = _solve_all(inst, wave_keys=wave_keys)
    assert got.solutions == ref.solutions
    for k in STAT_KEYS:
        assert getattr(got.stats, k) == getattr(ref.stats, k), k


@pytest.mark.parametrize("m,s", [(5, 1), (6, 4), (7, 1)])
def test_persistent_pipeline_matches_per_wave_launches(m, s):
    """The persistent wave pipeline (k_waves) and per-wave scatter + join launches agree exactly."""
    inst = msb.generate_instance(m, 100, s)
    ref = _solve_all(inst)
    opts = _native.make_options(mode="all", flags=_native.MSP_FLAG_WAVE_LAUNCHES)
    rc, xb, st = _native.solve_raw(inst.a, inst.d, opts)
    assert rc == 0, _native.last_error()
    got = sorted((tuple(int(v) for v in r) for r in xb), key=msb.solution_encoding)
    assert got == ref.solutions
    for k in STAT_KEYS:
        assert st[k] == getattr(ref.stats, k), k


def test_global_table_join_path_matches():
    """The fallback global-hash-table join gives identical results to the partitioned join."""
    for (m, s) in ((4, 11), (5, 1), (6, 4)):
        inst = msb.generate_instance(m, 100, s)
        ref = _solve_all(inst)
        opts = _native.make_options(mode="all", flags=_native.MSP_FLAG_JOIN_GLOBAL)
        rc, xb, st = _native.solve_raw(inst.a, inst.d, opts)
        assert rc == 0, _native.last_error()
        got = sorted((tuple(int(v) for v in r) for r in xb), key=msb.solution_encoding)
        assert got == ref.solutions
        for k in STAT_KEYS:
            assert st[k] == getattr(ref.stats, k), k


def test_first_mode():
    for (m, s) in ((4, 11), (5, 1), (6, 4)):
        inst = msb.generate_instance(m, 100, s)
        full = _solve_all(inst)
        first = msb.solve(inst, msb.SolverConfig(mode="first"))
        assert first.feasible == full.feasible
        if full.feasible:
            assert first.solutions[0] in full.solutions


@pytest.mark.slow
def test_m7_s1_full_against_reference():
    rec = load_golden("solve_7_100_1.json")
    inst = inst_from(rec["instance"])
    res = _solve_all(inst)
    assert _strings(res.solutions) == rec["solutions"]
    for k in STAT_KEYS:
        assert getattr(res.stats, k) == rec["stats"][k], k
    ref_rows = rec["batches"]
    assert res.stats.row1_candidate_pairs == sum(b[1] * b[2] for b in ref_rows)


@pytest.mark.slow
def test_m8_s1_full_against_golden():
    """(8,70) s1 full enumeration (two-level huge-batch path + persistent waves) against the pinned
    oracle's full run (tests/golden/make_golden_oracle.py): solutions and every counter."""
    rec = load_golden("solve_8_100_1.json")
    inst = inst_from(rec["instance"])
    res = _solve_all(inst)
    assert _strings(res.solutions) == rec["solutions"]
    for k in STAT_KEYS:
        assert getattr(res.stats, k) == rec["stats"][k], k
    assert res.stats.row1_candidate_pairs == rec["row1_candidate_pairs"]


@pytest.mark.parametrize("seed", [1, 2])
def test_planted_m6_matches_oracle(seed):
    """BASELINE configs[1]: planted-feasible (6,50) instances (SURVEY.md §8(d) recipe): the planted x*
    is found and solutions + every counter equal the pinned oracle's."""
    inst, x = msb.plant_instance(6, 100, seed)
    res = _solve_all(inst)
    assert tuple(x) in res.solutions
    ref = O.solve(inst.a, inst.d, mode="all", workers=8)
    assert res.solutions == ref.solutions
    for k in STAT_KEYS:
        assert getattr(res.stats, k) == ref.stats[k], k


@pytest.mark.slow
@pytest.mark.parametrize("m,seed", [(7, 3), (8, 1)])
def test_planted_large_found(m, seed):
    """Planted (7,60) and (8,70) instances: the planted x* is among the (verified) solutions."""
    inst, x = msb.plant_instance(m, 100, seed)
    res = _solve_all(inst)
    assert tuple(x) in res.solutions
    assert all(msb.verify_solution(inst, s) for s in res.solutions)


def test_cancel_word_stops_the_solve(tmp_path):
    """msp_options.cancel: a set word stops the solve (stats.cancelled, no solutions); unset is inert."""
    from paper_2507_05045_b200.distributed import CancelFlag
    from paper_2507_05045_b200.solver import native_solve

    inst = msb.generate_instance(6, 100, 4)
    flag = CancelFlag(f"msp_cancel_test_{tmp_path.name}", create=True)
    try:
        sols, st = native_solve(inst, "first", None, cancel=flag.address)
        assert len(sols) == 1 and st["cancelled"] == 0
        assert msb.verify_solution(inst, sols[0])
        flag.set()
        sols, st = native_solve(inst, "first", None, cancel=flag.address)
        assert sols == [] and st["cancelled"] == 1
    finally:
        flag.close(unlink=True)


def test_gpu_brute_force_agrees_with_table_path():
    """the GPU brute force (k_brute, n <= 28) as an independent conformance
    check of the table path on many small instances (and both against the oracle on a few)."""
    from paper_2507_05045_b200.solver import native_solve

    for seed in range(24):
        m, n = 2 + seed % 3, 12 + seed % 13
        inst = seeded_instance(7000 + seed, m=m, n=n, k=5 + seed % 30, d_mode="half" if seed % 2 else "random")
        brute, bst = native_solve(inst, "all", None, brute_force_max_n=28)
        table, tst = native_solve(inst, "all", None, brute_force_max_n=0,
                                  flags=_native.MSP_FLAG_FORCE_TABLE_PATH)
        assert bst["fallback"] == 1 and tst["fallback"] == 0
        key = msb.solution_encoding
        assert sorted(brute, key=key) == sorted(table, key=key), seed
        if seed < 6:
            ref = O.solve(inst.a, inst.d, mode="all")
            assert sorted(table, key=key) == ref.solutions, seed


def test_per_batch_stats_match_reference_stream():
    """MSP_FLAG_BATCH_STATS: every batch's (alpha, n_left, n_right, filtered, hash_hits) of a full
    solve equals the reference's per-batch ValidationStats (validate.py:63-71,316-379)."""
    for rec in load_golden("solves_medium.json"):
        if "batches" not in rec:
            continue
        inst = inst_from(rec["instance"])
        opts = _native.make_options(mode="all", flags=_native.MSP_FLAG_BATCH_STATS)
        rc, xb, st = _native.solve_raw(inst.a, inst.d, opts)
        assert rc == 0, _native.last_error()
        ref = [tuple(b[:5]) for b in rec["batches"]]
        assert st["batch_stats"] == ref, rec["name"]


@pytest.mark.slow
def test_alpha_groups_with_hits_9_80():
    """Hit-bearing (9,80) s1 batches (FNV collisions and solutions; all on the two-level join path)
    through msp_join_alpha against the streaming CPU oracle (tests/golden/make_golden_groups.py)."""
    g = load_golden("alpha_groups_9_100_1_hits.json")
    inst = inst_from(g["instance"])
    assert sum(grp["hash_hits"] for grp in g["groups"]) >= 10
    for grp in g["groups"]:
        opts = _native.make_options(mode="all")
        rc, xb, st = _native.solve_raw(inst.a, inst.d, opts, alpha=grp["alpha"])
        assert rc == 0, _native.last_error()
        assert (st["candidates_left"], st["candidates_right"]) == (grp["n_left"], grp["n_right"])
        assert st["filtered_residuals"] == grp["filtered"], grp["alpha"]
        assert (st["hash_hits"], st["exact_hits"]) == (grp["hash_hits"], grp["exact_hits"]), grp["alpha"]
        assert sorted("".join(map(str, r)) for r in xb.tolist()) == grp["solutions"]


@pytest.mark.slow
def test_full_9_80_hits_match_oracle_groups():
    """The headline (9,80) s1 full enumeration, batch by batch against the CPU oracle: the GPU's
    per-batch stats (MSP_FLAG_BATCH_STATS) put hash hits in exactly the 92 batches the oracle goldens
    hold (alpha_groups_9_100_1_hits*.json), each batch's (n_left, n_right, filtered, hash_hits) equals
    the oracle's, and the 7 solutions are the union of the oracle's per-batch solutions."""
    g10 = load_golden("alpha_groups_9_100_1_hits.json")
    gall = load_golden("alpha_groups_9_100_1_hits_all.json")
    inst = inst_from(g10["instance"])
    groups = {grp["alpha"]: grp for grp in g10["groups"] + gall["groups"]}
    opts = _native.make_options(mode="all", flags=_native.MSP_FLAG_BATCH_STATS)
    rc, xb, st = _native.solve_raw(inst.a, inst.d, opts)
    assert rc == 0, _native.last_error()
    assert st["hash_hits"] == 99 and st["exact_hits"] == 7 and st["batches"] == 1911
    gpu_hits = {b[0]: b for b in st["batch_stats"] if b[4] > 0}
    assert sorted(gpu_hits) == sorted(gall["hit_alphas"])
    for alpha, grp in groups.items():
        assert gpu_hits[alpha][1:] == (grp["n_left"], grp["n_right"], grp["filtered"], grp["hash_hits"]), alpha
    if len(groups) == len(gall["hit_alphas"]):  # every hit batch pinned: the totals and solutions too
        assert sum(grp["hash_hits"] for grp in groups.values()) == 99
        sols = sorted(s for grp in groups.values() for s in grp["solutions"])
        assert sorted("".join(map(str, r)) for r in xb.tolist()) == sols
    # the heap-free plan against the reference stream's 1911 batch headers (heap enumeration restated)
    stream = load_golden("stream_9_100_1.json")["headers"]
    assert [b[:3] for b in st["batch_stats"]] == [(h[0], h[2], h[3]) for h in stream]
    # every other batch's counters against the oracle's filter join (tests/golden/make_golden_batches_9_80.py)
    if not os.path.exists(os.path.join(os.path.dirname(__file__), "golden", "batches_9_100_1.json")):
        return
    gb = load_golden("batches_9_100_1.json")
    by_alpha = {b[0]: b for b in st["batch_stats"]}
    for alpha, nl, nr, filt, hh, eh in gb["records"]:
        assert by_alpha[alpha] == (alpha, nl, nr, filt, hh), alpha
        assert hh == 0 and eh == 0
    assert len(gb["records"]) + len(groups) == len(stream) or not gb["complete"]


@pytest.mark.slow
def test_planted_9_80_found():
    """BASELINE configs[4]: a planted-feasible (9,80) instance, full enumeration: x* is found."""
    inst, x = msb.plant_instance(9, 100, 1)
    res = _solve_all(inst)
    assert tuple(x) in res.solutions
    assert all(msb.verify_solution(inst, s) for s in res.solutions)
    assert res.stats.exact_hits == len(res.solutions) and res.stats.hash_hits >= res.stats.exact_hits


@pytest.mark.parametrize("world", [2, 4, 8])
def test_alpha_bands_through_cuda_band_solver(world):
    """SURVEY.md §8(e) sharding on one GPU: (7,60) s1 cut into `world` cost-balanced alpha-bands, each
    solved by the CUDA band solver (distributed.cuda_band_solver), merged by the same code as the
    multi-rank path (merge_band_results): solutions and every counter equal the reference golden."""
    from paper_2507_05045_b200.distributed import alpha_bands, cuda_band_solver, merge_band_results

    rec = load_golden("solve_7_100_1.json")
    inst = inst_from(rec["instance"])
    plan = _native.alpha_plan(inst.a, inst.d)
    bands = alpha_bands(plan, world)
    solver = cuda_band_solver(0)
    sols, per = [], []
    for band in bands:
        s, st = solver(inst, "all", band)
        sols += s
        per.append(st)
    res = merge_band_results(inst, sols, per)
    assert _strings(res.solutions) == rec["solutions"]
    for k in ("batches", "candidates_left", "candidates_right", "hash_hits", "exact_hits", "filtered_residuals"):
        assert getattr(res.stats, k) == rec["stats"][k], (world, k)
    assert res.stats.row1_candidate_pairs == sum(b[1] * b[2] for b in rec["batches"])


def _cuda_rank(rank, world, port, q):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_05045_b200.distributed import solve_sharded

        inst = msb.generate_instance(7, 100, 1)
        res = solve_sharded(inst, msb.SolverConfig(mode="all", device=0), dist=dist)
        q.put((rank, _strings(res.solutions), {k: getattr(res.stats, k) for k in STAT_KEYS}))
    except Exception as exc:  # surfaced by the parent
        q.put((rank, repr(exc), None))
    finally:
        dist.destroy_process_group()


def test_two_ranks_cuda_band_solver_gloo():
    """Two rank processes (gloo) sharing GPU 0, each solving its alpha-band of (7,60) s1 with the CUDA
    engine (solve_sharded's default band solver), gathered: both ranks return the golden result."""
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_cuda_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    rec = load_golden("solve_7_100_1.json")
    for rank, sols, st in out:
        assert st is not None, sols
        assert sols == rec["solutions"], rank
        for k in STAT_KEYS:
            assert st[k] == rec["stats"][k], (rank, k)


# Frozen feasible seeds of the reference's benchmark classes (test_acceptance.py:178-183) and the
# (7,60) seeds its README reports feasible (README.md:187-192).
FEASIBLE_SEEDS = {(3, 20): [27, 98, 99, 116], (4, 30): [11, 12, 15, 30], (5, 40): [1, 3, 14, 17],
                  (6, 50): [4, 5, 8, 9], (7, 60): [1, 2, 3, 4]}


def test_first_mode_frozen_feasible_seeds():
    """First mode (the reference's Table-1 mode, solver.py:278-279,391-392) on every frozen feasible
    seed: verdict feasible, exactly one solution, verified on the original instance."""
    for (m, n), seeds in FEASIBLE_SEEDS.items():
        for seed in seeds:
            inst = msb.generate_instance(m, 100, seed)
            assert inst.n == n
            res = msb.solve(inst, msb.SolverConfig(mode="first"))
            assert res.verdict == "feasible", (m, seed)
            assert len(res.solutions) == 1 and msb.verify_solution(inst, res.solutions[0]), (m, seed)


def test_first_mode_matches_all_mode_verdicts_and_membership():
    """First mode vs the reference goldens: same verdict, and the one solution is in the full set."""
    for rec in load_golden("solves_medium.json"):
        inst = inst_from(rec["instance"])
        res = msb.solve(inst, msb.SolverConfig(mode="first"))
        assert res.verdict == rec["verdict"], rec["name"]
        if res.solutions:
            assert _strings(res.solutions)[0] in rec["solutions"], rec["name"]


def test_time_limit_raises_mid_solve():
    """SolveTimeout (solver.py:54-56,263-264): a time limit far below the (8,70) solve time raises
    mid-solve; a generous one does not (test_solver.py:198-216)."""
    inst = msb.generate_instance(8, 100, 1)
    with pytest.raises(msb.SolveTimeout):
        msb.solve(inst, msb.SolverConfig(mode="all"), time_limit=0.05)
    with pytest.raises(msb.SolveTimeout):
        msb.solve(inst, msb.SolverConfig(mode="all"), time_limit=1e-9)
    small = msb.MspInstance([[1, 2, 3], [2, 1, 3]], [3, 3])
    assert msb.solve(small, msb.SolverConfig(mode="all"), time_limit=60.0).feasible


def test_massive_multiplicity_all_zero_instance():
    """The reference's hit-buffer regrowth case (test_validate.py:298-314): the all-zero 1x13 instance
    has 2^13 solutions, all in one batch with one repeated key (partitioned bucket overflow ->
    global-table re-join)."""
    inst = msb.MspInstance([[0] * 13], [0])
    res = _solve_all(inst)
    assert len(res.solutions) == 2 ** 13
    assert res.stats.hash_hits == res.stats.exact_hits == 2 ** 13


def test_hit_list_regrowth_subprocess():
    """The device hit list (distinct hit keys) regrows like fastval.join_pairs' output buffer
    (fastval.py:126-139): with a 16-key initial list, a duplicate-heavy instance with far more
    distinct hit keys re-runs with a grown list and matches the oracle."""
    import json
    import subprocess
    import sys

    code = (
        "import json, paper_2507_05045_b200 as msb\n"
        "from conftest import seeded_instance\n"
        "inst = seeded_instance(77, m=1, n=24, k=5)\n"
        "r = msb.solve(inst, msb.SolverConfig(mode='all'))\n"
        "print(json.dumps([len(r.solutions), r.stats.hash_hits, r.stats.batches]))\n"
    )
    import os

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, MSP_HIT_CAP="16",
               PYTHONPATH=os.pathsep.join([os.path.dirname(here), here, os.environ.get("PYTHONPATH", "")]))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=here,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    nsol, hh, nb = json.loads(out.stdout.strip().splitlines()[-1])
    inst = seeded_instance(77, m=1, n=24, k=5)
    ref = O.solve(inst.a, inst.d, mode="all")
    assert nsol == len(ref.solutions) and hh == ref.stats["hash_hits"]
    assert nb > 16  # more distinct hit keys (one per batch at m = 1) than the initial list holds


def test_engine_names_of_the_reference_run_the_cuda_engine():
    inst = msb.generate_instance(4, 100, 11)
    ref = _solve_all(inst)
    for engine in ("python", "jit", "cuda", None):
        res = msb.solve(inst, msb.SolverConfig(mode="all"), engine=engine)
        assert res.solutions == ref.solutions and res.stats.engine == "cuda"


def test_generic_weights_match_reference():
    """generic u64 weights through the CUDA engine -- K = 10^6 instances (P32
    companion layout + sparse alpha plan) and surrogate-reduced instances (reduce_rows 2, 3: u64 merged
    row 0, sparse plan) -- against the reference's solves: solutions and every counter."""
    for rec in load_golden("solves_generic.json"):
        inst = inst_from(rec["instance"])
        res = msb.solve(inst, msb.SolverConfig(mode="all", reduce_rows=rec["reduce_rows"]))
        assert _strings(res.solutions) == rec["solutions"], rec["name"]
        assert res.verdict == rec["verdict"]
        for k in STAT_KEYS:
            assert getattr(res.stats, k) == rec["stats"][k], (rec["name"], k)


def test_generic_weights_per_batch_stats():
    """Per-batch counters of K = 10^6 instances (sparse plan) equal the reference's per-batch stats."""
    for rec in load_golden("solves_generic.json"):
        if "batches" not in rec:
            continue
        inst = inst_from(rec["instance"])
        opts = _native.make_options(mode="all", flags=_native.MSP_FLAG_BATCH_STATS)
        rc, xb, st = _native.solve_raw(inst.a, inst.d, opts)
        assert rc == 0, _native.last_error()
        assert st.get("batch_stats", []) == [tuple(b[:5]) for b in rec["batches"]], rec["name"]


def test_sparse_plan_matches_dense_plan(monkeypatch):
    """The sparse (sorted pair-sum) alpha plan, forced on K = 100 instances, reproduces the dense
    plan exactly: batch headers, per-batch counters, solutions."""
    for (m, s) in ((4, 11), (5, 3), (6, 4), (7, 1)):
        inst = msb.generate_instance(m, 100, s)
        opts = _native.make_options(mode="all", flags=_native.MSP_FLAG_BATCH_STATS)
        monkeypatch.delenv("MSP_SPARSE_PLAN", raising=False)
        rc0, xb0, st0 = _native.solve_raw(inst.a, inst.d, opts)
        plan0 = _native.alpha_plan(inst.a, inst.d)
        monkeypatch.setenv("MSP_SPARSE_PLAN", "1")
        rc1, xb1, st1 = _native.solve_raw(inst.a, inst.d, opts)
        plan1 = _native.alpha_plan(inst.a, inst.d)
        monkeypatch.delenv("MSP_SPARSE_PLAN")
        assert rc0 == 0 and rc1 == 0, _native.last_error()
        assert plan1 == plan0, (m, s)
        assert st1["batch_stats"] == st0["batch_stats"], (m, s)
        assert sorted(map(tuple, xb1.tolist())) == sorted(map(tuple, xb0.tolist()))
        for k in STAT_KEYS:
            assert st1[k] == st0[k], (m, s, k)


def test_sparse_plan_alpha_windows(monkeypatch):
    """The sparse plan streamed through alpha windows (MSP_SPARSE_WINDOW_PAIRS run pairs per window
    side: 1 forces single-alpha windows past the budget, 37 .. 65536 cut the range into many windows)
    reproduces the one-window plan: batch headers, per-batch counters, solutions, counters -- on K = 100
    instances and the generic-weight (K = 10^6) goldens, and inside an alpha band."""
    cases = [(msb.generate_instance(5, 100, 3), ("1", "37", "4096")),
             (msb.generate_instance(6, 100, 4), ("37", "4096")), (msb.generate_instance(7, 100, 1), ("4096",))]
    cases += [(inst_from(r["instance"]), ("4096", "65536")) for r in load_golden("solves_generic.json")
              if r["reduce_rows"] == 1][:4]
    monkeypatch.setenv("MSP_SPARSE_PLAN", "1")
    for inst, budgets in cases:
        opts = _native.make_options(mode="all", flags=_native.MSP_FLAG_BATCH_STATS)
        monkeypatch.delenv("MSP_SPARSE_WINDOW_PAIRS", raising=False)
        rc0, xb0, st0 = _native.solve_raw(inst.a, inst.d, opts)
        plan0 = _native.alpha_plan(inst.a, inst.d)
        assert rc0 == 0, _native.last_error()
        alphas = [b[0] for b in st0["batch_stats"]]
        lo, hi = (alphas[len(alphas) // 3], alphas[2 * len(alphas) // 3]) if len(alphas) > 2 else (0, 0)
        band = _native.make_options(mode="all", flags=_native.MSP_FLAG_BATCH_STATS, alpha_lo=lo, alpha_hi=hi)
        for w in budgets:
            monkeypatch.setenv("MSP_SPARSE_WINDOW_PAIRS", w)
            rc1, xb1, st1 = _native.solve_raw(inst.a, inst.d, opts)
            assert rc1 == 0, _native.last_error()
            assert _native.alpha_plan(inst.a, inst.d) == plan0, w
            assert st1["batch_stats"] == st0["batch_stats"], w
            assert sorted(map(tuple, xb1.tolist())) == sorted(map(tuple, xb0.tolist()))
            for k in STAT_KEYS:
                assert st1[k] == st0[k], (w, k)
            if hi:
                rc2, _, st2 = _native.solve_raw(inst.a, inst.d, band)
                assert rc2 == 0, _native.last_error()
                assert st2["batch_stats"] == [b for b in st0["batch_stats"] if lo <= b[0] < hi], w


def test_one_sided_recovery_matches_two_sided(monkeypatch):
    """Hit recovery enumerates one side of a hit batch and finds the other side's exact pairs by
    table lookup; forcing the two-sided recovery (both sides enumerated, every pair of a hit key
    compared) gives the same solutions and counters -- on solution-bearing K = 100 instances,
    planted ones (equal-vector pairs on one side) and the hit-bearing (9,80) alpha-groups."""
    cases = [(msb.generate_instance(m, 100, s), None) for (m, s) in ((4, 11), (6, 4), (7, 1))]
    cases += [(msb.plant_instance(m, 100, s)[0], None) for (m, s) in ((5, 1), (6, 2))]
    g = load_golden("alpha_groups_9_100_1_hits.json")
    inst9 = inst_from(g["instance"])
    cases += [(inst9, grp["alpha"]) for grp in g["groups"] if grp["solutions"]][:2]
    for inst, alpha in cases:
        opts = _native.make_options(mode="all", flags=_native.MSP_FLAG_BATCH_STATS)
        monkeypatch.delenv("MSP_RECOVER_TWO_SIDED", raising=False)
        rc0, xb0, st0 = _native.solve_raw(inst.a, inst.d, opts, alpha=alpha)
        monkeypatch.setenv("MSP_RECOVER_TWO_SIDED", "1")
        rc1, xb1, st1 = _native.solve_raw(inst.a, inst.d, opts, alpha=alpha)
        monkeypatch.delenv("MSP_RECOVER_TWO_SIDED")
        assert rc0 == 0 and rc1 == 0, _native.last_error()
        assert sorted(map(tuple, xb0.tolist())) == sorted(map(tuple, xb1.tolist()))
        assert len(xb0) > 0
        for k in STAT_KEYS:
            assert st0[k] == st1[k], k


def test_time_limit_stops_the_running_kernels():
    """The deadline reaches the running kernels (host-mapped stop word polled at every task switch of
    the persistent pipeline): a (9,80) full enumeration (~40 s) with a 1 s limit raises SolveTimeout
    within a fraction of a second of the limit, not at the end of the enumeration."""
    import time

    inst = msb.generate_instance(9, 100, 1)
    msb.solve(msb.generate_instance(4, 100, 11), msb.SolverConfig(mode="all"))  # (context already up)
    t0 = time.perf_counter()
    with pytest.raises(msb.SolveTimeout):
        msb.solve(inst, msb.SolverConfig(mode="all"), time_limit=1.0)
    assert time.perf_counter() - t0 < 4.0
    # the device is usable right after an interrupted solve
    res = msb.solve(msb.generate_instance(6, 100, 4), msb.SolverConfig(mode="all"))
    assert len(res.solutions) == 2


def test_cancel_word_stops_a_running_solve(tmp_path):
    """Cross-rank early exit: a cancel word set while a (9,80) solve runs stops it
    within a task switch; the solve returns cancelled with partial counters."""
    import threading
    import time

    from paper_2507_05045_b200.distributed import CancelFlag
    from paper_2507_05045_b200.solver import native_solve

    inst = msb.generate_instance(9, 100, 1)
    flag = CancelFlag(f"msp_cancel_run_{tmp_path.name}", create=True)
    try:
        timer = threading.Timer(1.0, flag.set)
        timer.start()
        t0 = time.perf_counter()
        sols, st = native_solve(inst, "all", None, cancel=flag.address)
        dt = time.perf_counter() - t0
        timer.join()
        assert st["cancelled"] == 1 and dt < 5.0
    finally:
        flag.close(unlink=True)


def test_degenerate_hash_seam_counts_every_pair():
    """The reference's degenerate-hash injection (validate.py:161-162,208-216; test_validate.py:197-241):
    with every key hashed to one value, every unfiltered (left, right) pair of a batch is a hash hit,
    so hash_hits = sum over batches of n_left x (n_right - filtered); the exact confirmation still
    finds exactly the true solutions."""
    for (m, s) in ((3, 5), (4, 11), (4, 12)):
        inst = msb.generate_instance(m, 100, s) if m > 3 else seeded_instance(s, m=3, n=16, k=20)
        ref = _solve_all(inst)
        opts = _native.make_options(mode="all", flags=_native.MSP_FLAG_DEGENERATE_HASH | _native.MSP_FLAG_BATCH_STATS
                                    | _native.MSP_FLAG_FORCE_TABLE_PATH)
        rc, xb, st = _native.solve_raw(inst.a, inst.d, opts)
        assert rc == 0, _native.last_error()
        expect = sum(nl * (nr - filt) for _, nl, nr, filt, _ in st["batch_stats"])
        assert st["hash_hits"] == expect, (m, s)
        assert st["exact_hits"] == ref.stats.exact_hits
        assert sorted(map(tuple, xb.tolist())) == sorted(ref.solutions)
        assert st["filtered_residuals"] == ref.stats.filtered_residuals
