"""Multi-rank sharding on CPU: alpha-band partition + gloo all-gather, world size 2.

The per-band solver is the oracle restricted to the band (the GPU path is covered by -m gpu tests);
what is tested here is the sharding logic: bands tile the alpha axis exactly once, are cost-balanced,
and the gathered solutions and counters equal the single-rank solve.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import paper_2507_05045_b200 as msb
from paper_2507_05045_b200.distributed import alpha_bands, band_cost, solve_sharded

STATS = ("batches", "candidates_left", "candidates_right", "filtered_residuals", "hash_hits",
         "exact_hits", "row1_candidate_pairs")


def _plan(inst):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import plan_np

    return plan_np(inst)


def test_bands_cover_every_batch_once_and_balance():
    inst = msb.generate_instance(6, 100, 4)
    plan = _plan(inst)
    total = sum(p[2] + p[3] for p in plan)
    for world in (1, 2, 3, 4, 8):
        bands = alpha_bands(plan, world)
        assert len(bands) == world
        owners = []
        for p in plan:
            hit = [r for r, (lo, hi) in enumerate(bands) if p[0] >= lo and (hi == 0 or p[0] < hi) and not (hi and lo >= hi)]
            owners.append(hit)
        assert all(len(h) == 1 for h in owners), world
        costs = [band_cost(plan, b) if not (b[1] and b[0] >= b[1]) else 0 for b in bands]
        assert sum(costs) == total
        assert max(costs) <= total / world * 1.2 + max(p[2] + p[3] for p in plan)


def oracle_band_solver(inst, mode, band):
    from oracle import oracle as O

    lo, hi = band
    if hi and lo >= hi:
        return [], {}
    r = O.solve(inst.a, inst.d, mode=mode, alpha_lo=lo, alpha_hi=hi, workers=1)
    st = dict(r.stats)
    return r.solutions, st


def _worker(rank, world, port, m, seed, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inst = msb.generate_instance(m, 100, seed)
        plan = _plan(inst)
        res = solve_sharded(inst, msb.SolverConfig(mode="all"), dist=dist, plan=plan,
                            band_solver=oracle_band_solver)
        q.put((rank, [msb.solution_to_string(x) for x in res.solutions],
               {k: getattr(res.stats, k) for k in STATS}))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("m,seed", [(4, 11), (5, 3), (6, 4)])
def test_two_rank_gloo_solve_equals_single_rank(m, seed):
    import torch.multiprocessing as tmp
    from oracle import oracle as O

    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, m, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    inst = msb.generate_instance(m, 100, seed)
    ref = O.solve(inst.a, inst.d)
    ref_sols = ["".join(map(str, x)) for x in ref.solutions]
    for rank, sols, st in outs:
        assert sols == ref_sols, rank
        for k in STATS:
            assert st[k] == ref.stats[k], (rank, k)


def _first_worker(rank, world, port, m, seed, q):
    import torch.distributed as dist

    from paper_2507_05045_b200.distributed import shared_cancel_flag

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # the shared cancel word: set by rank 1, observed by rank 0 through its own mapping
        flag = shared_cancel_flag(dist)
        seen_before = flag.is_set()
        dist.barrier()
        if rank == 1:
            flag.set()
        dist.barrier()
        seen_after = flag.is_set()
        flag.close(unlink=rank == 0)
        inst = msb.generate_instance(m, 100, seed)
        res = solve_sharded(inst, msb.SolverConfig(mode="first"), dist=dist, plan=_plan(inst),
                            band_solver=oracle_band_solver)
        q.put((rank, seen_before, seen_after, [msb.solution_to_string(x) for x in res.solutions],
               res.verdict))
    finally:
        dist.destroy_process_group()


def test_two_rank_first_mode_shares_the_cancel_word():
    """First mode over 2 ranks (gloo): the cancel word is one shared int32; one verified solution."""
    import torch.multiprocessing as tmp

    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    m, seed = 6, 4  # feasible (SURVEY.md §8(c) frozen seeds)
    procs = [ctx.Process(target=_first_worker, args=(r, 2, port, m, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    inst = msb.generate_instance(m, 100, seed)
    sols = [s for _, _, _, s, _ in outs]
    assert sols[0] == sols[1] and len(sols[0]) == 1
    x = tuple(int(c) for c in sols[0][0])
    assert msb.verify_solution(inst, x)
    for rank, before, after, _, verdict in outs:
        assert not before and after and verdict == "feasible", rank
