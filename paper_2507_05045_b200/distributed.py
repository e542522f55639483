"""Multi-GPU sharding: one process per GPU, contiguous alpha-bands, one final gather.

SURVEY.md §8(e): a batch (alpha, beta = t - alpha) joins only L(alpha) with R(beta), so batches are
independent units.  Every rank rebuilds the (tiny) quarter tables and the plan, cuts the alpha axis
into contiguous bands of equal candidate-pair cost c(alpha) = n_left + n_right, and solves its band
with ``msp_solve(alpha_lo, alpha_hi)``.  No data-path collective exists; the only communication is the
final all-gather of solution bit vectors and of the per-rank counters (NCCL on GPUs, gloo in the
CPU tests).  The reference has no multi-device mode; its in-process analogue is
pipeline_run's result merge (solver.py:284-289,415-418).
"""

from __future__ import annotations

import os
import time
from typing import Callable, Sequence

import numpy as np

from .instances import MspInstance, solution_encoding, verify_solution
from .solver import SolveResult, SolverConfig, SolveStats, native_solve, stats_from_native

COUNTERS = ("batches", "candidates_left", "candidates_right", "filtered_residuals", "hash_hits",
            "exact_hits", "peak_table_entries", "peak_heap1", "peak_heap2", "kernel_launches", "waves",
            "cancelled")


def alpha_bands(plan: Sequence[tuple[int, int, int, int]], world: int) -> list[tuple[int, int]]:
    """Contiguous [alpha_lo, alpha_hi) bands with balanced n_left + n_right.

    ``plan`` is the batch header list (alpha, beta, n_left, n_right) in alpha order.  Band r starts
    at the first batch whose cost prefix reaches r/world of the total.  alpha_hi = 0 means unbounded.
    """
    if world <= 1 or not plan:
        return [(0, 0)] + [(1, 1)] * (world - 1) if world > 1 else [(0, 0)]
    cost = np.array([p[2] + p[3] for p in plan], dtype=np.float64)
    pre = np.concatenate([[0.0], np.cumsum(cost)])
    total = pre[-1]
    starts = [0]
    for r in range(1, world):
        idx = int(np.searchsorted(pre, total * r / world, side="left"))
        starts.append(min(max(idx, starts[-1]), len(plan)))
    bands = []
    for r in range(world):
        lo_i = starts[r]
        hi_i = starts[r + 1] if r + 1 < world else len(plan)
        if lo_i >= hi_i:
            bands.append((1, 1))  # empty band (alpha_lo == alpha_hi)
            continue
        lo = 0 if r == 0 else int(plan[lo_i][0])
        hi = 0 if hi_i == len(plan) else int(plan[hi_i][0])
        bands.append((lo, hi))
    return bands


def band_cost(plan, band) -> int:
    lo, hi = band
    return sum(p[2] + p[3] for p in plan if p[0] >= lo and (hi == 0 or p[0] < hi))


def _gather_solutions(sols: list[tuple[int, ...]], n: int, dist, device) -> list[tuple[int, ...]]:
    import torch

    world = dist.get_world_size()
    x = torch.tensor(np.array(sols, dtype=np.uint8).reshape(-1, n), device=device)
    cnt = torch.tensor([x.shape[0]], dtype=torch.int64, device=device)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt)
    maxc = max(int(c.item()) for c in cnts)
    pad = torch.zeros((max(maxc, 1), n), dtype=torch.uint8, device=device)
    pad[: x.shape[0]] = x
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    out = []
    for c, b in zip(cnts, bufs):
        out.extend(tuple(int(v) for v in row) for row in b[: int(c.item())].cpu().numpy())
    return out


def _gather_counters(st: dict, dist, device) -> list[dict]:
    import torch

    world = dist.get_world_size()
    row1 = int(st.get("row1_candidate_pairs", 0))
    vals = [int(st.get(k, 0)) for k in COUNTERS] + [row1 & ((1 << 62) - 1), row1 >> 62]
    t = torch.tensor(vals, dtype=torch.int64, device=device)
    bufs = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(bufs, t)
    out = []
    for b in bufs:
        v = b.cpu().tolist()
        d = dict(zip(COUNTERS, v[: len(COUNTERS)]))
        d["row1_candidate_pairs"] = v[-2] | (v[-1] << 62)
        out.append(d)
    return out


BandSolver = Callable[[MspInstance, str, tuple[int, int]], tuple[list[tuple[int, ...]], dict]]


class CancelFlag:
    """One int32 shared by the rank processes of a node (a /dev/shm mapping).

    First mode's cross-GPU early exit (the reference stops its one
    process at the first verified solution, solver.py:278-279,391-392): the rank that confirms a
    solution sets the word; every rank's ``msp_solve`` polls it at its wave checkpoints through
    ``msp_options.cancel`` and stops.  The word is host memory: a checkpoint already synchronises
    the host with the device, so polling costs nothing on the device.
    """

    def __init__(self, name: str, create: bool):
        import ctypes
        import mmap
        import tempfile

        base = "/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir()
        self.path = os.path.join(base, name)
        if create:
            with open(self.path, "wb") as fh:
                fh.write(b"\0" * 8)
        self._fh = open(self.path, "r+b")
        self._mm = mmap.mmap(self._fh.fileno(), 8)
        self._word = ctypes.c_int32.from_buffer(self._mm)
        self.address = ctypes.addressof(self._word)

    def set(self) -> None:
        self._word.value = 1

    def is_set(self) -> bool:
        return self._word.value != 0

    def close(self, unlink: bool = False) -> None:
        del self._word
        self._mm.close()
        self._fh.close()
        if unlink:
            try:
                os.unlink(self.path)
            except OSError:
                pass


def shared_cancel_flag(dist) -> CancelFlag:
    """Rank 0 creates the word, every rank maps it (collective over ``dist``)."""
    import uuid

    name = [f"msp_cancel_{uuid.uuid4().hex}" if dist.get_rank() == 0 else None]
    if dist.get_rank() == 0:
        flag = CancelFlag(name[0], create=True)
    dist.broadcast_object_list(name, src=0)
    if dist.get_rank() != 0:
        flag = CancelFlag(name[0], create=False)
    dist.barrier()
    return flag


def cuda_band_solver(device: int, time_limit: float | None = None, wave_keys: int = 0,
                     stream: int | None = None, cancel: CancelFlag | None = None) -> BandSolver:
    def run(work: MspInstance, mode: str, band: tuple[int, int]):
        lo, hi = band
        if hi != 0 and lo >= hi:  # empty band: nothing to enumerate on this rank
            return [], {}
        return native_solve(work, mode, time_limit, device=device, alpha_lo=lo, alpha_hi=hi,
                            wave_keys=wave_keys, stream=stream,
                            cancel=cancel.address if cancel is not None else None)
    return run


def merge_band_results(inst: MspInstance, sols: list[tuple[int, ...]], per_band: list[dict],
                       mode: str = "all") -> SolveResult:
    """Merge the bands' solutions and counters into one SolveResult (the reference's in-process
    merge: _merge_vstats solver.py:284-289, results sorted solver.py:238-241,415-418).  Counters
    add up over bands (every batch lives in exactly one band); the table peaks are per solve."""
    stats = SolveStats(engine="cuda")
    for k in ("batches", "candidates_left", "candidates_right", "filtered_residuals", "hash_hits",
              "exact_hits", "kernel_launches", "waves", "row1_candidate_pairs"):
        setattr(stats, k, sum(int(r.get(k, 0)) for r in per_band))
    for k in ("peak_table_entries", "peak_heap1", "peak_heap2"):
        setattr(stats, k, max((int(r.get(k, 0)) for r in per_band), default=0))
    stats.cancelled_ranks = int(sum(int(r.get("cancelled", 0)) for r in per_band))
    sols = list(sols)
    for x in sols:
        if not verify_solution(inst, x):
            raise RuntimeError("internal error: candidate failed original-system verification")
    sols.sort(key=solution_encoding)
    if len(set(sols)) != len(sols):
        raise RuntimeError("internal error: duplicate solutions emitted")
    if mode == "first":
        sols = sols[:1]
    return SolveResult("feasible" if sols else "infeasible", sols, stats)


def solve_sharded(inst: MspInstance, cfg: SolverConfig | None = None, dist=None,
                  plan: Sequence[tuple[int, int, int, int]] | None = None,
                  band_solver: BandSolver | None = None, device=None) -> SolveResult:
    """All-solutions solve of one instance over the ranks of ``dist`` (torch.distributed).

    Every rank returns the same merged SolveResult.  ``plan`` defaults to the device plan
    (``msp_alpha_plan``); ``band_solver`` defaults to the CUDA engine on ``cfg.device``.
    """
    from . import _native

    cfg = (cfg or SolverConfig(mode="all")).validated()
    if cfg.reduce_rows != 1:
        raise ValueError("sharded solve takes the unreduced instance")
    t0 = time.perf_counter()
    world = dist.get_world_size()
    rank = dist.get_rank()
    if plan is None:
        plan = _native.alpha_plan(inst.a, inst.d, device=cfg.device)
    bands = alpha_bands(plan, world)
    cancel = shared_cancel_flag(dist) if cfg.mode == "first" else None
    if band_solver is None:
        band_solver = cuda_band_solver(cfg.device, wave_keys=cfg.wave_keys, cancel=cancel)
    if cancel is not None and cancel.is_set():
        sols, st = [], {}
    else:
        sols, st = band_solver(inst, cfg.mode, bands[rank])
    if cancel is not None and sols:
        cancel.set()  # the other ranks stop at their next wave checkpoint
    if device is None:
        import torch
        device = torch.device("cuda", cfg.device) if dist.get_backend() == "nccl" else torch.device("cpu")
    all_sols = _gather_solutions(sols, inst.n, dist, device)
    per_rank = _gather_counters(st, dist, device)
    res = merge_band_results(inst, all_sols, per_rank, cfg.mode)
    stats = res.stats
    if cancel is not None:
        dist.barrier()
        cancel.close(unlink=rank == 0)
    stats.t_total = time.perf_counter() - t0
    return res
