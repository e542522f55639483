"""Drop-in ``solve()`` whose table path runs on one B200 through libmsp_b200.so.

Mirrors the reference driver ``pkg/src/marketsplit/solver.py``:

* ``SolverConfig``  <- solver.py:58-91 (same fields, same ``validated()`` errors; ``backend``
  gains ``"cuda"``, the only compute engine here -- ``"parallel"``/``"serial"`` are accepted as
  names of the engine being replaced and run on the GPU too)
* ``SolveStats``    <- solver.py:94-129 (same counters and ``as_dict`` schema, engine = "cuda")
* ``SolveResult``   <- solver.py:132-140
* ``SolveTimeout``  <- solver.py:54-56
* ``solve``         <- solver.py:170-245: surrogate reduction (host, integer only), first-mode
  zero-RHS shortcut (no compute), then ONE native call that covers both the n <= 12 brute-force
  branch (a GPU kernel) and the table path (K1..K6), then the reference's own final checks:
  every solution re-verified on the original instance (solver.py:248-253), all-mode sorted by
  ``solution_encoding`` with a duplicate check (solver.py:238-241).

There is no CPU fallback: if the CUDA library or device is missing, ``solve`` raises.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .instances import (
    MspInstance,
    SolutionVector,
    solution_encoding,
    surrogate_reduce,
    verify_solution,
)

BRUTE_FORCE_MAX_N = 12  # solver.py:48
DEFAULT_MEMORY_BUDGET = 512 * 2**20  # validate.py:37

_MODES = ("first", "all")
_BACKENDS = ("cuda", "parallel", "serial")
# The reference's engine names (solver.py:158-167: "jit" numba, "python" heap twin) select the
# enumerator it replaces; here every name runs the CUDA engine (the results are engine-independent
# in the reference too, test_solver.py:169-186).
_ENGINES = (None, "auto", "cuda", "jit", "python")


class SolveTimeout(Exception):
    """Raised when a time limit expires before a verdict is reached."""


@dataclass
class SolverConfig:
    """Solve knobs (reference solver.py:58-91).

    ``chunk_pairs``, ``pipeline_depth`` and ``worker_count`` are validated exactly as in the
    reference; on the GPU the join-wave planner replaces chunking and the thread pipeline, so they
    do not change results (the reference guarantees the same invariance).  ``device`` selects
    the CUDA ordinal.
    """

    mode: str = "first"
    reduce_rows: int = 1
    chunk_pairs: int | None = None
    backend: str = "cuda"
    pipeline_depth: int = 1
    worker_count: int = 0
    memory_budget_bytes: int = DEFAULT_MEMORY_BUDGET
    device: int = 0
    wave_keys: int = 0
    join: str = "auto"  # "auto" | "partitioned" | "global": join strategy of the CUDA engine

    def validated(self) -> "SolverConfig":
        if self.mode not in _MODES:
            raise ValueError(f"mode must be one of {_MODES}, got {self.mode!r}")
        if self.reduce_rows < 1:
            raise ValueError("reduce_rows must be >= 1")
        if self.chunk_pairs is not None and self.chunk_pairs < 1:
            raise ValueError("chunk_pairs must be >= 1")
        if self.pipeline_depth < 1:
            raise ValueError("pipeline_depth must be >= 1")
        if self.worker_count < 0:
            raise ValueError("worker_count must be >= 0")
        if self.memory_budget_bytes < 1:
            raise ValueError("memory_budget_bytes must be >= 1")
        if self.join not in ("auto", "partitioned", "global"):
            raise ValueError(f"unknown join {self.join!r}")
        if self.backend not in _BACKENDS:
            raise ValueError(f"unknown backend {self.backend!r}; choose from {sorted(_BACKENDS)}")
        return self


@dataclass
class SolveStats:
    batches: int = 0
    candidates_left: int = 0
    candidates_right: int = 0
    hash_hits: int = 0
    exact_hits: int = 0
    filtered_residuals: int = 0
    peak_table_entries: int = 0
    peak_heap1: int = 0
    peak_heap2: int = 0
    t_build: float = 0.0
    t_enumerate: float = 0.0
    t_validate: float = 0.0
    t_total: float = 0.0
    fallback: str = "none"
    engine: str = "none"
    # B200 additions (not in the reference schema's required keys)
    row1_candidate_pairs: int = 0
    waves: int = 0
    kernel_launches: int = 0
    cancelled_ranks: int = 0  # sharded first mode: ranks stopped early by another rank's solution
    dev_ms_total: float = 0.0
    t_init: float = 0.0  # one-time CUDA context/device init inside this solve (first call only)

    def as_dict(self) -> dict:
        return {
            "batches": self.batches,
            "candidates_left": self.candidates_left,
            "candidates_right": self.candidates_right,
            "hash_hits": self.hash_hits,
            "exact_hits": self.exact_hits,
            "filtered_residuals": self.filtered_residuals,
            "peak_table_entries": self.peak_table_entries,
            "peak_heap1": self.peak_heap1,
            "peak_heap2": self.peak_heap2,
            "t_build": round(self.t_build, 6),
            "t_enumerate": round(self.t_enumerate, 6),
            "t_validate": round(self.t_validate, 6),
            "t_total": round(self.t_total, 6),
            "fallback": self.fallback,
            "engine": self.engine,
        }


@dataclass
class SolveResult:
    verdict: str
    solutions: list[SolutionVector]
    stats: SolveStats

    @property
    def feasible(self) -> bool:
        return self.verdict == "feasible"


_FALLBACK = {0: "none", 1: "brute-force"}


def raise_for_status(rc: int, time_limit=None) -> None:
    """Map msp_status to the reference's exception types (include/msp_b200.h)."""
    if rc == _native.MSP_OK:
        return
    msg = _native.last_error()
    if rc == _native.MSP_TIMEOUT:
        raise SolveTimeout(f"time limit of {time_limit}s exceeded" if time_limit else msg)
    if rc in (_native.MSP_INVALID_ARGUMENT, _native.MSP_UNSUPPORTED):
        raise ValueError(msg)
    if rc == _native.MSP_INTERNAL and "alpha" in msg:
        raise AssertionError(msg)
    raise RuntimeError(f"CUDA solver failed ({rc}): {msg}")


def _check_verified(original: MspInstance, sols) -> None:  # solver.py:248-253
    for x in sols:
        if not verify_solution(original, x):
            raise RuntimeError("internal error: candidate failed original-system verification")


def native_solve(work: MspInstance, mode: str, time_limit: float | None, device: int = 0,
                 alpha_lo: int = 0, alpha_hi: int = 0, flags: int = 0, wave_keys: int = 0,
                 brute_force_max_n: int = BRUTE_FORCE_MAX_N, stream: int | None = None,
                 cancel: int | None = None):
    """One msp_solve call; returns (solution tuples, raw stats dict).

    ``cancel``: address of a shared int32 polled at wave checkpoints (cross-rank early exit).
    """
    opts = _native.make_options(mode=mode, device=device, time_limit=time_limit, alpha_lo=alpha_lo,
                                alpha_hi=alpha_hi, flags=flags, brute_force_max_n=brute_force_max_n,
                                wave_keys=wave_keys, stream=stream, cancel=cancel)
    rc, xb, st = _native.solve_raw(work.a, work.d, opts)
    raise_for_status(rc, time_limit)
    sols = [tuple(int(v) for v in row) for row in xb]
    return sols, st


def stats_from_native(st: dict, stats: SolveStats) -> None:
    for k in ("batches", "candidates_left", "candidates_right", "hash_hits", "exact_hits",
              "filtered_residuals", "peak_table_entries", "peak_heap1", "peak_heap2",
              "row1_candidate_pairs", "waves", "kernel_launches"):
        setattr(stats, k, int(st[k]))
    for k in ("t_build", "t_enumerate", "t_validate", "dev_ms_total", "t_init"):
        setattr(stats, k, float(st[k]))
    stats.fallback = _FALLBACK.get(int(st["fallback"]), "none")


def solve(
    inst: MspInstance,
    cfg: SolverConfig | None = None,
    time_limit: float | None = None,
    engine: str | None = None,
) -> SolveResult:
    """Solve an instance (reference solver.py:170-245) with the B200 engine."""
    cfg = (cfg or SolverConfig()).validated()
    if engine not in _ENGINES:
        raise ValueError(f"unknown enumerator engine {engine!r}")
    t_start = time.perf_counter()
    stats = SolveStats()
    work = inst
    if cfg.reduce_rows > 1:
        work = surrogate_reduce(inst, cfg.reduce_rows)

    if cfg.mode == "first" and not inst.d.any():  # solver.py:190-195
        zero = (0,) * inst.n
        assert verify_solution(inst, zero)
        stats.fallback = "zero-rhs"
        stats.t_total = time.perf_counter() - t_start
        return SolveResult("feasible", [zero], stats)

    if time_limit is not None and time_limit <= 0:
        raise SolveTimeout(f"time limit of {time_limit}s exceeded")
    flags = _native.MSP_FLAG_JOIN_GLOBAL if cfg.join == "global" else 0
    found, st = native_solve(work, cfg.mode, time_limit, device=cfg.device, wave_keys=cfg.wave_keys,
                             flags=flags)
    stats_from_native(st, stats)
    if stats.fallback == "none":
        stats.engine = "cuda"
    _check_verified(inst, found)
    if cfg.mode == "all":
        found.sort(key=solution_encoding)
        if len(set(found)) != len(found):
            raise RuntimeError("internal error: duplicate solutions emitted")
    elif found:
        found = sorted(found, key=solution_encoding)[:1]
    stats.t_total = time.perf_counter() - t_start
    if time_limit is not None and stats.t_total > time_limit:
        raise SolveTimeout(f"time limit of {time_limit}s exceeded")
    return SolveResult("feasible" if found else "infeasible", found, stats)
