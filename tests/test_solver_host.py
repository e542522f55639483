"""Host logic of the drop-in solve(): config validation and error mapping (pkg/tests/test_solver.py)."""

from __future__ import annotations

import pytest

import paper_2507_05045_b200 as msb
from paper_2507_05045_b200 import _native
from paper_2507_05045_b200.solver import raise_for_status


def test_config_validation():
    inst = msb.MspInstance([[1, 1, 1, 1]], [2])
    for bad in (dict(mode="some"), dict(pipeline_depth=0), dict(chunk_pairs=0), dict(backend="gpu"),
                dict(reduce_rows=0), dict(worker_count=-1), dict(memory_budget_bytes=0)):
        with pytest.raises(ValueError):
            msb.solve(inst, msb.SolverConfig(**bad))


def test_unknown_engine_rejected():
    with pytest.raises(ValueError):
        msb.solve(msb.MspInstance([[1, 2, 3, 4]], [5]), msb.SolverConfig(mode="all"), engine="numba-gpu")


def test_reduce_rows_out_of_range():
    with pytest.raises(ValueError, match="r out of range"):
        msb.solve(msb.MspInstance([[1, 2, 3, 4]], [5]), msb.SolverConfig(reduce_rows=2))


def test_zero_rhs_first_mode_needs_no_device():
    inst = msb.MspInstance([[3, 1, 4, 1, 5, 9, 2, 6]] * 2, [0, 0])
    res = msb.solve(inst, msb.SolverConfig(mode="first"))
    assert res.feasible and res.solutions == [(0,) * 8]
    assert res.stats.fallback == "zero-rhs"


def test_nonpositive_time_limit_times_out():
    with pytest.raises(msb.SolveTimeout):
        msb.solve(msb.generate_instance(4, 100, 1), msb.SolverConfig(mode="all"), time_limit=0)


def test_status_mapping(monkeypatch):
    monkeypatch.setattr(_native, "last_error", lambda: "boom alpha")
    raise_for_status(_native.MSP_OK)
    with pytest.raises(msb.SolveTimeout):
        raise_for_status(_native.MSP_TIMEOUT, 1.0)
    with pytest.raises(ValueError):
        raise_for_status(_native.MSP_INVALID_ARGUMENT)
    with pytest.raises(ValueError):
        raise_for_status(_native.MSP_UNSUPPORTED)
    with pytest.raises(AssertionError):
        raise_for_status(_native.MSP_INTERNAL)
    with pytest.raises(RuntimeError):
        raise_for_status(_native.MSP_CUDA_ERROR)


def test_stats_schema_matches_reference():
    keys = set(msb.SolveStats().as_dict())
    assert keys == {"batches", "candidates_left", "candidates_right", "hash_hits", "exact_hits",
                    "filtered_residuals", "peak_table_entries", "peak_heap1", "peak_heap2", "t_build",
                    "t_enumerate", "t_validate", "t_total", "fallback", "engine"}
