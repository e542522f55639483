"""Shared fixtures: golden-fixture loading, seeded instances, GPU marker."""

from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

from paper_2507_05045_b200.instances import MspInstance, SplitMix64  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libmsp_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_golden(name: str):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    with open(path) as fh:
        return json.load(fh)


def inst_from(rec) -> MspInstance:
    return MspInstance(rec["a"], rec["d"])


def seeded_instance(seed: int, m: int, n: int, k: int, d_mode: str = "half") -> MspInstance:
    """Same construction as the reference tests' helper (pkg/tests/conftest.py:10-26)."""
    rng = SplitMix64(seed)
    rows = [[rng.below(k) for _ in range(n)] for _ in range(m)]
    if d_mode == "half":
        d = [sum(r) // 2 for r in rows]
    else:
        d = [rng.below(sum(r) + 1) for r in rows]
    return MspInstance(rows, d, k_bound=k)


STAT_KEYS = ("batches", "candidates_left", "candidates_right", "hash_hits", "exact_hits",
             "filtered_residuals", "peak_table_entries", "peak_heap1", "peak_heap2")
