"""ctypes wrapper for the CPU oracle (liboracle.so, built from msp_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() (as the checker) and
bench.py's reference / cpu_baseline legs.  The product package never imports this module.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")


def build(force: bool = False) -> str:
    srcs = [os.path.join(HERE, f) for f in ("msp_oracle.c", "msp_oracle_groups.cc", "Makefile")]
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(map(os.path.getmtime, srcs)):
        subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB_PATH


class Options(C.Structure):
    _fields_ = [
        ("mode", C.c_int32),
        ("workers", C.c_int32),
        ("chunk_pairs", C.c_int64),
        ("bucket_bits_cap", C.c_int32),
        ("record_batches", C.c_int32),
        ("alpha_lo", C.c_uint64),
        ("alpha_hi", C.c_uint64),
        ("row", C.c_int32),
        ("brute_force_max_n", C.c_int32),
    ]


class Result(C.Structure):
    _fields_ = [
        ("batches", C.c_int64),
        ("candidates_left", C.c_int64),
        ("candidates_right", C.c_int64),
        ("filtered_residuals", C.c_int64),
        ("hash_hits", C.c_int64),
        ("exact_hits", C.c_int64),
        ("row1_pairs_lo", C.c_uint64),
        ("row1_pairs_hi", C.c_uint64),
        ("peak_table_entries", C.c_int64),
        ("peak_heap1", C.c_int64),
        ("peak_heap2", C.c_int64),
        ("t_build", C.c_double),
        ("t_enumerate", C.c_double),
        ("t_validate", C.c_double),
        ("t_total", C.c_double),
        ("fallback", C.c_int32),
        ("threads_used", C.c_int32),
        ("n_solutions", C.c_int64),
        ("xbits", C.POINTER(C.c_uint8)),
        ("n_batch_records", C.c_int64),
        ("batch_records", C.POINTER(C.c_int64)),
    ]


class GroupResult(C.Structure):
    _fields_ = [
        ("n_left", C.c_int64), ("n_right", C.c_int64), ("filtered", C.c_int64),
        ("hash_hits", C.c_int64), ("exact_hits", C.c_int64), ("passes", C.c_int64),
        ("n_hit_keys", C.c_int64), ("hit_keys", C.POINTER(C.c_uint64)),
        ("n_solutions", C.c_int64), ("xbits", C.POINTER(C.c_uint8)),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        L.oracle_splitmix64_next.restype = C.c_uint64
        L.oracle_splitmix64_next.argtypes = [C.POINTER(C.c_uint64)]
        L.oracle_splitmix64_below.restype = C.c_uint64
        L.oracle_splitmix64_below.argtypes = [C.POINTER(C.c_uint64), C.c_uint64]
        L.oracle_fnv_fold.restype = C.c_uint64
        L.oracle_fnv_fold.argtypes = [C.POINTER(C.c_uint64), C.c_int]
        L.oracle_block_sizes.argtypes = [C.c_int, C.POINTER(C.c_int32)]
        L.oracle_build_tables.restype = C.c_int
        L.oracle_build_tables.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_uint64), C.c_int,
                                          C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                          C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
        L.oracle_solve.restype = C.c_int
        L.oracle_solve.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                   C.POINTER(Options), C.POINTER(Result)]
        L.oracle_result_free.argtypes = [C.POINTER(Result)]
        L.oracle_stream.restype = C.c_int64
        L.oracle_stream.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                    C.c_int64, C.POINTER(C.c_int64), C.c_int64, C.POINTER(C.c_int64)]
        L.oracle_alpha_group.restype = C.c_int
        L.oracle_alpha_group.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                         C.c_uint64, C.c_int, C.c_int, C.POINTER(GroupResult)]
        L.oracle_group_result_free.argtypes = [C.POINTER(GroupResult)]
        L.oracle_groups_open.restype = C.c_void_p
        L.oracle_groups_open.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.oracle_groups_close.argtypes = [C.c_void_p]
        L.oracle_groups_run.restype = C.c_int
        L.oracle_groups_run.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_int, C.POINTER(GroupResult)]
        _lib = L
    return _lib


def _u64(arr) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(arr, dtype=np.uint64))


def _ptr(a: np.ndarray, ty=C.c_uint64):
    return a.ctypes.data_as(C.POINTER(ty))


def fnv_fold(vec) -> int:
    v = _u64(vec)
    return int(lib().oracle_fnv_fold(_ptr(v), len(v)))


def splitmix64(seed: int, count: int) -> list[int]:
    st = C.c_uint64(seed)
    return [int(lib().oracle_splitmix64_next(C.byref(st))) for _ in range(count)]


def splitmix64_below(seed: int, k: int, count: int) -> list[int]:
    st = C.c_uint64(seed)
    return [int(lib().oracle_splitmix64_below(C.byref(st), k)) for _ in range(count)]


def block_sizes(n: int) -> list[int]:
    out = (C.c_int32 * 4)()
    lib().oracle_block_sizes(n, out)
    return list(out)


def build_tables(a, row: int = 0):
    """Reference-order quarter tables: list of dicts(weights, masks, contribs, run_end)."""
    a = _u64(a)
    m, n = a.shape
    sizes = [1 << b for b in block_sizes(n)]
    outs = [dict(weights=np.zeros(s, np.uint64), masks=np.zeros(s, np.uint64),
                 contribs=np.zeros((s, m), np.uint64), run_end=np.zeros(s, np.int64)) for s in sizes]
    arr = lambda key: (C.c_void_p * 4)(*[o[key].ctypes.data for o in outs])  # noqa: E731
    rc = lib().oracle_build_tables(m, n, _ptr(a), row, arr("weights"), arr("masks"),
                                   arr("contribs"), arr("run_end"))
    if rc:
        raise ValueError("oracle_build_tables failed")
    return outs


@dataclass
class OracleSolve:
    solutions: list[tuple[int, ...]]
    stats: dict
    batch_records: np.ndarray = field(default_factory=lambda: np.zeros((0, 7), np.int64))
    status: int = 0


def solve(a, d, mode: str = "all", workers: int = 0, chunk_pairs: int = 0, bucket_bits_cap: int = 0,
          record_batches: bool = False, alpha_lo: int = 0, alpha_hi: int = 0, row: int = 0,
          brute_force_max_n: int = -1) -> OracleSolve:
    a = _u64(a)
    d = _u64(d)
    m, n = a.shape
    opt = Options(mode=1 if mode == "all" else 0, workers=workers, chunk_pairs=chunk_pairs,
                  bucket_bits_cap=bucket_bits_cap, record_batches=int(record_batches),
                  alpha_lo=alpha_lo, alpha_hi=alpha_hi, row=row, brute_force_max_n=brute_force_max_n)
    res = Result()
    rc = lib().oracle_solve(m, n, _ptr(a), _ptr(d), C.byref(opt), C.byref(res))
    try:
        ns = res.n_solutions
        xb = np.ctypeslib.as_array(res.xbits, shape=(ns * n,)).reshape(ns, n).copy() if ns else np.zeros((0, n), np.uint8)
        nb = res.n_batch_records
        br = (np.ctypeslib.as_array(res.batch_records, shape=(nb * 7,)).reshape(nb, 7).copy()
              if nb else np.zeros((0, 7), np.int64))
        stats = {k: getattr(res, k) for k in (
            "batches", "candidates_left", "candidates_right", "hash_hits", "exact_hits",
            "filtered_residuals", "peak_table_entries", "peak_heap1", "peak_heap2",
            "t_build", "t_enumerate", "t_validate", "t_total", "threads_used")}
        stats["row1_candidate_pairs"] = (res.row1_pairs_hi << 64) | res.row1_pairs_lo
        stats["fallback"] = {0: "none", 1: "brute-force", 2: "zero-rhs"}[res.fallback]
    finally:
        lib().oracle_result_free(C.byref(res))
    sols = sorted({tuple(int(v) for v in row) for row in xb},
                  key=lambda x: int("".join(map(str, x)) or "0", 2))
    if len(sols) != len(xb):
        raise RuntimeError("oracle emitted duplicate solutions")
    if br.size:
        br = br[np.argsort(br[:, 6], kind="stable")]
    return OracleSolve(solutions=sols, stats=stats, batch_records=br, status=rc)


def stream(a, d):
    """Reference batch stream: list of (alpha, beta, left_pairs, right_pairs)."""
    a = _u64(a)
    d = _u64(d)
    m, n = a.shape
    maxb, maxp = 1 << 16, 1 << 22
    hdr = np.zeros((maxb, 4), np.int64)
    pairs = np.zeros((maxp, 2), np.int64)
    nb = lib().oracle_stream(m, n, _ptr(a), _ptr(d), maxb, _ptr(hdr, C.c_int64), maxp, _ptr(pairs, C.c_int64))
    if nb < 0:
        raise ValueError("stream too large for oracle_stream buffers")
    out, pos = [], 0
    for al, be, nl, nr in hdr[:nb].tolist():
        lp = pairs[pos:pos + nl].tolist(); pos += nl
        rp = pairs[pos:pos + nr].tolist(); pos += nr
        out.append((al, be, lp, rp))
    return out


def stream_headers(a, d):
    """Batch headers (alpha, beta, n_left, n_right) of the reference stream, without the pairs."""
    a = _u64(a)
    d = _u64(d)
    m, n = a.shape
    maxb = 1 << 20
    hdr = np.zeros((maxb, 4), np.int64)
    nb = lib().oracle_stream(m, n, _ptr(a), _ptr(d), maxb, _ptr(hdr, C.c_int64), 0, None)
    nb = nb if nb >= 0 else -nb - 1  # (max_pairs 0: the count comes back encoded as -nb - 1)
    if nb > maxb:
        raise ValueError("too many batches for stream_headers")
    return [tuple(int(v) for v in row) for row in hdr[:nb].tolist()]


def _group_dict(res: GroupResult, n: int) -> dict:
    ns = res.n_solutions
    xb = np.ctypeslib.as_array(res.xbits, shape=(ns * n,)).reshape(ns, n).copy() if ns else np.zeros((0, n), np.uint8)
    keys = (np.ctypeslib.as_array(res.hit_keys, shape=(res.n_hit_keys,)).tolist() if res.n_hit_keys else [])
    out = {k: int(getattr(res, k)) for k in ("n_left", "n_right", "filtered", "hash_hits", "exact_hits", "passes")}
    out["hit_keys"] = [int(k) for k in keys]
    out["solutions"] = sorted("".join(str(int(v)) for v in row) for row in xb)
    return out


def alpha_group(a, d, alpha: int, threads: int = 0, passes: int = 0) -> dict:
    """One alpha-group (batch) of the instance through the streaming CPU restatement
    (msp_oracle_groups.cc): validate_chunked's per-batch counters + solutions, for batches too big
    to materialise.  Keys: n_left, n_right, filtered, hash_hits, exact_hits, hit_keys, solutions."""
    a = _u64(a)
    d = _u64(d)
    m, n = a.shape
    res = GroupResult()
    rc = lib().oracle_alpha_group(m, n, _ptr(a), _ptr(d), alpha, threads, passes, C.byref(res))
    try:
        if rc:
            raise ValueError("oracle_alpha_group failed")
        return _group_dict(res, n)
    finally:
        lib().oracle_group_result_free(C.byref(res))


class AlphaGroups:
    """An instance's quarter tables built once for many alpha-group runs (msp_oracle_groups.cc).
    run(alpha, method=1) is the filter join, method=0 the hash-range sort-merge of alpha_group();
    both compute validate_chunked's per-batch counters exactly."""

    def __init__(self, a, d):
        self.a, self.d = _u64(a), _u64(d)
        self.m, self.n = self.a.shape
        self.h = lib().oracle_groups_open(self.m, self.n, _ptr(self.a), _ptr(self.d))
        if not self.h:
            raise ValueError("oracle_groups_open failed")

    def run(self, alpha: int, method: int = 1, threads: int = 0, passes: int = 0) -> dict:
        res = GroupResult()
        rc = lib().oracle_groups_run(self.h, alpha, threads, method, passes, C.byref(res))
        try:
            if rc:
                raise ValueError("oracle_groups_run failed")
            return _group_dict(res, self.n)
        finally:
            lib().oracle_group_result_free(C.byref(res))

    def close(self):
        if self.h:
            lib().oracle_groups_close(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
