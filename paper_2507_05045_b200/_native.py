"""ctypes binding of libmsp_b200.so (C-ABI declared in include/msp_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA device is visible, every
entry point raises ``NativeUnavailable`` instead of computing anything on the host.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_NAME = "libmsp_b200.so"
LIB_PATH = os.path.join(PKG_DIR, LIB_NAME)
CSRC = os.path.join(PKG_DIR, "csrc")
INCLUDE = os.path.join(REPO_DIR, "include")

MSP_OK, MSP_TIMEOUT, MSP_INVALID_ARGUMENT, MSP_CUDA_ERROR, MSP_INTERNAL, MSP_UNSUPPORTED = range(6)
MSP_MODE_FIRST, MSP_MODE_ALL = 0, 1
MSP_FLAG_PROFILE = 1 << 0
MSP_FLAG_FORCE_TABLE_PATH = 1 << 1
MSP_FLAG_JOIN_GLOBAL = 1 << 2
MSP_FLAG_DIAG_HASH_ONLY = 1 << 3
MSP_FLAG_WAVE_LAUNCHES = 1 << 4
MSP_FLAG_BATCH_STATS = 1 << 5
MSP_FLAG_DEGENERATE_HASH = 1 << 6

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--expt-relaxed-constexpr",
]

EXPORTED_SYMBOLS = (
    "msp_solve", "msp_result_free", "msp_build_tables", "msp_alpha_plan", "msp_join_alpha",
    "msp_release", "msp_last_error", "msp_version", "msp_int32_peak", "msp_abi_sizes",
)


class NativeUnavailable(RuntimeError):
    """The CUDA library could not be loaded or used; there is deliberately no fallback."""


def sources() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every kernel + the C-ABI into the in-tree shared library (sm_100a)."""
    srcs = sources()
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hdrs.append(os.path.join(INCLUDE, "msp_b200.h"))
    newest = max(os.path.getmtime(p) for p in srcs + hdrs)
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= newest:
        return LIB_PATH
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not os.path.exists(nvcc):
        nvcc = "nvcc"
    import tempfile
    from concurrent.futures import ThreadPoolExecutor

    tmp = LIB_PATH + ".tmp"
    with tempfile.TemporaryDirectory(prefix="msp_build_") as td:
        objs = [os.path.join(td, os.path.basename(f) + ".o") for f in srcs]
        cmds = [[nvcc, *NVCC_FLAGS, "-I", INCLUDE, "-I", CSRC, "-c", "-o", o, f] for f, o in zip(srcs, objs)]
        if verbose:
            for c in cmds:
                print(" ".join(c), file=sys.stderr)
        with ThreadPoolExecutor(max_workers=len(cmds)) as ex:  # one nvcc per translation unit
            for f in [ex.submit(subprocess.check_call, c) for c in cmds]:
                f.result()
        subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs])
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


class Problem(C.Structure):
    _fields_ = [("m", C.c_int32), ("n", C.c_int32),
                ("a", C.POINTER(C.c_uint64)), ("d", C.POINTER(C.c_uint64))]


class Options(C.Structure):
    _fields_ = [
        ("mode", C.c_int32),
        ("device", C.c_int32),
        ("time_limit_s", C.c_double),
        ("alpha_lo", C.c_uint64),
        ("alpha_hi", C.c_uint64),
        ("flags", C.c_uint32),
        ("brute_force_max_n", C.c_int32),
        ("wave_keys", C.c_uint64),
        ("stream", C.c_void_p),
        ("cancel", C.c_void_p),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("batches", C.c_int64), ("candidates_left", C.c_int64), ("candidates_right", C.c_int64),
        ("filtered_residuals", C.c_int64), ("hash_hits", C.c_int64), ("exact_hits", C.c_int64),
        ("row1_pairs_lo", C.c_uint64), ("row1_pairs_hi", C.c_uint64),
        ("peak_table_entries", C.c_int64), ("peak_heap1", C.c_int64), ("peak_heap2", C.c_int64),
        ("t_build", C.c_double), ("t_enumerate", C.c_double), ("t_validate", C.c_double),
        ("t_total", C.c_double),
        ("fallback", C.c_int32), ("waves", C.c_int32), ("kernel_launches", C.c_int64),
        ("dev_ms_total", C.c_double), ("dev_ms_tables", C.c_double), ("dev_ms_join", C.c_double),
        ("dev_ms_hot", C.c_double), ("hot_launches", C.c_int64), ("hot_pairs", C.c_int64),
        ("hot_bytes", C.c_int64),
        ("cancelled", C.c_int32), ("reserved", C.c_int32), ("t_init", C.c_double),
    ]


class Result(C.Structure):
    _fields_ = [("n_solutions", C.c_int64), ("n", C.c_int32),
                ("xbits", C.POINTER(C.c_uint8)), ("stats", Stats),
                ("n_batch_stats", C.c_int64), ("batch_stats", C.POINTER(C.c_int64))]


_lib = None


def load(path: str | None = None):
    """Load (never build) the library; raise NativeUnavailable when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("MSP_B200_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    try:
        L = C.CDLL(path)
    except OSError as exc:
        raise NativeUnavailable(f"cannot load {path}: {exc}") from exc
    L.msp_solve.restype = C.c_int
    L.msp_solve.argtypes = [C.POINTER(Problem), C.POINTER(Options), C.POINTER(Result)]
    L.msp_result_free.restype = None
    L.msp_result_free.argtypes = [C.POINTER(Result)]
    L.msp_join_alpha.restype = C.c_int
    L.msp_join_alpha.argtypes = [C.POINTER(Problem), C.POINTER(Options), C.c_uint64, C.POINTER(Result)]
    L.msp_alpha_plan.restype = C.c_int64
    L.msp_alpha_plan.argtypes = [C.POINTER(Problem), C.c_int32, C.c_int64] + [C.POINTER(C.c_uint64)] * 4
    L.msp_build_tables.restype = C.c_int
    L.msp_build_tables.argtypes = [C.POINTER(Problem), C.c_int32] + [C.POINTER(C.c_void_p)] * 4
    L.msp_release.restype = None
    L.msp_release.argtypes = [C.c_int32]
    L.msp_last_error.restype = C.c_char_p
    L.msp_last_error.argtypes = []
    L.msp_version.restype = C.c_int32
    L.msp_int32_peak.restype = C.c_double
    L.msp_int32_peak.argtypes = [C.c_int32]
    L.msp_abi_sizes.restype = None
    L.msp_abi_sizes.argtypes = [C.POINTER(C.c_int32)]
    _lib = L
    return L


def last_error() -> str:
    return (load().msp_last_error() or b"").decode("utf-8", "replace")


class _ProblemArrays:
    """Keeps the contiguous u64 arrays alive for the duration of a call."""

    def __init__(self, a, d):
        self.a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
        self.d = np.ascontiguousarray(np.asarray(d, dtype=np.uint64))
        m, n = self.a.shape
        self.prob = Problem(m, n, self.a.ctypes.data_as(C.POINTER(C.c_uint64)),
                            self.d.ctypes.data_as(C.POINTER(C.c_uint64)))


def make_options(mode: str = "all", device: int = 0, time_limit: float | None = None,
                 alpha_lo: int = 0, alpha_hi: int = 0, flags: int = 0, brute_force_max_n: int = -1,
                 wave_keys: int = 0, stream: int | None = None, cancel: int | None = None) -> Options:
    """``cancel``: address of a shared int32 (CancelFlag.address) polled at wave checkpoints."""
    return Options(MSP_MODE_ALL if mode == "all" else MSP_MODE_FIRST, device,
                   float(time_limit) if time_limit else 0.0, alpha_lo, alpha_hi, flags,
                   brute_force_max_n, wave_keys, stream or None, cancel or None)


def solve_raw(a, d, opts: Options, alpha: int | None = None):
    """Call msp_solve (or msp_join_alpha); returns (status, xbits ndarray, stats dict)."""
    L = load()
    pa = _ProblemArrays(a, d)
    res = Result()
    if alpha is None:
        rc = L.msp_solve(C.byref(pa.prob), C.byref(opts), C.byref(res))
    else:
        rc = L.msp_join_alpha(C.byref(pa.prob), C.byref(opts), alpha, C.byref(res))
    try:
        n = pa.a.shape[1]
        ns = res.n_solutions if rc == MSP_OK else 0
        xb = (np.ctypeslib.as_array(res.xbits, shape=(ns * n,)).reshape(ns, n).copy()
              if ns else np.zeros((0, n), np.uint8))
        st = {name: getattr(res.stats, name) for name, _ in Stats._fields_}
        st["row1_candidate_pairs"] = (st.pop("row1_pairs_hi") << 64) | st.pop("row1_pairs_lo")
        nb = res.n_batch_stats if rc == MSP_OK else 0
        if nb:  # (alpha, n_left, n_right, filtered_residuals, hash_hits) per batch
            st["batch_stats"] = [tuple(int(v) for v in row) for row in
                                 np.ctypeslib.as_array(res.batch_stats, shape=(nb * 5,)).reshape(nb, 5)]
    finally:
        L.msp_result_free(C.byref(res))
    return rc, xb, st


def alpha_plan(a, d, device: int = 0):
    """Batch headers (alpha, beta, n_left, n_right) in alpha order, from the device plan."""
    L = load()
    pa = _ProblemArrays(a, d)
    cap = 1 << 16
    while True:
        bufs = [np.zeros(cap, np.uint64) for _ in range(4)]
        ptrs = [b.ctypes.data_as(C.POINTER(C.c_uint64)) for b in bufs]
        nb = L.msp_alpha_plan(C.byref(pa.prob), device, cap, *ptrs)
        if nb < 0:
            raise RuntimeError(f"msp_alpha_plan failed ({-nb}): {last_error()}")
        if nb <= cap:
            break
        cap = nb  # msp_alpha_plan returns the true count: retry with room for every batch
    cols = [b[:nb].tolist() for b in bufs]
    return list(zip(*cols))


def build_tables(a, d, device: int = 0):
    """Device-built quarter tables in the reference format (weights, masks, contribs, run_end)."""
    L = load()
    pa = _ProblemArrays(a, d)
    m, n = pa.a.shape
    q, r = divmod(n, 4)
    sizes = [1 << (q + 1 if i < r else q) for i in range(4)]
    outs = [dict(weights=np.zeros(s, np.uint64), masks=np.zeros(s, np.uint32),
                 contribs=np.zeros((s, m), np.uint64), run_end=np.zeros(s, np.int64)) for s in sizes]
    arr = lambda k: (C.c_void_p * 4)(*[o[k].ctypes.data for o in outs])  # noqa: E731
    rc = L.msp_build_tables(C.byref(pa.prob), device, arr("weights"), arr("masks"), arr("contribs"),
                            arr("run_end"))
    if rc:
        raise RuntimeError(f"msp_build_tables failed ({rc}): {last_error()}")
    return outs
