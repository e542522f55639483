"""The C-ABI library loads and exports every entry point include/msp_b200.h declares (no GPU needed)."""

from __future__ import annotations

import ctypes as C
import os
import re

import pytest

from paper_2507_05045_b200 import _native

HEADER = os.path.join(_native.INCLUDE, "msp_b200.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_native.LIB_PATH):
        _native.build()
    return _native.load()


def declared_functions() -> list[str]:
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(msp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_entry_points():
    names = declared_functions()
    for n in ("msp_solve", "msp_result_free", "msp_build_tables", "msp_alpha_plan", "msp_join_alpha",
              "msp_last_error", "msp_release"):
        assert n in names
    assert set(names) == set(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_struct_mirrors_match_the_c_layout(lib):
    out = (C.c_int32 * 4)()
    lib.msp_abi_sizes(out)
    assert list(out) == [C.sizeof(_native.Problem), C.sizeof(_native.Options),
                         C.sizeof(_native.Stats), C.sizeof(_native.Result)]


def test_version(lib):
    assert lib.msp_version() == 1


def test_library_is_built_for_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_a_gpu(lib):
    import paper_2507_05045_b200 as msb

    inst = msb.generate_instance(4, 100, 11)
    with pytest.raises(RuntimeError, match="CUDA"):
        msb.solve(inst, msb.SolverConfig(mode="all"))


def test_integration_stub_structs_match_the_abi(lib):
    """The ctypes stub INTEGRATION.md tells a reference maintainer to paste matches the C layout."""
    import re as _re

    text = open(os.path.join(os.path.dirname(_native.INCLUDE), "INTEGRATION.md")).read()
    code = _re.search(r"```python\n(import ctypes as C.*?)\n_cuda = None", text, flags=_re.S).group(1)
    ns: dict = {}
    exec(code, ns)  # noqa: S102 -- the documented stub itself
    out = (C.c_int32 * 4)()
    lib.msp_abi_sizes(out)
    assert list(out) == [C.sizeof(ns["_Problem"]), C.sizeof(ns["_Options"]), C.sizeof(ns["_Stats"]),
                         C.sizeof(ns["_Result"])]
