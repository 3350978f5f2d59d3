"""The C-ABI boundary on a CPU-only machine: the in-tree library loads, exports
every function include/tcfft_b200.h declares, and its host-only entry points
(planning, introspection, error strings) behave like the reference's plan
validation (reference plan.py:22-32,105-113).  No compute calls."""

import ctypes
import json
import re
from pathlib import Path

import pytest

from paper_2104_11471_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "tcfft_b200.h"

SUCCESS, INVALID_PLAN, INVALID_VALUE, INVALID_SIZE, NOT_SUPPORTED, NO_DEVICE = 0, 1, 3, 4, 6, 7


def _declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(tcfft[A-Za-z0-9_]+)\s*\(", text)))


def test_header_declares_the_reference_surface():
    names = _declared()
    for n in ("tcfftPlan1D", "tcfftPlan2D", "tcfftExecC2C", "tcfftDestroy"):
        assert n in names


def test_library_exports_every_declared_symbol():
    L = _lib.load(build_if_missing=False)
    missing = [n for n in _declared() if not hasattr(L, n)]
    assert not missing, missing
    assert set(_lib.EXPORTS) <= set(_declared())


def _describe(dims, nx, ny, batch):
    L = _lib.load(build_if_missing=False)
    buf = ctypes.create_string_buffer(1 << 16)
    st = L.tcfftDescribePlan(dims, nx, ny, batch, buf, len(buf))
    return st, (json.loads(buf.value.decode()) if st == SUCCESS else None)


@pytest.mark.parametrize("n", [2, 4, 8, 16, 256, 4096, 16384, 1 << 15, 1 << 18, 1 << 19, 1 << 22, 1 << 24, 1 << 25,
                               1 << 27, 1 << 30])
def test_describe_1d_passes(n):
    st, d = _describe(1, n, 0, 8 if n <= 1 << 24 else 1)
    assert st == SUCCESS
    want = 1 if n <= 16384 else (2 if n <= 1 << 22 else 3)  # 2^19..2^22: blocked two-pass
    assert len(d["passes"]) == want
    for p in d["passes"]:
        assert p["kernel"] == 1, p  # an sm_100a instantiation exists for every pass
        assert p["E"] % p["N"] == 0 or p["kind"] != "row"
        assert 1 <= p["ctas_per_sm"] <= 4 and p["nwg"] in (1, 2)
        assert p["tmem_cols"] in (32, 64, 128, 256, 512)
        assert p["smem_bytes"] * p["ctas_per_sm"] <= 233472


@pytest.mark.parametrize("nx,ny", [(2, 2), (512, 512), (4096, 4096), (8, 1024)])
def test_describe_2d_passes(nx, ny):
    st, d = _describe(2, nx, ny, 4)
    assert st == SUCCESS and len(d["passes"]) == 2
    assert d["passes"][0]["kind"] == "row" and d["passes"][1]["kind"] == "strip"
    assert all(p["kernel"] == 1 for p in d["passes"])


@pytest.mark.parametrize("nx,ny,kinds", [(8192, 16, ["row", "strip", "strip"]),
                                         (1 << 20, 16, ["row", "strip", "strip"]),
                                         (64, 32768, ["strip", "rowT", "strip"]),
                                         (4, 1 << 20, ["strip", "rowTB", "strip"]),
                                         (16384, 32768, ["strip", "rowT", "strip", "strip"])])
def test_describe_2d_large_sizes(nx, ny, kinds):
    """Sizes beyond one chunk per column / row (the reference accepts every
    power of two, plan.py:125-138): split column passes and multi-pass rows."""
    st, d = _describe(2, nx, ny, 1)
    assert st == SUCCESS
    assert [p["kind"] for p in d["passes"]] == kinds
    assert all(p["kernel"] == 1 for p in d["passes"])
    assert d["ws_bytes"] >= nx * ny * 4


@pytest.mark.parametrize("args,code", [((1, 3, 0, 1), INVALID_SIZE), ((1, 0, 0, 1), INVALID_SIZE),
                                       ((1, 1, 0, 1), INVALID_SIZE), ((2, 8, 6, 1), INVALID_SIZE),
                                       ((1, 256, 0, 0), INVALID_VALUE), ((1, 1 << 31, 0, 1), INVALID_SIZE),
                                       ((2, 8192, 8, 1), NOT_SUPPORTED), ((2, 1 << 21, 16, 1), NOT_SUPPORTED)])
def test_describe_rejects_like_the_reference(args, code):
    st, _ = _describe(*args)
    assert st == code


def test_plan_without_device_fails_cleanly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = _lib.load(build_if_missing=False)
    h = ctypes.c_void_p()
    assert L.tcfftPlan1D(ctypes.byref(h), 256, 4) == NO_DEVICE
    assert L.tcfftPlan1D(ctypes.byref(h), 3, 4) == INVALID_SIZE  # validation precedes device lookup
    assert L.tcfftExecC2C(None, None, None) == INVALID_PLAN
    assert L.tcfftDestroy(None) == INVALID_PLAN
    assert L.tcfftSetPassMask(None, 1) == INVALID_PLAN


def test_error_strings_and_version():
    L = _lib.load(build_if_missing=False)
    for code in range(8):
        assert _lib.error_string(code)
    assert L.tcfftGetVersion() > 0


def test_python_mirror_raises_reference_exceptions():
    import paper_2104_11471_b200 as tc

    with pytest.raises(tc.UnsupportedSizeError):
        tc.plan_1d(3, 1)
    with pytest.raises(tc.PlanArgumentError):
        tc.plan_1d(256, 0)
    with pytest.raises(tc.PlanArgumentError):
        tc.plan_1d(256, 1, continuous_size=7)
    with pytest.raises(tc.PlanArgumentError):
        tc.plan_2d(256, 256, 1, precision="single")
