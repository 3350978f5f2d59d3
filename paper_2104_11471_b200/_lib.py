"""ctypes binding of the C ABI in include/tcfft_b200.h.

The shared library is built in-tree (``paper_2104_11471_b200/libtcfft_b200.so``,
see build.py).  There is no fallback: if the library cannot be loaded the
import of the execution path fails loudly.
"""

from __future__ import annotations

import ctypes
import json
import os
from pathlib import Path

_LIB_PATH = Path(os.environ.get("TCFFT_LIB") or (Path(__file__).resolve().parent / "libtcfft_b200.so"))
_lib = None

TCFFT_SUCCESS = 0
TCFFT_INVALID_PLAN = 1
TCFFT_ALLOC_FAILED = 2
TCFFT_INVALID_VALUE = 3
TCFFT_INVALID_SIZE = 4
TCFFT_EXEC_FAILED = 5
TCFFT_NOT_SUPPORTED = 6
TCFFT_NO_DEVICE = 7

# every symbol include/tcfft_b200.h declares
EXPORTS = (
    "tcfftPlan1D", "tcfftPlan2D", "tcfftSetStream", "tcfftGetWorkspaceSize", "tcfftExecC2C", "tcfftExecC2CHost",
    "tcfftExecC2CStrided",
    "tcfftDestroy", "tcfftGetErrorString", "tcfftGetVersion", "tcfftDescribePlan", "tcfftPlanTables",
    "tcfftSetPassMask", "tcfftPlan1DDist", "tcfftExecDistPass", "tcfftDistUnpack", "tcfftDescribeDistPlan",
    "tcfftDistPlanTables", "tcfftPlan1DDistFused", "tcfftDistSetPeers", "tcfftIpcGetHandle", "tcfftIpcOpenHandle",
    "tcfftIpcCloseHandle", "tcfftDescribeDistPlanFused", "tcfftDistPlanTablesFused",
)


def lib_path() -> Path:
    return _LIB_PATH


def load(build_if_missing: bool = True):
    """Load (building first if needed) the sm_100a extension."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists() and build_if_missing and os.environ.get("TCFFT_NO_BUILD") != "1":
        from . import build as _build

        _build.build()
    if not _LIB_PATH.exists():
        raise ImportError(f"tcfft B200 extension not built: {_LIB_PATH} missing (run python -m "
                          "paper_2104_11471_b200.build)")
    L = ctypes.CDLL(str(_LIB_PATH))
    vp, ci, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    L.tcfftPlan1D.argtypes = [ctypes.POINTER(vp), ci, ci]
    L.tcfftPlan2D.argtypes = [ctypes.POINTER(vp), ci, ci, ci]
    L.tcfftSetStream.argtypes = [vp, vp]
    L.tcfftGetWorkspaceSize.argtypes = [vp, ctypes.POINTER(sz)]
    L.tcfftExecC2C.argtypes = [vp, vp, vp]
    L.tcfftSetPassMask.argtypes = [vp, ctypes.c_uint]
    if hasattr(L, "tcfftExecC2CStrided"):
        L.tcfftExecC2CStrided.argtypes = [vp, vp, vp, ctypes.c_longlong, ctypes.c_longlong]
    if hasattr(L, "tcfftExecC2CHost"):
        L.tcfftExecC2CHost.argtypes = [vp, vp, vp]
    L.tcfftDestroy.argtypes = [vp]
    L.tcfftGetErrorString.argtypes = [ci]
    L.tcfftGetErrorString.restype = ctypes.c_char_p
    L.tcfftGetVersion.argtypes = []
    L.tcfftDescribePlan.argtypes = [ci, ci, ci, ci, ctypes.c_char_p, sz]
    L.tcfftPlanTables.argtypes = [ci, ci, ci, ci, ci, vp, ctypes.POINTER(sz), vp, ctypes.POINTER(sz), vp,
                                  ctypes.POINTER(sz)]
    L.tcfftPlan1DDist.argtypes = [ctypes.POINTER(vp), ci, ci, ci]
    L.tcfftExecDistPass.argtypes = [vp, ci, vp, vp]
    L.tcfftDistUnpack.argtypes = [vp, ci, vp, vp]
    L.tcfftDescribeDistPlan.argtypes = [ci, ci, ci, ctypes.c_char_p, sz]
    L.tcfftDistPlanTables.argtypes = [ci, ci, ci, ci, vp, ctypes.POINTER(sz), vp, ctypes.POINTER(sz), vp,
                                      ctypes.POINTER(sz)]
    L.tcfftPlan1DDistFused.argtypes = [ctypes.POINTER(vp), ci, ci, ci]
    L.tcfftDistSetPeers.argtypes = [vp, ctypes.POINTER(vp), ci]
    L.tcfftIpcGetHandle.argtypes = [vp, vp, sz]
    L.tcfftIpcOpenHandle.argtypes = [vp, ctypes.POINTER(vp)]
    L.tcfftIpcCloseHandle.argtypes = [vp]
    L.tcfftDescribeDistPlanFused.argtypes = [ci, ci, ci, ctypes.c_char_p, sz]
    L.tcfftDistPlanTablesFused.argtypes = [ci, ci, ci, ci, vp, ctypes.POINTER(sz), vp, ctypes.POINTER(sz), vp,
                                           ctypes.POINTER(sz)]
    for name in EXPORTS:
        if name not in ("tcfftGetErrorString",) and hasattr(L, name):
            getattr(L, name).restype = ci
    _lib = L
    return L


def error_string(code: int) -> str:
    return load().tcfftGetErrorString(code).decode()


def describe(dims: int, nx: int, ny: int, batch: int) -> dict:
    L = load()
    buf = ctypes.create_string_buffer(1 << 16)
    L.tcfftDescribePlan(dims, nx, ny, batch, buf, len(buf))
    return json.loads(buf.value.decode())


def _tables(call):
    rb, bb, tb = ctypes.c_size_t(0), ctypes.c_size_t(0), ctypes.c_size_t(0)
    st = call(None, ctypes.byref(rb), None, ctypes.byref(bb), None, ctypes.byref(tb))
    if st != TCFFT_SUCCESS:
        raise RuntimeError(error_string(st))
    r = ctypes.create_string_buffer(rb.value)
    b = ctypes.create_string_buffer(bb.value)
    t = ctypes.create_string_buffer(max(tb.value, 1))
    call(r, ctypes.byref(rb), b, ctypes.byref(bb), t, ctypes.byref(tb))
    return r.raw, b.raw, t.raw[: tb.value]


def plan_tables(dims: int, nx: int, ny: int, batch: int, pass_index: int):
    """Host tables of one pass as raw bytes: (rows, bmats, twiddles)."""
    L = load()
    return _tables(lambda *a: L.tcfftPlanTables(dims, nx, ny, batch, pass_index, *a))


def describe_dist(nx: int, rank: int, world: int, fused: bool = False) -> dict:
    """The distributed single-transform plan of one rank (tcfftDescribeDistPlan[Fused])."""
    L = load()
    buf = ctypes.create_string_buffer(1 << 16)
    (L.tcfftDescribeDistPlanFused if fused else L.tcfftDescribeDistPlan)(nx, rank, world, buf, len(buf))
    return json.loads(buf.value.decode())


def dist_plan_tables(nx: int, rank: int, world: int, pass_index: int, fused: bool = False):
    L = load()
    f = L.tcfftDistPlanTablesFused if fused else L.tcfftDistPlanTables
    return _tables(lambda *a: f(nx, rank, world, pass_index, *a))
