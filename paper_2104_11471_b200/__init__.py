"""B200-native tcFFT: batched FP16 complex-to-complex forward FFT on sm_100a.

Python host mirror of the reference package's plan/execute surface
(reference ``pkg/src/tcfft/__init__.py:8-49``, ``plan.py``, ``executor.py``)
over the C ABI in ``include/tcfft_b200.h``.  Data lives in torch CUDA tensors
(interleaved fp16 pairs: ``torch.complex32`` or ``float16[..., 2]``); torch is
only the device-memory / stream plumbing, every transform runs in the
hand-written sm_100a kernels of ``libtcfft_b200.so``.

    plan = plan_1d(4096, batch=16384)
    execute(plan, x)            # in place, natural order, like the reference
    y = execute(plan, x, out=y) # out of place
"""

from __future__ import annotations

import ctypes
import json
import math
import threading
from dataclasses import dataclass, field
from functools import reduce

import numpy as np

from . import _lib

__version__ = "0.1.0"

KERNEL_CATALOG = tuple(2 ** k for k in range(1, 14))  # reference kernels.py:27
VALID_CONT_SIZES = (4, 8, 16, 32, 64)                 # reference kernels.py:29
MAX_KERNEL_RADIX = 8192                               # reference plan.py:18


class UnsupportedSizeError(ValueError):
    """Transform size is not a power of two >= 2 (reference plan.py:22)."""


class PlanArgumentError(ValueError):
    """Bad batch / continuous_size / precision (reference plan.py:26)."""


class ExecuteError(ValueError):
    """Data does not match the plan, or the device execution failed
    (reference executor.py:21)."""


def _check_pow2(n: int, what: str) -> None:
    if not isinstance(n, int) or n < 2 or n & (n - 1):
        raise UnsupportedSizeError(f"{what} must be a power of two >= 2, got {n}")


def schedule_radices(n: int) -> tuple:
    """The reference's greedy kernel schedule (plan.py:35-44), kept for plan
    JSON / API compatibility.  The B200 pass decomposition is chosen
    separately (``Plan.passes``); results need not be bit-identical across
    schedules."""
    _check_pow2(n, "transform length")
    out, rem = [], n
    while rem > MAX_KERNEL_RADIX:
        out.append(MAX_KERNEL_RADIX)
        rem //= MAX_KERNEL_RADIX
    out.append(rem)
    return tuple(out)


def _validate_schedule(schedule, n: int) -> tuple:
    schedule = tuple(int(r) for r in schedule)
    for r in schedule:
        if r not in KERNEL_CATALOG:
            raise UnsupportedSizeError(f"radix {r} not in the kernel catalog")
    if reduce(lambda a, b: a * b, schedule, 1) != n:
        raise UnsupportedSizeError(f"schedule {schedule} does not multiply to {n}")
    return schedule


def _common_checks(batch, continuous_size, precision):
    if not isinstance(batch, int) or batch < 1:
        raise PlanArgumentError(f"batch must be >= 1, got {batch}")
    if continuous_size not in VALID_CONT_SIZES:
        raise PlanArgumentError(f"continuous_size must be one of {VALID_CONT_SIZES}")
    if precision not in ("half", "double"):
        raise PlanArgumentError("precision must be 'half' or 'double'")
    if precision != "half":
        raise PlanArgumentError("precision 'double' is a CPU reference mode; the B200 path computes in fp16 "
                                "storage / fp32 accumulation only (no CPU fallback)")


_STATUS_EXC = {
    _lib.TCFFT_INVALID_SIZE: UnsupportedSizeError,
    _lib.TCFFT_INVALID_VALUE: PlanArgumentError,
    _lib.TCFFT_NOT_SUPPORTED: UnsupportedSizeError,
}


@dataclass(eq=False)
class Plan:
    """Immutable transform configuration (reference plan.py:57-102) owning a
    device plan handle (twiddle tables, DFT matrices, launch geometry)."""

    dims: int
    nx: int
    ny: int | None
    batch: int
    schedule_x: tuple
    schedule_y: tuple | None
    continuous_size: int = 32
    precision: str = "half"
    _handle: object = field(default=None, repr=False)
    _desc: dict = field(default_factory=dict, repr=False)
    _device: int = field(default=-1, repr=False)
    # tcfftSetStream + exec form one critical section (include/tcfft_b200.h):
    # ctypes releases the GIL, so two threads sharing a plan would otherwise
    # launch on each other's stream
    _lock: object = field(default_factory=threading.Lock, repr=False)

    @property
    def n_logical(self) -> int:
        return self.nx if self.dims == 1 else self.nx * self.ny

    @property
    def passes(self) -> list:
        """B200 pass decomposition (one persistent kernel launch each)."""
        return self._desc.get("passes", [])

    def to_json(self) -> str:
        return json.dumps({
            "dims": self.dims, "nx": self.nx, "ny": self.ny, "batch": self.batch,
            "schedule_x": list(self.schedule_x),
            "schedule_y": list(self.schedule_y) if self.schedule_y else None,
            "continuous_size": self.continuous_size, "precision": self.precision,
        })

    def describe(self) -> dict:
        return dict(self._desc)

    def destroy(self) -> None:
        h = self._handle
        if h is not None and h.value:
            _lib.load().tcfftDestroy(h)
            self._handle = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def _current_device() -> int:
    try:
        import torch

        return torch.cuda.current_device() if torch.cuda.is_available() else -1
    except Exception:
        return -1


def _create(dims, nx, ny, batch):
    L = _lib.load()
    h = ctypes.c_void_p()
    st = L.tcfftPlan1D(ctypes.byref(h), nx, batch) if dims == 1 else L.tcfftPlan2D(ctypes.byref(h), nx, ny, batch)
    if st != _lib.TCFFT_SUCCESS:
        exc = _STATUS_EXC.get(st, ExecuteError)
        raise exc(f"tcfftPlan{dims}D failed: {_lib.error_string(st)}")
    return h


def plan_1d(nx: int, batch: int, *, continuous_size: int = 32, precision: str = "half",
            schedule=None) -> Plan:
    """Plan a batch of 1D transforms of power-of-two length nx
    (reference plan.py:116-122).  ``continuous_size`` and ``schedule`` are
    validated as in the reference; the B200 kernels pick their own TMA box
    widths and radix passes (results are invariant to both, reference
    test_acceptance.py:128-138)."""
    _check_pow2(nx, "nx")
    _common_checks(batch, continuous_size, precision)
    sched = schedule_radices(nx) if schedule is None else _validate_schedule(schedule, nx)
    desc = _lib.describe(1, nx, 0, batch)
    h = _create(1, nx, 0, batch)
    return Plan(1, nx, None, batch, sched, None, continuous_size, precision, h, desc, _current_device())


def plan_2d(nx: int, ny: int, batch: int, *, continuous_size: int = 32, precision: str = "half") -> Plan:
    """Plan batched 2D transforms over row-major (nx, ny) data: the contiguous
    dimension (ny) first, then nx down the columns (reference plan.py:125-138)."""
    _check_pow2(nx, "nx")
    _check_pow2(ny, "ny")
    _common_checks(batch, continuous_size, precision)
    desc = _lib.describe(2, nx, ny, batch)
    h = _create(2, nx, ny, batch)
    return Plan(2, nx, ny, batch, schedule_radices(nx), schedule_radices(ny), continuous_size, precision, h, desc,
                _current_device())


def _as_pairs(t):
    """View a torch complex32 / float16[..., 2] CUDA tensor as its interleaved
    storage; returns (storage tensor, total complex elements)."""
    import torch

    if not isinstance(t, torch.Tensor):
        raise ExecuteError(f"expected a torch CUDA tensor, got {type(t).__name__}")
    if not t.is_cuda:
        raise ExecuteError("data must be a CUDA tensor (the B200 path has no CPU fallback)")
    if t.dtype == torch.complex32:
        n = t.numel()
    elif t.dtype == torch.float16:
        if t.dim() == 0 or t.shape[-1] != 2:
            raise ExecuteError(f"float16 data must have a trailing dimension of 2 (re, im), got {tuple(t.shape)}")
        n = t.numel() // 2
    else:
        raise ExecuteError(f"plan precision half needs complex32 / float16 pair storage, got {t.dtype}")
    if not t.is_contiguous():
        raise ExecuteError("data must be contiguous (interleaved pairs, batch-major)")
    if t.data_ptr() % 16:
        raise ExecuteError("data must be 16-byte aligned")
    return t, n


def _check_device(plan: Plan, t) -> None:
    if plan._device >= 0 and t.device.index != plan._device:
        raise ExecuteError(f"data is on {t.device}, the plan was created on cuda:{plan._device}")


def execute(plan: Plan, data, out=None, stream=None):
    """Run the planned forward transform (reference executor.py:152-190).

    In place by default (returns ``data``); with ``out`` writes there and
    returns ``out``.  Natural order in and out, unnormalised.  Asynchronous on
    the current torch CUDA stream (or ``stream``)."""
    import torch

    if plan._handle is None:
        raise ExecuteError("plan has been destroyed")
    from .tensor import BatchedTensor

    if _is_host_view(data):
        return _execute_host_view(plan, data, stream)
    if isinstance(data, np.ndarray):
        raise ExecuteError("host numpy data: pass a BatchedTensor view of it (the reference API) or use execute_host")
    if isinstance(data, BatchedTensor):
        return _execute_view(plan, data, stream)
    t, n = _as_pairs(data)
    if n != plan.batch * plan.n_logical:
        raise ExecuteError(f"data holds {n} complex elements, plan needs batch={plan.batch} x "
                           f"len={plan.n_logical}")
    if out is None:
        o = t
    else:
        o, no = _as_pairs(out)
        if no != n:
            raise ExecuteError("out must hold as many elements as data")
        if o.device != t.device:
            raise ExecuteError("data and out must be on the same device")
    _check_device(plan, t)
    L = _lib.load()
    s = stream if stream is not None else torch.cuda.current_stream(t.device)
    with torch.cuda.device(t.device), plan._lock:
        st = L.tcfftSetStream(plan._handle, ctypes.c_void_p(s.cuda_stream))
        if st == _lib.TCFFT_SUCCESS:
            st = L.tcfftExecC2C(plan._handle, ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(o.data_ptr()))
    if st != _lib.TCFFT_SUCCESS:
        raise ExecuteError(f"tcfftExecC2C failed: {_lib.error_string(st)}")
    return o if out is not None else data


def _is_host_view(data) -> bool:
    """A BatchedTensor-shaped object over a host numpy buffer: ours, or the
    reference's own ``tcfft.BatchedTensor`` (executor.py:25-74)."""
    return all(hasattr(data, a) for a in ("pairs", "batch", "length", "stride", "batch_stride")) and \
        isinstance(data.pairs, np.ndarray)


def _execute_host_view(plan: Plan, data, stream=None):
    """Reference-style execute on host data (executor.py:152-190): the view's
    numpy buffer is transformed in place.  Contiguous batches go through the
    pipelined host-buffer path (tcfftExecC2CHost); other views copy the
    buffer to the plan's device, run the strided device path and copy back
    (the device path leaves elements outside the view untouched)."""
    import torch

    p = data.pairs
    if p.dtype != np.float16:
        raise ExecuteError(f"plan precision half needs {np.dtype(np.float16)} storage, got {p.dtype}")
    if p.ndim != 2 or p.shape[1] != 2:
        raise ExecuteError(f"pairs must be (total, 2), got {p.shape}")
    if data.length != plan.n_logical or data.batch != plan.batch:
        raise ExecuteError(f"data shape (batch={data.batch}, len={data.length}) does not match plan "
                           f"(batch={plan.batch}, len={plan.n_logical})")
    if plan.dims == 2 and data.stride != 1:
        raise ExecuteError("2D execution requires contiguous row-major data")
    n = data.batch * data.length
    if data.stride == 1 and (data.batch == 1 or data.batch_stride == data.length) and p.flags.c_contiguous:
        execute_host(plan, torch.from_numpy(p[:n]), stream=stream)
        return data
    dev = torch.device("cuda", plan._device if plan._device >= 0 else torch.cuda.current_device())
    d = torch.from_numpy(np.ascontiguousarray(p)).to(dev)
    from .tensor import BatchedTensor

    _execute_view(plan, BatchedTensor(d, data.batch, data.length, data.stride, data.batch_stride), stream)
    np.copyto(p, d.cpu().numpy())  # (synchronises)
    return data


def _execute_view(plan: Plan, data, stream=None):
    """In-place transform of a strided BatchedTensor view (executor.py:152-190)."""
    import torch

    if data.length != plan.n_logical or data.batch != plan.batch:
        raise ExecuteError(f"data shape (batch={data.batch}, len={data.length}) does not match plan "
                           f"(batch={plan.batch}, len={plan.n_logical})")
    if plan.dims == 2 and data.stride != 1:
        raise ExecuteError("2D execution requires contiguous row-major data")
    t = data.pairs
    if not t.is_cuda or t.dtype != torch.float16 or not t.is_contiguous():
        raise ExecuteError("BatchedTensor pairs must be a contiguous float16 CUDA tensor")
    _check_device(plan, t)
    L = _lib.load()
    s = stream if stream is not None else torch.cuda.current_stream(t.device)
    with torch.cuda.device(t.device), plan._lock:
        st = L.tcfftSetStream(plan._handle, ctypes.c_void_p(s.cuda_stream))
        if st == _lib.TCFFT_SUCCESS:
            ptr = ctypes.c_void_p(t.data_ptr())
            st = L.tcfftExecC2CStrided(plan._handle, ptr, ptr, data.stride, data.batch_stride)
    if st != _lib.TCFFT_SUCCESS:
        raise ExecuteError(f"tcfftExecC2CStrided failed: {_lib.error_string(st)}")
    return data


def execute_host(plan: Plan, data, out=None, stream=None):
    """Transform HOST data (torch CPU tensor, ideally pinned): the batch is
    sliced and H2D / transform / D2H of successive slices are pipelined
    (``tcfftExecC2CHost``).  In place by default; returns the host tensor.
    Synchronises the stream before returning (the result is on the host)."""
    import torch

    if plan._handle is None:
        raise ExecuteError("plan has been destroyed")
    need = plan.batch * plan.n_logical
    for what, t in (("data", data),) + ((("out", out),) if out is not None else ()):
        if not isinstance(t, torch.Tensor) or t.is_cuda:
            raise ExecuteError("execute_host needs CPU (host) tensors")
        if t.dtype not in (torch.complex32, torch.float16) or not t.is_contiguous():
            raise ExecuteError("host data must be contiguous complex32 / float16[..., 2]")
        if t.dtype == torch.float16 and (t.dim() == 0 or t.shape[-1] != 2):
            raise ExecuteError(f"float16 {what} must have a trailing dimension of 2 (re, im), got {tuple(t.shape)}")
        # tcfftExecC2CHost reads and writes batch * len * 4 bytes: an undersized
        # buffer would be overrun
        n = t.numel() // (1 if t.dtype == torch.complex32 else 2)
        if n != need:
            raise ExecuteError(f"{what} holds {n} complex elements, plan needs {need}")
    o = data if out is None else out
    L = _lib.load()
    dev = plan._device if plan._device >= 0 else torch.cuda.current_device()
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.device(dev), plan._lock:
        st = L.tcfftSetStream(plan._handle, ctypes.c_void_p(s.cuda_stream))
        if st == _lib.TCFFT_SUCCESS:
            st = L.tcfftExecC2CHost(plan._handle, ctypes.c_void_p(data.data_ptr()), ctypes.c_void_p(o.data_ptr()))
    if st != _lib.TCFFT_SUCCESS:
        raise ExecuteError(f"tcfftExecC2CHost failed: {_lib.error_string(st)}")
    s.synchronize()
    return o


def flops_5nlogn(n_total: int, batch: int) -> float:
    """Headline flop count of the project metric: 5 N log2 N per transform."""
    return 5.0 * n_total * math.log2(n_total) * batch


from .tcf import read_tcf, write_tcf  # noqa: E402  (TCF1 files, executor.py:203-230)
from .tensor import BatchedTensor  # noqa: E402  (strided views, executor.py:25-74)
from .dist import DistPlan  # noqa: E402  (distributed single transforms)

__all__ = [
    "BatchedTensor", "DistPlan", "read_tcf", "write_tcf",
    "ExecuteError", "Plan", "PlanArgumentError", "UnsupportedSizeError", "execute", "execute_host", "flops_5nlogn",
    "plan_1d", "plan_2d", "schedule_radices",
]
