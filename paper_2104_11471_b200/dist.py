"""Distributed single 1D transform over the ranks of a torch.distributed group
(the reference has no multi-GPU transform:
/root/reference/SPEC.md:14,467).

One transform of length N = N1 N2 (N1 = 2^floor(log2 N / 2)) is split over G
ranks, one process per GPU, as a four-step with ONE all-to-all between the
two local passes (plan.cpp build_plan_dist):

    rank g input   column slab  x[N2 n1 + n2], n2 in [g N2/G, (g+1) N2/G)   [N1][N2/G]
    pass 0         length-N1 column FFTs + twiddle W_N^{n2 k1} (global n2)   in place
    exchange       all-to-all of the slab's N1/G-row blocks                 (NCCL)
    unpack         received [G][N1/G][N2/G] -> rows [N1/G][N2]               (device copies)
    pass 1         length-N2 row FFTs, transposed store                     [N2][N1/G]
    rank g output  X[k1 + N1 k2], k1 in [g N1/G, (g+1) N1/G)

Both passes are the single-GPU sm_100a kernels of the four-step plans.  The
input and output distributions are the slab layouts of this decomposition
(`scatter_slab` / `gather_output` convert from / to the natural-order
transform).  The local steps are a small interface (`CudaLocal`) so that the
exchange logic can be exercised on CPU ranks (gloo) with the planner's tables
replayed by the test emulator (tests/test_dist.py); the product path is
`CudaLocal`, which has no CPU fallback.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from . import ExecuteError, PlanArgumentError, UnsupportedSizeError, _STATUS_EXC, _check_pow2

__all__ = ["DistPlan", "CudaLocal", "scatter_slab", "gather_output", "dist_geometry"]


def dist_geometry(nx: int, world: int):
    """(N1, N2, slab shape, output shape) of the distributed plan."""
    _check_pow2(nx, "nx")
    lg = nx.bit_length() - 1
    n1, n2 = 1 << (lg // 2), 1 << (lg - lg // 2)
    if world < 1 or world & (world - 1):
        raise PlanArgumentError(f"world size must be a power of two, got {world}")
    if n1 % world or n2 % world or n1 > 4096 or n2 > 4096:
        raise UnsupportedSizeError(f"distributed N={nx} over {world} ranks: needs N1={n1}, N2={n2} <= 4096 "
                                   "and divisible by the world size")
    return n1, n2, (n1, n2 // world), (n2, n1 // world)


def scatter_slab(x: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Rank `rank`'s input slab of the natural-order transform x (N, ...)."""
    n1, n2, _, _ = dist_geometry(x.shape[0], world)
    c = n2 // world
    return np.ascontiguousarray(x.reshape(n1, n2, *x.shape[1:])[:, rank * c:(rank + 1) * c])


def gather_output(parts, nx: int) -> np.ndarray:
    """Natural-order spectrum X[k] from every rank's [N2][N1/G] output."""
    world = len(parts)
    n1, n2, _, _ = dist_geometry(nx, world)
    r = n1 // world
    tail = parts[0].shape[2:]
    out = np.empty((n2, n1) + tail, dtype=parts[0].dtype)  # X[k1 + N1 k2] = out[k2][k1]
    for g, p in enumerate(parts):
        out[:, g * r:(g + 1) * r] = p
    return out.reshape((nx,) + tail)


class CudaLocal:
    """The local steps on this rank's GPU through the C ABI
    (tcfftPlan1DDist / tcfftExecDistPass / tcfftDistUnpack)."""

    def __init__(self, nx: int, rank: int, world: int):
        import torch

        self.torch = torch
        self.world = world
        L = _lib.load()
        h = ctypes.c_void_p()
        st = L.tcfftPlan1DDist(ctypes.byref(h), nx, rank, world)
        if st != _lib.TCFFT_SUCCESS:
            raise _STATUS_EXC.get(st, ExecuteError)(f"tcfftPlan1DDist failed: {_lib.error_string(st)}")
        self._h = h
        self._L = L
        self.device = torch.cuda.current_device()

    def _check(self, st, what):
        if st != _lib.TCFFT_SUCCESS:
            raise ExecuteError(f"{what} failed: {_lib.error_string(st)}")

    def _stream(self):
        s = self.torch.cuda.current_stream(self.device)
        self._check(self._L.tcfftSetStream(self._h, ctypes.c_void_p(s.cuda_stream)), "tcfftSetStream")

    def pass0(self, slab):
        self._stream()
        self._check(self._L.tcfftExecDistPass(self._h, 0, ctypes.c_void_p(slab.data_ptr()),
                                              ctypes.c_void_p(slab.data_ptr())), "pass 0")
        return slab

    def unpack(self, recv, rows):
        self._stream()
        self._check(self._L.tcfftDistUnpack(self._h, self.world, ctypes.c_void_p(recv.data_ptr()),
                                            ctypes.c_void_p(rows.data_ptr())), "unpack")
        return rows

    def pass1(self, rows, out):
        self._stream()
        self._check(self._L.tcfftExecDistPass(self._h, 1, ctypes.c_void_p(rows.data_ptr()),
                                              ctypes.c_void_p(out.data_ptr())), "pass 1")
        return out

    def destroy(self):
        if self._h is not None:
            self._L.tcfftDestroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class DistPlan:
    """A single transform of length `nx` split over the ranks of `group`.

    ``execute(slab)`` takes this rank's column slab (float16 [N1, N2/G, 2] or
    complex32, on this rank's GPU), transforms it in place through pass 0,
    exchanges the row blocks with one all-to-all, and returns this rank's
    [N2, N1/G] block of the spectrum.  Every rank must call it (collective)."""

    def __init__(self, nx: int, group=None, local=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.nx = nx
        self.n1, self.n2, self.slab_shape, self.out_shape = dist_geometry(nx, self.world)
        self.local = local if local is not None else CudaLocal(nx, self.rank, self.world)

    def _exchange(self, send):
        """All-to-all of equal row blocks (NCCL for CUDA tensors; CPU tensors
        and gloo groups stage through host memory)."""
        import torch

        if self.world == 1:
            return send.clone()
        backend = self.dist.get_backend(self.group)
        if backend == "nccl" or not send.is_cuda:
            recv = torch.empty_like(send)
            self.dist.all_to_all_single(recv, send, group=self.group)
            return recv
        host = send.cpu()
        recv = torch.empty_like(host)
        self.dist.all_to_all_single(recv, host, group=self.group)
        return recv.to(send.device)

    def execute(self, slab, out=None):
        import torch

        n1, c = self.slab_shape
        elems = slab.numel() // (2 if slab.dtype == torch.float16 else 1)
        if slab.dtype not in (torch.float16, torch.complex32) or elems != n1 * c:
            raise ExecuteError(f"slab must hold [{n1}][{c}] fp16 complex elements, got {tuple(slab.shape)} "
                               f"{slab.dtype}")
        if not slab.is_contiguous():
            raise ExecuteError("slab must be contiguous")
        y = self.local.pass0(slab)
        recv = self._exchange(y)  # [G][N1/G][N2/G]: row blocks in rank order
        rows = torch.empty_like(recv)
        rows = self.local.unpack(recv, rows)
        if out is None:
            out = torch.empty_like(rows)
        return self.local.pass1(rows, out)
