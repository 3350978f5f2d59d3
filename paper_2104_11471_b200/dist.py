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

Both passes are the single-GPU sm_100a kernels of the four-step plans.

Fused exchange (default when the size allows it, 2^14 .. 2^22 on <= 8 ranks):
pass 0's own TMA stores are the exchange.  Each rank's receive buffer is
mapped into every other rank (CUDA IPC; over NVLink / NVSwitch between GPUs),
and pass 0 stores each N1/G-row slice of every staging tile straight into the
owning rank's buffer, in the blocked layout [N2/C][N1/G][C] of the
single-GPU two-pass plan; after a barrier, pass 1 is that plan's blocked-rows
pass.  No collective and no unpack copy touch the data
(plan.cpp build_plan_dist, fft_kernel.cuh issue_store kIoPeer).

The input and output distributions are the slab layouts of this decomposition
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

    def __init__(self, nx: int, rank: int, world: int, fused: bool = False):
        import torch

        self.torch = torch
        self.world = world
        self.fused = fused
        L = _lib.load()
        h = ctypes.c_void_p()
        make = L.tcfftPlan1DDistFused if fused else L.tcfftPlan1DDist
        st = make(ctypes.byref(h), nx, rank, world)
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

    def set_peers(self, ptrs):
        arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
        self._check(self._L.tcfftDistSetPeers(self._h, arr, len(ptrs)), "tcfftDistSetPeers")

    def pass0(self, slab):
        """Unfused: transforms the slab in place and returns it (to be
        exchanged).  Fused: stores the slices into every rank's receive
        buffer and returns None (nothing left to exchange)."""
        self._stream()
        self._check(self._L.tcfftExecDistPass(self._h, 0, ctypes.c_void_p(slab.data_ptr()),
                                              ctypes.c_void_p(slab.data_ptr())), "pass 0")
        return None if self.fused else slab

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

    def __init__(self, nx: int, group=None, local=None, fused=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.nx = nx
        self.n1, self.n2, self.slab_shape, self.out_shape = dist_geometry(nx, self.world)
        if fused is None:
            fused = (local is None and self.world > 1 and self.world <= 8
                     and "error" not in _lib.describe_dist(nx, self.rank, self.world, fused=True))
        self.fused = bool(fused) if local is None else bool(getattr(local, "fused", False))
        self.local = local if local is not None else CudaLocal(nx, self.rank, self.world, fused=self.fused)
        self._recv = None
        self._opened = []
        if self.fused and local is None:
            self._map_receive_buffers()

    def _map_receive_buffers(self):
        """Allocate this rank's receive buffer and map every rank's into this
        process (CUDA IPC handles exchanged once, at plan time)."""
        import torch

        n1, c = self.slab_shape
        self._recv = torch.empty((n1 * c, 2), dtype=torch.float16, device="cuda")
        L = _lib.load()
        hb = ctypes.create_string_buffer(64)
        st = L.tcfftIpcGetHandle(ctypes.c_void_p(self._recv.data_ptr()), hb, 64)
        if st != _lib.TCFFT_SUCCESS:
            raise ExecuteError(f"tcfftIpcGetHandle failed: {_lib.error_string(st)}")
        handles = [None] * self.world
        self.dist.all_gather_object(handles, hb.raw, group=self.group)
        ptrs = []
        for h, raw in enumerate(handles):
            if h == self.rank:
                ptrs.append(self._recv.data_ptr())
                continue
            p = ctypes.c_void_p()
            st = L.tcfftIpcOpenHandle(ctypes.create_string_buffer(raw, 64), ctypes.byref(p))
            if st != _lib.TCFFT_SUCCESS:
                raise ExecuteError(f"tcfftIpcOpenHandle (rank {h}) failed: {_lib.error_string(st)}")
            self._opened.append(p.value)
            ptrs.append(p.value)
        self.local.set_peers(ptrs)

    def _sync(self):
        import torch

        if torch.cuda.is_available() and torch.cuda.is_initialized():
            torch.cuda.current_stream().synchronize()
        if self.world > 1:
            self.dist.barrier(group=self.group)

    def destroy(self):
        if self._opened:
            L = _lib.load()
            for p in self._opened:
                L.tcfftIpcCloseHandle(ctypes.c_void_p(p))
            self._opened = []
        if hasattr(self.local, "destroy"):
            self.local.destroy()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

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
        if self.fused:
            # every rank's previous pass 1 is done with its receive buffer ...
            self._sync()
            sent = self.local.pass0(slab)
            if sent is not None:
                # (emulated peers in CPU tests: deliver the slices the kernel
                # would have stored, [G][blocks][N1/G][C] in rank order)
                self._recv = self._exchange(sent)
            # ... and every rank's slices have landed in this one
            self._sync()
            return self.local.pass1(self._recv, self._out_like(slab) if out is None else out)
        y = self.local.pass0(slab)
        recv = self._exchange(y)  # [G][N1/G][N2/G]: row blocks in rank order
        rows = torch.empty_like(recv)
        rows = self.local.unpack(recv, rows)
        return self.local.pass1(rows, self._out_like(slab) if out is None else out)

    def _out_like(self, slab):
        """This rank's [N2][N1/G] output block, same element type as the slab."""
        import torch

        if slab.dtype == torch.complex32:
            return torch.empty(self.out_shape, dtype=slab.dtype, device=slab.device)
        return torch.empty((*self.out_shape, 2), dtype=slab.dtype, device=slab.device)
