"""Distributed single 1D transform (paper_2104_11471_b200.dist, SURVEY.md
8(f) rank 4): one transform split over world_size ranks with one all-to-all
between the two local passes.

CPU leg: world_size 2 over gloo, the local passes replayed from the planner's
own tables by the test emulator (tests/emulator.py EmulatedDistLocal), the
exchange / unpack / layout logic exactly as the GPU path runs it; checked
against the FP64 FFT and the reference restatement.  GPU leg: the CUDA path
with world_size 1 and with 2 ranks sharing one GPU (gloo exchange)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import restate as R
from paper_2104_11471_b200 import _lib
from paper_2104_11471_b200.dist import dist_geometry, gather_output, scatter_slab


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("nx,world", [(1 << 14, 2), (1 << 16, 4), (1 << 20, 8), (1 << 24, 2)])
def test_dist_plan_geometry(nx, world):
    n1, n2, slab, out = dist_geometry(nx, world)
    assert n1 * n2 == nx and slab == (n1, n2 // world) and out == (n2, n1 // world)
    for rank in range(world):
        d = _lib.describe_dist(nx, rank, world)
        p0, p1 = d["passes"]
        assert p0["kind"] == "strip" and p0["N"] == n1 and p0["tw4_total"] == nx
        assert p0["tw4_col0"] == rank * (n2 // world)
        assert p1["kind"] == "rowT" and p1["N"] == n2
        assert p0["kernel"] == 1 and p1["kernel"] == 1


def test_scatter_gather_roundtrip():
    nx, world = 1 << 12, 4
    x = np.arange(nx * 2, dtype=np.int64).reshape(nx, 2)
    n1, n2, _, _ = dist_geometry(nx, world)
    slabs = [scatter_slab(x, g, world) for g in range(world)]
    assert np.array_equal(np.concatenate(slabs, axis=1).reshape(nx, 2), x)
    # gather_output places rank g's [N2][N1/G] block at k1 in block g
    parts = [np.full((n2, n1 // world, 2), g) for g in range(world)]
    X = gather_output(parts, nx).reshape(n2, n1, 2)
    assert all((X[:, g * (n1 // world):(g + 1) * (n1 // world)] == g).all() for g in range(world))


def _worker(rank, world, port, nx, q, fused=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2104_11471_b200.dist import DistPlan
        from tests.emulator import EmulatedDistLocal, EmulatedDistLocalFused

        x = R.random_pairs([71, nx], 1, nx)[0]  # every rank regenerates the global input
        local = (EmulatedDistLocalFused if fused else EmulatedDistLocal)(nx, rank, world)
        plan = DistPlan(nx, local=local)
        assert plan.fused == fused
        slab = torch.from_numpy(scatter_slab(x, rank, world))
        out = plan.execute(slab)
        parts = [torch.empty_like(out) for _ in range(world)]
        dist.all_gather(parts, out)
        if rank == 0:
            X = gather_output([p.numpy() for p in parts], nx)
            q.put(X)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nx,world,fused", [(1 << 14, 2, False), (1 << 16, 2, False), (1 << 14, 2, True),
                                            (1 << 16, 2, True), (1 << 16, 4, True)])
def test_dist_transform_gloo_emulated(nx, world, fused):
    """fused: the peer-store layout (each rank's pass-0 slices land blocked
    [N2/C][N1/G][C] in the owning rank, read by the blocked-rows pass), the
    kernel's stores modelled by an all-to-all of the slices."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nx, q, fused)) for r in range(world)]
    for p in procs:
        p.start()
    X = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = R.random_pairs([71, nx], 1, nx)
    got = R.to_complex(X[None])[0]
    f64 = R.fft64(x, nx)[0]
    ref = R.to_complex(R.fft_half(x))[0]
    assert R.rel_l2(got, f64) < 1.5e-3
    assert R.rel_l2(got, ref) < 2e-3


# ---------------------------------------------------------------- GPU leg
def _gpu_run(nx, rank, world, fused=None):
    from paper_2104_11471_b200.dist import DistPlan

    x = R.random_pairs([72, nx], 1, nx)[0]
    plan = DistPlan(nx, fused=fused)
    assert fused is None or plan.fused == fused
    slab = torch.from_numpy(scatter_slab(x, rank, world)).cuda()
    out = plan.execute(slab)
    torch.cuda.synchronize()
    return x, out.cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("nx", [1 << 14, 1 << 16, 1 << 20, 1 << 24])
def test_dist_transform_world1_gpu(nx):
    x, out = _gpu_run(nx, 0, 1)
    X = gather_output([out], nx)
    got = R.to_complex(X[None])[0]
    assert R.rel_l2(got, R.fft64(x[None], nx)[0]) < 1.5e-3
    # one rank: the same two passes as the single-GPU four-step plan, bit for bit
    import paper_2104_11471_b200 as tc

    if (1 << 15) <= nx <= (1 << 18):
        t = torch.from_numpy(np.ascontiguousarray(x[None])).cuda()
        tc.execute(tc.plan_1d(nx, 1), t)
        assert np.array_equal(t.cpu().numpy()[0].view(np.uint16), X.view(np.uint16))


def _gpu_worker(rank, world, port, nx, q, fused=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, out = _gpu_run(nx, rank, world, fused)
        parts = [torch.empty_like(torch.from_numpy(out)) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(out))
        if rank == 0:
            q.put(gather_output([p.numpy() for p in parts], nx))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("nx,fused", [(1 << 16, False), (1 << 22, False), (1 << 16, True), (1 << 20, True),
                                      (1 << 22, True), (1 << 24, None)])
def test_dist_transform_two_ranks_one_gpu(nx, fused):
    """Two ranks sharing one GPU.  fused: pass 0 stores its slices into both
    ranks' receive buffers through CUDA IPC mappings (the peer-memory path,
    here on one device); None: the default choice (2^24: NCCL-style exchange)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, nx, q, fused)) for r in range(world)]
    for p in procs:
        p.start()
    X = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x = R.random_pairs([72, nx], 1, nx)
    got = R.to_complex(X[None])[0]
    assert R.rel_l2(got, R.fft64(x, nx)[0]) < 1.5e-3
    if nx <= 1 << 16:
        assert R.rel_l2(got, R.to_complex(R.fft_half(x))[0]) < 2e-3


@pytest.mark.gpu
def test_dist_plan_rejects_regular_exec():
    """A distributed plan's passes only run through tcfftExecDistPass; the
    single-GPU entry points and the wrong variant's calls are refused."""
    import ctypes

    L = _lib.load()
    for fused in (False, True):
        h = ctypes.c_void_p()
        make = L.tcfftPlan1DDistFused if fused else L.tcfftPlan1DDist
        assert make(ctypes.byref(h), 1 << 16, 0, 2) == 0
        buf = torch.empty((1 << 16, 2), dtype=torch.float16, device="cuda")
        ptr = ctypes.c_void_p(buf.data_ptr())
        assert L.tcfftExecC2C(h, ptr, ptr) == 3  # TCFFT_INVALID_VALUE
        if fused:
            assert L.tcfftDistUnpack(h, 2, ptr, ptr) == 3
            assert L.tcfftExecDistPass(h, 0, ptr, ptr) == 3  # peers not set yet
        else:
            arr = (ctypes.c_void_p * 2)(buf.data_ptr(), buf.data_ptr())
            assert L.tcfftDistSetPeers(h, arr, 2) == 3
        assert L.tcfftDestroy(h) == 0
