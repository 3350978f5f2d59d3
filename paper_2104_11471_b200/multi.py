"""Single-process multi-device execution: one batch, several GPUs.

Every transform of a batch is independent (reference SPEC.md:317: disjoint
batch segments may run concurrently), so a batch spread over D devices is D
contiguous shards (``shard.shard_range``), each transformed by its own
per-device plan on its own stream.  No data crosses between devices: there is
no collective on this path.

    mp = plan_many(4096, batch=16384, devices=[0, 1, 2, 3])
    execute_many(mp, [x0, x1, x2, x3])   # shard i resident on devices[i]
    execute_many_host(mp, h)             # one pinned host batch: every device
                                         # pipelines H2D / FFT / D2H of its
                                         # slice concurrently

The multi-process equivalent (one process per GPU under torchrun) is
``shard.my_shard`` + an ordinary plan, as ``bench.py --scaling strong`` does.
A device may appear more than once (two shards on one GPU, two streams).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

from . import ExecuteError, _lib, execute, plan_1d, plan_2d
from .shard import shard_range


@dataclass(eq=False)
class MultiPlan:
    dims: int
    nx: int
    ny: int | None
    batch: int
    devices: tuple
    shards: tuple            # (start, stop) per device slot
    plans: tuple             # Plan per device slot (None for an empty shard)
    streams: tuple = field(default=(), repr=False)

    @property
    def n_logical(self) -> int:
        return self.nx if self.dims == 1 else self.nx * self.ny

    def destroy(self) -> None:
        for p in self.plans:
            if p is not None:
                p.destroy()


def plan_many(nx: int, batch: int, devices, ny: int | None = None, **kw) -> MultiPlan:
    """Plan `batch` transforms (1D of length nx, or 2D nx x ny) split into
    contiguous, balanced shards over `devices` (CUDA indices)."""
    import torch

    devices = tuple(int(d) for d in devices)
    if not devices:
        raise ExecuteError("plan_many needs at least one device")
    if not isinstance(batch, int) or batch < 1:
        from . import PlanArgumentError

        raise PlanArgumentError(f"batch must be >= 1, got {batch}")
    shards, plans, streams = [], [], []
    for i, d in enumerate(devices):
        s0, s1 = shard_range(batch, i, len(devices))
        shards.append((s0, s1))
        with torch.cuda.device(d):
            if s1 > s0:
                plans.append(plan_1d(nx, s1 - s0, **kw) if ny is None else plan_2d(nx, ny, s1 - s0, **kw))
            else:
                plans.append(None)
            streams.append(torch.cuda.Stream(device=d))
    return MultiPlan(1 if ny is None else 2, nx, ny, batch, devices, tuple(shards), tuple(plans), tuple(streams))


def execute_many(mp: MultiPlan, shards, outs=None):
    """Transform device-resident shards: ``shards[i]`` holds transforms
    ``mp.shards[i]`` on ``cuda:mp.devices[i]``.  Launches on every device's
    stream (ordered after each device's current stream), then makes each
    current stream wait for them.  In place unless ``outs`` is given."""
    import torch

    if len(shards) != len(mp.devices) or (outs is not None and len(outs) != len(shards)):
        raise ExecuteError(f"expected {len(mp.devices)} shards")
    res = []
    for i, (d, p, st) in enumerate(zip(mp.devices, mp.plans, mp.streams)):
        x = shards[i]
        o = None if outs is None else outs[i]
        if p is None:
            res.append(o if o is not None else x)
            continue
        with torch.cuda.device(d):
            cur = torch.cuda.current_stream(d)
            st.wait_stream(cur)
            res.append(execute(p, x, out=o, stream=st))
    for d, p, st in zip(mp.devices, mp.plans, mp.streams):
        if p is not None:
            torch.cuda.current_stream(d).wait_stream(st)
    return res


def execute_many_host(mp: MultiPlan, data, out=None):
    """Transform one HOST batch (contiguous torch CPU tensor, ideally pinned):
    device slot i runs ``tcfftExecC2CHost`` on its slice of the host buffer,
    all devices concurrently; returns after every slice is back on the host."""
    import torch

    for what, t in (("data", data),) + ((("out", out),) if out is not None else ()):
        if not isinstance(t, torch.Tensor) or t.is_cuda or not t.is_contiguous():
            raise ExecuteError(f"{what} must be a contiguous host tensor")
        if t.dtype not in (torch.complex32, torch.float16):
            raise ExecuteError(f"{what} must be complex32 / float16[..., 2]")
        n = t.numel() // (1 if t.dtype == torch.complex32 else 2)
        if n != mp.batch * mp.n_logical:
            raise ExecuteError(f"{what} holds {n} complex elements, the plan needs {mp.batch * mp.n_logical}")
    o = data if out is None else out
    L = _lib.load()
    per = mp.n_logical * 4  # bytes per transform
    launched = []
    for (s0, s1), d, p, st in zip(mp.shards, mp.devices, mp.plans, mp.streams):
        if p is None:
            continue
        with torch.cuda.device(d), p._lock:
            r = L.tcfftSetStream(p._handle, ctypes.c_void_p(st.cuda_stream))
            if r == _lib.TCFFT_SUCCESS:
                r = L.tcfftExecC2CHost(p._handle, ctypes.c_void_p(data.data_ptr() + s0 * per),
                                       ctypes.c_void_p(o.data_ptr() + s0 * per))
        if r != _lib.TCFFT_SUCCESS:
            for s in launched:
                s.synchronize()
            raise ExecuteError(f"tcfftExecC2CHost on cuda:{d} failed: {_lib.error_string(r)}")
        launched.append(st)
    for s in launched:
        s.synchronize()
    return o


__all__ = ["MultiPlan", "plan_many", "execute_many", "execute_many_host"]
