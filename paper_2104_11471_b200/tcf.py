"""TCF1 binary interchange files, read/written straight through pinned host
memory (reference ``pkg/src/tcfft/executor.py:203-230``).

Layout: ``"TCF1"`` + ``<4sIIII`` header (magic, dims, nx, ny, batch), then
little-endian binary16 ``(re, im)`` pairs, batch-major -- i.e. exactly the
interleaved buffer ``execute`` consumes, so a file can be read into a pinned
host tensor and copied to the device without any reformatting.
"""

from __future__ import annotations

import struct

from . import ExecuteError

TCF_MAGIC = b"TCF1"
_HEADER = struct.Struct("<4sIIII")


def write_tcf(path, pairs, dims: int, nx: int, ny: int = 1) -> None:
    """Write (batch, nx*ny, 2) fp16 pairs (torch tensor on any device, or a
    numpy array) as a TCF1 file (executor.py:207-215)."""
    import numpy as np
    import torch

    if isinstance(pairs, torch.Tensor):
        t = pairs.detach()
        if t.dtype == torch.complex32:
            t = torch.view_as_real(t) if hasattr(torch, "view_as_real") else t.view(torch.float16)
        if t.dtype != torch.float16:
            raise ExecuteError(f"expected float16 pairs, got {t.dtype}")
        host = t.to("cpu", non_blocking=False).contiguous()
        arr = host.numpy()
    else:
        arr = np.ascontiguousarray(pairs, dtype=np.float16)
    if arr.ndim != 3 or arr.shape[2] != 2 or arr.shape[1] != nx * ny:
        raise ExecuteError(f"expected (batch, {nx * ny}, 2) data, got {tuple(arr.shape)}")
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(TCF_MAGIC, dims, nx, ny, arr.shape[0]))
        fh.write(arr.view(np.uint16).astype("<u2", copy=False).tobytes())


def read_tcf(path, device=None, pin_memory: bool = True):
    """Read a TCF1 file into a (batch, nx*ny, 2) float16 tensor: pinned host
    memory (``device=None``) or, via that pinned buffer, a CUDA device.
    Returns ``(pairs, dims, nx, ny)`` like the reference (executor.py:218-230)."""
    import torch

    with open(path, "rb") as fh:
        head = fh.read(_HEADER.size)
        if len(head) != _HEADER.size:
            raise ExecuteError("truncated TCF header")
        magic, dims, nx, ny, batch = _HEADER.unpack(head)
        if magic != TCF_MAGIC:
            raise ExecuteError(f"bad magic {magic!r}, expected {TCF_MAGIC!r}")
        n = nx * ny
        host = torch.empty((batch, n, 2), dtype=torch.float16,
                           pin_memory=pin_memory and torch.cuda.is_available())
        view = memoryview(host.numpy()).cast("B")
        got = fh.readinto(view)
        if got != batch * n * 4 or fh.read(1):
            raise ExecuteError("truncated TCF payload" if got != batch * n * 4 else "trailing bytes in TCF payload")
    if device is not None:
        return host.to(device, non_blocking=True), dims, nx, ny
    return host, dims, nx, ny
