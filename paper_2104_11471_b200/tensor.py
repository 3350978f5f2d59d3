"""``BatchedTensor``: the reference's strided batch view, on a CUDA tensor
(reference ``pkg/src/tcfft/executor.py:25-74``).

Logical element j of sequence b lives at ``pairs[b*batch_stride + j*stride]``;
``pairs`` is a ``(total, 2)`` float16 array with re at ``[..., 0]``: a CUDA
tensor (device view), or, as in the reference, a host numpy array.
``execute(plan, BatchedTensor)`` transforms the view in place: device views
through ``tcfftExecC2CStrided`` (contiguous and row-pitched views run directly,
other views via a plan-owned contiguous scratch), host views through the
host-buffer pipeline (``tcfftExecC2CHost``) or a device copy of the buffer.
The reference's own ``BatchedTensor`` objects (numpy ``pairs``) are accepted
by ``execute`` as they are.
"""

from __future__ import annotations

import numpy as np

from . import ExecuteError


class BatchedTensor:
    def __init__(self, pairs, batch: int, length: int, stride: int = 1, batch_stride: int | None = None):
        import torch

        ok = (isinstance(pairs, torch.Tensor) and pairs.dim() == 2) or (isinstance(pairs, np.ndarray) and pairs.ndim == 2)
        if not ok or pairs.shape[1] != 2:
            shape = tuple(pairs.shape) if hasattr(pairs, "shape") else type(pairs).__name__
            raise ExecuteError(f"pairs must be (total, 2), got {shape}")
        if batch_stride is None:
            batch_stride = length * stride
        needed = batch_stride * (batch - 1) + stride * (length - 1) + 1
        if pairs.shape[0] < needed:
            raise ExecuteError(f"buffer of {pairs.shape[0]} elements too small for batch={batch} len={length} "
                               f"stride={stride}")
        if stride < 1 or (batch > 1 and batch_stride < stride * length):
            raise ExecuteError("logical elements must not alias")
        self.pairs = pairs
        self.batch = batch
        self.length = length
        self.stride = stride
        self.batch_stride = batch_stride

    @classmethod
    def zeros(cls, batch: int, length: int, device="cuda") -> "BatchedTensor":
        import torch

        return cls(torch.zeros((batch * length, 2), dtype=torch.float16, device=device), batch, length)

    @classmethod
    def from_complex(cls, z, device="cuda") -> "BatchedTensor":
        """Pack a (batch, length) complex array, RNE to fp16 (executor.py:57-65)."""
        import torch

        z = np.atleast_2d(np.asarray(z))
        batch, length = z.shape
        pairs = np.empty((batch * length, 2), dtype=np.float16)
        pairs[:, 0] = z.real.reshape(-1).astype(np.float16)
        pairs[:, 1] = z.imag.reshape(-1).astype(np.float16)
        return cls(torch.from_numpy(pairs).to(device), batch, length)

    def offsets(self) -> np.ndarray:
        return np.arange(self.batch, dtype=np.int64) * self.batch_stride

    def to_complex(self) -> np.ndarray:
        """Gather the logical (batch, length) sequences as complex128 (host)."""
        idx = self.offsets()[:, None] + np.arange(self.length) * self.stride
        p = self.pairs if isinstance(self.pairs, np.ndarray) else self.pairs.detach().cpu().numpy()
        vals = p[idx]
        return vals[..., 0].astype(np.float64) + 1j * vals[..., 1].astype(np.float64)
