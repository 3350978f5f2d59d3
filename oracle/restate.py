"""CPU restatement of the tcFFT reference half-precision pipeline.

TEST INFRASTRUCTURE ONLY.  This module is the parity checker for the B200
kernels: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import it.  The product path
(``paper_2104_11471_b200``) never imports or calls anything under ``oracle/``.

It is a vectorised numpy restatement of the reference's algorithm, written to
be bit-identical to it (pinned by ``tests/test_oracle.py`` against golden
vectors produced by running the reference itself, see ``oracle/gen_golden.py``):

* schedule: greedy radix-8192 kernels then a remainder kernel
  (reference ``pkg/src/tcfft/plan.py:35-44``); each kernel's sub-radices are
  16s first, then 2 / 4 / (4, 2) (``pkg/src/tcfft/kernels.py:48-62``);
* input digit reversal over the flat sub-radix list, last radix outermost
  (``pkg/src/tcfft/plan.py:141-158``, applied ``executor.py:80-127``);
* per stage (radix r, sub-length n2): position ``blk*r*n2 + m*n2 + k`` holds
  input m of butterfly (blk, k); twiddle ``W_{r*n2}^(m*k)`` with the exponent
  reduced exactly in int64, fp64 trig, RNE to fp16 (``twiddle.py:21-42``);
  twiddled input = fp32 complex product rounded once to fp16
  (``half.py:70-82``, ``kernels.py:212-225``);
* radix 16: ``re = Fr.Xr + (-Fi).Xi``, ``im = Fi.Xr + Fr.Xi`` as two chained
  16x16x16 fp32 MMAs, ascending-k accumulation without FMA contraction,
  rounded once to fp16 at store (``kernels.py:227-246``, ``fragments.py:225-244``,
  ``_core.pyx:10-20``);
* radix 2 / 4: fp32 adds of the fp16 twiddled inputs, rounded once
  (``kernels.py:264-310``);
* 2D: rows (contiguous ny) first, then columns (nx at stride ny)
  (``executor.py:180-190``).  The column pass equals a transposed row pass
  bit-for-bit (reference test ``test_executor.py:183-200``).
"""

from __future__ import annotations

import math
from functools import lru_cache

import numpy as np

MAX_KERNEL_RADIX = 8192  # plan.py:18


def schedule_radices(n: int) -> tuple:
    """Greedy kernel schedule (plan.py:35-44)."""
    if n < 2 or n & (n - 1):
        raise ValueError(f"transform length must be a power of two >= 2, got {n}")
    out, rem = [], n
    while rem > MAX_KERNEL_RADIX:
        out.append(MAX_KERNEL_RADIX)
        rem //= MAX_KERNEL_RADIX
    out.append(rem)
    return tuple(out)


def sub_radices_for(radix: int) -> tuple:
    """16s first, then the {2,4,8} remainder, 8 = (4, 2) (kernels.py:48-62)."""
    subs, rem = [], radix
    while rem % 16 == 0 and rem >= 16:
        subs.append(16)
        rem //= 16
    if rem == 8:
        subs += [4, 2]
    elif rem in (2, 4):
        subs.append(rem)
    return tuple(subs)


def sub_radix_list(n: int, schedule=None) -> tuple:
    sched = schedule_radices(n) if schedule is None else tuple(schedule)
    subs = []
    for r in sched:
        subs.extend(sub_radices_for(r))
    return tuple(subs)


def digit_reversal_destinations(n: int, subs) -> np.ndarray:
    """dest[t] = position of input t before the first merge (plan.py:141-158)."""
    t = np.arange(n, dtype=np.int64)
    dest = np.zeros(n, dtype=np.int64)
    for r in reversed(tuple(subs)):
        dest = dest * r + t % r
        t //= r
    return dest


def _round_half(x):
    with np.errstate(over="ignore", under="ignore", invalid="ignore"):
        return np.asarray(x).astype(np.float16)


def twiddle_block(rows, cols, n: int, dtype=np.float16) -> np.ndarray:
    """W_n^(m*k) as (..., 2) pairs (twiddle.py:21-42)."""
    m = np.asarray(rows, dtype=np.int64)
    k = np.asarray(cols, dtype=np.int64)
    e = np.remainder(m * np.remainder(k, n), n)
    ang = (-2.0 * np.pi / n) * e.astype(np.float64)
    out = np.empty(e.shape + (2,), dtype=np.float64)
    out[..., 0] = np.cos(ang)
    out[..., 1] = np.sin(ang)
    if dtype == np.float64:
        return out
    return _round_half(out)


@lru_cache(maxsize=None)
def _f16_tables():
    j = np.arange(16)
    f = twiddle_block(j[:, None], j[None, :], 16)  # (16, 16, 2) fp16
    fr = f[..., 0].astype(np.float32)
    fi = f[..., 1].astype(np.float32)
    fin = (-f[..., 1]).astype(np.float32)
    return fr, fi, fin


def complex_mul_pairs(a, b):
    """fp32 products, one fp32 rounding of the sum, RNE to fp16 (half.py:70-82)."""
    ar = a[..., 0].astype(np.float32)
    ai = a[..., 1].astype(np.float32)
    br = b[..., 0].astype(np.float32)
    bi = b[..., 1].astype(np.float32)
    out = np.empty(np.broadcast_shapes(a.shape, b.shape), dtype=np.float16)
    out[..., 0] = _round_half(ar * br - ai * bi)
    out[..., 1] = _round_half(ar * bi + ai * br)
    return out


def _mma_chain(a_first, b_first, a_second, b_second):
    """d = (0 + sum_k a1[j,k] b1[k]) + sum_k a2[j,k] b2[k]; fp32, ascending k,
    no FMA (fragments.py:225-244 -> _core.pyx:15-20), chained through the
    fp32 accumulator fragment (kernels.py:237-240).

    b_* have shape (..., 16[k], n2); result (..., 16[j], n2) float32."""
    shape = b_first.shape
    acc = np.zeros(shape[:-2] + (16, shape[-1]), dtype=np.float32)
    for a, b in ((a_first, b_first), (a_second, b_second)):
        for k in range(16):
            acc = acc + a[:, k][:, None] * b[..., k : k + 1, :]
    return acc


def apply_stage(x: np.ndarray, radix: int, n2: int) -> np.ndarray:
    """One sub-merge over every sequence (kernels.py:323-356 semantics).

    x: (B, N, 2) fp16, already in the stage's in-place layout.  Returns the
    new (B, N, 2) fp16 array."""
    B, N, _ = x.shape
    nblk = N // (radix * n2)
    v = x.reshape(B, nblk, radix, n2, 2)
    m = np.arange(radix)
    k = np.arange(n2)
    tw = twiddle_block(m[:, None], k[None, :], radix * n2)  # (r, n2, 2)
    xt = complex_mul_pairs(v, tw[None, None])  # (B, nblk, r, n2, 2) fp16
    out = np.empty_like(v)
    if radix == 16:
        fr, fi, fin = _f16_tables()
        xr = xt[..., 0].astype(np.float32)
        xi = xt[..., 1].astype(np.float32)
        re = _mma_chain(fr, xr, fin, xi)
        im = _mma_chain(fi, xr, fr, xi)
        out[..., 0] = _round_half(re)
        out[..., 1] = _round_half(im)
    elif radix == 2:
        u = xt.astype(np.float32)
        out[:, :, 0] = _round_half(u[:, :, 0] + u[:, :, 1])
        out[:, :, 1] = _round_half(u[:, :, 0] - u[:, :, 1])
    elif radix == 4:
        u = xt.astype(np.float32)
        a = u[:, :, 0] + u[:, :, 2]
        b = u[:, :, 1] + u[:, :, 3]
        c = u[:, :, 0] - u[:, :, 2]
        d = u[:, :, 1] - u[:, :, 3]
        out[:, :, 0] = _round_half(a + b)
        out[:, :, 2] = _round_half(a - b)
        out[:, :, 1, :, 0] = _round_half(c[..., 0] + d[..., 1])
        out[:, :, 1, :, 1] = _round_half(c[..., 1] - d[..., 0])
        out[:, :, 3, :, 0] = _round_half(c[..., 0] - d[..., 1])
        out[:, :, 3, :, 1] = _round_half(c[..., 1] + d[..., 0])
    else:
        raise ValueError(f"no sub-merge for radix {radix}")
    return out.reshape(B, N, 2)


def fft_half(pairs: np.ndarray, schedule=None) -> np.ndarray:
    """Forward half-precision transform of (B, N, 2) fp16 pairs along axis 1,
    natural order in and out (executor.py:133-140, 152-178)."""
    pairs = np.ascontiguousarray(pairs, dtype=np.float16)
    B, N, _ = pairs.shape
    subs = sub_radix_list(N, schedule)
    dest = digit_reversal_destinations(N, subs)
    x = np.empty_like(pairs)
    x[:, dest] = pairs
    n2 = 1
    for r in subs:
        x = apply_stage(x, r, n2)
        n2 *= r
    assert n2 == N
    return x


def fft2_half(pairs: np.ndarray, nx: int, ny: int) -> np.ndarray:
    """Batched 2D transform of (B, nx*ny, 2) row-major pairs: rows (ny) first,
    then columns (nx) (executor.py:180-190)."""
    B = pairs.shape[0]
    v = np.ascontiguousarray(pairs, dtype=np.float16).reshape(B * nx, ny, 2)
    v = fft_half(v).reshape(B, nx, ny, 2)
    t = np.ascontiguousarray(v.transpose(0, 2, 1, 3)).reshape(B * ny, nx, 2)
    t = fft_half(t).reshape(B, ny, nx, 2)
    return np.ascontiguousarray(t.transpose(0, 2, 1, 3)).reshape(B, nx * ny, 2)


# -- inputs and metrics ------------------------------------------------------


def random_pairs(seed, batch: int, total: int) -> np.ndarray:
    """Seeded U[-1,1) re/im rounded RNE to fp16 (cli.py:40-43, executor.py:57-65)."""
    rng = np.random.default_rng(seed)
    re = rng.uniform(-1.0, 1.0, (batch, total))
    im = rng.uniform(-1.0, 1.0, (batch, total))
    out = np.empty((batch, total, 2), dtype=np.float16)
    out[..., 0] = re.astype(np.float16)
    out[..., 1] = im.astype(np.float16)
    return out


def to_complex(pairs: np.ndarray) -> np.ndarray:
    p = np.asarray(pairs)
    return p[..., 0].astype(np.float64) + 1j * p[..., 1].astype(np.float64)


def fft64(pairs: np.ndarray, nx: int, ny: int | None = None) -> np.ndarray:
    """FP64 spectra of the fp16 inputs actually consumed (cli.py:46-59)."""
    z = to_complex(pairs)
    if ny is None:
        return np.fft.fft(z, axis=-1)
    B = z.shape[0]
    return np.fft.fft2(z.reshape(B, nx, ny)).reshape(B, nx * ny)


def relative_error(x, x_ref) -> float:
    """Eq.5 mean per-bin relative deviation, 1e-6*peak floor (oracle.py:64-75)."""
    x = np.asarray(x, dtype=np.complex128)
    x_ref = np.asarray(x_ref, dtype=np.complex128)
    mag = np.abs(x_ref)
    floor = 1e-6 * mag.max()
    return float(np.mean(np.abs(x_ref - x) / np.maximum(mag, floor)))


def rel_l2(x, x_ref) -> float:
    x = np.asarray(x, dtype=np.complex128)
    x_ref = np.asarray(x_ref, dtype=np.complex128)
    return float(np.linalg.norm(x - x_ref) / max(np.linalg.norm(x_ref), 1e-300))


def flops_5nlogn(n_total: int, batch: int) -> float:
    return 5.0 * n_total * math.log2(n_total) * batch
