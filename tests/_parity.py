"""Parity gates shared by the GPU tests.

On identical fp16 inputs, with ``ref`` = the reference's output (the
bit-identical restatement ``oracle/restate.py`` or the stored reference
outputs) and ``fp64`` = numpy's FP64 FFT of the fp16 input:

  G1  relL2(gpu, ref) <= 2e-3 for every checked transform
  G2  mean relL2(gpu, fp64) <= 1.25 x mean relL2(ref, fp64), and
      mean Eq.5(gpu, fp64) <= 1.25 x mean Eq.5(ref, fp64), where Eq.5 is the
      reference's ``relative_error`` (mean per-bin relative deviation with the
      denominator floored at 1e-6 of the peak, reference oracle.py:64-75)
  G3  every output finite
"""

import numpy as np

from oracle import restate as R

G1_TOL = 2e-3
G2_FACTOR = 1.25


def gates(y, x, nx, ny=None, ref=None):
    """y: GPU output pairs (batch, n, 2); x: the fp16 input pairs."""
    ref = (R.fft_half(x) if ny is None else R.fft2_half(x, nx, ny)) if ref is None else ref
    g, r = R.to_complex(y), R.to_complex(ref)
    f = R.fft64(x, nx, ny)
    assert np.isfinite(g).all(), "G3: non-finite outputs"
    e_ref = np.array([R.rel_l2(g[i], r[i]) for i in range(len(g))])
    e_gpu64 = np.mean([R.rel_l2(g[i], f[i]) for i in range(len(g))])
    e_ref64 = np.mean([R.rel_l2(r[i], f[i]) for i in range(len(g))])
    q_gpu64 = np.mean([R.relative_error(g[i], f[i]) for i in range(len(g))])
    q_ref64 = np.mean([R.relative_error(r[i], f[i]) for i in range(len(g))])
    assert e_ref.max() <= G1_TOL, f"G1: relL2(gpu, ref) max {e_ref.max():.3e}"
    assert e_gpu64 <= G2_FACTOR * e_ref64, f"G2 rel-L2: gpu {e_gpu64:.3e} vs ref {e_ref64:.3e}"
    assert q_gpu64 <= G2_FACTOR * q_ref64, f"G2 Eq.5: gpu {q_gpu64:.3e} vs ref {q_ref64:.3e}"
    return e_ref.max(), e_gpu64, e_ref64
