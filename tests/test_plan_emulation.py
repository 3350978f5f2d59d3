"""CPU check of the planner's tables: emulate the kernel dataflow on CPU
(tests/emulator.py) and compare with the FP64 FFT and the reference
restatement.  No GPU needed; exercises the real C planner through the C ABI."""

import numpy as np
import pytest

from oracle import restate as R
from tests.emulator import PassTables, run_fourstep, run_pass_row, run_pass_strip

SIZES_1D = [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384]


def _errs(y_pairs, x_pairs, nx, ny=None):
    got = R.to_complex(y_pairs)
    ref = R.fft64(x_pairs, nx, ny)
    return max(R.rel_l2(got[b], ref[b]) for b in range(got.shape[0]))


@pytest.mark.parametrize("n", SIZES_1D)
def test_row_pass_emulation_matches_fft(n):
    batch = max(2, min(6, 8192 // n)) if n >= 4 else 6
    x = R.random_pairs([7, n], batch, n)
    pt = PassTables(1, n, 0, batch, 0)
    y = run_pass_row(pt, x)
    assert np.isfinite(R.to_complex(y)).all()
    e64 = _errs(y, x, n)
    ref = R.to_complex(R.fft_half(x))
    e_ref = max(R.rel_l2(R.to_complex(y)[b], ref[b]) for b in range(batch))
    assert e64 < 1.5e-3, e64
    assert e_ref < 2e-3, e_ref


@pytest.mark.parametrize("nx,ny,batch", [(16, 16, 3), (64, 32, 2), (32, 64, 2), (256, 256, 1), (512, 512, 1),
                                         (1024, 8, 1), (8, 256, 1)])
def test_2d_emulation_matches_fft2(nx, ny, batch):
    x = R.random_pairs([9, nx, ny], batch, nx * ny)
    p0 = PassTables(2, nx, ny, batch, 0)
    p1 = PassTables(2, nx, ny, batch, 1)
    rows = run_pass_row(p0, x.reshape(batch * nx, ny, 2))
    y = run_pass_strip(p1, rows.reshape(batch, nx, ny, 2)).reshape(batch, nx * ny, 2)
    e64 = _errs(y, x, nx, ny)
    assert e64 < 2e-3, e64


def test_bank_conflicts_report(capsys):
    lines = []
    for dims, nx, ny in [(1, 256, 0), (1, 4096, 0), (1, 512, 0), (1, 1024, 0), (1, 8192, 0), (2, 512, 512)]:
        for pi in range(2 if dims == 2 else 1):
            pt = PassTables(dims, nx, ny, 1, pi)
            stats = {}
            if pt.d["kind"] == "row":
                N = pt.d["N"]
                x = R.random_pairs([1], pt.d["T"], N)
                run_pass_row(pt, x, stats)
            else:
                x = R.random_pairs([1], 1, nx * ny).reshape(1, nx, ny, 2)
                run_pass_strip(pt, x, stats)
            for k, (tot, cnt, ideal) in stats.items():
                lines.append(f"{dims}d {nx}x{ny} pass{pi} {k}: {tot / cnt:.2f} wavefronts/instr (ideal {ideal})")
                assert tot / cnt <= 4 * ideal, (k, tot / cnt)
    with capsys.disabled():
        print("\n" + "\n".join(lines))


@pytest.mark.parametrize("n,batch", [(1 << 15, 2), (1 << 16, 1), (1 << 17, 1)])
def test_fourstep_emulation_matches_fft(n, batch):
    x = R.random_pairs([11, n], batch, n)
    y = run_fourstep(n, x)
    assert np.isfinite(R.to_complex(y)).all()
    e64 = _errs(y, x, n)
    assert e64 < 1.5e-3, e64
