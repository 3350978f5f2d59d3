"""Pin the CPU restatement (oracle/restate.py) to the reference itself.

The golden file was produced by running the reference package
(/root/reference/pkg/src/tcfft) through oracle/gen_golden.py; every case must
match bit-for-bit (uint16 view)."""

import hashlib
from pathlib import Path

import numpy as np
import pytest

from oracle import restate as R

GOLD = np.load(Path(__file__).parent / "golden" / "reference_outputs.npz")


def _cases():
    for rec in GOLD["meta"]:
        tag, nx, ny, b, cfg, sha = str(rec).split("|")
        yield tag, int(nx), int(ny), int(b), int(cfg), sha


@pytest.mark.parametrize("case", list(_cases()), ids=lambda c: f"{c[0]}-{c[1]}x{c[2]}-b{c[3]}")
def test_restatement_bit_identical_to_reference(case):
    tag, nx, ny, b, cfg, sha = case
    x = R.random_pairs([cfg, 0], b, nx * (ny or 1))
    y = R.fft_half(x) if ny == 0 else R.fft2_half(x, nx, ny)
    assert hashlib.sha256(y.view(np.uint16).tobytes()).hexdigest() == sha
    key = f"{tag}_{nx}_{ny}_out"
    if key in GOLD:
        assert np.array_equal(GOLD[key].view(np.uint16), y.view(np.uint16))


def test_impulse_flat_spectrum_kat():
    # reference test_executor.py:87-92
    z = np.zeros((1, 16, 2), np.float16)
    z[0, 0, 0] = 1
    y = R.fft_half(z)
    assert np.array_equal(y.view(np.uint16), GOLD["impulse16_out"].view(np.uint16))
    assert np.array_equal(R.to_complex(y)[0], np.ones(16))


def test_tone_kat():
    # reference test_executor.py:95-103
    y = R.fft_half(GOLD["tone256_in"])
    assert np.array_equal(y.view(np.uint16), GOLD["tone256_out"].view(np.uint16))
    mag = np.abs(R.to_complex(y)[0])
    assert mag.argmax() == 256 - 5


def test_2d_impulse_kat():
    z = np.zeros((1, 256, 2), np.float16)
    z[0, 0, 0] = 1
    y = R.fft2_half(z, 16, 16)
    assert np.array_equal(y.view(np.uint16), GOLD["impulse2d16_out"].view(np.uint16))


def test_radix2_exact_kat():
    # reference test_kernels.py:93-100: (0.5+0.25j, 0.25-0.5j) -> (0.75-0.25j, 0.25+0.75j)
    x = np.array([[[0.5, 0.25], [0.25, -0.5]]], np.float16)
    y = R.to_complex(R.fft_half(x))[0]
    assert y[0] == 0.75 - 0.25j and y[1] == 0.25 + 0.75j


def test_schedule_examples():
    # reference test_plan.py:14-27
    assert R.schedule_radices(1 << 16) == (8192, 8)
    assert R.schedule_radices(1 << 26) == (8192, 8192)
    assert R.sub_radix_list(512) == (16, 16, 2)
    assert R.sub_radix_list(1 << 17) == (16, 16, 16, 2, 16)


def test_reference_error_envelope_matches_recorded():
    # reference pkg/test_output.txt:243: 1D 4096 mean Eq.5 error 0.078% over 20 seeds
    rng = np.random.default_rng(4096)
    z = rng.uniform(-1, 1, (20, 4096)) + 1j * rng.uniform(-1, 1, (20, 4096))
    x = np.empty((20, 4096, 2), np.float16)
    x[..., 0] = z.real.astype(np.float16)
    x[..., 1] = z.imag.astype(np.float16)
    y = R.to_complex(R.fft_half(x))
    ref = R.fft64(x, 4096)
    err = np.mean([R.relative_error(y[b], ref[b]) for b in range(20)])
    assert abs(100 * err - 0.078) < 0.0015
