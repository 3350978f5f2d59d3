"""TCF1 files (reference test_executor.py:228-257), read through pinned host memory."""

import numpy as np
import pytest

import paper_2104_11471_b200 as tc
from oracle import restate as R


def test_tcf_round_trip(tmp_path):
    rng = np.random.default_rng(7)
    pairs = rng.uniform(-1, 1, (3, 64, 2)).astype(np.float16)
    path = tmp_path / "data.tcf"
    tc.write_tcf(path, pairs, 1, 64)
    got, dims, nx, ny = tc.read_tcf(path, pin_memory=False)
    assert (dims, nx, ny) == (1, 64, 1)
    assert np.array_equal(got.numpy().view(np.uint16), pairs.view(np.uint16))


def test_tcf_bytes_match_reference_format(tmp_path):
    # header <4sIIII then LE fp16 pairs, exactly as the reference writes them
    pairs = R.random_pairs([1], 2, 16 * 8).reshape(2, 128, 2)
    path = tmp_path / "x.tcf"
    tc.write_tcf(path, pairs, 2, 16, 8)
    raw = path.read_bytes()
    assert raw[:4] == b"TCF1"
    assert np.frombuffer(raw[4:20], "<u4").tolist() == [2, 16, 8, 2]
    assert raw[20:] == pairs.astype("<f2").tobytes()


def test_tcf_rejects_bad_magic(tmp_path):
    path = tmp_path / "bad.tcf"
    path.write_bytes(b"NOPE" + b"\x00" * 16)
    with pytest.raises(tc.ExecuteError):
        tc.read_tcf(path, pin_memory=False)


def test_tcf_rejects_truncated_payload(tmp_path):
    path = tmp_path / "short.tcf"
    tc.write_tcf(path, np.zeros((1, 64, 2), np.float16), 1, 64)
    path.write_bytes(path.read_bytes()[:-8])
    with pytest.raises(tc.ExecuteError):
        tc.read_tcf(path, pin_memory=False)


def test_tcf_shape_validation(tmp_path):
    with pytest.raises(tc.ExecuteError):
        tc.write_tcf(tmp_path / "x.tcf", np.zeros((1, 63, 2), np.float16), 1, 64)


@pytest.mark.gpu
def test_tcf_to_device_transform_and_back(tmp_path):
    import torch

    x = R.random_pairs([3, 4096], 4, 4096)
    tc.write_tcf(tmp_path / "in.tcf", x, 1, 4096)
    d, dims, nx, ny = tc.read_tcf(tmp_path / "in.tcf", device="cuda")
    plan = tc.plan_1d(nx, d.shape[0])
    tc.execute(plan, d)
    tc.write_tcf(tmp_path / "out.tcf", d, 1, nx)
    y, *_ = tc.read_tcf(tmp_path / "out.tcf", pin_memory=False)
    ref = R.to_complex(R.fft_half(x))
    g = R.to_complex(y.numpy())
    assert max(R.rel_l2(g[b], ref[b]) for b in range(4)) < 2e-3
