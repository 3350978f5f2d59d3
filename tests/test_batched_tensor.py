"""BatchedTensor strided views (reference test_executor.py:27-52 and the
strided-pass tests :168-200)."""

import numpy as np
import pytest

from oracle import restate as R
from tests._parity import gates

torch = pytest.importorskip("torch")
import paper_2104_11471_b200 as tc  # noqa: E402


def test_tensor_rejects_bad_pair_shape():
    with pytest.raises(tc.ExecuteError):
        tc.BatchedTensor(torch.zeros((8, 3), dtype=torch.float16), 1, 8)


def test_tensor_rejects_short_buffer():
    with pytest.raises(tc.ExecuteError):
        tc.BatchedTensor(torch.zeros((7, 2), dtype=torch.float16), 1, 8)


def test_tensor_rejects_aliasing_batches():
    with pytest.raises(tc.ExecuteError):
        tc.BatchedTensor(torch.zeros((16, 2), dtype=torch.float16), 2, 8, batch_stride=4)


def test_tensor_strided_view_addresses():
    data = tc.BatchedTensor(torch.zeros((64, 2), dtype=torch.float16), 2, 4, stride=8, batch_stride=32)
    assert data.offsets().tolist() == [0, 32]


def test_tensor_complex_round_trip_cpu():
    z = np.array([[0.5 + 0.25j, -1.0, 2.0j]])
    d = tc.BatchedTensor.from_complex(z, device="cpu")
    assert np.array_equal(d.to_complex(), z)


def _strided_case(n, batch, stride, bstride, seed):
    x = R.random_pairs([seed, n], batch, n)  # logical sequences
    total = bstride * (batch - 1) + stride * (n - 1) + 1
    buf = np.full((total + 5, 2), np.float16(7.0))  # sentinel outside the view
    idx = (np.arange(batch)[:, None] * bstride + np.arange(n)[None, :] * stride)
    buf[idx] = x
    return x, buf, idx


@pytest.mark.gpu
@pytest.mark.parametrize("n,batch,stride,bstride", [(256, 8, 1, 256), (256, 8, 1, 260), (1024, 3, 1, 1100),
                                                      (512, 4, 3, 2000), (4, 2, 8, 32), (4096, 4, 2, 8195),
                                                      (1 << 15, 2, 1, (1 << 15) + 16),
                                                      # row-pitched 3D tensor maps (swizzled row plans):
                                                      (4096, 5, 1, 4100), (2048, 7, 1, 2052), (8192, 3, 1, 8200),
                                                      (32, 300, 1, 36), (256, 10001, 1, 260), (4096, 3, 1, 4098),
                                                      # two-pass plans, box tensor maps at the view's image stride:
                                                      (1 << 16, 3, 1, (1 << 16) + 4), (1 << 18, 2, 1, (1 << 18) + 256),
                                                      (1 << 20, 2, 1, (1 << 20) + 64), (1 << 22, 2, 1, (1 << 22) + 8)])
def test_strided_views_equal_contiguous(n, batch, stride, bstride):
    x, buf, idx = _strided_case(n, batch, stride, bstride, 3)
    t = torch.from_numpy(buf).cuda()
    view = tc.BatchedTensor(t, batch, n, stride=stride, batch_stride=bstride)
    tc.execute(tc.plan_1d(n, batch), view)
    got = t.cpu().numpy()
    y = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    tc.execute(tc.plan_1d(n, batch), y)
    want = y.cpu().numpy()
    assert np.array_equal(got[idx].view(np.uint16), want.view(np.uint16))
    gates(got[idx], x, n)  # and against the reference restatement (oracle)
    mask = np.ones(len(buf), bool)
    mask[idx.reshape(-1)] = False
    assert np.all(got[mask] == np.float16(7.0))  # nothing outside the view touched


def test_interleaved_view_aliases_like_reference():
    # the reference forbids batch_stride < stride*length for batch > 1
    # (executor.py:45-46); interleaved columns are the 2D column pass instead
    with pytest.raises(tc.ExecuteError):
        tc.BatchedTensor(torch.zeros((64, 2), dtype=torch.float16), 4, 16, stride=4, batch_stride=1)


def test_host_view_validation_cpu():
    """numpy-backed views (the reference's BatchedTensor storage) are accepted
    by the constructor and checked like the reference before any device work."""
    v = tc.BatchedTensor(np.zeros((16, 2), np.float16), 2, 8)
    assert v.offsets().tolist() == [0, 8] and v.to_complex().shape == (2, 8)
    with pytest.raises(tc.ExecuteError):
        tc.BatchedTensor(np.zeros((16, 3), np.float16), 2, 8)


def _reference_batched_tensor_cls():
    """The reference's own BatchedTensor class when its package is installed
    (baseline/_ref, not on every box), else ours."""
    import importlib
    import sys
    from pathlib import Path

    ref = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
    if (ref / "tcfft").is_dir():
        sys.path.insert(0, str(ref))
        try:
            return importlib.import_module("tcfft").BatchedTensor
        except Exception:
            pass
        finally:
            sys.path.remove(str(ref))
    return tc.BatchedTensor


@pytest.mark.gpu
@pytest.mark.parametrize("n,batch,stride,bstride", [(4096, 8, 1, 4096), (256, 8, 1, 260), (512, 4, 3, 2000),
                                                      (1 << 16, 2, 1, 1 << 16), (64, 16, 2, 200)])
def test_execute_on_host_views_like_reference(n, batch, stride, bstride):
    """execute(plan, view) on a HOST numpy buffer, as a reference caller does
    (executor.py:152-190): the reference's own BatchedTensor object when
    available, transformed in place, nothing outside the view touched."""
    BT = _reference_batched_tensor_cls()
    x, buf, idx = _strided_case(n, batch, stride, bstride, 11)
    view = BT(buf, batch, n, stride=stride, batch_stride=bstride)
    out = tc.execute(tc.plan_1d(n, batch), view)
    assert out is view
    got = view.pairs
    gates(got[idx], x, n)
    mask = np.ones(len(buf), bool)
    mask[idx.reshape(-1)] = False
    assert np.all(got[mask] == np.float16(7.0))


@pytest.mark.gpu
def test_execute_host_view_rejects_wrong_dtype():
    BT = _reference_batched_tensor_cls()
    view = BT(np.zeros((64, 2), np.float64), 4, 16)
    with pytest.raises(tc.ExecuteError):
        tc.execute(tc.plan_1d(16, 4), view)


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,batch,bstride", [(512, 512, 3, 512 * 512 + 64), (256, 1024, 2, 256 * 1024 + 4),
                                                  (1024, 4096, 2, 1024 * 4096 + 16), (64, 64, 5, 4100),
                                                  (2048, 2048, 2, 2048 * 2048 + 32)])
def test_2d_row_pitched_views(nx, ny, batch, bstride):
    """2D batches at a padded image stride (executor.py:180-190 allows any
    batch_stride with stride 1; gather -> transform -> scatter), against the
    contiguous path and the oracle, nothing outside the view touched."""
    n = nx * ny
    x, buf, idx = _strided_case(n, batch, 1, bstride, 5)
    t = torch.from_numpy(buf).cuda()
    tc.execute(tc.plan_2d(nx, ny, batch), tc.BatchedTensor(t, batch, n, batch_stride=bstride))
    got = t.cpu().numpy()
    y = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    tc.execute(tc.plan_2d(nx, ny, batch), y)
    assert np.array_equal(got[idx].view(np.uint16), y.cpu().numpy().view(np.uint16))
    gates(got[idx][:2], x[:2], nx, ny)
    mask = np.ones(len(buf), bool)
    mask[idx.reshape(-1)] = False
    assert np.all(got[mask] == np.float16(7.0))
