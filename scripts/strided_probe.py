"""Strided BatchedTensor views: device time of the same
transform on a contiguous batch, on a row-pitched view (batch_stride = N + 4:
row-pitched tensor maps / padded-pitch bulk copies, one HBM pass) and on a
general view (stride 2: gather -> transform -> scatter).  One JSON line per
case: ms and the HBM fraction of the FFT's own passes (8 B per element per
pass; the general view's gather / scatter copies come on top).

    python scripts/strided_probe.py
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2104_11471_b200 as tc  # noqa: E402


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(bench.HOLD_CYCLES)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    peak, _ = bench._peaks()
    cases = [((n, None), b) for n, b in ((4096, 16384), (2048, 32768), (256, 262144), (1024, 65536),
                                          (1 << 16, 1024), (1 << 22, 16))]
    cases += [((512, 512), 256), ((2048, 2048), 16)]
    for (nx, ny), batch in cases:
        n = nx * (ny or 1)
        plan = tc.plan_1d(nx, batch) if ny is None else tc.plan_2d(nx, ny, batch)
        views = (("contiguous", 1, n), ("row-pitched", 1, n + 4), ("general", 2, 2 * n + 4))
        if ny:  # 2D: stride 1 only (executor.py:180-181); the general case is an unaligned pitch
            views = (("contiguous", 1, n), ("row-pitched", 1, n + 4), ("general", 1, n + 2))
        for name, stride, bstride in views:
            total = bstride * (batch - 1) + stride * (n - 1) + 1
            t = (torch.rand((total, 2), device="cuda") * 2 - 1).half()
            if name == "contiguous":
                ms = timed(lambda: tc.execute(plan, t))
            else:
                v = tc.BatchedTensor(t, batch, n, stride=stride, batch_stride=bstride)
                ms = timed(lambda: tc.execute(plan, v))
            gbs = batch * n * 8 * len(plan.passes) / (ms * 1e-3) / 1e9
            print(json.dumps({"nx": nx, "ny": ny, "batch": batch, "view": name, "stride": stride, "batch_stride": bstride,
                              "passes": len(plan.passes), "ms": round(ms, 4),
                              "hbm_gbs_fft_passes": round(gbs, 1), "frac": round(gbs / peak, 3)}), flush=True)
            del t


if __name__ == "__main__":
    main()
