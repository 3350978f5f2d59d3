"""C5 size sweep (BASELINE.json configs[4]): 1D N=2^8..2^24 and 2D 256^2..4096^2,
batch chosen so batch*N ~ 2^27 elements (512 MiB in + out, > 4x L2), device
time with CUDA events; prints one JSON line per size.

    python scripts/sweep.py [--dims 1|2|both] [--reps 10]
"""
import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_11471_b200 as tc  # noqa: E402


def run(nx, ny, reps, peak, elems=1 << 27):
    n = nx * (ny or 1)
    batch = max(1, elems // n)
    plan = tc.plan_1d(nx, batch) if ny is None else tc.plan_2d(nx, ny, batch)
    x = (torch.rand((batch, n, 2), device="cuda") * 2 - 1).half()
    y = torch.empty_like(x)
    for _ in range(3):
        tc.execute(plan, x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        tc.execute(plan, x, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    passes = len(plan.passes)
    gbs = batch * n * 8 * passes / (ms * 1e-3) / 1e9
    return {"dims": 1 if ny is None else 2, "nx": nx, "ny": ny, "batch": batch, "passes": passes,
            "ms": round(ms, 4), "gflops_5nlogn": round(5 * n * math.log2(n) * batch / (ms * 1e-3) / 1e9, 1),
            "hbm_gbs": round(gbs, 1), "roofline_frac": round(gbs / peak, 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="both")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--sizes", type=int, nargs="*")
    ap.add_argument("--elems-log2", type=int, nargs="*", help="batch sweep: total elements 2^k per size")
    a = ap.parse_args()
    peak = 6549.4
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peak = json.load(open(p))["hbm_gbs"]
    if a.elems_log2:
        for k in a.sizes:
            for e in a.elems_log2:
                print(json.dumps(run(1 << k, None, a.reps, peak, 1 << e)), flush=True)
        return
    if a.dims in ("1", "both"):
        for k in (a.sizes or range(8, 25)):
            print(json.dumps(run(1 << k, None, a.reps, peak)), flush=True)
    if a.dims in ("2", "both"):
        for k in (a.sizes or range(8, 13)):
            print(json.dumps(run(1 << k, 1 << k, a.reps, peak)), flush=True)


if __name__ == "__main__":
    main()
