"""PDL / tail timeline probe (trace build only): per-CTA start, PDL-wait
return and end stamps of each pass of the last execution.

    TCFFT_DEFINES=TCFFT_TRACE python -m paper_2104_11471_b200.build -o /tmp/libtrace.so
    TCFFT_LIB=/tmp/libtrace.so python scripts/trace_probe.py c3
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_11471_b200 as tc  # noqa: E402
from paper_2104_11471_b200 import _lib  # noqa: E402

CFG = {"c1": (1, 256, None, 4096), "c2": (1, 4096, None, 16384), "c3": (1, 1 << 22, None, 64),
       "c4": (2, 512, 512, 1024)}


def main():
    dims, nx, ny, batch = CFG[sys.argv[1] if len(sys.argv) > 1 else "c3"]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    plan = tc.plan_1d(nx, batch) if dims == 1 else tc.plan_2d(nx, ny, batch)
    n = nx * (ny or 1)
    x = (torch.rand((batch, n, 2), device="cuda") * 2 - 1).half()
    y = torch.empty_like(x)
    for _ in range(3):
        tc.execute(plan, x, out=y)
    torch.cuda.synchronize()
    for _ in range(steps):
        tc.execute(plan, x, out=y)
    torch.cuda.synchronize()
    L = _lib.load()
    L.tcfftDebugTrace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
    res = []
    t_min = None
    for i in range(len(plan.passes)):
        buf = np.zeros((4096, 8), dtype=np.uint64)
        g = L.tcfftDebugTrace(plan._handle, i, buf.ctypes.data, buf.nbytes)
        a = buf[:g].astype(np.int64)
        t_min = a[:, 0].min() if t_min is None else min(t_min, a[:, 0].min())
        res.append(a)
    for i, a in enumerate(res):
        st, wt, en = (a[:, 0] - t_min) / 1e3, (a[:, 1] - t_min) / 1e3, (a[:, 2] - t_min) / 1e3
        q = lambda v: [round(float(np.percentile(v, p)), 1) for p in (0, 5, 50, 95, 100)]
        per_sm = np.bincount(a[:, 3], minlength=148)
        ld, m0, so, bw = ((a[:, k] - t_min) / 1e3 for k in (4, 5, 6, 7))
        print(json.dumps({"pass": i, "grid": len(a), "start_us_pctl": q(st), "wait_us_pctl": q(wt), "end_us_pctl": q(en),
                          "ctas_per_sm_min_max": [int(per_sm.min()), int(per_sm.max())],
                          "dur_us_pctl": q(en - wt),
                          "first_chunk": {"load_done": q(ld - wt), "mma0_done": q(m0 - wt), "store_issued": q(so - wt),
                                          "final_wait_start": q(bw - wt)}}))


if __name__ == "__main__":
    main()
