"""Small executions covering every pass-kernel family the planner emits, for
compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python scripts/sanitize.py [--quick]

Covers: 1D single-pass rows 2..16384 (swizzled, unswizzled 4..16-point rows,
padded-pitch 64..1024, small-batch 2048-element chunks, one-CTA-per-SM
two-warpgroup 16384), pipelined 1024 rows, ticketed (dynamic) chunk
scheduling, four-step 2^15..2^18, two-pass blocked 2^19..2^22, three-step
2^23 / 2^25, 2D rows + column strips (3D / 4D boxes, 256-column strips for
nx <= 8, radix-64 strips), 2D split columns (nx >= 8192) and multi-pass rows
(ny > 16384), the distributed plan's two passes + unpack (one rank),
out-of-place, host-buffer pipeline, strided views."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_11471_b200 as tc  # noqa: E402


def run(nx, ny, batch, oop=False):
    n = nx * (ny or 1)
    x = (torch.rand((batch, n, 2), device="cuda") * 2 - 1).half()
    plan = tc.plan_1d(nx, batch) if ny is None else tc.plan_2d(nx, ny, batch)
    if oop:
        y = torch.empty_like(x)
        tc.execute(plan, x, out=y)
    else:
        y = tc.execute(plan, x)
    torch.cuda.synchronize()
    assert torch.isfinite(y.float()).all().item(), (nx, ny, batch)
    plan.destroy()
    print("ok", nx, ny, batch, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--views", action="store_true", help="only the strided-view cases")
    a = ap.parse_args()
    if a.views:
        views()
        return
    cases = [(n, None, b) for n, b in [(2, 1024), (4, 512), (4, 3), (8, 257), (16, 33), (32, 64), (64, 64),
                                        (128, 40), (256, 16), (256, 4096), (512, 24), (1024, 12), (1024, 200),
                                        (2048, 8), (4096, 4), (4096, 4096), (8192, 4), (16384, 4)]]
    cases += [(1 << k, None, 2) for k in range(15, 19)]
    cases += [(1 << k, None, 1) for k in range(19, 23 if not a.quick else 20)]
    cases += [(16, 16, 3), (64, 32, 2), (8, 256, 2), (2, 4096, 1), (512, 512, 2), (1024, 1024, 1),
              (2048, 2048, 1), (256, 256, 64)]
    if not a.quick:
        cases += [(4096, 4096, 1)]
    cases += [(1 << 23, None, 1), (8192, 16, 1), (16384, 64, 1), (16, 32768, 1)]
    if not a.quick:
        cases += [(1 << 25, None, 1)]
    for c in cases:
        run(*c)
    # distributed single transform, one rank: pass 0, unpack, pass 1
    from paper_2104_11471_b200.dist import DistPlan

    for nx in (1 << 14, 1 << 20):
        dp = DistPlan(nx)
        out = dp.execute((torch.rand((dp.slab_shape[0], dp.slab_shape[1], 2), device="cuda") * 2 - 1).half())
        torch.cuda.synchronize()
        assert torch.isfinite(out.float()).all().item()
        print("ok dist", nx, flush=True)
    run(4096, None, 64, oop=True)
    # host-buffer pipeline (several slices) and a strided view (scratch path)
    plan = tc.plan_1d(4096, 2048)
    h = (torch.rand((2048, 4096, 2)) * 2 - 1).half().pin_memory()
    tc.execute_host(plan, h)
    views()
    print("sanitize cases done", flush=True)


def views():
    # general view (gather / scatter), padded-pitch bulk copies, row-pitched
    # 3D tensor maps (full and partial last chunk)
    wide = torch.zeros((8, 2 * 4096, 2), device="cuda", dtype=torch.float16)
    v = tc.BatchedTensor(wide.view(-1, 2), 8, 4096, stride=2, batch_stride=2 * 4096)
    tc.execute(tc.plan_1d(4096, 8), v)
    for n, b, bs in ((1024, 4, 1100), (4096, 5, 4100), (32, 300, 36), (256, 10001, 260), (8192, 3, 8200)):
        pv = tc.BatchedTensor((torch.rand((b * bs, 2), device="cuda") * 2 - 1).half(), b, n, batch_stride=bs)
        tc.execute(tc.plan_1d(n, b), pv)
        torch.cuda.synchronize()
        print("ok view", n, b, bs, flush=True)


if __name__ == "__main__":
    main()
