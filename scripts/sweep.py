"""C5 size sweep (BASELINE.json configs[4]): 1D N=2^8..2^24 and 2D 256^2..4096^2,
batch chosen so batch*N ~ 2^27 elements (512 MiB in + out, > 4x L2); prints
one JSON line per size (rank 0).

Per size:
* ms / gflops_5nlogn / roofline_frac: one burst of --reps executes timed from
  an idle GPU with CUDA events on the launch stream (barrier + synchronize on
  both sides, max over ranks), as bench.py's `value`;
* sustained: the same burst repeated back to back for ~0.5 s (power-capped
  steady state), median;
* clocks: nvidia-smi SM clock / throttle reasons sampled over both
  (bench.ClockSampler);
* cpu_baseline (rank 0, unless --no-cpu): the reference algorithm's
  bit-identical CPU restatement (oracle/restate.py, kind "port") on all host
  cores, bounded sample of the same size (bench.cpu_baseline).

Multi-GPU (torchrun, one process per GPU, bench.Dist): --scaling strong
(default) gives each rank a contiguous shard of the size's batch
(shard.my_shard), weak the whole batch per rank; no collective on the data
path, value = all ranks' transforms / max over ranks of the device time.

    python scripts/sweep.py [--dims 1|2|both] [--reps 10] [--sizes 8 9 ..] [--no-cpu]
    torchrun --nproc-per-node 8 scripts/sweep.py --scaling strong
"""
import argparse
import json
import math
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (ClockSampler, Dist, cpu_baseline)
import paper_2104_11471_b200 as tc  # noqa: E402
from paper_2104_11471_b200 import shard  # noqa: E402


def run(nx, ny, reps, peak, D, scaling="strong", cpu=True, elems=1 << 27, sustain_s=0.5):
    n = nx * (ny or 1)
    batch = max(1, elems // n)
    if D.world > 1 and scaling == "strong":
        b0, b1 = shard.shard_range(batch, D.rank, D.world)
        mine = b1 - b0
    else:
        mine = batch
    total = mine * D.world if scaling == "weak" or D.world == 1 else batch
    plan = tc.plan_1d(nx, mine) if ny is None else tc.plan_2d(nx, ny, mine)
    x = (torch.rand((mine, n, 2), device=D.dev) * 2 - 1).half()
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream(D.dev)
    for _ in range(3):
        tc.execute(plan, x, out=y)

    def timed():
        torch.cuda.synchronize()
        D.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(bench.HOLD_CYCLES)  # the host enqueues while the stream is held
        e0.record(stream)
        for _ in range(reps):
            tc.execute(plan, x, out=y)
        e1.record(stream)
        torch.cuda.synchronize()
        return D.max(e0.elapsed_time(e1) / reps)

    clk = bench.ClockSampler()
    clk.start()
    time.sleep(0.25)
    ms = timed()
    sus = []
    t_end = time.perf_counter() + sustain_s
    while time.perf_counter() < t_end or len(sus) < 3:
        sus.append(timed())
    clocks = clk.stop(D.local)
    passes = len(plan.passes)
    flop = 5 * n * math.log2(n) * total
    gbs = total * n * 8 * passes / (ms * 1e-3) / 1e9
    ms_s = statistics.median(sus)
    rec = {"dims": 1 if ny is None else 2, "nx": nx, "ny": ny, "batch": total, "batch_per_gpu": mine,
           "n_gpus": D.world, "scaling": scaling if D.world > 1 else "weak", "passes": passes,
           "ms": round(ms, 4), "gflops_5nlogn": round(flop / (ms * 1e-3) / 1e9, 1),
           "hbm_gbs": round(gbs, 1), "roofline_frac": round(gbs / peak, 3),
           "sustained": {"ms": round(ms_s, 4), "gflops_5nlogn": round(flop / (ms_s * 1e-3) / 1e9, 1),
                         "bursts": len(sus)},
           "clocks": clocks}
    del x, y, plan
    if cpu and D.rank == 0:
        cfg = {"dims": rec["dims"], "nx": nx, "ny": ny, "batch": total}
        rec["cpu_baseline"] = bench.cpu_baseline(cfg, target_s=1.0)
        rec["gpu_over_cpu"] = round(rec["gflops_5nlogn"] / max(rec["cpu_baseline"]["value"], 1e-9), 1)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="both")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--sizes", type=int, nargs="*")
    ap.add_argument("--elems-log2", type=int, nargs="*", help="batch sweep: total elements 2^k per size")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong")
    ap.add_argument("--no-cpu", action="store_true", help="skip the per-size CPU baseline")
    a = ap.parse_args()
    peak, _ = bench._peaks()
    D = bench.Dist()
    cpu = not a.no_cpu

    def emit(rec):
        if D.rank == 0:
            print(json.dumps(rec), flush=True)

    if a.elems_log2:
        for k in a.sizes:
            for e in a.elems_log2:
                emit(run(1 << k, None, a.reps, peak, D, a.scaling, cpu, 1 << e))
    else:
        if a.dims in ("1", "both"):
            for k in (a.sizes or range(8, 25)):
                emit(run(1 << k, None, a.reps, peak, D, a.scaling, cpu))
        if a.dims in ("2", "both"):
            for k in (a.sizes or range(8, 13)):
                emit(run(1 << k, 1 << k, a.reps, peak, D, a.scaling, cpu))
    D.close()


if __name__ == "__main__":
    main()
