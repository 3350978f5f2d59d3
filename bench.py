"""Benchmark of the B200 tcFFT hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One "step" = one forward FP16 C2C execute over the whole configured batch
(default C2 = configs[1]: 1D N=4096 x batch 16384, the metric's headline
config that fits one GPU).  Prints ONE JSON line (rank 0).

* value / ms_per_step: device time (CUDA events on the launch stream), inputs
  already resident in HBM, max over ranks; GFLOP/s at 5 N log2 N per transform.
* e2e: the same metric through the public API with HOST (pinned) buffers:
  H2D of the step's input, execute, D2H of the step's spectrum, all timed.
* roofline: dominant kernel's algorithmic HBM bytes (8 B per complex element
  per pass: 4 read + 4 written) / its measured launch time, against the
  measured copy bandwidth in MEASURED_PEAKS.json.
* cpu_baseline (rank 0, N=1): the reference algorithm's CPU restatement
  (oracle/restate.py, bit-identical to the reference) on the host cores, on a
  bounded sample of the same workload.
* --impl reference: times that CPU implementation alone (all host cores).

Multi-GPU (torchrun, one process per GPU): every rank runs the full config on
its own GPU (batch-sharded, no collectives) -> "scaling": "weak".
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c1": dict(dims=1, nx=256, ny=None, batch=4096, name="C1: batched 1D C2C FP16 FFT N=256 batch=4096"),
    "c2": dict(dims=1, nx=4096, ny=None, batch=16384, name="C2: batched 1D C2C FP16 FFT N=4096 batch=16384"),
    "c3": dict(dims=1, nx=1 << 22, ny=None, batch=64, name="C3: 1D C2C FP16 FFT N=2^22 batch=64"),
    "c4": dict(dims=2, nx=512, ny=512, batch=1024, name="C4: batched 2D C2C FP16 FFT 512x512 batch=1024"),
}
METRIC = "FP16 C2C FFT GFLOP/s (5N*log2N/t)"
HOLD_CYCLES = 4_000_000  # ~2 ms spin at 1.9 GHz before each timed region
PROFILE_SUMMARY = ROOT / "profiles" / "ncu_summary.json"


def _flops(cfg) -> float:
    n = cfg["nx"] * (cfg["ny"] or 1)
    return 5.0 * n * math.log2(n) * cfg["batch"]


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# --------------------------------------------------------------- CPU leg
def _cpu_worker(args):
    import numpy as np

    from oracle import restate as R

    cfg, count, seed = args
    n = cfg["nx"] * (cfg["ny"] or 1)
    x = R.random_pairs([seed], count, n)
    t0 = time.perf_counter()
    if cfg["ny"]:
        R.fft2_half(x, cfg["nx"], cfg["ny"])
    else:
        R.fft_half(x)
    return time.perf_counter() - t0, count


def cpu_baseline(cfg, target_s: float = 12.0):
    """Reference algorithm (bit-exact restatement) on all host cores, bounded
    sample sized for ~target_s of CPU work.  Returns dict."""
    import multiprocessing as mp

    import numpy as np  # noqa: F401

    cores = len(os.sched_getaffinity(0))
    n = cfg["nx"] * (cfg["ny"] or 1)
    # calibrate on one transform
    dt, _ = _cpu_worker((cfg, 1, 999))
    per = max(1, int(target_s / max(dt, 1e-4) / cores)) if cores > 1 else max(1, int(target_s / max(dt, 1e-4)))
    per = min(per, max(1, cfg["batch"] // cores))
    per = max(per, 1)
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        res = pool.map(_cpu_worker, [(cfg, per, 1000 + i) for i in range(cores)])
    wall = time.perf_counter() - t0
    transforms = sum(c for _, c in res)
    gflops = 5.0 * n * math.log2(n) * transforms / wall / 1e9
    return {
        "value": gflops,
        "unit": "GFLOP/s",
        "cores": cores,
        "kind": "port",
        "sample": f"{transforms} of {cfg['batch']} transforms ({per} per process x {cores} processes), "
                  f"oracle/restate.py (bit-identical restatement of the reference), wall {wall:.2f} s",
        "seconds_per_transform": wall / transforms * cores,
    }


# --------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self):
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout
                    for line in out.strip().splitlines():
                        f = [x.strip() for x in line.split(",")]
                        self.samples.append(f)
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self, device_index=0):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        rows = [s for s in self.samples if s and s[0] == str(device_index)]
        if not rows:
            return None
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        # median over the samples taken under load (power draw > 300 W), if any
        loaded = [r for r in rows if (num(r[3]) or 0.0) > 300.0]
        sm = [num(r[1]) for r in (loaded or rows) if num(r[1]) is not None]
        smax = max(num(r[2]) for r in rows if num(r[2]) is not None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows), "samples_under_load": len(loaded),
                "power_w_max": max((num(r[3]) or 0.0) for r in rows)}


# --------------------------------------------------------------- GPU leg
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2104_11471_b200 as tc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; TCFFT_BENCH_BACKEND=gloo (test hook) lets several
    # ranks share one GPU to exercise the multi-rank timing path
    backend = os.environ.get("TCFFT_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    if world > 1:
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg)

    n = cfg["nx"] * (cfg["ny"] or 1)
    batch = cfg["batch"]
    elems = n * batch
    plan = tc.plan_1d(cfg["nx"], batch) if cfg["dims"] == 1 else tc.plan_2d(cfg["nx"], cfg["ny"], batch)
    passes = len(plan.passes)
    stream = torch.cuda.current_stream(dev)

    # rotate buffers so that every step's working set exceeds L2
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    step_bytes = elems * 4 * 2
    nbuf = max(1, math.ceil(4 * l2 / step_bytes))
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    ins = [(torch.rand((batch, n, 2), device=dev, generator=g) * 2 - 1).half() for _ in range(nbuf)]
    outs = [torch.empty_like(ins[0]) for _ in range(nbuf)]

    def step(i):
        tc.execute(plan, ins[i % nbuf], out=outs[i % nbuf])

    use_graph = args.graph or (step_bytes < 64 << 20)
    graph = None
    if use_graph:
        reps = nbuf
        for i in range(reps):
            step(i)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):  # captured on torch's side stream, replayed on `stream`
            for i in range(reps):
                step(i)

    def run_steps(k):
        if graph is None:
            for i in range(k):
                step(i)
        else:
            done = 0
            while done < k:
                graph.replay()
                done += nbuf

    steps = args.steps if graph is None else max(args.steps, nbuf) // nbuf * nbuf
    for _ in range(max(args.warmup, 3)):
        run_steps(1 if graph is None else nbuf)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler()
    clk.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # hold the stream for ~2 ms with a spin kernel (outside the timed region)
    # while the host enqueues the K steps: the timed region then measures
    # back-to-back device execution, not the first launch's host latency
    torch.cuda._sleep(HOLD_CYCLES)
    e0.record(stream)
    run_steps(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        t = torch.tensor([ms], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        dist.barrier()

    # per-pass kernel time: each pass launched on its own (tcfftSetPassMask),
    # K launches bracketed by CUDA events on the launch stream; the dominant
    # (slowest) pass is the roofline kernel
    pass_ms = None
    per_pass = None
    if passes == 1:
        pass_ms = ms
    else:
        from paper_2104_11471_b200 import _lib

        L = _lib.load()
        per_pass = []
        for i in range(passes):
            L.tcfftSetPassMask(plan._handle, 1 << i)
            for w in range(2):
                step(w)
            torch.cuda._sleep(HOLD_CYCLES)
            e0.record(stream)
            for j in range(steps):
                step(j)
            e1.record(stream)
            torch.cuda.synchronize()
            per_pass.append(e0.elapsed_time(e1) / steps)
        L.tcfftSetPassMask(plan._handle, 0xFFFFFFFF)
        pass_ms = max(per_pass)
    # e2e: the public host-buffer API (tcfftExecC2CHost via execute_host):
    # pinned host input -> sliced, pipelined H2D / transform / D2H -> pinned
    # host output, all inside the timed region, every step.
    h_in = torch.empty((batch, n, 2) if not args.no_e2e else (1, n, 2), dtype=torch.float16, pin_memory=True)
    h_in.copy_(ins[0][: h_in.shape[0]].cpu())
    h_out = torch.empty_like(h_in, pin_memory=True)
    e2e_steps = max(1, min(args.steps, 5))
    eplan = plan if not args.no_e2e else (tc.plan_1d(cfg["nx"], 1) if cfg["dims"] == 1 else tc.plan_2d(cfg["nx"], cfg["ny"], 1))
    xh = (lambda: tc.execute_host(eplan, h_in, out=h_out)) if hasattr(tc, "execute_host") and not args.no_e2e else (lambda: None)
    xh()  # warm (builds the slice pipeline)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(e2e_steps):
        xh()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    e2e_wall_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = t.item()

    # context for `frac`: a torch copy_ moving the same bytes as one pass
    # (read + write = 8 B/element), L2 flushed before each, best of 10
    copy_gbs = None
    try:
        src_c = torch.empty(elems * 4, dtype=torch.uint8, device=dev)
        dst_c = torch.empty_like(src_c)
        fl = torch.empty(2 * l2, dtype=torch.uint8, device=dev)
        best = 1e30
        for _ in range(10):
            fl.zero_()
            e0.record(stream)
            dst_c.copy_(src_c)
            e1.record(stream)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        copy_gbs = round(elems * 8 / (best * 1e-3) / 1e9, 1)
        del src_c, dst_c, fl
    except Exception:
        copy_gbs = None

    # sustained (measured last, so that the per-pass, e2e and copy figures
    # above see the same idle-start conditions as `value`): ~1 s of
    # back-to-back steps (the 1 kW part settles under its power cap), then the
    # same K-step timed region; the clock record spans the whole measurement
    # (sm_mhz = median of the samples taken under load)
    t_load = time.perf_counter()
    while time.perf_counter() - t_load < 1.0:
        run_steps(1 if graph is None else nbuf)
        torch.cuda.synchronize()
    torch.cuda._sleep(HOLD_CYCLES)
    e0.record(stream)
    run_steps(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_sus = e0.elapsed_time(e1) / steps
    clocks = clk.stop(local)
    if world > 1:
        t = torch.tensor([ms_sus], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_sus = t.item()
    flops = _flops(cfg)
    value = flops * world / (ms * 1e-3) / 1e9
    e2e_val = flops * world / (e2e_ms * 1e-3) / 1e9
    peak, peak_kind = _peaks()
    roof = None
    achieved = elems * 8 / (pass_ms * 1e-3) / 1e9
    traffic = None
    if PROFILE_SUMMARY.exists():
        try:
            prof = json.loads(PROFILE_SUMMARY.read_text()).get(args.config, {})
            traffic = prof.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured"
            else "fallback 6650 GB/s (B200_PROFILING.md)",
            "algorithmic_bytes_per_launch": elems * 8, "same_size_copy_gbs": copy_gbs}
    if per_pass is not None:
        dom = max(range(passes), key=lambda i: per_pass[i])
        roof["kernel"] = f"pass {dom} of {passes} (slowest); per-pass ms {[round(x, 4) for x in per_pass]}"
        roof["per_pass_frac"] = [round(elems * 8 / (x * 1e-3) / 1e9 / peak, 4) for x in per_pass]
        roof["step_frac"] = round(elems * 8 * passes / (ms * 1e-3) / 1e9 / peak, 4)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GFLOP/s", "n_gpus": world, "steps": steps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp16", "data": "synthetic (U[-1,1) fp16 pairs)",
            "config": {"workload": cfg["name"], "dims": cfg["dims"], "nx": cfg["nx"], "ny": cfg["ny"],
                       "batch_per_gpu": batch, "passes": passes,
                       "l2": f"{nbuf} rotating in/out buffer pairs, {nbuf * step_bytes / 2**20:.0f} MiB "
                             f"(>= 4x L2 {l2 / 2**20:.0f} MiB) per cycle",
                       "cuda_graph": graph is not None, "parallelism": f"batch-sharded x{world}"},
            "e2e": {"value": round(e2e_val, 1), "unit": "GFLOP/s", "h2d_bytes_per_step": elems * 4,
                    "d2h_bytes_per_step": elems * 4, "ms_per_step": round(e2e_ms, 4),
                    "wall_ms_per_step": round(e2e_wall_ms, 4),
                    "api": "execute_host -> tcfftExecC2CHost (pinned host in/out, pipelined slices)"},
            "gpu_launches": steps * passes,
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "sustained": {"value": round(flops * world / (ms_sus * 1e-3) / 1e9, 1), "unit": "GFLOP/s",
                          "ms_per_step": round(ms_sus, 5),
                          "note": "same K steps after ~1 s of back-to-back steps (power-capped steady "
                                  "state); `value` is the same region timed from an idle GPU"},
            "hbm_gbs_effective": round(elems * 8 * passes / (ms * 1e-3) / 1e9, 1),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(args, cfg):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    per_step = []
    info = None
    for i in range(max(args.warmup, 0) + args.steps):
        info = cpu_baseline(cfg, target_s=args.ref_seconds)
        if i >= args.warmup:
            per_step.append(info["value"])
    val = statistics.median(per_step)
    n = cfg["nx"] * (cfg["ny"] or 1)
    ms = _flops(cfg) / (val * 1e9) * 1e3
    line = {
        "metric": METRIC, "value": round(val, 4), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp16", "data": "synthetic (U[-1,1) fp16 pairs)",
        "config": {"workload": cfg["name"], "dims": cfg["dims"], "nx": cfg["nx"], "ny": cfg["ny"],
                   "batch_per_gpu": cfg["batch"], "parallelism": "host cores"},
        "impl": "reference",
        "cpu_baseline": {"value": round(val, 4), "unit": "GFLOP/s", "cores": info["cores"], "kind": "port",
                         "sample": info["sample"]},
        "e2e": {"value": round(val, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
