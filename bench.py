"""Benchmark of the B200 tcFFT hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
                    [--impl ours|reference] [--scaling strong|weak] [--no-nested]

One "step" = one forward FP16 C2C execute over the configured batch.  The
headline workload is C3 (configs[2]: 1D N=2^22 x batch 64, 2^28 elements =
1 GiB, the largest single-GPU configuration, tied with C4, and the multi-pass
path); C1, C2 and C4 are measured in the same run and carried as nested
records under "configs" (same fields: value, roofline.per_pass_frac, clocks,
e2e, cpu_baseline).  Prints ONE JSON line (rank 0).

* value / ms_per_step: device time (CUDA events on the launch stream, K steps
  bracketed by barrier + synchronize), inputs already resident in HBM, max
  over ranks; GFLOP/s at 5 N log2 N per transform, whole job.
* e2e: the same metric through the public API with HOST (pinned) buffers:
  execute_host -> tcfftExecC2CHost, H2D of the step's input, transform, D2H
  of the step's spectrum, all inside the timed region.
* roofline: the slowest pass kernel's algorithmic HBM bytes (8 B per complex
  element per pass: 4 read + 4 written) / its measured launch time (each pass
  launched alone through tcfftSetPassMask), against MEASURED_PEAKS.json.
* cpu_baseline (rank 0): the reference algorithm's CPU restatement
  (oracle/restate.py, bit-identical to the reference: kind "port") on the host
  cores, on a bounded sample of the same workload.
* --impl reference: the UNMODIFIED reference package (baseline/_ref, its
  compiled Cython backend) through its own public API (plan_1d / plan_2d /
  execute on BatchedTensor), on all host cores, same config and metric.

Multi-GPU (torchrun, one process per GPU): --scaling strong (default) shards
the config's batch into contiguous per-rank shards (shard.my_shard; each rank
plans batch/world), --scaling weak runs the full config batch on every rank.
No collective touches the data path; value = all ranks' transforms / max over
ranks of the device time.
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
HEADLINE = "c3"
METRIC = "FP16 C2C FFT GFLOP/s (5N*log2N/t)"
HOLD_CYCLES = 4_000_000  # ~2 ms spin at 1.9 GHz before each timed region
PROFILE_SUMMARY = ROOT / "profiles" / "ncu_summary.json"
REF_DIR = ROOT / "baseline" / "_ref"


def _n(cfg) -> int:
    return cfg["nx"] * (cfg["ny"] or 1)


def _flops_per_transform(cfg) -> float:
    n = _n(cfg)
    return 5.0 * n * math.log2(n)


def _config_dict(key, cfg, world, scaling):
    """The workload description, identical for both arms (implementation
    details live under "impl")."""
    per = cfg["batch"] // world if scaling == "strong" and world > 1 else cfg["batch"]
    return {"workload": cfg["name"], "config_id": key, "dims": cfg["dims"], "nx": cfg["nx"], "ny": cfg["ny"],
            "batch": cfg["batch"] * (world if scaling == "weak" else 1), "batch_per_gpu": per,
            "elements_per_transform": _n(cfg)}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback 6650 GB/s (B200_PROFILING.md)"


# --------------------------------------------------------------- CPU port leg (cpu_baseline)
def _port_worker(args):
    from oracle import restate as R

    cfg, count, seed = args
    x = R.random_pairs([seed], count, _n(cfg))
    t0 = time.perf_counter()
    if cfg["ny"]:
        R.fft2_half(x, cfg["nx"], cfg["ny"])
    else:
        R.fft_half(x)
    return time.perf_counter() - t0, count


def cpu_baseline(cfg, target_s: float = 8.0):
    """The reference algorithm's bit-identical restatement (oracle/restate.py)
    on all host cores, one process per core, on a bounded sample sized for
    ~target_s of wall time.  Throughput = sample flops / sample wall time."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    dt, _ = _port_worker((cfg, 1, 999))  # calibrate on one transform
    per = max(1, min(int(target_s / max(dt, 1e-4)), max(1, cfg["batch"] // cores)))
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        res = pool.map(_port_worker, [(cfg, per, 1000 + i) for i in range(cores)])
    wall = time.perf_counter() - t0
    transforms = sum(c for _, c in res)
    return {
        "value": round(_flops_per_transform(cfg) * transforms / wall / 1e9, 4),
        "unit": "GFLOP/s",
        "cores": cores,
        "kind": "port",
        "sample": f"{transforms} transforms of the workload ({per} per process x {cores} processes), "
                  f"oracle/restate.py (bit-identical restatement of the reference), wall {wall:.2f} s",
        "extrapolated": False,
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
                        self.samples.append([x.strip() for x in line.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.1)

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
        smax = max((num(r[2]) for r in rows if num(r[2]) is not None), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows), "samples_under_load": len(loaded),
                "power_w_max": max((num(r[3]) or 0.0) for r in rows)}


# --------------------------------------------------------------- GPU leg
class Dist:
    """Rank context: one process per GPU (torchrun), NCCL for the timing
    collectives; TCFFT_BENCH_BACKEND=gloo (test hook) lets several ranks share
    one GPU to exercise the multi-rank path."""

    def __init__(self):
        import torch
        import torch.distributed as dist

        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = os.environ.get("TCFFT_BENCH_BACKEND", "nccl")
        if self.backend != "nccl":
            local = local % torch.cuda.device_count()
        self.local = local
        self.dev = torch.device("cuda", local)
        torch.cuda.set_device(self.dev)
        if self.world > 1:
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group(self.backend)
        self.dist = dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64, device=self.dev if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def measure(key, args, D: Dist, headline: bool):
    import torch

    import paper_2104_11471_b200 as tc
    from paper_2104_11471_b200 import _lib
    from paper_2104_11471_b200.shard import shard_range

    cfg = CONFIGS[key]
    world, rank, dev = D.world, D.rank, D.dev
    scaling = args.scaling if world > 1 else "weak"
    n = _n(cfg)
    if scaling == "strong":
        s0, s1 = shard_range(cfg["batch"], rank, world)
        batch = s1 - s0
        total_transforms = cfg["batch"]
    else:
        s0, batch = 0, cfg["batch"]
        total_transforms = cfg["batch"] * world
    elems = n * batch
    plan = tc.plan_1d(cfg["nx"], batch) if cfg["dims"] == 1 else tc.plan_2d(cfg["nx"], cfg["ny"], batch)
    passes = len(plan.passes)
    stream = torch.cuda.current_stream(dev)

    # rotate buffers so that every cycle's working set exceeds 4x L2
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    step_bytes = elems * 4 * 2
    nbuf = max(1, math.ceil(4 * l2 / step_bytes))
    g = torch.Generator(device=dev).manual_seed(1234 + 7 * s0)
    ins = [(torch.rand((batch, n, 2), device=dev, generator=g) * 2 - 1).half() for _ in range(nbuf)]
    outs = [torch.empty_like(ins[0]) for _ in range(nbuf)]

    def step(i):
        tc.execute(plan, ins[i % nbuf], out=outs[i % nbuf])

    # small working sets: replay a CUDA graph of nbuf steps (launch-bound otherwise)
    graph = None
    if args.graph or step_bytes < (64 << 20):
        for i in range(nbuf):
            step(i)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for i in range(nbuf):
                step(i)

    def run_steps(k):
        if graph is None:
            for i in range(k):
                step(i)
        else:
            for _ in range(k // nbuf):
                graph.replay()

    steps = args.steps if graph is None else max(args.steps, nbuf) // nbuf * nbuf
    warm = max(args.warmup, 3)

    def direct_steps(k):
        for i in range(k):
            step(i)

    def timed(k, runner=run_steps):
        """K steps bracketed by barrier + synchronize, CUDA events on the
        launch stream; a spin kernel holds the stream while the host enqueues
        (timed region = back-to-back device execution).  Max over ranks."""
        torch.cuda.synchronize()
        D.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(HOLD_CYCLES)
        e0.record(stream)
        runner(k)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        return D.max(ms)

    for _ in range(warm):
        run_steps(1 if graph is None else nbuf)
    clk = ClockSampler()
    clk.start()
    time.sleep(0.3)
    ms = timed(steps)

    # per-pass kernel times: each pass launched alone (tcfftSetPassMask); the
    # slowest pass is the roofline kernel
    per_pass = [ms]
    if passes > 1:
        L = _lib.load()
        per_pass = []
        for i in range(passes):
            L.tcfftSetPassMask(plan._handle, 1 << i)
            direct_steps(2)
            per_pass.append(timed(args.steps, direct_steps))
        L.tcfftSetPassMask(plan._handle, 0xFFFFFFFF)

    # e2e through the public host-buffer API (pinned host in / out)
    e2e = None
    if not args.no_e2e:
        h_in = torch.empty((batch, n, 2), dtype=torch.float16, pin_memory=True)
        h_in.copy_(ins[0].cpu())
        h_out = torch.empty_like(h_in, pin_memory=True)
        tc.execute_host(plan, h_in, out=h_out)  # warm (builds the slice pipeline)
        e2e_steps = max(1, min(args.steps, 5))
        torch.cuda.synchronize()
        D.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(e2e_steps):
            tc.execute_host(plan, h_in, out=h_out)  # synchronises: the spectrum is on the host
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = D.max(e0.elapsed_time(e1) / e2e_steps)
        e2e_wall = D.max((time.perf_counter() - t0) * 1e3 / e2e_steps)
        e2e = {"value": round(_flops_per_transform(cfg) * total_transforms / (e2e_ms * 1e-3) / 1e9, 1),
               "unit": "GFLOP/s", "h2d_bytes_per_step": elems * 4, "d2h_bytes_per_step": elems * 4,
               "ms_per_step": round(e2e_ms, 4), "wall_ms_per_step": round(e2e_wall, 4), "steps": e2e_steps,
               "api": "execute_host -> tcfftExecC2CHost (pinned host in/out, pipelined H2D / FFT / D2H slices)"}
        del h_in, h_out

    # sustained (headline only, measured last so every figure above sees the
    # same idle-start conditions as `value`): ~1 s of back-to-back steps (the
    # 1 kW part settles under its power cap), then the same K-step region
    sustained = None
    if headline:
        t_load = time.perf_counter()
        while time.perf_counter() - t_load < 1.0:
            run_steps(1 if graph is None else nbuf)
            torch.cuda.synchronize()
        ms_sus = timed(steps)
        sustained = {"value": round(_flops_per_transform(cfg) * total_transforms / (ms_sus * 1e-3) / 1e9, 1),
                     "unit": "GFLOP/s", "ms_per_step": round(ms_sus, 5),
                     "note": "same K steps after ~1 s of back-to-back steps (power-capped steady state); "
                             "`value` is the same region timed from an idle GPU"}
    clocks = clk.stop(D.local)

    peak, peak_src = _peaks()
    dom = max(range(len(per_pass)), key=lambda i: per_pass[i])
    achieved = elems * 8 / (per_pass[dom] * 1e-3) / 1e9
    traffic = None
    if PROFILE_SUMMARY.exists():
        try:
            traffic = json.loads(PROFILE_SUMMARY.read_text()).get(key, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
            "kernel": f"pass {dom} of {passes} (slowest)", "per_pass_ms": [round(x, 5) for x in per_pass],
            "algorithmic_bytes_per_launch": elems * 8,
            "per_pass_frac": [round(elems * 8 / (x * 1e-3) / 1e9 / peak, 4) for x in per_pass],
            "step_frac": round(elems * 8 * passes / (ms * 1e-3) / 1e9 / peak, 4)}
    rec = {
        "value": round(_flops_per_transform(cfg) * total_transforms / (ms * 1e-3) / 1e9, 1),
        "unit": "GFLOP/s", "ms_per_step": round(ms, 5), "steps": steps, "warmup": warm,
        "config": _config_dict(key, cfg, world, scaling),
        "impl": {"passes": passes, "plan": [{k: p[k] for k in ("kind", "N", "E", "chunks", "ctas_per_sm")}
                                            for p in plan.passes],
                 "l2": f"{nbuf} rotating in/out buffer pairs, {nbuf * step_bytes / 2**20:.0f} MiB per cycle "
                       f"(>= 4x L2 {l2 / 2**20:.0f} MiB: inputs larger than L2, no flush needed)",
                 "cuda_graph": graph is not None, "parallelism": f"batch-sharded x{world} ({scaling})"},
        "e2e": e2e, "gpu_launches": steps * passes, "roofline": roof, "clocks": clocks,
        "hbm_gbs_effective": round(elems * 8 * passes / (ms * 1e-3) / 1e9, 1),
    }
    if sustained:
        rec["sustained"] = sustained
    plan.destroy()
    del ins, outs, graph
    torch.cuda.empty_cache()
    return rec


def run_ours(args):
    D = Dist()
    scaling = args.scaling if D.world > 1 else "weak"
    head = measure(args.config, args, D, headline=True)
    nested = {}
    if not args.no_nested:
        for key in sorted(CONFIGS):
            if key != args.config:
                nested[key] = measure(key, args, D, headline=False)
    cpu = {}
    if D.rank == 0 and not args.no_cpu:
        cpu[args.config] = cpu_baseline(CONFIGS[args.config], target_s=args.cpu_seconds)
        for key in nested:
            cpu[key] = cpu_baseline(CONFIGS[key], target_s=max(1.0, args.cpu_seconds / 4))
    if D.rank == 0:
        for key, rec in nested.items():
            rec["cpu_baseline"] = cpu.get(key)
        line = {
            "metric": METRIC, "value": head["value"], "unit": "GFLOP/s", "n_gpus": D.world,
            "steps": head["steps"], "warmup": head["warmup"], "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "fp16",
            "data": "synthetic (U[-1,1) fp16 pairs, seeded)",
            "config": head["config"], "impl": head["impl"], "e2e": head["e2e"],
            "gpu_launches": head["gpu_launches"], "roofline": head["roofline"],
            "cpu_baseline": cpu.get(args.config), "clocks": head["clocks"],
            "sustained": head.get("sustained"), "hbm_gbs_effective": head["hbm_gbs_effective"],
            "configs": nested,
        }
        print(json.dumps(line), flush=True)
    D.close()


# --------------------------------------------------------------- reference arm
_REF = {}


def _ref_init(ref_dir):
    """Worker initialiser: import the unmodified reference package
    (baseline/_ref) with its compiled Cython MMA backend."""
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["TCFFT_BACKEND"] = "ext"
    sys.path.insert(0, ref_dir)
    import tcfft  # the reference package

    _REF["tcfft"] = tcfft


def _ref_task(task):
    """One task: `count` transforms of the workload through the reference's
    own public API (plan_1d / plan_2d, BatchedTensor, execute)."""
    import numpy as np

    tcfft = _REF["tcfft"]
    dims, nx, ny, count, seed = task
    n = nx * (ny or 1)
    rng = np.random.default_rng([2104, seed])
    x = rng.uniform(-1.0, 1.0, size=(count * n, 2)).astype(np.float16)
    data = tcfft.BatchedTensor(x, count, n)
    plan = tcfft.plan_1d(nx, count) if dims == 1 else tcfft.plan_2d(nx, ny, count)
    t0 = time.perf_counter()
    tcfft.execute(plan, data)
    dt = time.perf_counter() - t0
    return dt, count, tcfft.backend.active_backend(), tcfft.__file__


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import multiprocessing as mp

    cfg = CONFIGS[args.config]
    scaling = args.scaling if world > 1 else "weak"
    cores = len(os.sched_getaffinity(0))
    if not (REF_DIR / "tcfft").exists():
        print(json.dumps({"impl": "reference", "unavailable": f"reference not installed in {REF_DIR}"}), flush=True)
        return
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores, initializer=_ref_init, initargs=(str(REF_DIR),)) as pool:
        # warm-up: every worker imports the reference and runs one small task
        # of the workload (one transform) to size the per-task batch
        warm = pool.map(_ref_task, [(cfg["dims"], cfg["nx"], cfg["ny"], 1, 10_000 + i) for i in range(cores)],
                        chunksize=1)
        backend, ref_file = warm[0][2], warm[0][3]
        t_one = statistics.median(w[0] for w in warm)
        per_task = max(1, min(int(args.ref_task_seconds / max(t_one, 1e-4)), max(1, cfg["batch"] // cores)))
        # K steps: every step is one task of `per_task` transforms; the tasks
        # run concurrently on all host cores (a process per core), so the
        # timed queue is padded to a multiple of the core count (every core
        # busy until the end) and ms_per_step is the wall time / K
        tasks = cores * math.ceil(args.steps / cores)
        jobs = [(cfg["dims"], cfg["nx"], cfg["ny"], per_task, i) for i in range(tasks)]
        t0 = time.perf_counter()
        res = pool.map(_ref_task, jobs, chunksize=1)
        wall = time.perf_counter() - t0
    transforms = sum(r[1] for r in res)
    val = _flops_per_transform(cfg) * transforms / wall / 1e9
    sample = (f"{tasks} tasks x {per_task} transform(s) = {transforms} transforms of the workload "
              f"(batch {cfg['batch']}), one reference process per host core ({cores}), "
              f"reference tcfft.execute ({backend} backend, {ref_file}), timed wall {wall:.1f} s; "
              f"warm-up: one 1-transform task per process")
    line = {
        "metric": METRIC, "value": round(val, 4), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": 1, "ms_per_step": round(wall * 1e3 / args.steps, 1), "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "fp16", "data": "synthetic (U[-1,1) fp16 pairs, seeded)",
        "config": _config_dict(args.config, cfg, world, scaling),
        "impl": "reference",
        "cpu_baseline": {"value": round(val, 4), "unit": "GFLOP/s", "cores": cores, "kind": "reference",
                         "sample": sample, "extrapolated": False},
        "e2e": {"value": round(val, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "seconds_per_transform_per_core": round(wall * cores / transforms, 3),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=HEADLINE, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-nested", action="store_true", help="measure only --config")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--ref-task-seconds", type=float, default=2.0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
