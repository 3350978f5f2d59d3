"""Multi-device execution of one batch (paper_2104_11471_b200.multi) and the
multi-rank bench path (strong-scaling shards, torchrun).

One GPU is available in this pool, so the device lists repeat cuda:0 (two
shards, two streams, two plans on one GPU): the sharding, stream ordering and
host-slice addressing are the same code a multi-GPU box runs."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2104_11471_b200 as tc  # noqa: E402
from paper_2104_11471_b200 import multi  # noqa: E402
from oracle import restate as R  # noqa: E402
from tests._parity import gates  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent


def test_plan_many_shards_cover_batch_cpu_only():
    # pure host logic: shard ranges of a MultiPlan are contiguous and balanced
    from paper_2104_11471_b200.shard import shard_range

    b, d = 1001, 3
    r = [shard_range(b, i, d) for i in range(d)]
    assert r[0][0] == 0 and r[-1][1] == b and all(r[i][1] == r[i + 1][0] for i in range(d - 1))
    assert max(e - s for s, e in r) - min(e - s for s, e in r) <= 1


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,batch,devs", [(4096, None, 101, [0, 0]), (1 << 16, None, 3, [0, 0, 0]),
                                                (512, 512, 6, [0, 0]), (256, None, 2, [0, 0, 0])])
def test_execute_many_matches_single_plan(nx, ny, batch, devs):
    total = nx * (ny or 1)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = (torch.rand((batch, total, 2), device="cuda", generator=g) * 2 - 1).half()
    ref = torch.empty_like(x)
    tc.execute(tc.plan_1d(nx, batch) if ny is None else tc.plan_2d(nx, ny, batch), x, out=ref)
    mp = multi.plan_many(nx, batch, devs, ny=ny)
    parts = [x[s:e].clone() for s, e in mp.shards]
    multi.execute_many(mp, parts)
    torch.cuda.synchronize()
    got = torch.cat(parts)
    assert torch.equal(got.view(torch.int16), ref.view(torch.int16))
    # host path: one pinned batch, every slot transforms its slice
    h = x.cpu().pin_memory()
    ho = torch.empty_like(h).pin_memory()
    multi.execute_many_host(mp, h, out=ho)
    assert torch.equal(ho.view(torch.int16), ref.cpu().view(torch.int16))
    xs = x[:2].cpu().numpy()
    gates(ho[:2].numpy(), xs, nx, ny)
    mp.destroy()


@pytest.mark.gpu
def test_bench_two_ranks_strong_scaling_json():
    """bench.py under torchrun with 2 ranks (gloo timing collectives, both
    ranks on the one GPU): strong scaling shards the config batch."""
    env = dict(os.environ, TCFFT_BENCH_BACKEND="gloo", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", str(ROOT / "bench.py"), "--gpus", "2",
           "--config", "c2", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-nested", "--no-e2e"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["batch"] == 16384 and d["config"]["batch_per_gpu"] == 8192
    assert d["value"] > 0 and d["gpu_launches"] == d["steps"]


@pytest.mark.gpu
def test_sweep_one_size_json_with_cpu_baseline_and_clocks():
    """scripts/sweep.py (C5): one JSON line per size with the burst and
    sustained device figures, the clock record and the per-size CPU baseline."""
    cmd = [sys.executable, str(ROOT / "scripts" / "sweep.py"), "--dims", "1", "--sizes", "10", "--reps", "3"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    d = json.loads([l for l in res.stdout.splitlines() if l.startswith("{")][0])
    assert d["nx"] == 1024 and d["n_gpus"] == 1 and d["batch"] == (1 << 27) // 1024
    assert d["gflops_5nlogn"] > 0 and d["sustained"]["gflops_5nlogn"] > 0 and d["sustained"]["bursts"] >= 3
    assert d["clocks"] is None or "sm_mhz" in d["clocks"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] > 0


@pytest.mark.gpu
def test_sweep_two_ranks_strong_scaling_json():
    """scripts/sweep.py under torchrun with 2 ranks (gloo timing collectives,
    both ranks on the one GPU): strong scaling shards each size's batch."""
    env = dict(os.environ, TCFFT_BENCH_BACKEND="gloo", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29519", str(ROOT / "scripts" / "sweep.py"),
           "--dims", "2", "--sizes", "8", "--reps", "3", "--no-cpu"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["batch"] == (1 << 27) // 65536 and d["batch_per_gpu"] == d["batch"] // 2
    assert "cpu_baseline" not in d
