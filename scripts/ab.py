"""Interleaved A/B of env variants on bench.py configs (device time only).

    python scripts/ab.py --configs c2 c1 --variants "TCFFT_PDL=0" "TCFFT_PDL=1" --rounds 3
Also times a same-size torch copy (read+write bytes = the pass's traffic).
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(cfg, env, steps):
    e = dict(os.environ, TCFFT_EXPERIMENTS="1")
    for kv in env.split():
        k, v = kv.split("=", 1)
        e[k] = v
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", str(steps),
                          "--warmup", "5", "--no-cpu", "--no-e2e", "--no-nested"], capture_output=True, text=True, env=e, cwd=ROOT)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
        return d["value"], d["ms_per_step"]
    except Exception:
        return None, out.stderr[-300:]


def copy_time(nbytes):
    import torch
    a = torch.empty(nbytes // 2, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    best = 1e9
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["c2"])
    ap.add_argument("--variants", nargs="+", required=True)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--copy-bytes", type=int, nargs="*", default=[])
    a = ap.parse_args()
    res = {}
    for r in range(a.rounds):
        for c in a.configs:
            for v in a.variants:
                val, ms = run(c, v, a.steps)
                res.setdefault((c, v), []).append(val)
                print(f"round {r} {c} [{v}] {val} {ms}", flush=True)
    for (c, v), vals in res.items():
        ok = [x for x in vals if x]
        print(json.dumps({"config": c, "variant": v, "values": ok, "mean": round(sum(ok) / max(1, len(ok)), 1)}))
    for nb in a.copy_bytes:
        ms = copy_time(nb)
        print(json.dumps({"copy_bytes": nb, "ms": round(ms, 4), "gbs": round(nb / (ms * 1e-3) / 1e9, 1)}))


if __name__ == "__main__":
    main()
