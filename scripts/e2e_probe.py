import torch, time, sys, os
sys.path.insert(0, '.')
import paper_2104_11471_b200 as tc
n, b = 4096, 16384
plan = tc.plan_1d(n, b)
h = torch.empty((b, n, 2), dtype=torch.float16, pin_memory=True); h.uniform_(-1, 1)
o = torch.empty_like(h, pin_memory=True)
for _ in range(2): tc.execute_host(plan, h, out=o)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5): tc.execute_host(plan, h, out=o)
dt = (time.perf_counter() - t) / 5
d = torch.empty(b, n, 2, dtype=torch.float16, device='cuda')
t = time.perf_counter()
for _ in range(5): d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); h2d = (time.perf_counter() - t) / 5
t = time.perf_counter()
for _ in range(5): o.copy_(d, non_blocking=True)
torch.cuda.synchronize(); d2h = (time.perf_counter() - t) / 5
print(f"slice {os.environ.get('TCFFT_SLICE_MB','32')} MB: e2e {dt*1e3:.2f} ms  ({5*n*12*b/dt/1e9:.0f} GFLOP/s)  h2d {256/1024/h2d:.1f} GB/s  d2h {256/1024/d2h:.1f} GB/s")
