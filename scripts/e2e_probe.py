import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1608_03589_b200 as p
N = 64
hin = torch.empty((N, 2048, 2048), dtype=torch.float32, pin_memory=True); hin.normal_()
hout = torch.empty((N, 2048, 2048), dtype=torch.float32, pin_memory=True)
d_in = torch.empty((16, 2048, 2048), device="cuda"); d_out = torch.empty_like(d_in)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def copies():
    for k in range(0, N, 16):
        with torch.cuda.stream(s1): d_in.copy_(hin[k:k+16], non_blocking=True)
        with torch.cuda.stream(s2): hout[k:k+16].copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
copies(); t = time.perf_counter(); copies(); dt = time.perf_counter() - t
print(f"raw concurrent H2D+D2H: {N*16.78e6/dt/1e9:.1f} GB/s each way -> {N/dt:.0f} slices/s ceiling")
def h2d():
    for k in range(0, N, 16): d_in.copy_(hin[k:k+16], non_blocking=True)
    torch.cuda.synchronize()
h2d(); t = time.perf_counter(); h2d(); dt = time.perf_counter() - t
print(f"H2D alone: {N*16.78e6/dt/1e9:.1f} GB/s")
plan = p.get_plan(2048, 2048, 2048, None, None, (0.0, 1.0))
for ch in (4, 8, 16):
    plan.execute_host(hin, hout, chunk=ch)
    t = time.perf_counter()
    for _ in range(2): plan.execute_host(hin, hout, chunk=ch)
    dt = (time.perf_counter() - t) / 2
    print(f"execute_host chunk={ch}: {N/dt:.0f} slices/s")
