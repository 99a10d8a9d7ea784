"""Quick per-stage timing of the pipeline at a given size (CUDA events, warm)."""
import sys, os, time, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1608_03589_b200 as p
from paper_1608_03589_b200 import _native as N
ap = argparse.ArgumentParser(); ap.add_argument('--n', type=int, default=2048); ap.add_argument('--batch', type=int, default=16); ap.add_argument('--fbp', type=int, default=1)
a = ap.parse_args()
n = a.n
t0 = time.time(); plan = p.LogPolarPlan(n, n, n, filter_spec=(0.0, 1.0) if a.fbp else None); print('plan create s', time.time() - t0, plan.info)
g = torch.randn(a.batch, n, n, device='cuda').cumsum(1) * 0.01
ws_bytes = plan.workspace_bytes(a.batch); ws = torch.empty(ws_bytes, dtype=torch.uint8, device='cuda')
out = torch.empty(a.batch, n, n, device='cuda')
for _ in range(3): plan.execute(g, out=out, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
R = 5
for _ in range(R): plan.execute(g, out=out, workspace=ws)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
print(f'full pipeline: {ms:.3f} ms per batch of {a.batch} -> {ms/a.batch*1000:.1f} us/slice, {a.batch/ms*1000:.0f} slices/s')
