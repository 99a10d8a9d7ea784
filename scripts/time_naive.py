"""Time the direct O(n^2 ntheta) backprojector at config-4 size and its LP gap."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1608_03589_b200 as p
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
x = p.synth.config_batch(4, range(B), torch.device("cuda"))
for _ in range(2): p.backproject_naive_batch(x, 2048)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); nv = p.backproject_naive_batch(x, 2048); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"naive: {ms/B:.3f} ms/slice  {B/ms*1000:.1f} slices/s  {2048**3/(ms/B*1e-3)/1e9:.1f} Glerp/s")
lp = p.logpolar_backproject_batch(x, 2048)
xs = -1.0 + (np.arange(2048) + 0.5) * (2.0 / 2048)
X, Y = np.meshgrid(xs, xs); disk = torch.from_numpy(np.hypot(X, Y) <= 1.0).cuda()
d = (lp - nv)[:, disk]; r = (d.norm() / nv[:, disk].norm()).item()
print(f"LP vs direct rel-L2 in unit disk: {r:.3e}")
