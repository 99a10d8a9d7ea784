"""Per-stage timing (CUDA events, warm) of one plan geometry: python scripts/time_geometry.py NT NTHETA N [BATCH]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1608_03589_b200 as p

nt, nth, n = (int(v) for v in sys.argv[1:4])
batch = int(sys.argv[4]) if len(sys.argv) > 4 else 8
plan = p.LogPolarPlan(nt, nth, n, filter_spec=(0.0, 1.0))
g = torch.randn(batch, nt, nth, device="cuda")
ws = torch.empty(plan.workspace_bytes(batch), dtype=torch.uint8, device="cuda")
out = torch.empty(batch, n, n, device="cuda")
for _ in range(2):
    plan.execute(g, out=out, workspace=ws)
torch.cuda.synchronize()
plan.profile(True)
for _ in range(3):
    plan.execute(g, out=out, workspace=ws)
st = plan.profile_read()
plan.profile(False)
print(f"{nt} x {nth} -> {n}^2, phi_q {plan.info['phi_q']}")
for k, v in st.items():
    print(f"  {k:14s} {v['ms'] / v['slices'] * 1000:8.1f} us/slice")
