"""Per-stage timing of the pipeline (CUDA events around each launch, warm)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1608_03589_b200 as p

ap = argparse.ArgumentParser()
ap.add_argument('--n', type=int, default=2048); ap.add_argument('--batch', type=int, default=16)
ap.add_argument('--fbp', type=int, default=1); ap.add_argument('--reps', type=int, default=5)
a = ap.parse_args()
n = a.n
t0 = time.time(); plan = p.LogPolarPlan(n, n, n, filter_spec=(0.0, 1.0) if a.fbp else None)
print('plan create s %.2f' % (time.time() - t0))
g = p.synth.config_batch(3 if a.fbp else 2, range(a.batch), torch.device('cuda')) if n == 2048 else torch.randn(a.batch, n, n, device='cuda')
ws = torch.empty(plan.workspace_bytes(a.batch), dtype=torch.uint8, device='cuda')
out = torch.empty(a.batch, n, n, device='cuda')
for _ in range(3): plan.execute(g, out=out, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(a.reps): plan.execute(g, out=out, workspace=ws)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
print(f'full pipeline: {ms:.3f} ms per batch of {a.batch} -> {ms/a.batch*1000:.1f} us/slice, {a.batch/ms*1000:.0f} slices/s')
plan.profile(True)
for _ in range(a.reps): plan.execute(g, out=out, workspace=ws)
st = plan.profile_read(); plan.profile(False)
ab = p.algorithmic_bytes(plan)
for k, v in st.items():
    us = v['ms'] / v['slices'] * 1000
    by = ab[k]['per_slice'] + ab[k]['per_launch'] * v['launches'] / v['slices']
    print(f'  {k:12s} {us:8.1f} us/slice  {by/1e6:8.2f} MB/slice  {by/us/1e3:7.0f} GB/s')
