"""Small end-to-end run of every kernel for compute-sanitizer (memcheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1608_03589_b200 as p
from oracle import phantoms
g0 = torch.from_numpy(np.stack([phantoms.config_sinogram(0, i) for i in range(3)])).cuda()
g1 = torch.from_numpy(np.stack([phantoms.config_sinogram(1, i) for i in range(2)])).cuda()
for n in (256, 255, 64):
    p.logpolar_backproject_batch(g0, n)
p.logpolar_backproject_batch(g0, 256, p.LogPolarOptions(rho0=-0.1, nrho=40))
plan = p.get_plan(512, 512, 512, None, None, (0.0, 1.0))
plan.execute(g1, chunk=1); plan.filter(g1); lp = plan.logpolar(g1); plan.readout(lp)
plan.execute_host(g1.cpu().numpy(), chunk=1)
p.backproject_naive_batch(g0, 200)
p.VolumeReconstructor(256, 256, 256, devices=[0, 0]).run(g0.cpu().numpy())
# K3 with its TMEM-held operands (L = 4096 at 1024^2) and the mixed-radix row DFTs (nphi = 1536 = 3 x 512,
# 2560 = 5 x 512, 6400 = 25 x 256) in both directions
g2 = torch.randn(2, 1024, 1024, device="cuda")
p.get_plan(1024, 1024, 1024, None, None, (0.0, 1.0)).execute(g2)
for nth in (768, 1280, 3200):
    gm = torch.randn(2, 96, nth, device="cuda")
    p.get_plan(96, nth, 64, None, None, (0.0, 1.0)).execute(gm)
torch.cuda.synchronize()
print("sanitize run ok")
