"""Mixed-radix row-DFT smoke over several angle counts, with LPBP_MIXED=1 / 0 (Bluestein) and
CUDA_LAUNCH_BLOCKING=1 so a failing kernel names its stage: python scripts/dbg_mixed.py."""
import os, sys, subprocess
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1608_03589_b200 as p
nth = int(sys.argv[1]); nt, n = 96, 64
g = torch.randn(1, nt, nth, device="cuda")
try:
    plan = p.get_plan(nt, nth, n, None, None, None)
    out = plan.execute(g); torch.cuda.synchronize()
    print(nth, "ok", plan.info["phi_q"], plan.info["L"], float(out.abs().max()))
except Exception as e:
    print(nth, "FAIL", str(e)[:200])
'''
for mixed in ("1", "0"):
    for nth in (768, 1280, 1536, 2304, 2560, 3200, 3840):
        env = dict(os.environ, LPBP_MIXED=mixed, CUDA_LAUNCH_BLOCKING="1")
        r = subprocess.run([sys.executable, "-c", code, str(nth)], env=env, capture_output=True, text=True)
        print("mixed", mixed, r.stdout.strip(), r.stderr.strip()[-300:] if r.returncode else "")
