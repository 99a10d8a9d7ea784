"""Time the BST engine (fbp default) at 2048^2 against the log-polar FBP on the same
batch (CUDA events, device-resident).  usage: python scripts/time_bst.py [--batch 8] [--n 2048]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1608_03589_b200 as p  # noqa: E402
from oracle import fastbp_oracle as O  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    B = a.batch
    sino = p.synth.config_batch(3, range(B), device="cuda")
    bst = p.BstPlan(2048, 2048, p.BstOptions(n_out=2048), filter_spec=(0.0, 1.0))
    lp = p.LogPolarPlan(2048, 2048, 2048, filter_spec=(0.0, 1.0))
    out = torch.empty(B, 2048, 2048, device="cuda")
    t_bst = timed(lambda: bst.execute(sino, out=out, chunk=B), a.reps)
    t_lp = timed(lambda: lp.execute(sino, out=out, chunk=B), a.reps)
    print(f"fbp bst: {1e3 * t_bst / B:.1f} us/slice   fbp logpolar: {1e3 * t_lp / B:.1f} us/slice   "
          f"(L={bst.info['L']}, m_need={bst.info['m_need']}, big={bst.info['big']})")
    if a.check:
        img = bst.execute(sino[:1])[0].cpu().numpy()
        ref = O.fbp_bst(sino[0].double().cpu().numpy(), 2048)
        print(f"fbp bst 2048 vs oracle: rel_l2 {O.relative_l2(img, ref):.3e}")


if __name__ == "__main__":
    main()
