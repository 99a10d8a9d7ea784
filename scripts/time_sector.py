"""Time the sector (partial) backprojection at 2048^2 against the full log-polar
backprojection on the same inputs (CUDA events, device-resident batch).

usage: python scripts/time_sector.py [--batch 16] [--reps 5] [--sectors 4] [--a 0.25]
"""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1608_03589_b200 as p  # noqa: E402


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
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--sectors", type=int, default=4)
    ap.add_argument("--a", type=float, default=0.25)
    ap.add_argument("--n", type=int, default=2048)
    a = ap.parse_args()
    n, B = a.n, a.batch
    sino = p.synth.config_batch(2, range(B), device="cuda") if n == 2048 else torch.randn(B, n, n, device="cuda")
    k = a.sectors
    sectors = [(i * math.pi / k, math.pi / (2 * k), a.a) for i in range(k)]
    sp = p.SectorPlan(n, n, n, sectors)
    full = p.LogPolarPlan(n, n, n)
    out = torch.empty(B, n, n, device="cuda")
    ms_sec = timed(lambda: sp.execute(sino, out=out, chunk=B), a.reps)
    ms_full = timed(lambda: full.execute(sino, out=out, chunk=B), a.reps)
    print(f"sector x{k} (a_r={a.a}): {1e3 * ms_sec / B:.1f} us/slice   full log-polar BP: {1e3 * ms_full / B:.1f} us/slice")
    for i, inf in enumerate(sp.info):
        print(f"  sector {i}: jc={inf['jc']} nrho={inf['nrho']} L={inf['L']} rho0={inf['rho0']:.4f}")
    # stages of sector 0 and the readout
    work = sp.prepare(0, sino)
    t_prep = timed(lambda: sp.prepare(0, sino), a.reps)
    t_lp = timed(lambda: sp.logpolar(0, work), a.reps)
    print(f"  per sector: prep {1e3 * t_prep / B:.1f} us/slice, log-polar stage {1e3 * t_lp / B:.1f} us/slice; "
          f"readout (rest) ~{1e3 * (ms_sec - k * (t_prep + t_lp)) / B:.1f} us/slice")


if __name__ == "__main__":
    main()
