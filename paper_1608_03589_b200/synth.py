"""Seeded synthetic sinograms generated on the device (benchmark harness).

Ellipse parameters are drawn on the host exactly as documented in
oracle/phantoms.py (numpy Generator(PCG64(seed)); u, v, a, b, tilt, rho in that
order), and the exact line integrals (fastbp radon.py:38-61) are evaluated in
fp64 by liblpbp's lpbp_radon_ellipses kernel.  Gaussian noise (sigma = noise *
max g) comes from torch's device generator seeded per slice, so noisy device
sinograms are statistically — not bitwise — identical to oracle/phantoms'."""

from __future__ import annotations

import math
from ctypes import c_void_p

import numpy as np
import torch

from ._native import check, lib

CONFIGS = {
    0: dict(nt=256, ntheta=256, n=256, k=10, amin=0.05, amax=0.35, noise=0.0, fbp=False, slices=1),
    1: dict(nt=512, ntheta=512, n=512, k=20, amin=0.05, amax=0.35, noise=0.01, fbp=True, slices=16),
    2: dict(nt=2048, ntheta=2048, n=2048, k=50, amin=0.01, amax=0.3, noise=0.01, fbp=False, slices=64),
    3: dict(nt=2048, ntheta=2048, n=2048, k=50, amin=0.01, amax=0.3, noise=0.01, fbp=True, slices=2048),
    4: dict(nt=2048, ntheta=2048, n=2048, k=50, amin=0.01, amax=0.3, noise=0.01, fbp=False, slices=64),
}
BASE_SEED = 20261019


def ellipse_params(seed: int, k: int, amin: float, amax: float) -> np.ndarray:
    """[k][6] = (cx, cy, a, b, tilt, rho)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    u = rng.random(k)
    v = rng.random(k)
    rad = 0.6 * np.sqrt(u)
    a = rng.uniform(amin, amax, k)
    b = rng.uniform(amin, amax, k)
    tilt = rng.uniform(0.0, math.pi, k)
    rho = rng.uniform(-0.5, 1.0, k)
    return np.stack([rad * np.cos(2.0 * math.pi * v), rad * np.sin(2.0 * math.pi * v), a, b, tilt, rho], axis=1)


def radon_ellipses(params: np.ndarray, nt: int, ntheta: int, device) -> torch.Tensor:
    """params [B][k][6] -> noiseless float32 sinograms [B][nt][ntheta] on `device`."""
    params = np.ascontiguousarray(params, dtype=np.float64)
    bsz, k, _ = params.shape
    dp = torch.from_numpy(params).to(device)
    out = torch.empty((bsz, nt, ntheta), dtype=torch.float32, device=device)
    with torch.cuda.device(device):
        check(lib().lpbp_radon_ellipses(c_void_p(dp.data_ptr()), k, nt, ntheta, bsz, c_void_p(out.data_ptr()),
                                        c_void_p(torch.cuda.current_stream(device).cuda_stream)))
    return out


def config_batch(cfg: int, slice_ids, device, gen_chunk: int = 64) -> torch.Tensor:
    """Sinograms of config `cfg` for the given global slice indices (seed = BASE_SEED
    + 7919*cfg + index, as oracle/phantoms.config_sinogram)."""
    c = CONFIGS[cfg]
    ids = list(slice_ids)
    out = torch.empty((len(ids), c["nt"], c["ntheta"]), dtype=torch.float32, device=device)
    for lo in range(0, len(ids), gen_chunk):
        part = ids[lo:lo + gen_chunk]
        seeds = [BASE_SEED + 7919 * cfg + i for i in part]
        prm = np.stack([ellipse_params(s, c["k"], c["amin"], c["amax"]) for s in seeds])
        g = radon_ellipses(prm, c["nt"], c["ntheta"], device)
        if c["noise"] > 0:
            for j, s in enumerate(seeds):
                gen = torch.Generator(device=device)
                gen.manual_seed(s)
                noise = torch.randn(g.shape[1:], generator=gen, device=device, dtype=torch.float32)
                g[j].add_(noise, alpha=float(c["noise"] * g[j].max()))
        out[lo:lo + len(part)] = g
    return out
