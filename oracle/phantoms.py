"""Seeded synthetic inputs for the benchmark configurations (TEST/BENCH HARNESS).

The reference has no random-ellipse generator and no Gaussian noise model
(SURVEY §0 finding 9); both are defined here on top of the reference's exact
ellipse line integral (radon.py:38-61, restated in radon_ellipses below).

Draw order (numpy.random.Generator(PCG64(seed)), one call per quantity, each of
shape (K,)):
  u = random(K); v = random(K)           -> centre 0.6*sqrt(u)*(cos 2 pi v, sin 2 pi v)
  a = uniform(amin, amax, K); b = uniform(amin, amax, K)     semi-axes
  tilt = uniform(0, pi, K); rho = uniform(-0.5, 1.0, K)      tilt, density
Noise (configs 1-4): a second Generator(PCG64(seed + NOISE_SEED_OFFSET)) draws
standard_normal((nt, ntheta)) * 0.01 * max(g).  The sinogram is then rounded
to float32; the oracle receives those float32 values upcast to float64.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

NOISE_SEED_OFFSET = 1_000_003


@dataclass(frozen=True)
class EllipseParams:
    cx: np.ndarray
    cy: np.ndarray
    a: np.ndarray
    b: np.ndarray
    tilt: np.ndarray
    rho: np.ndarray


def random_ellipses(seed: int, k: int, amin: float, amax: float) -> EllipseParams:
    rng = np.random.Generator(np.random.PCG64(seed))
    u = rng.random(k)
    v = rng.random(k)
    rad = 0.6 * np.sqrt(u)
    cx = rad * np.cos(2.0 * math.pi * v)
    cy = rad * np.sin(2.0 * math.pi * v)
    a = rng.uniform(amin, amax, k)
    b = rng.uniform(amin, amax, k)
    tilt = rng.uniform(0.0, math.pi, k)
    rho = rng.uniform(-0.5, 1.0, k)
    return EllipseParams(cx, cy, a, b, tilt, rho)


def radon_ellipses(e: EllipseParams, nt: int, ntheta: int) -> np.ndarray:
    """Exact line integrals of an additive ellipse phantom (radon.py:38-61):
    2 rho A B sqrt(w^2 - tau^2) / w^2 with tau = t - c.xi, w^2 = A^2 cos^2(theta-gamma)
    + B^2 sin^2(theta-gamma); t_i = -1 + 2i/nt, theta_j = j pi/ntheta."""
    t = (-1.0 + np.arange(nt) * (2.0 / nt))[:, None]
    th = (np.arange(ntheta) * (math.pi / ntheta))[None, :]
    out = np.zeros((nt, ntheta))
    for i in range(len(e.a)):
        ang = th - e.tilt[i]
        w2 = (e.a[i] * np.cos(ang)) ** 2 + (e.b[i] * np.sin(ang)) ** 2
        tau = t - (e.cx[i] * np.cos(th) + e.cy[i] * np.sin(th))
        under = w2 - tau ** 2
        out += np.where(under > 0.0, 2.0 * e.rho[i] * e.a[i] * e.b[i] * np.sqrt(np.maximum(under, 0.0)) / w2, 0.0)
    return out


def sinogram(seed: int, nt: int, ntheta: int, k: int, amin: float, amax: float, noise: float) -> np.ndarray:
    """float32 sinogram [nt][ntheta] of a seeded random-ellipse phantom plus
    Gaussian noise with sigma = noise * max(g)."""
    g = radon_ellipses(random_ellipses(seed, k, amin, amax), nt, ntheta)
    if noise > 0:
        rng = np.random.Generator(np.random.PCG64(seed + NOISE_SEED_OFFSET))
        g = g + rng.standard_normal(g.shape) * (noise * float(np.max(g)))
    return g.astype(np.float32)


# BASELINE.json configs: (nt, ntheta, n, K, amin, amax, noise, filter)
CONFIGS = {
    0: dict(nt=256, ntheta=256, n=256, k=10, amin=0.05, amax=0.35, noise=0.0, fbp=False, slices=1),
    1: dict(nt=512, ntheta=512, n=512, k=20, amin=0.05, amax=0.35, noise=0.01, fbp=True, slices=16),
    2: dict(nt=2048, ntheta=2048, n=2048, k=50, amin=0.01, amax=0.3, noise=0.01, fbp=False, slices=64),
    3: dict(nt=2048, ntheta=2048, n=2048, k=50, amin=0.01, amax=0.3, noise=0.01, fbp=True, slices=2048),
    4: dict(nt=2048, ntheta=2048, n=2048, k=50, amin=0.01, amax=0.3, noise=0.01, fbp=False, slices=64),
}
BASE_SEED = 20261019


def config_seed(cfg: int, slice_index: int) -> int:
    """Per-slice seed.  Config 4 runs on "the same 64-slice inputs as config 2"
    (BASELINE.json configs[4]), so it takes config 2's seeds."""
    return BASE_SEED + 7919 * (2 if cfg == 4 else cfg) + slice_index


def config_sinogram(cfg: int, slice_index: int = 0) -> np.ndarray:
    c = CONFIGS[cfg]
    return sinogram(config_seed(cfg, slice_index), c["nt"], c["ntheta"], c["k"], c["amin"], c["amax"], c["noise"])
