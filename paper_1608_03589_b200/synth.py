"""Analytic ellipse-phantom sinograms on the device: the reference's
radon_ellipses(EllipseSet, nt, ntheta) -> Sinogram (radon.py:38-61, with the
Ellipse / EllipseSet containers of phantoms.py:36-62) and the seeded synthetic
configs the benchmark uses.

Ellipse parameters are drawn on the host exactly as documented in
oracle/phantoms.py (numpy Generator(PCG64(seed)); u, v, a, b, tilt, rho in that
order), and the exact line integrals (fastbp radon.py:38-61) are evaluated in
fp64 by liblpbp's lpbp_radon_ellipses kernel.  Gaussian noise (sigma = noise *
max g) comes from torch's device generator seeded per slice, so noisy device
sinograms are statistically — not bitwise — identical to oracle/phantoms'."""

from __future__ import annotations

import math
from ctypes import c_void_p
from dataclasses import dataclass

import numpy as np
import torch

from ._native import check, lib
from .grids import Sinogram


@dataclass(frozen=True)
class Ellipse:
    """Additive ellipse: center, semi-axes (A, B), tilt in radians, intensity (phantoms.py:36-47)."""

    center: tuple[float, float]
    semi_axes: tuple[float, float]
    tilt: float
    intensity: float

    def __post_init__(self):
        if self.semi_axes[0] <= 0 or self.semi_axes[1] <= 0:
            raise ValueError("semi-axes must be positive")


@dataclass(frozen=True)
class EllipseSet:
    """Nonempty tuple of ellipses (phantoms.py:50-62)."""

    ellipses: tuple[Ellipse, ...]

    def __post_init__(self):
        if len(self.ellipses) == 0:
            raise ValueError("EllipseSet must be nonempty")

    def __iter__(self):
        return iter(self.ellipses)

    def __len__(self):
        return len(self.ellipses)

    def params(self) -> np.ndarray:
        """[k][6] float64 rows (cx, cy, A, B, tilt, intensity): the kernel's parameter layout."""
        return np.array([[e.center[0], e.center[1], e.semi_axes[0], e.semi_axes[1], e.tilt, e.intensity]
                         for e in self.ellipses], dtype=np.float64)


def _device(device) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("radon_ellipses runs on the GPU (liblpbp.so); no CUDA device is available")
    return torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)


def radon_ellipses(ellipse_set: EllipseSet, nt: int, ntheta: int, device=None) -> Sinogram:
    """Exact line integrals of an additive ellipse phantom (radon.py:38-61), evaluated in
    fp64 on the GPU with the reference's per-ellipse accumulation order; returns the
    reference's Sinogram (float64 values).  Agreement with the reference is to the last
    few ulps (device cos/sin vs the host libm)."""
    dev = _device(device)
    out = radon_ellipses_batch(ellipse_set.params()[None], int(nt), int(ntheta), dev, dtype=torch.float64)
    return Sinogram(int(nt), int(ntheta), out[0].cpu().numpy())

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


def radon_ellipses_batch(params: np.ndarray, nt: int, ntheta: int, device, dtype=torch.float32) -> torch.Tensor:
    """params [B][k][6] (cx, cy, A, B, tilt, intensity) -> noiseless sinograms [B][nt][ntheta]
    (float32 or float64) on `device`."""
    params = np.ascontiguousarray(params, dtype=np.float64)
    bsz, k, _ = params.shape
    if dtype not in (torch.float32, torch.float64):
        raise ValueError("dtype must be torch.float32 or torch.float64")
    dp = torch.from_numpy(params).to(device)
    out = torch.empty((bsz, nt, ntheta), dtype=dtype, device=device)
    fn = lib().lpbp_radon_ellipses if dtype == torch.float32 else lib().lpbp_radon_ellipses_f64
    with torch.cuda.device(device):
        check(fn(c_void_p(dp.data_ptr()), k, nt, ntheta, bsz, c_void_p(out.data_ptr()),
                 c_void_p(torch.cuda.current_stream(device).cuda_stream)))
    return out


def config_batch(cfg: int, slice_ids, device, gen_chunk: int = 64, geometry: tuple[int, int] | None = None) -> torch.Tensor:
    """Sinograms of config `cfg` for the given global slice indices (seed = BASE_SEED
    + 7919*cfg + index, as oracle/phantoms.config_sinogram; config 4 reuses config 2's
    seeds: BASELINE.json configs[4] runs on the same 64 slices)."""
    c = dict(CONFIGS[cfg])
    if geometry is not None:  # the config's phantoms sampled at another (nt, ntheta)
        c.update(nt=int(geometry[0]), ntheta=int(geometry[1]))
    ids = list(slice_ids)
    out = torch.empty((len(ids), c["nt"], c["ntheta"]), dtype=torch.float32, device=device)
    for lo in range(0, len(ids), gen_chunk):
        part = ids[lo:lo + gen_chunk]
        seeds = [BASE_SEED + 7919 * (2 if cfg == 4 else cfg) + i for i in part]
        prm = np.stack([ellipse_params(s, c["k"], c["amin"], c["amax"]) for s in seeds])
        g = radon_ellipses_batch(prm, c["nt"], c["ntheta"], device)
        if c["noise"] > 0:
            for j, s in enumerate(seeds):
                gen = torch.Generator(device=device)
                gen.manual_seed(s)
                noise = torch.randn(g.shape[1:], generator=gen, device=device, dtype=torch.float32)
                g[j].add_(noise, alpha=float(c["noise"] * g[j].max()))
        out[lo:lo + len(part)] = g
    return out
