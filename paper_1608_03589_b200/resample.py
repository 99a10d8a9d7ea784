"""The log-polar path's resampling steps as standalone device operations, with
the reference's names, containers and ValueError texts (fastbp.grids:290-347,
399-443; fastbp.logpolar:66-81, 138-145).  The fused pipeline
(logpolar_backproject) computes these implicitly; these entry points serve
code that calls the steps one by one.  Computed in liblpbp.so; inputs are
rounded to float32 on the device, outputs come back as float64 containers.
"""

from __future__ import annotations

import math
from ctypes import c_void_p
from dataclasses import dataclass, field

import numpy as np
import torch

from ._native import check, lib
from .grids import CartesianImage, LogPolarImage, Sinogram, _frozen_f64

__all__ = ["PolarSinogram", "PolarSpectrum", "FrequencyImage", "sinogram_to_semipolar", "semipolar_to_logpolar",
           "logpolar_to_cartesian", "polar_to_cartesian_frequency", "make_logpolar_kernel", "truncation_error_bound"]


@dataclass(frozen=True)
class PolarSinogram:
    """Semi-polar samples on s_i = i/(ns-1) in [0, 1], phi_k = k 2 pi / nphi (grids.py:125-154)."""

    ns: int
    nphi: int
    values: np.ndarray = field(repr=False)

    def __post_init__(self):
        if self.ns < 2 or self.nphi < 2:
            raise ValueError("ns and nphi must be >= 2")
        object.__setattr__(self, "values", _frozen_f64(self.values, (self.ns, self.nphi), "(ns, nphi)"))

    @property
    def ds(self) -> float:
        return 1.0 / (self.ns - 1)

    @property
    def dphi(self) -> float:
        return 2.0 * math.pi / self.nphi

    def s(self) -> np.ndarray:
        return np.arange(self.ns) * self.ds

    def phi(self) -> np.ndarray:
        return np.arange(self.nphi) * self.dphi


def _frozen_c128(values, shape, label) -> np.ndarray:
    arr = np.array(values, dtype=np.complex128, copy=True)
    if arr.shape != shape:
        raise ValueError(f"values must have shape {label} = {shape}")
    if not np.all(np.isfinite(arr.view(np.float64))):
        raise ValueError("values must contain only finite values")
    arr = np.ascontiguousarray(arr)
    arr.setflags(write=False)
    return arr


@dataclass(frozen=True)
class PolarSpectrum:
    """Complex samples on radial frequency rays sigma_m = m dsigma, values[nsigma][ntheta] (grids.py:200-229)."""

    nsigma: int
    ntheta: int
    dsigma: float
    values: np.ndarray = field(repr=False)

    def __post_init__(self):
        if self.nsigma < 2 or self.ntheta < 2:
            raise ValueError("nsigma and ntheta must be >= 2")
        if not self.dsigma > 0:
            raise ValueError("dsigma must be positive")
        object.__setattr__(self, "values", _frozen_c128(self.values, (self.nsigma, self.ntheta), "(nsigma, ntheta)"))

    @property
    def dtheta(self) -> float:
        return 2.0 * math.pi / self.ntheta

    def sigma(self) -> np.ndarray:
        return np.arange(self.nsigma) * self.dsigma

    @property
    def sigma_max(self) -> float:
        return (self.nsigma - 1) * self.dsigma


@dataclass(frozen=True)
class FrequencyImage:
    """Cartesian frequency samples in FFT layout, values[ny][nx]; bin k holds omega = pi k (grids.py:232-246)."""

    nx: int
    ny: int
    values: np.ndarray = field(repr=False)

    def __post_init__(self):
        if self.nx < 2 or self.ny < 2:
            raise ValueError("nx and ny must be >= 2")
        object.__setattr__(self, "values", _frozen_c128(self.values, (self.ny, self.nx), "(ny, nx)"))


def _dev(values: np.ndarray) -> torch.Tensor:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1608_03589_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch.from_numpy(np.ascontiguousarray(values, dtype=np.float32)).cuda()


def _stream() -> c_void_p:
    return c_void_p(torch.cuda.current_stream().cuda_stream)


def sinogram_to_semipolar(g: Sinogram, ns: int | None = None) -> PolarSinogram:
    """Unfold onto the semi-polar grid: p(s, phi) = g(s, phi) for phi < pi, g(-s, phi - pi)
    otherwise, linear in t, zero outside the t range (grids.py:290-311)."""
    ns = g.nt // 2 if ns is None else int(ns)
    if ns < 2:
        raise ValueError("ns must be >= 2")
    src = _dev(g.values)
    out = torch.empty((ns, 2 * g.ntheta), dtype=torch.float32, device=src.device)
    check(lib().lpbp_sinogram_to_semipolar(c_void_p(src.data_ptr()), c_void_p(out.data_ptr()), g.nt, g.ntheta, ns, 1,
                                           _stream()))
    return PolarSinogram(ns, 2 * g.ntheta, out.double().cpu().numpy())


def semipolar_to_logpolar(p: PolarSinogram, rho0: float, nrho: int) -> LogPolarImage:
    """Resample radial profiles at s = e^rho_i (grids.py:332-347)."""
    if nrho < 2:
        raise ValueError("nrho must be >= 2")
    if not rho0 < 0:
        raise ValueError("rho0 must be negative")
    src = _dev(p.values)
    out = torch.empty((nrho, p.nphi), dtype=torch.float32, device=src.device)
    check(lib().lpbp_semipolar_to_logpolar(c_void_p(src.data_ptr()), c_void_p(out.data_ptr()), p.ns, p.nphi,
                                           float(rho0), int(nrho), 1, _stream()))
    return LogPolarImage(int(nrho), p.nphi, float(rho0), out.double().cpu().numpy())


def logpolar_to_cartesian(l: LogPolarImage, nx: int, ny: int) -> CartesianImage:
    """Bilinear log-polar samples at the pixel centres of an nx x ny image; zero for
    r > 1, r = 0 or ln r < rho0 (grids.py:399-443)."""
    if nx < 2 or ny < 2:
        raise ValueError("nx and ny must be >= 2")
    src = _dev(l.values)
    out = torch.empty((ny, nx), dtype=torch.float32, device=src.device)
    check(lib().lpbp_logpolar_to_cartesian(c_void_p(src.data_ptr()), c_void_p(out.data_ptr()), l.nrho, l.nphi,
                                           float(l.rho0), int(nx), int(ny), 1, _stream()))
    return CartesianImage(int(nx), int(ny), out.double().cpu().numpy())


def polar_to_cartesian_frequency(ps: PolarSpectrum, nx: int, ny: int, dw: float = math.pi) -> FrequencyImage:
    """Bilinear (sigma, theta) gridding onto the lattice omega = dw k with the Hermitian
    average F(k) = (G(k) + conj G(-k)) / 2 (grids.py:456-508), fp64 coordinates on the device."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1608_03589_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    src = torch.from_numpy(np.ascontiguousarray(ps.values, dtype=np.complex64)).cuda()
    out = torch.empty((int(ny), int(nx)), dtype=torch.complex64, device=src.device)
    check(lib().lpbp_polar_to_cartesian_frequency(c_void_p(src.data_ptr()), c_void_p(out.data_ptr()), ps.nsigma,
                                                  ps.ntheta, ps.ntheta, 1, ps.nsigma * ps.ntheta, float(ps.dsigma),
                                                  int(nx), int(ny), float(dw), 1.0, 1, _stream()))
    return FrequencyImage(int(nx), int(ny), out.cpu().numpy().astype(np.complex128))


def make_logpolar_kernel(nrho: int, nphi: int, drho: float) -> np.ndarray:
    """Box-discretised kernel on the lag mesh (logpolar.py:66-81): 1/drho where
    |e^{i drho} cos(-pi + j 2pi/nphi) - 1| <= drho (built in fp64 by liblpbp)."""
    if nrho < 2 or nphi < 2:
        raise ValueError("kernel mesh must be at least 2 x 2")
    if not drho > 0:
        raise ValueError("drho must be positive")
    out = np.empty((int(nrho), int(nphi)), dtype=np.float64)
    check(lib().lpbp_logpolar_kernel(int(nrho), int(nphi), float(drho), c_void_p(out.ctypes.data)))
    return out


def truncation_error_bound(rho0: float, c: float) -> float:
    """2 pi c^2 e^{2 rho0}: squared-L2 bound on what cutting the mesh at rho0 loses (logpolar.py:138-145)."""
    if c < 0:
        raise ValueError("c must be >= 0")
    return 2.0 * math.pi * c * c * math.exp(2.0 * rho0)
