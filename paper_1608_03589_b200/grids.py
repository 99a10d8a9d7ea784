"""Containers and mesh sizing of the drop-in API.

Same fields, validation and error messages as fastbp.grids (grids.py:61-197,
372-391) so code written against the reference runs unchanged; values are
float64 numpy arrays, frozen after construction.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


def _frozen_f64(values, shape: tuple[int, int], label: str) -> np.ndarray:
    arr = np.array(values, dtype=np.float64, copy=True)
    if arr.shape != shape:
        raise ValueError(f"values must have shape {label} = {shape}")
    if not np.all(np.isfinite(arr)):
        raise ValueError("values must contain only finite values")
    arr = np.ascontiguousarray(arr)
    arr.setflags(write=False)
    return arr


@dataclass(frozen=True)
class CartesianImage:
    """Image on [-1, 1]^2, values[ny][nx], pixel centres -1 + (j + 1/2) * 2/n (grids.py:61-91)."""

    nx: int
    ny: int
    values: np.ndarray = field(repr=False)

    def __post_init__(self):
        if self.nx < 2 or self.ny < 2:
            raise ValueError("nx and ny must be >= 2")
        object.__setattr__(self, "values", _frozen_f64(self.values, (self.ny, self.nx), "(ny, nx)"))

    @property
    def dx(self) -> float:
        return 2.0 / self.nx

    @property
    def dy(self) -> float:
        return 2.0 / self.ny

    def x_centers(self) -> np.ndarray:
        return -1.0 + (np.arange(self.nx) + 0.5) * self.dx

    def y_centers(self) -> np.ndarray:
        return -1.0 + (np.arange(self.ny) + 0.5) * self.dy


@dataclass(frozen=True)
class Sinogram:
    """g(t_i, theta_j), values[nt][ntheta], t_i = -1 + 2i/nt, theta_j = j pi/ntheta (grids.py:93-122)."""

    nt: int
    ntheta: int
    values: np.ndarray = field(repr=False)

    def __post_init__(self):
        if self.nt < 2 or self.ntheta < 1:
            raise ValueError("nt must be >= 2 and ntheta >= 1")
        object.__setattr__(self, "values", _frozen_f64(self.values, (self.nt, self.ntheta), "(nt, ntheta)"))

    @property
    def dt(self) -> float:
        return 2.0 / self.nt

    @property
    def dtheta(self) -> float:
        return math.pi / self.ntheta

    def t(self) -> np.ndarray:
        return -1.0 + np.arange(self.nt) * self.dt

    def theta(self) -> np.ndarray:
        return np.arange(self.ntheta) * self.dtheta


@dataclass(frozen=True)
class LogPolarImage:
    """Samples on rho_i = rho0 + (i+1) drho, drho = -rho0/nrho, phi_j = j 2pi/nphi (grids.py:157-197)."""

    nrho: int
    nphi: int
    rho0: float
    values: np.ndarray = field(repr=False)

    def __post_init__(self):
        if self.nrho < 2 or self.nphi < 2:
            raise ValueError("nrho and nphi must be >= 2")
        if not self.rho0 < 0:
            raise ValueError("rho0 must be negative")
        object.__setattr__(self, "values", _frozen_f64(self.values, (self.nrho, self.nphi), "(nrho, nphi)"))

    @property
    def drho(self) -> float:
        return -self.rho0 / self.nrho

    @property
    def dphi(self) -> float:
        return 2.0 * math.pi / self.nphi

    def rho(self) -> np.ndarray:
        return self.rho0 + (np.arange(self.nrho) + 1) * self.drho

    def phi(self) -> np.ndarray:
        return np.arange(self.nphi) * self.dphi

    @property
    def fovea_radius(self) -> float:
        return math.exp(self.rho0)


def compute_nrho(ns: int, nx: int, ny: int) -> int:
    """Radial mesh count for an (nx, ny) target (grids.py:372-382)."""
    if ns < 2 or nx < 2 or ny < 2:
        raise ValueError("all counts must be >= 2")
    v = math.ceil(math.log(min(1.0 / nx, 1.0 / ny)) / math.log(1.0 - 2.0 / ns))
    return int(min(max(v, 2), 64 * ns))


def adaptive_rho0(nx: int, ny: int) -> float:
    """ln(min(dx, dy)) - ln 2 (grids.py:385-391)."""
    if nx < 2 or ny < 2:
        raise ValueError("counts must be >= 2")
    return math.log(min(2.0 / nx, 2.0 / ny)) - math.log(2.0)
