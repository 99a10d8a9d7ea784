"""Log-polar backprojection engine — drop-in for fastbp.logpolar's hot path.

logpolar_backproject keeps the reference signature (logpolar.py:121-136) and
runs on the sm_100a pipeline in liblpbp.so: sinogram row DFTs, per-frequency
resampling + rho-axis FFT convolution with the precomputed kernel spectrum,
inverse row DFTs and the Cartesian readout.  Inputs are rounded to float32 on
the device; outputs come back as float64 containers like the reference's.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .grids import CartesianImage, LogPolarImage, Sinogram, adaptive_rho0
from .plan import LogPolarPlan, get_plan

__all__ = [
    "LOGPOLAR_SCALE",
    "LogPolarOptions",
    "logpolar_backproject",
    "logpolar_backproject_batch",
    "logpolar_convolve",
    "mesh_for",
    "partial_backproject",
]

LOGPOLAR_SCALE = 0.5  # logpolar.py:47 (folded into the plan's kernel spectrum)


@dataclass(frozen=True)
class LogPolarOptions:
    """rho0 None -> adaptive inner radius; nrho None -> resolution-rule mesh
    (logpolar.py:50-63)."""

    rho0: float | None = None
    nrho: int | None = None

    def __post_init__(self):
        if self.rho0 is not None and not self.rho0 < 0:
            raise ValueError("rho0 must be negative")
        if self.nrho is not None and self.nrho < 2:
            raise ValueError("nrho must be >= 2")


def mesh_for(ns: int, rho0: float, nrho: int | None) -> int:
    """Radial count obeying 1 - e^{-drho} <= 2/ns (logpolar.py:84-97)."""
    step = 2.0 / ns
    if nrho is None:
        nrho = max(2, int(math.ceil(-rho0 / -math.log1p(-step))))
    drho = -rho0 / nrho
    if 1.0 - math.exp(-drho) > step * (1.0 + 1e-9):
        raise ValueError(
            "log-polar mesh too coarse: largest radial step "
            f"{1.0 - math.exp(-drho):.3e} exceeds the sinogram step {step:.3e}"
        )
    return nrho


def _to_device(g: Sinogram) -> torch.Tensor:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1608_03589_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch.from_numpy(np.ascontiguousarray(g.values, dtype=np.float32)).cuda().unsqueeze(0)


def plan_for(nt: int, ntheta: int, n_out: int, opts: LogPolarOptions | None,
             filter_spec: tuple[float, float] | None = None) -> LogPolarPlan:
    opts = opts or LogPolarOptions()
    return get_plan(nt, ntheta, n_out, opts.rho0, opts.nrho, filter_spec)


def logpolar_backproject(g: Sinogram, n_out: int, opts: LogPolarOptions | None = None) -> CartesianImage:
    """Backproject a sinogram through the log-polar pipeline (logpolar.py:121-136).
    Pixels inside the fovea (radius below e^rho0) and outside the unit disk are zero."""
    if n_out < 2:
        raise ValueError("n_out must be >= 2")
    plan = plan_for(g.nt, g.ntheta, n_out, opts)
    img = plan.execute(_to_device(g))
    return CartesianImage(n_out, n_out, img[0].double().cpu().numpy())


def logpolar_backproject_batch(sino: torch.Tensor, n_out: int, opts: LogPolarOptions | None = None,
                               out: torch.Tensor | None = None) -> torch.Tensor:
    """Batched device entry point: [B, nt, ntheta] float32 CUDA -> [B, n_out, n_out]."""
    if n_out < 2:
        raise ValueError("n_out must be >= 2")
    plan = plan_for(sino.shape[1], sino.shape[2], n_out, opts)
    return plan.execute(sino, out=out)


def logpolar_convolve(g: Sinogram, n_out: int, opts: LogPolarOptions | None = None) -> LogPolarImage:
    """The convolved log-polar image of g, i.e. fastbp's
    _logpolar_convolve(sinogram_to_semipolar(g), rho0, nrho) (logpolar.py:100-118)."""
    plan = plan_for(g.nt, g.ntheta, n_out, opts)
    lp = plan.logpolar(_to_device(g))
    return LogPolarImage(plan.nrho, plan.nphi, plan.rho0, lp[0].double().cpu().numpy())


def partial_backproject(g: Sinogram, sectors, n_out: int) -> CartesianImage:
    """fastbp.logpolar.partial_backproject (logpolar.py:210-299); see sector.py."""
    from .sector import partial_backproject as _pb
    return _pb(g, sectors, n_out)


def make_logpolar_kernel(nrho: int, nphi: int, drho: float):
    """fastbp.logpolar.make_logpolar_kernel (logpolar.py:66-81); see resample.py."""
    from .resample import make_logpolar_kernel as _k
    return _k(nrho, nphi, drho)


def truncation_error_bound(rho0: float, c: float) -> float:
    """fastbp.logpolar.truncation_error_bound (logpolar.py:138-145)."""
    from .resample import truncation_error_bound as _t
    return _t(rho0, c)
