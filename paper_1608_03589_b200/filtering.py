"""Filtered backprojection — drop-in for fastbp.filtering's path (filtering.py:27-98).

filter_sinogram / fbp keep the reference signatures.  engine="logpolar" runs the
fused device pipeline (ramp filter kernel + log-polar backprojection, 1/(2 pi)
applied in the readout); engine="bst" (the reference's default) runs the BST
engine of bst.py with the ramp filter in front (lpbp_bst_*); engine="naive"
filters on the device and runs the direct backprojector.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .grids import CartesianImage, Sinogram
from .logpolar import LogPolarOptions, _to_device, plan_for
from .plan import naive_backproject

__all__ = ["FBP_SCALE", "FilterSpec", "filter_sinogram", "fbp", "fbp_batch"]

FBP_SCALE = 1.0 / (2.0 * math.pi)  # filtering.py:27


@dataclass(frozen=True)
class FilterSpec:
    """|sigma| / (1 + lam |sigma|), hard low-pass at cutoff * Nyquist (filtering.py:30-51)."""

    lam: float = 0.0
    kind: str = "tikhonov"
    cutoff: float = 1.0

    def __post_init__(self):
        if self.lam < 0:
            raise ValueError("lambda must be >= 0")
        if self.kind not in ("ramp", "tikhonov"):
            raise ValueError("kind must be 'ramp' or 'tikhonov'")
        if not (0.0 < self.cutoff <= 1.0):
            raise ValueError("cutoff must lie in (0, 1]")
        if self.kind == "ramp" and self.lam != 0.0:
            raise ValueError("ramp filter has lambda = 0")

    def response(self, sigma: np.ndarray) -> np.ndarray:
        a = np.abs(sigma)
        return a / (1.0 + self.lam * a)


def _spec_key(spec: FilterSpec) -> tuple[float, float]:
    return (float(spec.lam), float(spec.cutoff))


def filter_sinogram(g: Sinogram, spec: FilterSpec) -> Sinogram:
    """Per-angle filtering along t (filtering.py:54-70) on the device."""
    # The filter taps do not depend on the output size; any valid n works for the plan.
    plan = plan_for(g.nt, g.ntheta, g.nt, None, _spec_key(spec))
    out = plan.filter(_to_device(g))
    return Sinogram(g.nt, g.ntheta, out[0].double().cpu().numpy())


def fbp(g: Sinogram, spec: FilterSpec, engine: str = "bst", n: int = 256, engine_options=None) -> CartesianImage:
    """Filtered backprojection (filtering.py:73-98)."""
    if engine == "logpolar":
        opts = engine_options if isinstance(engine_options, LogPolarOptions) else LogPolarOptions()
        if n < 2:
            raise ValueError("n_out must be >= 2")
        plan = plan_for(g.nt, g.ntheta, n, opts, _spec_key(spec))
        img = plan.execute(_to_device(g))
        return CartesianImage(n, n, img[0].double().cpu().numpy())
    if engine == "naive":
        if n < 2:
            raise ValueError("n must be >= 2")
        plan = plan_for(g.nt, g.ntheta, g.nt, None, _spec_key(spec))
        fg = plan.filter(_to_device(g))
        img = naive_backproject(fg, n) * FBP_SCALE
        return CartesianImage(n, n, img[0].double().cpu().numpy())
    if engine == "bst":
        from .bst import BstOptions, get_bst_plan
        opts = engine_options if isinstance(engine_options, BstOptions) else BstOptions(n_out=n)
        if opts.n_out != n:
            opts = BstOptions(n_out=n, beta=opts.beta, zero_pad=opts.zero_pad, dc_mode=opts.dc_mode)
        plan = get_bst_plan(g.nt, g.ntheta, opts, _spec_key(spec))
        img = plan.execute(_to_device(g))
        return CartesianImage(n, n, img[0].double().cpu().numpy())
    raise ValueError("engine must be 'naive', 'bst' or 'logpolar'")


def fbp_batch(sino: torch.Tensor, spec: FilterSpec, n: int, opts: LogPolarOptions | None = None,
              out: torch.Tensor | None = None) -> torch.Tensor:
    """Batched device FBP: [B, nt, ntheta] float32 CUDA -> [B, n, n]."""
    if n < 2:
        raise ValueError("n_out must be >= 2")
    plan = plan_for(sino.shape[1], sino.shape[2], n, opts, _spec_key(spec))
    return plan.execute(sino, out=out)
