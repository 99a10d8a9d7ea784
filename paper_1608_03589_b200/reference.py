"""Direct pixel-driven backprojector (fastbp.reference.backproject_naive,
reference.py:21-37) on the device — the accuracy cross-check for the log-polar path."""

from __future__ import annotations

import numpy as np
import torch

from .grids import CartesianImage, Sinogram
from .plan import naive_backproject

__all__ = ["backproject_naive", "backproject_naive_batch"]


def backproject_naive(g: Sinogram, n: int) -> CartesianImage:
    """b(x) = dtheta * sum_k g(x . xi_k, theta_k), linear interpolation in t,
    zero past the sampled range; covers the whole square."""
    if n < 2:
        raise ValueError("n must be >= 2")
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1608_03589_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    sino = torch.from_numpy(np.ascontiguousarray(g.values, dtype=np.float32)).cuda().unsqueeze(0)
    return CartesianImage(n, n, naive_backproject(sino, n)[0].double().cpu().numpy())


def backproject_naive_batch(sino: torch.Tensor, n: int) -> torch.Tensor:
    if n < 2:
        raise ValueError("n must be >= 2")
    return naive_backproject(sino, n)
