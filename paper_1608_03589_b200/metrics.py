"""Parity metrics (fastbp.metrics.relative_l2, metrics.py:29-36, plus max-abs)."""

from __future__ import annotations

import numpy as np

from .grids import CartesianImage

__all__ = ["relative_l2", "max_abs_error"]


def _values(a) -> np.ndarray:
    return a.values if isinstance(a, CartesianImage) else np.asarray(a, dtype=np.float64)


def relative_l2(a, b) -> float:
    """||a - b||_2 / ||b||_2 (b is the reference)."""
    x, y = _values(a), _values(b)
    if x.shape != y.shape:
        raise ValueError(f"dimension mismatch: {x.shape} vs {y.shape}")
    den = np.linalg.norm(y)
    if den == 0.0:
        return 0.0 if np.linalg.norm(x) == 0.0 else float("inf")
    return float(np.linalg.norm(x - y) / den)


def max_abs_error(a, b) -> float:
    x, y = _values(a), _values(b)
    if x.shape != y.shape:
        raise ValueError(f"dimension mismatch: {x.shape} vs {y.shape}")
    return float(np.max(np.abs(x - y))) if x.size else 0.0
