"""Worker for tests/test_gpu_sweep.py (TEST INFRASTRUCTURE): reconstructs one
downloaded device-generated sinogram with the CPU oracle and compares it with the
GPU image of the same input.  Runs in spawned processes, one slice per task."""

from __future__ import annotations

import os


def oracle_compare(job):
    """job = (label, slice_id, fbp, n, sino_path, img_path) -> (label, slice_id, rel_l2, max_abs, ref_max)."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np

    from oracle import fastbp_oracle as O

    label, sid, fbp, n, sino_path, img_path = job
    g = np.load(sino_path).astype(np.float64)
    got = np.load(img_path)
    ref = O.fbp_logpolar(g, n) if fbp else O.logpolar_backproject(g, n)
    return label, sid, O.relative_l2(got, ref), O.max_abs(got, ref), float(np.max(np.abs(ref)))
