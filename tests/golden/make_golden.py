"""Generate the golden vectors pinned by the test suite, by running the REFERENCE
implementation (fastbp, /root/reference/pkg/src) on seeded inputs.

Run in the build container (where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
The outputs are committed; the GPU box never needs /root/reference.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import fastbp as fb  # noqa: E402  (the reference)
from fastbp.logpolar import _logpolar_convolve, _mesh_for, make_logpolar_kernel  # noqa: E402

from oracle import phantoms  # noqa: E402


def lp_stage(g: np.ndarray, n: int):
    s = fb.Sinogram(*g.shape, g)
    rho0 = fb.adaptive_rho0(n, n)
    nrho = _mesh_for(g.shape[0] // 2, rho0, None)
    return _logpolar_convolve(fb.sinogram_to_semipolar(s), rho0, nrho).values


def main() -> None:
    out = {}
    # config 0: BP 256x256 -> 256 (BASELINE.json configs[0])
    g0 = phantoms.config_sinogram(0).astype(np.float64)
    s0 = fb.Sinogram(*g0.shape, g0)
    np.savez_compressed(
        os.path.join(HERE, "cfg0.npz"),
        sino=g0.astype(np.float32),
        bp=fb.logpolar_backproject(s0, 256).values,
        lp=lp_stage(g0, 256).astype(np.float32),
        naive=fb.backproject_naive(s0, 256).values.astype(np.float32),
        fbp=fb.fbp(s0, fb.FilterSpec(), engine="logpolar", n=256).values.astype(np.float32),
        filtered=fb.filter_sinogram(s0, fb.FilterSpec()).values.astype(np.float32),
    )
    # config 1: FBP 512x512 -> 512, slice 0 of the 16-slice batch (configs[1])
    g1 = phantoms.config_sinogram(1, 0).astype(np.float64)
    s1 = fb.Sinogram(*g1.shape, g1)
    np.savez_compressed(
        os.path.join(HERE, "cfg1.npz"),
        sino=g1.astype(np.float32),
        fbp=fb.fbp(s1, fb.FilterSpec(), engine="logpolar", n=512).values.astype(np.float32),
        filtered=fb.filter_sinogram(s1, fb.FilterSpec()).values.astype(np.float32),
        fbp_tik=fb.fbp(s1, fb.FilterSpec(lam=0.02, cutoff=0.9), engine="logpolar", n=512).values.astype(np.float32),
    )
    # non-square / explicit options: 512 bins x 256 angles -> 256, rho0 = -4, nrho = 600
    g2 = phantoms.sinogram(77, 512, 256, 12, 0.05, 0.35, 0.01).astype(np.float64)
    s2 = fb.Sinogram(*g2.shape, g2)
    np.savez_compressed(
        os.path.join(HERE, "opts.npz"),
        sino=g2.astype(np.float32),
        bp_default=fb.logpolar_backproject(s2, 256).values.astype(np.float32),
        bp_opts=fb.logpolar_backproject(s2, 256, fb.LogPolarOptions(rho0=-4.0, nrho=600)).values.astype(np.float32),
        bp_n300=fb.logpolar_backproject(s2, 300).values.astype(np.float32),
    )
    # known answers: mesh sizes and kernel supports at the three benchmark sizes,
    # compute_nrho(1024,...) = 3546, scratch_lp.py constant-sinogram means
    kat = {"compute_nrho_1024": fb.compute_nrho(1024, 1024, 1024)}
    for nt, n in ((256, 256), (512, 512), (2048, 2048)):
        rho0 = fb.adaptive_rho0(n, n)
        nrho = _mesh_for(nt // 2, rho0, None)
        drho = -rho0 / nrho
        kern = np.roll(make_logpolar_kernel(nrho, 2 * nt, drho), -nt, axis=1)
        rows = np.nonzero(kern.any(axis=1))[0]
        kat[f"mesh_{nt}"] = {"rho0": rho0, "nrho": nrho, "drho": drho, "nnz": int(np.count_nonzero(kern)),
                             "kmax": int(rows.max()), "cells_checksum": int(np.sum(np.nonzero(kern)[0] * 7919 + np.nonzero(kern)[1]))}
    for nt, nth, n in ((128, 90, 64), (256, 180, 128)):
        g = fb.Sinogram(nt, nth, np.ones((nt, nth)))
        b = fb.logpolar_backproject(g, n)
        xs = -1.0 + (np.arange(n) + 0.5) * (2.0 / n)
        X, Y = np.meshgrid(xs, xs)
        R = np.hypot(X, Y)
        inner = (R > 2 * math.exp(fb.adaptive_rho0(n, n))) & (R <= 0.8)
        kat[f"const_mean_{nt}_{nth}_{n}"] = float(b.values[inner].mean())
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1, sort_keys=True)
    print("wrote goldens:", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
