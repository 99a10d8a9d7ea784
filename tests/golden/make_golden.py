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


def sector_goldens() -> None:
    """partial_backproject (logpolar.py:210-299) on seeded inputs, with the stage
    intermediates of one sector from the reference's own helpers."""
    import warnings

    from fastbp.logpolar import _rescale_support, _roll_angles, partial_backproject
    from fastbp.radon import shift_sinogram

    cases = {
        "a": (phantoms.sinogram(101, 256, 180, 10, 0.05, 0.35, 0.0), 128,
              [(k * math.pi / 4, math.pi / 8, 0.25) for k in range(4)]),
        "b": (phantoms.sinogram(102, 256, 256, 10, 0.05, 0.35, 0.01), 256, [(0.0, math.pi / 2, 0.25)]),
        "c": (phantoms.config_sinogram(0), 256,
              [(0.3, math.pi / 6, 0.2), (0.3 + math.pi / 3, math.pi / 6, 0.3), (0.3 + 2 * math.pi / 3, math.pi / 6, 0.35)]),
    }
    arrays = {}
    kat = {}
    for key, (g, n, sectors) in cases.items():
        g = g.astype(np.float32).astype(np.float64)
        s = fb.Sinogram(*g.shape, g)
        with warnings.catch_warnings(record=True) as caught:
            warnings.simplefilter("always")
            pb = partial_backproject(s, sectors, n).values
        n_warn = sum(1 for w in caught if issubclass(w.category, RuntimeWarning))
        arrays[f"{key}_sino"] = g.astype(np.float32)
        arrays[f"{key}_sectors"] = np.asarray(sectors, dtype=np.float64)
        arrays[f"{key}_n"] = np.asarray(n)
        arrays[f"{key}_pb"] = pb
        # stage intermediates of sector 0: rotated/weighted/shrunk/shifted sinogram and its log-polar image
        theta0, beta, a_r = sectors[0]
        dth = math.pi / g.shape[1]
        jc = int(round((theta0 + beta) / dth))
        theta = np.arange(g.shape[1]) * dth
        masks = [np.abs(np.mod(theta - (t0 + b) + math.pi / 2, math.pi) - math.pi / 2) <= b + 2 * dth + 1e-12
                 for t0, b, _ in sectors]
        cover = np.sum(masks, axis=0).astype(np.float64)
        rot = (np.arange(g.shape[1]) + jc) % g.shape[1]
        w = np.zeros(g.shape[1])
        w[masks[0][rot]] = 1.0
        w /= cover[rot]
        gr = _roll_angles(s, jc)
        gr = fb.Sinogram(gr.nt, gr.ntheta, gr.values * w[None, :])
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            gsh = shift_sinogram(_rescale_support(gr, a_r), (1.0 - a_r, 0.0)).values
        support_min = (1.0 - a_r) * math.cos(min(beta + 2 * dth, math.pi / 2)) - a_r
        rho0_s = (min(math.log(support_min), math.log(1 - 2 * a_r)) - 0.2 if support_min > 0.05
                  else math.log(a_r) + fb.adaptive_rho0(n, n))
        nrho_s = _mesh_for(g.shape[0] // 2, rho0_s, None)
        lp0 = _logpolar_convolve(fb.sinogram_to_semipolar(fb.Sinogram(*gsh.shape, gsh)), rho0_s, nrho_s).values
        arrays[f"{key}_sec0_sino"] = gsh
        arrays[f"{key}_sec0_lp"] = lp0
        kat[f"sector_{key}"] = {"jc0": jc, "rho0_0": rho0_s, "nrho_0": nrho_s, "runtime_warnings": n_warn}
        if key == "a":  # the reference's own sector experiment (scratch_fbp.py:33-49), on this seeded phantom
            nv = fb.backproject_naive(s, n).values
            lp = fb.logpolar_backproject(s, n).values
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                pb1 = partial_backproject(s, [(0.0, math.pi / 2, 0.25)], n).values
            xs = -1.0 + (np.arange(n) + 0.5) * (2.0 / n)
            R = np.hypot(*np.meshgrid(xs, xs))
            m = (R > 2 * math.exp(fb.adaptive_rho0(n, n))) & (R <= 1.0)
            kat["sector_a"]["annulus_vs_naive"] = float(np.linalg.norm(pb[m] - nv[m]) / np.linalg.norm(nv[m]))
            kat["sector_a"]["single_vs_lp"] = float(np.linalg.norm(pb1[m] - lp[m]) / np.linalg.norm(lp[m]))
            arrays["a_single_pb"] = pb1
    np.savez_compressed(os.path.join(HERE, "sector.npz"), **arrays)
    with open(os.path.join(HERE, "kat_sector.json"), "w") as f:
        json.dump(kat, f, indent=1, sort_keys=True)


def bst_goldens() -> None:
    """The BST engine (bst.py:120-206) and fbp's default engine, from the reference."""
    from fastbp.bst import BstOptions, _radial_spectra, bst_backproject, mean_backprojection
    from fastbp.grids import PolarSpectrum, polar_to_cartesian_frequency

    arrays, kat = {}, {}
    g0 = phantoms.config_sinogram(0).astype(np.float64)
    s0 = fb.Sinogram(*g0.shape, g0)
    arrays["cfg0_bp"] = bst_backproject(s0, BstOptions(n_out=256)).values
    arrays["cfg0_fbp"] = fb.fbp(s0, fb.FilterSpec(), n=256).values           # default engine = "bst"
    g1 = phantoms.config_sinogram(1, 0).astype(np.float64)
    s1 = fb.Sinogram(*g1.shape, g1)
    arrays["cfg1_fbp"] = fb.fbp(s1, fb.FilterSpec(), n=512).values.astype(np.float32)
    arrays["cfg1_fbp_tik"] = fb.fbp(s1, fb.FilterSpec(lam=0.02, cutoff=0.9), n=512).values.astype(np.float32)
    g2 = phantoms.sinogram(201, 256, 180, 10, 0.05, 0.35, 0.01).astype(np.float32).astype(np.float64)
    s2 = fb.Sinogram(*g2.shape, g2)
    arrays["opt_sino"] = g2.astype(np.float32)
    arrays["opt_beta4_zp3_cap"] = bst_backproject(s2, BstOptions(n_out=128, beta=4.0, zero_pad=3.0,
                                                                dc_mode="kernel_cap")).values
    arrays["opt_beta2"] = bst_backproject(s2, BstOptions(n_out=128, beta=2.0)).values
    g3 = phantoms.sinogram(202, 200, 96, 8, 0.05, 0.35, 0.01).astype(np.float32).astype(np.float64)
    s3 = fb.Sinogram(*g3.shape, g3)
    arrays["odd_sino"] = g3.astype(np.float32)
    arrays["odd_n101"] = bst_backproject(s3, BstOptions(n_out=101)).values
    # stage intermediates on the small case: radial spectra and the padded cartesian grid
    g4 = phantoms.sinogram(203, 128, 90, 6, 0.05, 0.35, 0.0).astype(np.float32).astype(np.float64)
    s4 = fb.Sinogram(*g4.shape, g4)
    H, dsig = _radial_spectra(s4, 2.0, 0.0, 64)
    arrays["small_sino"] = g4.astype(np.float32)
    arrays["small_H"] = H
    ps = PolarSpectrum(H.shape[0], H.shape[1], dsig, H)
    arrays["small_grid"] = polar_to_cartesian_frequency(ps, 128, 128, dw=math.pi / 2).values
    arrays["small_bp"] = bst_backproject(s4, BstOptions(n_out=64)).values
    from fastbp.bst import bst_spectrum
    arrays["small_spectrum"] = bst_spectrum(s4, BstOptions(n_out=64)).values
    kat["small_dsigma"] = dsig
    kat["mean_bp_cfg0"] = mean_backprojection(s0)
    try:
        bst_backproject(fb.Sinogram(64, 32, np.ones((64, 32))), BstOptions(n_out=256))
    except ValueError as e:
        kat["too_fine_message"] = str(e)
    np.savez_compressed(os.path.join(HERE, "bst.npz"), **arrays)
    with open(os.path.join(HERE, "kat_bst.json"), "w") as f:
        json.dump(kat, f, indent=1, sort_keys=True)


def radon_goldens() -> None:
    """The input generator radon_ellipses (radon.py:38-61) on EllipseSets (phantoms.py:36-62)."""
    from fastbp.phantoms import Ellipse, EllipseSet
    from fastbp.radon import radon_ellipses

    arrays, kat = {}, {}
    rng = np.random.Generator(np.random.PCG64(4242))

    def random_set(k):
        return [((rng.uniform(-0.7, 0.7), rng.uniform(-0.7, 0.7)), (rng.uniform(0.02, 0.5), rng.uniform(0.02, 0.5)),
                 rng.uniform(0.0, math.pi), rng.uniform(-1.0, 1.0)) for _ in range(k)]

    cases = {
        # hand-picked: one ellipse crossing the unit circle, one thin tilted, one at the origin
        "small": ([((0.0, 0.0), (0.6, 0.4), 0.3, 1.0), ((0.8, 0.1), (0.5, 0.2), 1.1, -0.5),
                   ((-0.2, 0.35), (1e-3, 0.3), math.pi / 3, 2.0), ((0.1, -0.5), (0.05, 0.05), 0.0, 0.7),
                   ((-0.45, -0.2), (0.25, 0.1), 2.9, 0.25)], 64, 45),
        "many": (random_set(300), 100, 70),      # > 256 ellipses, ragged 64-row / 32-angle tiles
        "odd": (random_set(7), 33, 17),
    }
    for name, (ell, nt, nth) in cases.items():
        es = EllipseSet(tuple(Ellipse(c, ab, t, r) for c, ab, t, r in ell))
        arrays[f"{name}_params"] = np.array([[c[0], c[1], ab[0], ab[1], t, r] for c, ab, t, r in ell])
        arrays[f"{name}_sino"] = radon_ellipses(es, nt, nth).values
    for key, fn in (("semi_axes_message", lambda: Ellipse((0.0, 0.0), (0.0, 0.1), 0.0, 1.0)),
                    ("empty_set_message", lambda: EllipseSet(()))):
        try:
            fn()
        except ValueError as e:
            kat[key] = str(e)
    np.savez_compressed(os.path.join(HERE, "radon.npz"), **arrays)
    with open(os.path.join(HERE, "kat_radon.json"), "w") as f:
        json.dump(kat, f, indent=1, sort_keys=True)


def main() -> None:
    if "--only-radon" in sys.argv:
        radon_goldens()
        print("wrote radon goldens")
        return
    if "--only-bst" in sys.argv:
        bst_goldens()
        print("wrote bst goldens")
        return
    if "--only-sector" in sys.argv:
        sector_goldens()
        print("wrote sector goldens")
        return
    sector_goldens()
    bst_goldens()
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
    sector_goldens()
    bst_goldens()
    radon_goldens()
    print("wrote goldens:", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
