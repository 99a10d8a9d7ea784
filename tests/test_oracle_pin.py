"""Pin the CPU oracle (oracle/fastbp_oracle.py) to the reference: against the
committed golden vectors made by the reference itself (tests/golden/make_golden.py)
and, where the reference is importable, against it directly."""

import json
import math
import os

import numpy as np
import pytest

from oracle import fastbp_oracle as O
from oracle import phantoms

from conftest import GOLDEN

TOL = 1e-12  # fp64 restatement: agreement to rounding


def rel(a, b):
    return O.relative_l2(a, b)


def test_inputs_regenerate_bitwise(golden):
    assert np.array_equal(phantoms.config_sinogram(0), golden("cfg0.npz")["sino"])
    assert np.array_equal(phantoms.config_sinogram(1, 0), golden("cfg1.npz")["sino"])


def test_cfg0_backprojection(golden):
    z = golden("cfg0.npz")
    g = z["sino"].astype(np.float64)
    assert rel(O.logpolar_backproject(g, 256), z["bp"]) < TOL


def test_cfg0_stages(golden):
    z = golden("cfg0.npz")
    g = z["sino"].astype(np.float64)
    assert rel(O.logpolar_stage(g, 256), z["lp"]) < 1e-6  # golden stored as float32
    assert rel(O.ramp_filter(g), z["filtered"]) < 1e-6
    assert rel(O.fbp_logpolar(g, 256), z["fbp"]) < 1e-6


def test_cfg1_fbp(golden):
    z = golden("cfg1.npz")
    g = z["sino"].astype(np.float64)
    assert rel(O.fbp_logpolar(g, 512), z["fbp"]) < 1e-6
    assert rel(O.ramp_filter(g), z["filtered"]) < 1e-6
    assert rel(O.fbp_logpolar(g, 512, lam=0.02, cutoff=0.9), z["fbp_tik"]) < 1e-6


def test_options_and_nonsquare(golden):
    z = golden("opts.npz")
    g = z["sino"].astype(np.float64)
    assert rel(O.logpolar_backproject(g, 256), z["bp_default"]) < 1e-6
    assert rel(O.logpolar_backproject(g, 256, rho0=-4.0, nrho=600), z["bp_opts"]) < 1e-6
    assert rel(O.logpolar_backproject(g, 300), z["bp_n300"]) < 1e-6


def test_naive_cfg0(golden):
    z = golden("cfg0.npz")
    g = z["sino"].astype(np.float64)
    rows = np.arange(0, 256, 17)
    assert rel(O.backproject_naive(g, 256, rows=rows), z["naive"][rows]) < 1e-6


def test_known_answers():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        kat = json.load(f)
    assert O.compute_nrho(1024, 1024, 1024) == kat["compute_nrho_1024"] == 3546
    for nt in (256, 512, 2048):
        m = kat[f"mesh_{nt}"]
        ns, r0, nr, drho = O.lp_geometry(nt, nt)
        assert (r0, nr) == (m["rho0"], m["nrho"])
        kern = np.roll(O.lp_kernel(nr, 2 * nt, drho), -nt, axis=1)
        k, l = np.nonzero(kern)
        assert len(k) == m["nnz"] and int(k.max()) == m["kmax"]
        assert int(np.sum(k * 7919 + l)) == m["cells_checksum"]
    for nt, nth, n in ((128, 90, 64), (256, 180, 128)):
        b = O.logpolar_backproject(np.ones((nt, nth)), n)
        xs = -1.0 + (np.arange(n) + 0.5) * (2.0 / n)
        X, Y = np.meshgrid(xs, xs)
        R = np.hypot(X, Y)
        inner = (R > 2 * math.exp(O.adaptive_rho0(n, n))) & (R <= 0.8)
        assert abs(b[inner].mean() - kat[f"const_mean_{nt}_{nth}_{n}"]) < 1e-12


def test_errors_match_reference():
    with pytest.raises(ValueError, match="n_out must be >= 2"):
        O.logpolar_backproject(np.ones((16, 8)), 1)
    with pytest.raises(ValueError, match="rho0 must be negative"):
        O.logpolar_backproject(np.ones((16, 8)), 8, rho0=0.5)
    with pytest.raises(ValueError, match="log-polar mesh too coarse"):
        O.logpolar_backproject(np.ones((64, 8)), 8, nrho=3)


def test_against_reference_directly(reference):
    fb = reference
    rng = np.random.default_rng(5)
    g = rng.standard_normal((128, 96)).cumsum(0) * 0.01
    s = fb.Sinogram(*g.shape, g)
    assert rel(O.logpolar_backproject(g, 100), fb.logpolar_backproject(s, 100).values) < TOL
    assert rel(O.ramp_filter(g, 0.1, 0.7), fb.filter_sinogram(s, fb.FilterSpec(lam=0.1, cutoff=0.7)).values) < TOL
    assert rel(O.backproject_naive(g, 40), fb.backproject_naive(s, 40).values) < TOL
    p = fb.sinogram_to_semipolar(s)
    assert np.abs(O.semipolar(g) - p.values).max() == 0.0
    lp = fb.semipolar_to_logpolar(p, -3.0, 300)
    assert np.abs(O.logpolar_resample(p.values, -3.0, 300) - lp.values).max() == 0.0
    assert np.abs(O.lp_readout(lp.values, -3.0, 50, 50) - fb.logpolar_to_cartesian(lp, 50, 50).values).max() < 1e-15
