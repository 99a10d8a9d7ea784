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


# ---- sector (partial) backprojection, logpolar.py:153-299 ----

def _sector_case(z, key):
    return (z[f"{key}_sino"].astype(np.float64), [tuple(s) for s in z[f"{key}_sectors"]], int(z[f"{key}_n"]))


@pytest.mark.parametrize("key", ["a", "b", "c"])
def test_sector_backprojection(golden, key):
    z = golden("sector.npz")
    g, sectors, n = _sector_case(z, key)
    out, stages = O.partial_backproject(g, sectors, n, return_stages=True)
    assert rel(out, z[f"{key}_pb"]) < TOL
    assert rel(stages[0]["sino"], z[f"{key}_sec0_sino"]) < TOL
    assert rel(stages[0]["lp"], z[f"{key}_sec0_lp"]) < TOL
    with open(os.path.join(GOLDEN, "kat_sector.json")) as f:
        kat = json.load(f)[f"sector_{key}"]
    assert (stages[0]["jc"], stages[0]["rho0"], stages[0]["nrho"]) == (kat["jc0"], kat["rho0_0"], kat["nrho_0"])


def test_sector_known_answers(golden):
    """The reference's own sector experiment (scratch_fbp.py:33-49) on the seeded phantom of case a."""
    z = golden("sector.npz")
    g, sectors, n = _sector_case(z, "a")
    with open(os.path.join(GOLDEN, "kat_sector.json")) as f:
        kat = json.load(f)["sector_a"]
    xs = -1.0 + (np.arange(n) + 0.5) * (2.0 / n)
    R = np.hypot(*np.meshgrid(xs, xs))
    m = (R > 2 * math.exp(O.adaptive_rho0(n, n))) & (R <= 1.0)
    pb = O.partial_backproject(g, sectors, n)
    nv = O.backproject_naive(g, n)
    assert abs(np.linalg.norm(pb[m] - nv[m]) / np.linalg.norm(nv[m]) - kat["annulus_vs_naive"]) < 1e-12
    pb1 = O.partial_backproject(g, [(0.0, math.pi / 2, 0.25)], n)
    assert rel(pb1, z["a_single_pb"]) < TOL
    lp = O.logpolar_backproject(g, n)
    assert abs(np.linalg.norm(pb1[m] - lp[m]) / np.linalg.norm(lp[m]) - kat["single_vs_lp"]) < 1e-12


def test_sector_errors_match_reference():
    g = np.ones((64, 32))
    with pytest.raises(ValueError, match="n_out must be >= 2"):
        O.partial_backproject(g, [(0.0, math.pi / 2, 0.25)], 1)
    with pytest.raises(ValueError, match="at least one sector is required"):
        O.partial_backproject(g, [], 16)
    with pytest.raises(ValueError, match=r"sector half-width beta must lie in \(0, pi/2\]"):
        O.partial_backproject(g, [(0.0, 2.0, 0.25)], 16)
    with pytest.raises(ValueError, match=r"sector rescale a_r must lie in \(0, 1/2\)"):
        O.partial_backproject(g, [(0.0, 1.0, 0.5)], 16)
    with pytest.raises(ValueError, match="sectors do not cover the angle range: theta = 1.6690 uncovered"):
        O.partial_backproject(g, [(0.0, 0.7, 0.25)], 16)


def test_sector_against_reference_directly(reference):
    import warnings

    from fastbp.logpolar import partial_backproject
    fb = reference
    rng = np.random.default_rng(11)
    g = rng.standard_normal((128, 96)).cumsum(0) * 0.01
    sectors = [(0.1, 0.6, 0.3), (1.3, 0.5, 0.2), (2.2, 0.6, 0.4)]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ref = partial_backproject(fb.Sinogram(*g.shape, g), sectors, 70).values
    assert rel(O.partial_backproject(g, sectors, 70), ref) < TOL
    with pytest.raises(ValueError) as e_ref:
        partial_backproject(fb.Sinogram(64, 32, np.ones((64, 32))), [(0.0, 0.7, 0.25)], 16)
    with pytest.raises(ValueError) as e_or:
        O.partial_backproject(np.ones((64, 32)), [(0.0, 0.7, 0.25)], 16)
    assert str(e_ref.value) == str(e_or.value)


# ---- BST engine (bst.py:120-206), fbp's default engine ----

def test_bst_cfg_goldens(golden):
    z = golden("bst.npz")
    g0 = phantoms.config_sinogram(0).astype(np.float64)
    assert rel(O.bst_backproject(g0, 256), z["cfg0_bp"]) < TOL
    assert rel(O.fbp_bst(g0, 256), z["cfg0_fbp"]) < TOL
    g1 = phantoms.config_sinogram(1, 0).astype(np.float64)
    assert rel(O.fbp_bst(g1, 512), z["cfg1_fbp"]) < 1e-6            # stored as float32
    assert rel(O.fbp_bst(g1, 512, lam=0.02, cutoff=0.9), z["cfg1_fbp_tik"]) < 1e-6


def test_bst_options_and_odd_size(golden):
    z = golden("bst.npz")
    g = z["opt_sino"].astype(np.float64)
    assert rel(O.bst_backproject(g, 128, beta=4.0, zero_pad=3.0, dc_mode="kernel_cap"), z["opt_beta4_zp3_cap"]) < TOL
    assert rel(O.bst_backproject(g, 128, beta=2.0), z["opt_beta2"]) < TOL
    assert rel(O.bst_backproject(z["odd_sino"].astype(np.float64), 101), z["odd_n101"]) < TOL


def test_bst_stages_and_known_answers(golden):
    z = golden("bst.npz")
    with open(os.path.join(GOLDEN, "kat_bst.json")) as f:
        kat = json.load(f)
    g = z["small_sino"].astype(np.float64)
    H, dsig = O.bst_radial_spectra(g, 64)
    assert dsig == kat["small_dsigma"]
    assert rel(H, z["small_H"]) < TOL
    assert rel(O.polar_to_cartesian(H, dsig, 128, 128, math.pi / 2), z["small_grid"]) < TOL
    assert rel(O.bst_backproject(g, 64), z["small_bp"]) < TOL
    assert abs(O.mean_backprojection(phantoms.config_sinogram(0)) - kat["mean_bp_cfg0"]) < 1e-15
    with pytest.raises(ValueError) as e:
        O.bst_backproject(np.ones((64, 32)), 256)
    assert str(e.value) == kat["too_fine_message"]
    for kw, msg in ((dict(n_out=1), "n_out must be >= 2"), (dict(n_out=8, beta=-1.0), "beta must be >= 0"),
                    (dict(n_out=8, zero_pad=0.5), "zero_pad must be >= 1"),
                    (dict(n_out=8, dc_mode="x"), "dc_mode must be 'subtract_mean' or 'kernel_cap'")):
        with pytest.raises(ValueError, match=msg):
            O.bst_validate(**kw)


def test_bst_against_reference_directly(reference):
    from fastbp.bst import BstOptions, bst_backproject
    fb = reference
    rng = np.random.default_rng(21)
    g = rng.standard_normal((160, 120)).cumsum(0) * 0.01
    s = fb.Sinogram(*g.shape, g)
    for kw in ({}, dict(beta=3.0, zero_pad=1.5), dict(dc_mode="kernel_cap")):
        assert rel(O.bst_backproject(g, 90, **kw), bst_backproject(s, BstOptions(n_out=90, **kw)).values) < TOL
    assert rel(O.fbp_bst(g, 90, 0.1, 0.8), fb.fbp(s, fb.FilterSpec(lam=0.1, cutoff=0.8), n=90).values) < TOL


def _direct_stencil(lp: np.ndarray, drho: float) -> np.ndarray:
    """The log-polar convolution summed directly over the kernel's cells: causal in rho,
    circular in phi (the definition the FFT form of logpolar.py:100-118 implements)."""
    nrho, nphi = lp.shape
    kern = np.roll(O.lp_kernel(nrho, nphi, drho), -(nphi // 2), axis=1)
    out = np.zeros_like(lp)
    for k, l in zip(*np.nonzero(kern)):
        out[k:, :] += kern[k, l] * np.roll(lp[:nrho - k, :], l, axis=1)
    return 0.5 * drho * (2.0 * math.pi / nphi) * out


def test_fft_convolution_equals_direct_stencil():
    """SPEC's invariant (FFT convolution = direct spatial convolution) on the oracle."""
    rng = np.random.default_rng(9)
    for nrho, nphi in ((16, 16), (40, 64), (353, 512)):
        lp = rng.standard_normal((nrho, nphi))
        drho = 5.545177 / nrho
        assert rel(O.lp_convolve(lp, drho), _direct_stencil(lp, drho)) < 1e-10


# ---- SPEC.md examples and invariants, on the oracle ----

def test_spec_kernel_examples():
    for nrho, nphi, drho in ((353, 512, 1.570872e-2), (64, 90, 0.05)):
        k = O.lp_kernel(nrho, nphi, drho)            # columns theta_j = -pi + j 2pi/nphi
        j0 = nphi // 2                               # theta = 0
        assert k[0, j0] == 1.0 / drho
        if nphi % 4 == 0:
            assert not k[:, nphi // 4 + j0 if nphi // 4 + j0 < nphi else nphi // 4].any()  # theta = pi/2
    # support count grows linearly with nrho at fixed rho0 (ratio within [0.5, 2] per doubling)
    rho0 = -5.0
    counts = [int(np.count_nonzero(O.lp_kernel(nr, 512, -rho0 / nr))) for nr in (200, 400, 800)]
    for a, b in zip(counts, counts[1:]):
        assert 0.5 <= (b / a) / 2.0 <= 2.0


def test_spec_truncation_bound_examples():
    assert abs(2 * math.pi / 1024 ** 2 - 5.99e-6) < 5e-9
    from paper_1608_03589_b200.resample import truncation_error_bound as tb
    assert tb(-math.log(1024.0), 1.0) == pytest.approx(2 * math.pi / 1024 ** 2, rel=1e-15)
    assert tb(-3.0 - math.log(2.0), 1.3) == pytest.approx(tb(-3.0, 1.3) / 4.0, rel=1e-14)
    assert tb(-745.0, 1.0) == 0.0 or tb(-745.0, 1.0) < 1e-300


def test_spec_mesh_rule_every_size():
    """Delta rho <= Delta s for every mesh the adaptive rule builds (1 - e^{-drho} <= 2/ns)."""
    for nt in (64, 128, 200, 256, 512, 1000, 2048):
        for n in (32, 64, 100, 256, 512, 2048):
            ns, r0, nr, drho = O.lp_geometry(nt, n)
            assert 1.0 - math.exp(-drho) <= (2.0 / ns) * (1.0 + 1e-9)


def test_spec_truncation_error_is_bounded():
    """The squared-L2 change between two rho0 choices stays under the bound at the shallower
    rho0 with c = max |B g| near the origin (inequality direction only)."""
    g = phantoms.sinogram(31, 128, 90, 6, 0.05, 0.35, 0.0).astype(np.float64)
    n = 64
    r_deep = O.adaptive_rho0(n, n)
    r_shallow = r_deep + math.log(4.0)
    a = O.logpolar_backproject(g, n, rho0=r_deep)
    b = O.logpolar_backproject(g, n, rho0=r_shallow)
    xs = -1.0 + (np.arange(n) + 0.5) * (2.0 / n)
    R = np.hypot(*np.meshgrid(xs, xs))
    c = float(np.abs(a[R <= 2 * math.exp(r_shallow)]).max())
    err2 = float(np.sum((a - b) ** 2)) * (2.0 / n) ** 2
    assert err2 <= 2 * math.pi * c * c * math.exp(2 * r_shallow)


def test_oracle_radon_ellipses_pinned_to_reference(golden):
    """oracle/phantoms.radon_ellipses (the harness generator) vs the reference's radon_ellipses
    on the committed EllipseSet goldens (hand-picked, 300 ellipses, odd sizes)."""
    z = golden("radon.npz")
    for name in ("small", "many", "odd"):
        p = z[f"{name}_params"]
        ref = z[f"{name}_sino"]
        e = phantoms.EllipseParams(*(p[:, i].copy() for i in range(6)))
        got = phantoms.radon_ellipses(e, *ref.shape)
        assert np.max(np.abs(got - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref))), name
