"""GPU parity of the BST engine (fastbp.bst, bst.py:120-206) and of fbp's default
engine, through liblpbp.so's lpbp_bst_* C ABI: against the reference's golden
vectors (tests/golden/bst.npz, made by the reference itself) and the CPU oracle.
Bar: relative L2 <= 1e-4 in fp32, max-abs reported."""

import json
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fastbp_oracle as O
from oracle import phantoms

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

RTOL = 1e-4


@pytest.fixture(scope="module")
def pkg():
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    import paper_1608_03589_b200 as p
    return p


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def report(name, got, ref):
    r = O.relative_l2(got, ref)
    print(f"{name}: rel_l2={r:.3e} max_abs={O.max_abs(got, ref):.3e}")
    return r


def test_bst_cfg0_vs_reference_golden(pkg, golden):
    z = golden("bst.npz")
    g = phantoms.config_sinogram(0).astype(np.float64)
    s = pkg.Sinogram(*g.shape, g)
    assert report("bst cfg0", pkg.bst_backproject(s, pkg.BstOptions(n_out=256)).values, z["cfg0_bp"]) <= RTOL
    # fbp's default engine is "bst"
    assert report("fbp(bst) cfg0", pkg.fbp(s, pkg.FilterSpec(), n=256).values, z["cfg0_fbp"]) <= RTOL


def test_bst_cfg1_fbp_vs_reference_golden(pkg, golden):
    z = golden("bst.npz")
    g = phantoms.config_sinogram(1, 0).astype(np.float64)
    s = pkg.Sinogram(*g.shape, g)
    assert report("fbp(bst) cfg1", pkg.fbp(s, pkg.FilterSpec(), n=512).values, z["cfg1_fbp"]) <= RTOL
    tik = pkg.fbp(s, pkg.FilterSpec(lam=0.02, cutoff=0.9), engine="bst", n=512).values
    assert report("fbp(bst) cfg1 tikhonov", tik, z["cfg1_fbp_tik"]) <= RTOL


def test_bst_options(pkg, golden):
    z = golden("bst.npz")
    g = z["opt_sino"].astype(np.float64)
    s = pkg.Sinogram(*g.shape, g)
    assert report("bst beta=2", pkg.bst_backproject(s, pkg.BstOptions(n_out=128, beta=2.0)).values,
                  z["opt_beta2"]) <= RTOL
    cap = pkg.bst_backproject(s, pkg.BstOptions(n_out=128, beta=4.0, dc_mode="kernel_cap")).values
    assert report("bst kernel_cap beta=4", cap, O.bst_backproject(g, 128, beta=4.0, dc_mode="kernel_cap")) <= RTOL
    zp = pkg.bst_backproject(s, pkg.BstOptions(n_out=128, zero_pad=1.0)).values
    assert report("bst zero_pad=1", zp, O.bst_backproject(g, 128, zero_pad=1.0)) <= RTOL


@pytest.mark.parametrize("nt,nth,n,kw", [(256, 180, 64, dict(zero_pad=2.0)), (256, 180, 64, dict(zero_pad=4.0, beta=8.0)),
                                         (128, 90, 64, {}), (512, 360, 128, dict(zero_pad=8.0))])
def test_bst_reference_script_sizes(pkg, nt, nth, n, kw):
    """The sizes and options the reference's own BST experiments use (n 64/128, z 2/4/8)."""
    g = phantoms.sinogram(700 + nt + n, nt, nth, 8, 0.05, 0.35, 0.01).astype(np.float64)
    img = pkg.bst_backproject(pkg.Sinogram(nt, nth, g), pkg.BstOptions(n_out=n, **kw)).values
    assert report(f"bst {nt}x{nth}->{n} {kw}", img, O.bst_backproject(g, n, **kw)) <= RTOL


def test_bst_generic_sizes_vs_reference_golden(pkg, golden):
    """Non-power-of-two radial lengths and padded sides run through Bluestein convolutions."""
    z = golden("bst.npz")
    g = z["opt_sino"].astype(np.float64)  # 256 x 180, zero_pad = 3 -> L = 1536
    img = pkg.bst_backproject(pkg.Sinogram(*g.shape, g),
                              pkg.BstOptions(n_out=128, beta=4.0, zero_pad=3.0, dc_mode="kernel_cap")).values
    assert report("bst zero_pad=3 (L=1536) kernel_cap beta=4", img, z["opt_beta4_zp3_cap"]) <= RTOL
    g3 = z["odd_sino"].astype(np.float64)  # 200 x 96 -> n = 101 (padded side 202)
    img = pkg.bst_backproject(pkg.Sinogram(*g3.shape, g3), pkg.BstOptions(n_out=101)).values
    assert report("bst 200x96 -> 101", img, z["odd_n101"]) <= RTOL
    img = pkg.fbp(pkg.Sinogram(*g3.shape, g3), pkg.FilterSpec(lam=0.01), n=75).values
    assert report("fbp(bst) 200x96 -> 75", img, O.fbp_bst(g3, 75, lam=0.01)) <= RTOL


def test_bst_radial_stage(pkg, golden):
    z = golden("bst.npz")
    g = z["opt_sino"].astype(np.float64)
    plan = pkg.BstPlan(256, 180, pkg.BstOptions(n_out=128, dc_mode="kernel_cap"))
    got = plan.radial(dev(g)[None])[0].cpu().numpy().T  # -> [m][ray]
    H, dsig = O.bst_radial_spectra(g, 128)
    kern = np.empty(H.shape[0])
    kern[0] = 1.0 / dsig
    kern[1:] = 1.0 / (np.arange(1, H.shape[0]) * dsig)
    assert got.shape == H.shape
    assert report("bst radial stage", got, 0.5 * H * kern[:, None]) <= RTOL


def test_bst_batch_host_and_linearity(pkg):
    sino = np.stack([phantoms.sinogram(500 + i, 512, 512, 12, 0.05, 0.35, 0.01) for i in range(4)])
    plan = pkg.BstPlan(512, 512, pkg.BstOptions(n_out=512), filter_spec=(0.0, 1.0))
    full = plan.execute(dev(sino))
    for chunk in (1, 3):
        assert torch.equal(plan.execute(dev(sino), chunk=chunk), full)
    assert np.array_equal(plan.execute_host(sino, chunk=2), full.cpu().numpy())
    assert plan.last_launches >= 4
    ref = O.fbp_bst(sino[1].astype(np.float64), 512)
    assert report("fbp(bst) 512 batch slice 1", full[1].cpu().numpy(), ref) <= RTOL
    # linearity (the mean restoration is linear too)
    a, b = dev(sino[0]), dev(sino[2])
    ia, ib, iab = (plan.execute(x[None])[0].double() for x in (a, b, 2 * a - 3 * b))
    assert O.relative_l2((2 * ia - 3 * ib).cpu().numpy(), iab.cpu().numpy()) < 1e-5


def test_bst_profiling_and_pipelined_host_path(pkg):
    """Stage events cover ramp / radial / grid_x / grid_y once per chunk; the pipelined host path
    (two staging slots, H2D / compute / D2H streams) is bitwise equal to the device path for ragged
    chunking and for a chunk size change between calls (the staging is re-sized)."""
    sino = np.stack([phantoms.sinogram(700 + i, 256, 256, 8, 0.05, 0.35, 0.01) for i in range(7)])
    plan = pkg.BstPlan(256, 256, pkg.BstOptions(n_out=256), filter_spec=(0.0, 1.0))
    plan.profile(True)
    full = plan.execute(dev(sino), chunk=3)
    st = plan.profile_read()
    plan.profile(False)
    assert set(st) == {"ramp_filter", "bst_radial", "bst_grid_x", "bst_grid_y"}
    assert all(v["launches"] == 3 and v["slices"] == 7 and v["ms"] > 0 for v in st.values())
    ref = full.cpu().numpy()
    for chunk in (2, 5, 3):
        got = plan.execute_host(sino, chunk=chunk)
        assert np.array_equal(got, ref), chunk
    assert plan.last_launches == 4 * 3


def test_bst_2048_fbp_vs_oracle(pkg):
    """Config-3 geometry through fbp's default engine."""
    g = phantoms.config_sinogram(3, 5)
    img = pkg.fbp(pkg.Sinogram(*g.shape, g.astype(np.float64)), pkg.FilterSpec(), n=2048).values
    ref = O.fbp_bst(g.astype(np.float64), 2048)
    assert report("fbp(bst) 2048", img, ref) <= RTOL


def test_bst_errors(pkg):
    with open(os.path.join(GOLDEN, "kat_bst.json")) as f:
        kat = json.load(f)
    with pytest.raises(ValueError) as e:
        pkg.bst_backproject(pkg.Sinogram(64, 32, np.ones((64, 32))), pkg.BstOptions(n_out=256))
    assert str(e.value) == kat["too_fine_message"]
    for kw, msg in ((dict(n_out=1), "n_out must be >= 2"), (dict(n_out=8, beta=-1.0), "beta must be >= 0"),
                    (dict(n_out=8, zero_pad=0.5), "zero_pad must be >= 1"),
                    (dict(n_out=8, dc_mode="x"), "dc_mode must be 'subtract_mean' or 'kernel_cap'")):
        with pytest.raises(ValueError, match=msg):
            pkg.BstOptions(**kw)
    # sizes this build does not instantiate fail loudly (no fallback)
    with pytest.raises(NotImplementedError):  # odd nt
        pkg.bst_backproject(pkg.Sinogram(129, 96, np.ones((129, 96))), pkg.BstOptions(n_out=64))
    with pytest.raises(NotImplementedError):  # zero_pad = 3 at nt = 2048: L = 12288 > 4096 and not a power of two
        pkg.bst_backproject(pkg.Sinogram(2048, 64, np.ones((2048, 64))), pkg.BstOptions(n_out=512, zero_pad=3.0))


def test_bst_helpers(pkg, golden):
    z = golden("bst.npz")
    with open(os.path.join(GOLDEN, "kat_bst.json")) as f:
        kat = json.load(f)
    g = z["small_sino"].astype(np.float64)  # 128 x 90
    # polar_to_cartesian_frequency on the reference's own polar spectrum, padded lattice (dw = pi/2)
    H = z["small_H"]
    ps = pkg.PolarSpectrum(H.shape[0], H.shape[1], kat["small_dsigma"], H)
    grid = pkg.polar_to_cartesian_frequency(ps, 128, 128, dw=math.pi / 2)
    assert report("polar_to_cartesian_frequency", grid.values, z["small_grid"]) <= 1e-6
    # bst_spectrum: the engine's native product on the n_out lattice
    spec = pkg.bst_spectrum(pkg.Sinogram(*g.shape, g), pkg.BstOptions(n_out=64))
    assert report("bst_spectrum", spec.values, z["small_spectrum"]) <= RTOL
    # exact mean through <g, chord>
    m = pkg.mean_backprojection(pkg.Sinogram(256, 256, phantoms.config_sinogram(0).astype(np.float64)))
    assert abs(m - kat["mean_bp_cfg0"]) <= 1e-6 * abs(kat["mean_bp_cfg0"])
    with pytest.raises(ValueError, match="polar spectrum reaches sigma"):
        pkg.polar_to_cartesian_frequency(ps, 1024, 1024)
