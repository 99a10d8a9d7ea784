"""GPU parity of the path's standalone resampling steps (grids.py:290-347, 399-443)
against the oracle (pinned to the reference to ~1e-16 in tests/test_oracle_pin.py)."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fastbp_oracle as O
from oracle import phantoms

pytestmark = pytest.mark.gpu
RTOL = 1e-6  # pure resampling in fp32 with fp64 positions


@pytest.fixture(scope="module")
def pkg():
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    import paper_1608_03589_b200 as p
    return p


def report(name, got, ref):
    r = O.relative_l2(got, ref)
    print(f"{name}: rel_l2={r:.3e} max_abs={O.max_abs(got, ref):.3e}")
    return r


@pytest.mark.parametrize("nt,nth,ns", [(256, 256, None), (200, 90, None), (128, 96, 250)])
def test_sinogram_to_semipolar(pkg, nt, nth, ns):
    g = phantoms.sinogram(900 + nt, nt, nth, 8, 0.05, 0.35, 0.01).astype(np.float64)
    p = pkg.sinogram_to_semipolar(pkg.Sinogram(nt, nth, g), ns)
    assert p.values.shape == ((ns or nt // 2), 2 * nth)
    assert report(f"semipolar {nt}x{nth} ns={ns}", p.values, O.semipolar(g, ns)) <= RTOL


@pytest.mark.parametrize("rho0,nrho", [(-5.545177, 353), (-3.0, 300), (-1.2, 64)])
def test_semipolar_to_logpolar(pkg, rho0, nrho):
    g = phantoms.config_sinogram(0).astype(np.float64)
    p = O.semipolar(g)
    lp = pkg.semipolar_to_logpolar(pkg.PolarSinogram(*p.shape, p), rho0, nrho)
    assert (lp.nrho, lp.nphi, lp.rho0) == (nrho, p.shape[1], rho0)
    assert report(f"semi->lp rho0={rho0} nrho={nrho}", lp.values, O.logpolar_resample(p, rho0, nrho)) <= RTOL


@pytest.mark.parametrize("nx,ny", [(256, 256), (300, 170), (65, 64)])
def test_logpolar_to_cartesian(pkg, nx, ny):
    g = phantoms.config_sinogram(0).astype(np.float64)
    lp = O.logpolar_stage(g, 256)
    rho0 = O.adaptive_rho0(256, 256)
    img = pkg.logpolar_to_cartesian(pkg.LogPolarImage(*lp.shape, rho0, lp), nx, ny)
    assert img.values.shape == (ny, nx)
    assert report(f"lp->cart {nx}x{ny}", img.values, O.lp_readout(lp, rho0, nx, ny)) <= RTOL


def test_composition_equals_fused_stage(pkg):
    """semipolar -> logpolar on the device equals the oracle's composition on 2048^2 sizes too."""
    g = phantoms.config_sinogram(2, 0).astype(np.float64)
    ns, r0, nr, _ = O.lp_geometry(2048, 2048)
    p = pkg.sinogram_to_semipolar(pkg.Sinogram(2048, 2048, g))
    lp = pkg.semipolar_to_logpolar(p, r0, nr)
    assert report("2048 semipolar", p.values, O.semipolar(g)) <= RTOL
    assert report("2048 semi->lp", lp.values, O.logpolar_resample(O.semipolar(g), r0, nr)) <= RTOL


def test_resample_errors(pkg):
    g = pkg.Sinogram(64, 32, np.ones((64, 32)))
    with pytest.raises(ValueError, match="ns must be >= 2"):
        pkg.sinogram_to_semipolar(g, 1)
    p = pkg.sinogram_to_semipolar(g)
    with pytest.raises(ValueError, match="nrho must be >= 2"):
        pkg.semipolar_to_logpolar(p, -2.0, 1)
    with pytest.raises(ValueError, match="rho0 must be negative"):
        pkg.semipolar_to_logpolar(p, 0.5, 10)
    lp = pkg.semipolar_to_logpolar(p, -2.0, 40)
    with pytest.raises(ValueError, match="nx and ny must be >= 2"):
        pkg.logpolar_to_cartesian(lp, 1, 8)


def test_logpolar_stage_vs_direct_stencil(pkg):
    """GPU log-polar stage (row DFTs + FFT convolution + inverse DFTs) against the convolution
    summed directly over the 507 kernel cells of config 0 (no FFT in the check)."""
    from test_oracle_pin import _direct_stencil
    g = phantoms.config_sinogram(0).astype(np.float64)
    ns, r0, nr, drho = O.lp_geometry(256, 256)
    direct = _direct_stencil(O.logpolar_resample(O.semipolar(g), r0, nr), drho)
    plan = pkg.get_plan(256, 256, 256, None, None, None)
    got = plan.logpolar(torch.from_numpy(g.astype(np.float32)).cuda()[None])[0].cpu().numpy()
    assert report("logpolar stage vs direct stencil", got, direct) <= 1e-4
