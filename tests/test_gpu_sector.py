"""GPU parity of the sector (partial) backprojection, fastbp.logpolar.partial_backproject
(logpolar.py:210-299), through liblpbp.so's lpbp_sector_* C ABI: against the
reference's golden vectors (tests/golden/sector.npz, made by the reference itself)
and the CPU oracle.  Bar: relative L2 <= 1e-4 in fp32, max-abs reported."""

import json
import math
import os
import warnings

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


def case(golden, key):
    z = golden("sector.npz")
    return z, z[f"{key}_sino"], [tuple(s) for s in z[f"{key}_sectors"]], int(z[f"{key}_n"])


@pytest.mark.parametrize("key", ["a", "b", "c"])
def test_sector_vs_reference_golden(pkg, golden, key):
    z, g, sectors, n = case(golden, key)
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        img = pkg.partial_backproject(pkg.Sinogram(*g.shape, g.astype(np.float64)), sectors, n)
    with open(os.path.join(GOLDEN, "kat_sector.json")) as f:
        kat = json.load(f)[f"sector_{key}"]
    assert sum(1 for w in caught if issubclass(w.category, RuntimeWarning)) == kat["runtime_warnings"]
    assert img.values.shape == (n, n)
    assert report(f"sector {key}", img.values, z[f"{key}_pb"]) <= RTOL


@pytest.mark.parametrize("key", ["a", "b", "c"])
def test_sector_stages(pkg, golden, key):
    """Sector 0's working-frame sinogram and its convolved log-polar image."""
    z, g, sectors, n = case(golden, key)
    plan = pkg.SectorPlan(g.shape[0], g.shape[1], n, sectors)
    with open(os.path.join(GOLDEN, "kat_sector.json")) as f:
        kat = json.load(f)[f"sector_{key}"]
    inf = plan.info[0]
    assert (inf["jc"], inf["nrho"]) == (kat["jc0"], kat["nrho_0"])
    assert inf["rho0"] == kat["rho0_0"]
    work = plan.prepare(0, dev(g)[None])
    assert report(f"sector {key} prep", work[0].cpu().numpy(), z[f"{key}_sec0_sino"]) <= 1e-6
    lp = plan.logpolar(0, dev(z[f"{key}_sec0_sino"])[None])[0].cpu().numpy()
    assert report(f"sector {key} logpolar", lp, z[f"{key}_sec0_lp"]) <= RTOL


def test_sector_single_covering_sector(pkg, golden):
    z, g, _, n = case(golden, "a")
    img = pkg.partial_backproject(pkg.Sinogram(*g.shape, g.astype(np.float64)), [(0.0, math.pi / 2, 0.25)], n)
    assert report("sector single", img.values, z["a_single_pb"]) <= RTOL


def test_sector_batch_and_chunk_invariance(pkg):
    """Slices are independent: any batch split / chunking gives bitwise-identical images."""
    sino = torch.stack([dev(phantoms.sinogram(300 + i, 256, 180, 8, 0.05, 0.35, 0.01)) for i in range(5)])
    sectors = [(k * math.pi / 3, math.pi / 6, 0.3) for k in range(3)]
    plan = pkg.SectorPlan(256, 180, 128, sectors)
    full = plan.execute(sino)
    for chunk in (1, 2, 5):
        assert torch.equal(plan.execute(sino, chunk=chunk), full)
    one = torch.cat([plan.execute(sino[i:i + 1]) for i in range(5)])
    assert torch.equal(one, full)
    assert plan.last_launches >= 1
    for i in (0, 4):
        ref = O.partial_backproject(sino[i].double().cpu().numpy(), sectors, 128)
        assert report(f"sector batch slice {i}", full[i].cpu().numpy(), ref) <= RTOL


def test_sector_host_path_matches_device(pkg):
    sino = np.stack([phantoms.sinogram(400 + i, 256, 180, 8, 0.05, 0.35, 0.01) for i in range(3)])
    sectors = [(k * math.pi / 4, math.pi / 8, 0.25) for k in range(4)]
    plan = pkg.SectorPlan(256, 180, 128, sectors)
    dev_out = plan.execute(dev(sino)).cpu().numpy()
    for chunk in (2, 1, 3):  # pipelined host path: ragged chunks, staging re-sized between calls
        assert np.array_equal(plan.execute_host(sino, chunk=chunk), dev_out), chunk


def test_sector_linearity_and_zero(pkg):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((128, 96)).cumsum(0).astype(np.float32) * 0.01
    b = rng.standard_normal((128, 96)).cumsum(0).astype(np.float32) * 0.01
    sectors = [(0.0, math.pi / 6, 0.3), (math.pi / 3, math.pi / 6, 0.2), (2 * math.pi / 3, math.pi / 6, 0.4)]
    plan = pkg.SectorPlan(128, 96, 80, sectors)
    ia, ib, iab = (plan.execute(dev(x)[None])[0].double() for x in (a, b, 2.0 * a - 3.0 * b))
    assert O.relative_l2((2 * ia - 3 * ib).cpu().numpy(), iab.cpu().numpy()) < 1e-5
    assert float(plan.execute(torch.zeros(1, 128, 96, device="cuda")).abs().max()) == 0.0
    ref = O.partial_backproject(a.astype(np.float64), sectors, 80)
    assert report("sector 128x96->80", ia.cpu().numpy(), ref) <= RTOL


def test_sector_2048_vs_oracle(pkg):
    """Config-2 geometry (2048 x 2048 -> 2048) with the reference experiment's four sectors."""
    g = phantoms.config_sinogram(2, 0)
    sectors = [(k * math.pi / 4, math.pi / 8, 0.25) for k in range(4)]
    img = pkg.partial_backproject_batch(dev(g)[None], sectors, 2048)[0].cpu().numpy()
    ref = O.partial_backproject(g.astype(np.float64), sectors, 2048)
    assert report("sector 2048 x4", img, ref) <= RTOL


def test_sector_errors(pkg):
    g = pkg.Sinogram(64, 32, np.ones((64, 32)))
    with pytest.raises(ValueError, match="n_out must be >= 2"):
        pkg.partial_backproject(g, [(0.0, math.pi / 2, 0.25)], 1)
    with pytest.raises(ValueError, match="at least one sector is required"):
        pkg.partial_backproject(g, [], 16)
    with pytest.raises(ValueError, match=r"sector half-width beta must lie in \(0, pi/2\]"):
        pkg.partial_backproject(g, [(0.0, 2.0, 0.25)], 16)
    with pytest.raises(ValueError, match=r"sector rescale a_r must lie in \(0, 1/2\)"):
        pkg.partial_backproject(g, [(0.0, 1.0, 0.5)], 16)
    with pytest.raises(ValueError, match="sectors do not cover the angle range: theta = 1.6690 uncovered"):
        pkg.partial_backproject(g, [(0.0, 0.7, 0.25)], 16)
