"""Direct pixel-driven backprojector (reference.py:21-37, configs[4]'s accuracy
cross-check) on the GPU through the C ABI (lpbp_naive_backproject): parity with
the oracle and with the reference's own 2048^2 output, slice-group invariance,
window geometry at extreme nt / n ratios, and the LP-vs-direct gap pinned to
the value the reference itself produces on the same slice."""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fastbp_oracle as O
from oracle import phantoms

pytestmark = pytest.mark.gpu
RTOL = 1e-4  # north_star: relative L2 <= 1e-4 in fp32
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


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


# (nt, ntheta, n, batch): square, ragged groups of 4, odd sizes, nt >> n (wide windows,
# fewer angles per stage), n >> nt (narrow windows), a single angle
CASES = [(256, 256, 256, 1), (128, 90, 64, 5), (200, 96, 101, 3), (512, 64, 48, 2), (64, 48, 300, 1),
         (255, 77, 129, 6), (96, 1, 40, 2)]


@pytest.mark.parametrize("nt,ntheta,n,batch", CASES)
def test_direct_vs_oracle(pkg, nt, ntheta, n, batch):
    sinos = np.stack([phantoms.sinogram(900 + i, nt, ntheta, 8, 0.05, 0.35, 0.01) for i in range(batch)])
    out = pkg.backproject_naive_batch(dev(sinos), n).cpu().numpy()
    assert out.shape == (batch, n, n)
    for i in range(batch):
        ref = O.backproject_naive(sinos[i].astype(np.float64), n)
        assert report(f"direct {nt}x{ntheta}->{n} slice {i}", out[i], ref) <= RTOL


def test_direct_group_invariance(pkg):
    """Slices are packed 4 per group; a slice's image must not depend on its group mates
    or its position (bitwise)."""
    sinos = np.stack([phantoms.sinogram(950 + i, 256, 180, 8, 0.05, 0.35, 0.01) for i in range(7)])
    d = dev(sinos)
    full = pkg.backproject_naive_batch(d, 200)
    for i in (0, 3, 4, 6):
        one = pkg.backproject_naive_batch(d[i:i + 1].clone(), 200)[0]
        assert torch.equal(one, full[i]), i
    rev = pkg.backproject_naive_batch(d.flip(0).contiguous(), 200)
    assert torch.equal(rev.flip(0), full)


def test_direct_zero_and_linearity(pkg):
    z = torch.zeros((2, 128, 64), device="cuda")
    assert torch.count_nonzero(pkg.backproject_naive_batch(z, 96)) == 0
    a = dev(phantoms.sinogram(970, 128, 64, 6, 0.05, 0.35, 0.0))
    b = dev(phantoms.sinogram(971, 128, 64, 6, 0.05, 0.35, 0.0))
    ia, ib, iab = (pkg.backproject_naive_batch(x[None], 96)[0].double() for x in (a, b, 2 * a - 3 * b))
    assert O.relative_l2((2 * ia - 3 * ib).cpu().numpy(), iab.cpu().numpy()) < 1e-6


def test_direct_errors(pkg):
    with pytest.raises(ValueError, match="n must be >= 2"):
        pkg.backproject_naive(pkg.Sinogram(16, 8, np.ones((16, 8))), 1)


@pytest.mark.slow
def test_cfg4_direct_vs_reference_rows_and_gap(pkg, golden):
    """configs[4] on config-2 slice 0: the GPU direct image against the REFERENCE's own
    backproject_naive rows (tests/golden/make_cfg4.py), and the LP-vs-direct gap against
    the reference's gap on the same slice (both GPU images are <= 1e-6 from the oracle,
    so the gaps agree to well under 1 %)."""
    z = golden("cfg4.npz")
    s = phantoms.config_sinogram(4, 0)
    d = dev(s)[None]
    nv = pkg.backproject_naive_batch(d, 2048)[0].cpu().numpy()
    rows = z["rows"]
    assert report("cfg4 direct rows vs reference", nv[rows], z["naive_rows"]) <= RTOL
    lp = pkg.logpolar_backproject_batch(d, 2048)[0].cpu().numpy()
    assert report("cfg4 LP rows vs reference", lp[rows], z["lp_rows"]) <= RTOL
    xs = -1.0 + (np.arange(2048) + 0.5) * (2.0 / 2048)
    X, Y = np.meshgrid(xs, xs)
    disk = np.hypot(X, Y) <= 1.0
    gap = O.relative_l2(lp[disk], nv[disk])
    full = O.relative_l2(lp, nv)
    ref_gap, ref_full = float(z["gap_disk"]), float(z["gap_full"])
    print(f"cfg4 LP vs direct: unit disk {gap:.4e} (reference {ref_gap:.4e}), full {full:.4e} (reference {ref_full:.4e})")
    assert abs(gap - ref_gap) <= 0.01 * ref_gap
    assert abs(full - ref_full) <= 0.01 * ref_full


@pytest.mark.slow
def test_cfg4_direct_four_slices_vs_oracle(pkg):
    """Four config-4 (= config-2) slices at 2048^2 in one call (one slice group) against the
    oracle on sampled rows."""
    ids = [0, 1, 2, 3]
    sinos = np.stack([phantoms.config_sinogram(4, i) for i in ids])
    out = pkg.backproject_naive_batch(dev(sinos), 2048).cpu().numpy()
    rows = np.arange(11, 2048, 173)
    for i in range(len(ids)):
        ref = O.backproject_naive(sinos[i].astype(np.float64), 2048, rows=rows)
        assert report(f"cfg4 slice {i} rows", out[i][rows], ref) <= RTOL


def test_cfg4_golden_metadata():
    with open(os.path.join(GOLDEN, "kat_cfg4.json")) as f:
        kat = json.load(f)
    assert 1e-3 < kat["gap_disk"] < 5e-3  # ~2e-3 in the unit disk at 2048^2
