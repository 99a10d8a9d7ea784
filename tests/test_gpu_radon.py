"""GPU parity of the input generator radon_ellipses (radon.py:38-61) through
liblpbp.so's lpbp_radon_ellipses{,_f64}: against the reference's own outputs
(tests/golden/radon.npz, made by tests/golden/make_golden.py --only-radon).
fp64 path: agreement to a few ulps (device vs host libm cos/sin); fp32 path:
rounding of the fp64 sum."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    import paper_1608_03589_b200 as p
    return p


def ellipse_set(p, prm):
    return p.EllipseSet(tuple(p.Ellipse((r[0], r[1]), (r[2], r[3]), r[4], r[5]) for r in prm))


@pytest.mark.parametrize("name", ["small", "many", "odd"])
def test_radon_ellipses_vs_reference_golden(pkg, golden, name):
    z = golden("radon.npz")
    prm, ref = z[f"{name}_params"], z[f"{name}_sino"]
    s = pkg.radon_ellipses(ellipse_set(pkg, prm), *ref.shape)
    assert isinstance(s, pkg.Sinogram) and s.values.dtype == np.float64 and s.values.shape == ref.shape
    scale = max(1.0, float(np.max(np.abs(ref))))
    err = float(np.max(np.abs(s.values - ref)))
    print(f"radon {name} ({len(prm)} ellipses, {ref.shape}): max_abs={err:.3e}")
    assert err <= 1e-12 * scale
    # fp32 batch path: two copies in one launch, rounding of the fp64 sums only
    got = pkg.synth.radon_ellipses_batch(np.stack([prm, prm]), *ref.shape, torch.device("cuda"))
    assert got.dtype == torch.float32
    for b in range(2):
        assert np.max(np.abs(got[b].cpu().numpy() - ref)) <= 1e-6 * scale


def test_radon_ellipses_feeds_the_path(pkg, golden):
    """Generator output straight into the drop-in backprojection: same result as the
    reference-generated sinogram."""
    z = golden("radon.npz")
    prm, ref = z["small_params"], z["small_sino"]
    s = pkg.radon_ellipses(ellipse_set(pkg, prm), *ref.shape)
    a = pkg.logpolar_backproject(s, 32).values
    b = pkg.logpolar_backproject(pkg.Sinogram(*ref.shape, ref), 32).values
    assert np.max(np.abs(a - b)) <= 1e-6 * max(1.0, float(np.max(np.abs(b))))


def test_radon_ellipses_host_abi(pkg, golden):
    """lpbp_radon_ellipses_host: numpy buffers in and out, as the INTEGRATION.md ctypes stub calls it."""
    from ctypes import c_void_p
    from paper_1608_03589_b200._native import check, lib
    z = golden("radon.npz")
    prm, ref = z["many_params"], z["many_sino"]
    params = np.ascontiguousarray(np.stack([prm, prm[::-1]]), dtype=np.float64)
    out = np.empty((2,) + ref.shape, dtype=np.float64)
    check(lib().lpbp_radon_ellipses_host(c_void_p(params.ctypes.data), prm.shape[0], ref.shape[0], ref.shape[1], 2,
                                         c_void_p(out.ctypes.data), 0))
    scale = max(1.0, float(np.max(np.abs(ref))))
    assert np.max(np.abs(out[0] - ref)) <= 1e-12 * scale
    assert np.max(np.abs(out[1] - ref)) <= 1e-11 * scale  # reversed order: sums re-associated
