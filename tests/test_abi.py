"""C-ABI checks that need no GPU: the library loads, exports every symbol of
include/lpbp.h, validates arguments with the reference's messages, and its
host-only plans (device = -1) build fp64 tables that reproduce the oracle when
the device dataflow is emulated in numpy."""

import ctypes
import math
import os
import re
from ctypes import byref, c_size_t, c_void_p

import numpy as np
import pytest

from oracle import fastbp_oracle as O
from paper_1608_03589_b200 import _native as N

from conftest import REPO


def header_symbols():
    text = open(os.path.join(REPO, "include", "lpbp.h")).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\*]+\s+)+\**(lpbp_\w+)\s*\(", text, flags=re.M)))


def test_exports_every_header_symbol():
    lib = N.lib()
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(N.SIGNATURES) == syms
    assert lib.lpbp_version() >= 100


def make(nt, ntheta, n, rho0=None, nrho=None, filt=None, device=-1):
    p = N.Params()
    p.nt, p.ntheta, p.n_out = nt, ntheta, n
    p.has_rho0, p.rho0 = (0, 0.0) if rho0 is None else (1, rho0)
    p.nrho = nrho or 0
    p.filter, (p.lam, p.cutoff) = (0, (0.0, 1.0)) if filt is None else (1, filt)
    p.device = device
    h = c_void_p()
    N.check(N.lib().lpbp_plan_create(byref(p), byref(h)))
    return h


class HostPlan:
    def __init__(self, *a, **k):
        self.h = make(*a, **k)
        self.info = N.PlanInfo()
        N.check(N.lib().lpbp_plan_get_info(self.h, byref(self.info)))

    def __del__(self):
        N.lib().lpbp_plan_destroy(self.h)

    def table(self, which, dtype, width=1):
        n = c_size_t()
        N.check(N.lib().lpbp_plan_table(self.h, which.encode(), None, 0, byref(n)))
        a = np.zeros(n.value * width, dtype=dtype)
        N.check(N.lib().lpbp_plan_table(self.h, which.encode(), c_void_p(a.ctypes.data), n.value, byref(n)))
        return a.reshape(-1, width) if width > 1 else a


@pytest.mark.parametrize("nt,n", [(256, 256), (512, 512), (2048, 2048)])
def test_geometry_and_kernel_support(nt, n):
    hp = HostPlan(nt, nt, n, filt=(0.0, 1.0))
    ns, r0, nr, drho = O.lp_geometry(nt, n)
    i = hp.info
    assert (i.ns, i.nrho, i.nphi) == (ns, nr, 2 * nt)
    assert i.rho0 == r0 and i.drho == drho
    kern = np.roll(O.lp_kernel(nr, 2 * nt, drho), -nt, axis=1)
    k, l = np.nonzero(kern)
    cells = hp.table("kernel_cells", np.int32, 2)
    assert np.array_equal(cells[:, 0], k) and np.array_equal(cells[:, 1], l)
    assert i.kmax == k.max() and i.L >= nr + i.kmax and (i.L & (i.L - 1)) == 0
    assert i.M == 2 * nt and abs(i.out_scale - 1 / (2 * math.pi)) < 1e-15


def emulate_device(hp, g):
    """numpy (fp64) emulation of the K2..K5 dataflow using the plan's tables."""
    i = hp.info
    nt, nth = g.shape
    nphi, nh, nrho, L, ns = i.nphi, i.nphi // 2 + 1, i.nrho, i.L, i.ns
    G = np.fft.rfft(g, n=nphi, axis=1).T  # [m][t]     (K2)
    ab = hp.table("ab", np.int32, 2)
    wab = hp.table("wab", np.float32, 4).astype(np.float64)
    ki = hp.table("ki", np.int32)
    wi = hp.table("wi", np.float32, 2).astype(np.float64)
    khat = hp.table("khat", np.complex64).reshape(nh, L).astype(np.complex128)
    sg = np.where(np.arange(nh) % 2 == 1, -1.0, 1.0)[:, None]
    p = (wab[:, 0] * G[:, ab[:, 0]] + wab[:, 1] * G[:, ab[:, 0] + 1]
         + sg * (wab[:, 2] * G[:, ab[:, 1]] + wab[:, 3] * G[:, ab[:, 1] + 1]))      # [m][k]   (K3 p)
    x = wi[:, 0] * p[:, ki] + wi[:, 1] * p[:, ki + 1]                              # [m][i]
    y = np.fft.ifft(np.fft.fft(x, n=L, axis=1) * khat, axis=1)[:, :nrho] * L       # unnormalised inverse
    yt = y.T.copy()
    yt[:, 0] = yt[:, 0].real
    yt[:, -1] = yt[:, -1].real
    lp = np.fft.irfft(yt, n=nphi, axis=1) * nphi                                   # (K4)
    return lp


def emulate_readout(hp, lp):
    i = hp.info
    n, nrho, nphi = i.n_out, i.nrho, i.nphi
    qidx = hp.table("qidx", np.uint32)
    qw = hp.table("qw", np.float32, 2)
    c = n // 2
    nq = n - c
    iy, jx = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    yneg, xneg = iy < c, jx < c
    qy = np.where(yneg, (n - 1 - iy) - c, iy - c)
    qx = np.where(xneg, (n - 1 - jx) - c, jx - c)
    e = qidx[qy * nq + qx]
    w = qw[qy * nq + qx].astype(np.float64)
    valid = e != 0xFFFFFFFF
    i0 = (e & 0xFFFF).astype(np.int64)
    jr = np.where(valid, (e >> 16).astype(np.int64), 0)
    wjr = w[..., 1]
    Q = np.where(xneg & ~yneg, nphi // 2, nphi)
    refl = xneg ^ yneg
    j0 = np.where(~refl, np.where(xneg & yneg, nphi // 2 + jr, jr), np.where(wjr == 0, Q - jr, Q - jr - 1))
    wj = np.where(~refl, wjr, np.where(wjr == 0, 0.0, 1.0 - wjr))
    j0 = np.where(j0 >= nphi, j0 - nphi, j0)
    j1 = np.where(j0 + 1 == nphi, 0, j0 + 1)
    i0 = np.where(valid, i0, 0)
    i1 = np.minimum(i0 + 1, nrho - 1)
    wi = w[..., 0]
    r0 = lp[i0, j0] + wj * (lp[i0, j1] - lp[i0, j0])
    r1 = lp[i1, j0] + wj * (lp[i1, j1] - lp[i1, j0])
    return np.where(valid, (r0 + wi * (r1 - r0)) * i.out_scale, 0.0)


@pytest.mark.parametrize("nt,nth,n,rho0,nrho", [(256, 256, 256, None, None), (512, 256, 300, None, None),
                                                (512, 256, 256, -4.0, 600), (256, 128, 255, None, None)])
def test_tables_reproduce_oracle(golden, nt, nth, n, rho0, nrho):
    rng = np.random.default_rng(nt + n)
    g = rng.standard_normal((nt, nth)).cumsum(axis=0) * 0.05
    hp = HostPlan(nt, nth, n, rho0=rho0, nrho=nrho)
    lp = emulate_device(hp, g)
    ref_lp = O.logpolar_stage(g, n, rho0, nrho)
    assert O.relative_l2(lp, ref_lp) < 2e-6  # fp32-rounded tables
    img = emulate_readout(hp, ref_lp)
    ref = O.lp_readout(ref_lp, hp.info.rho0, n, n)
    assert O.relative_l2(img, ref) < 1e-6
    assert np.array_equal(img == 0, ref == 0)


def test_ramp_table_reproduces_filter_sinogram():
    nt, nth = 512, 64
    rng = np.random.default_rng(3)
    g = rng.standard_normal((nt, nth))
    for lam, cut in ((0.0, 1.0), (0.05, 0.8)):
        hp = HostPlan(nt, nth, 128, filt=(lam, cut))
        H = hp.table("ramp", np.float32).astype(np.float64)
        M = hp.info.M
        out = np.fft.ifft(np.fft.fft(g, n=M, axis=0) * H[:, None], axis=0).real[:nt] * M
        assert O.relative_l2(out, O.ramp_filter(g, lam, cut)) < 1e-6


def test_validation_messages():
    with pytest.raises(ValueError, match="n_out must be >= 2"):
        make(256, 256, 1)
    with pytest.raises(ValueError, match="rho0 must be negative"):
        make(256, 256, 64, rho0=0.25)
    with pytest.raises(ValueError, match="nrho must be >= 2"):
        make(256, 256, 64, nrho=1)
    with pytest.raises(ValueError, match="log-polar mesh too coarse"):
        make(64, 16, 16, nrho=3)
    with pytest.raises(ValueError, match="nt must be >= 2"):
        make(1, 16, 16)
    with pytest.raises(ValueError, match="cutoff must lie in"):
        make(256, 256, 64, filt=(0.0, 1.5))
    with pytest.raises(ValueError, match="lambda must be >= 0"):
        make(256, 256, 64, filt=(-1.0, 1.0))


def test_host_only_plan_refuses_execution():
    hp = HostPlan(256, 256, 256)
    buf = (ctypes.c_float * 16)()
    with pytest.raises(ValueError, match="host-only"):
        N.check(N.lib().lpbp_execute(hp.h, ctypes.addressof(buf), ctypes.addressof(buf), 1, None, 0, None))
    ws = c_size_t()
    N.check(N.lib().lpbp_workspace_bytes(hp.h, 4, byref(ws)))
    assert ws.value >= 4 * (hp.info.workspace_per_slice - 256) - 1024


@pytest.mark.parametrize("nt,nth,n,rho0", [(256, 256, 256, None), (512, 256, 255, None), (512, 256, 300, -4.0),
                                           (2048, 2048, 2048, None)])
def test_fused_readout_bands_cover_every_pixel_once(nt, nth, n, rho0):
    """Quad lists of the streaming fused inverse-DFT + readout kernel: every output
    pixel is written exactly once, zero exactly where the reference readout is zero,
    and each pixel's taps (i0, i0+1) lie in its quad's rows or the carried row above."""
    hp = HostPlan(nt, nth, n, rho0=rho0)
    i = hp.info
    off = hp.table("band_off", np.uint32).astype(np.int64)
    ent = hp.table("band_entries", np.uint32)
    qidx = hp.table("qidx", np.uint32)
    assert len(off) == i.nbands + 1 and off[-1] == len(ent) == len(qidx)
    c, nq = n // 2, n - n // 2
    writes = np.zeros((n, n), dtype=np.int32)
    zero = np.zeros((n, n), dtype=bool)
    for b in range(i.nbands):
        e = ent[off[b]:off[b + 1]]
        q = (e & 0x7FFFFFFF).astype(np.int64)
        z = (e & 0x80000000) != 0
        qy, qx = q // nq, q % nq
        r0 = i.row_min + b * i.band_rows
        assert r0 % 4 == 0
        qi = qidx[q[~z]]
        assert np.all(qi[qi != 0xFFFFFFFF] != 0xFFFFFFFF)
        i0 = (qi & 0xFFFF).astype(np.int64)
        assert np.all(i0 >= r0 - 1) and np.all(i0 < r0 + i.band_rows - 1)  # taps: carry row + own rows
        assert np.all(qidx[q[z]] == 0xFFFFFFFF)
        iyp, iyn, jxp, jxn = c + qy, n - 1 - c - qy, c + qx, n - 1 - c - qx
        dupy, dupx = iyn == iyp, jxn == jxp  # odd n: centre row/column mirror onto themselves
        for iy, jx, keep in ((iyp, jxp, np.ones_like(dupx)), (iyp, jxn, ~dupx), (iyn, jxp, ~dupy), (iyn, jxn, ~dupx & ~dupy)):
            pix = (iy * n + jx)[keep]
            np.add.at(writes.reshape(-1), pix, 1)
            zero.reshape(-1)[(iy * n + jx)[keep & z]] = True
    assert writes.min() == 1 and writes.max() == 1
    # bands whose rows no pixel taps carry no entries (the fused kernel skips them); every tapped
    # row's band is flagged
    need = hp.table("band_need", np.uint32)
    assert len(need) == i.nbands
    assert np.all(off[1:][need == 0] == off[:-1][need == 0])
    qv = qidx[qidx != 0xFFFFFFFF]
    i0 = (qv & 0xFFFF).astype(np.int64)
    for r in (i0, np.minimum(i0 + 1, i.nrho - 1)):
        assert np.all(need[(r - i.row_min) // i.band_rows] == 1)
    if (nt, n) == (2048, 2048):
        assert need.sum() < 0.7 * i.nbands  # ~1/3 of the bands lie between the innermost pixels' radii
    # work units: contiguous band ranges, outermost first, covering every band once, <= 24 bands each
    units = hp.table("units", np.uint32).reshape(-1, 2).astype(np.int64)
    assert units[0, 1] == i.nbands and units[-1, 0] == 0
    assert np.all(units[:-1, 0] == units[1:, 1]) and np.all(units[:, 1] > units[:, 0])
    assert np.all(units[:, 1] - units[:, 0] <= 24)
    xs = -1.0 + (np.arange(n) + 0.5) * (2.0 / n)
    X, Y = np.meshgrid(xs, xs)
    R = np.hypot(X, Y)
    ref_zero = ~((R <= 1.0) & (R > 0) & (np.log(np.maximum(R, 1e-300)) >= i.rho0))
    assert np.array_equal(zero, ref_zero)


@pytest.mark.parametrize("nt,nth", [(128, 90), (256, 180), (200, 96)])
def test_generic_size_bluestein_tables(nt, nth):
    """Generic sizes: the chirp / chirp-filter spectra make an MB-point circular
    convolution equal the length-nphi DFT (forward and inverse), and the ramp is
    embedded on M = pow2 >= 2 nt."""
    hp = HostPlan(nt, nth, 64, filt=(0.0, 1.0))
    i = hp.info
    nphi = 2 * nth
    assert i.generic == 1 and i.MB >= 2 * nphi and (i.MB & (i.MB - 1)) == 0
    assert i.M >= 2 * nt and (i.M & (i.M - 1)) == 0
    c = hp.table("chirp", np.complex64).astype(np.complex128)
    bf = hp.table("bhat_f", np.complex64).astype(np.complex128)
    bi = hp.table("bhat_i", np.complex64).astype(np.complex128)
    rng = np.random.default_rng(nphi)
    x = rng.standard_normal(nphi) + 1j * rng.standard_normal(nphi)
    MB = i.MB
    conv = np.fft.ifft(np.fft.fft(x * c, MB) * bf * MB)   # block_conv: unnormalised inverse, 1/MB in bhat
    X = c * conv[:nphi]
    assert np.abs(X - np.fft.fft(x)).max() / np.abs(X).max() < 1e-5
    conv = np.fft.ifft(np.fft.fft(x * np.conj(c), MB) * bi * MB)
    xi = np.conj(c) * conv[:nphi]
    assert np.abs(xi - np.fft.ifft(x) * nphi).max() / np.abs(xi).max() < 1e-5
    g = rng.standard_normal((nt, nth))
    H = hp.table("ramp", np.float32).astype(np.float64)
    out = np.fft.ifft(np.fft.fft(g, n=i.M, axis=0) * H[:, None], axis=0).real[:nt] * i.M
    assert O.relative_l2(out, O.ramp_filter(g)) < 1e-6


# ---- sector (partial) backprojection plans, host-only (no GPU needed) ----

def _sector_plan(nt, nth, n, sectors):
    arr = (N.Sector * max(1, len(sectors)))()
    for i, (t0, b, a) in enumerate(sectors):
        arr[i].theta0, arr[i].beta, arr[i].a_r = t0, b, a
    h = c_void_p()
    rc = N.lib().lpbp_sector_plan_create(nt, nth, n, arr, len(sectors), -1, byref(h))
    return rc, h


@pytest.mark.parametrize("nt,nth,n,sectors", [
    (256, 180, 128, [(k * math.pi / 4, math.pi / 8, 0.25) for k in range(4)]),
    (256, 256, 256, [(0.0, math.pi / 2, 0.25)]),
    (2048, 2048, 2048, [(k * math.pi / 4, math.pi / 8, 0.25) for k in range(4)]),
    (128, 96, 80, [(-0.4, math.pi / 6, 0.3), (math.pi / 3 - 0.4, math.pi / 6, 0.2), (2 * math.pi / 3 - 0.4, math.pi / 6, 0.45)]),
])
def test_sector_geometry_matches_oracle(nt, nth, n, sectors):
    rc, h = _sector_plan(nt, nth, n, sectors)
    assert rc == N.LPBP_OK, N.lib().lpbp_last_error()
    try:
        for k, (t0, b, a) in enumerate(sectors):
            inf = N.SectorInfo()
            assert N.lib().lpbp_sector_get_info(h, k, byref(inf)) == N.LPBP_OK
            jc, theta_c, rho0, nrho = O.sector_geometry(nt, nth, n, t0, b, a)
            assert (inf.jc, inf.nrho, inf.nphi) == (jc, nrho, 2 * nth)
            assert inf.theta_c == pytest.approx(theta_c, abs=1e-15)
            assert inf.rho0 == pytest.approx(rho0, abs=1e-15)
            assert inf.drho == pytest.approx(-rho0 / nrho, rel=1e-15)
            assert inf.L >= 2 * nrho - 1 and inf.L & (inf.L - 1) == 0
        ws = c_size_t()
        assert N.lib().lpbp_sector_workspace_bytes(h, 2, byref(ws)) == N.LPBP_OK and ws.value > 0
        # host-only plans refuse to execute
        assert N.lib().lpbp_sector_execute(h, c_void_p(16), c_void_p(16), 1, None, 0, None) == N.LPBP_EINVAL
    finally:
        N.lib().lpbp_sector_plan_destroy(h)


def test_sector_validation_messages_match_oracle():
    cases = [
        (16, [(0.0, math.pi / 2, 0.25)], "n_out must be >= 2", 1),
        (16, [], "at least one sector is required", None),
        (16, [(0.0, 2.0, 0.25)], "sector half-width beta must lie in (0, pi/2]", None),
        (16, [(0.0, 0.0, 0.25)], "sector half-width beta must lie in (0, pi/2]", None),
        (16, [(0.0, 1.0, 0.5)], "sector rescale a_r must lie in (0, 1/2)", None),
        (16, [(0.0, 0.7, 0.25)], None, None),
        (16, [(0.0, 0.5, 0.2), (2.0, 0.5, 0.2)], None, None),
    ]
    for n, sectors, msg, n_override in cases:
        nn = n_override or n
        rc, h = _sector_plan(64, 32, nn, sectors)
        with pytest.raises(ValueError) as e:
            O.partial_backproject(np.ones((64, 32)), sectors, nn)
        assert rc == N.LPBP_EINVAL
        got = N.lib().lpbp_last_error().decode()
        assert got == str(e.value)
        if msg:
            assert got == msg
    rc, _ = _sector_plan(64, 32, 16, [(0.0, math.pi / 2, 0.25)] * 33)
    assert rc == N.LPBP_EINVAL and "at most 32 sectors" in N.lib().lpbp_last_error().decode()


# ---- BST engine plans, host-only ----

def _bst_plan(nt, nth, n, beta=0.0, zero_pad=2.0, dc_mode=0, filt=0):
    p = N.BstParams()
    p.nt, p.ntheta, p.n_out, p.beta, p.zero_pad, p.dc_mode, p.filter = nt, nth, n, beta, zero_pad, dc_mode, filt
    p.lam, p.cutoff, p.device = 0.0, 1.0, -1
    h = c_void_p()
    return N.lib().lpbp_bst_plan_create(byref(p), byref(h)), h


@pytest.mark.parametrize("nt,nth,n,zp,supported", [(256, 256, 256, 2.0, 1), (512, 512, 512, 2.0, 1),
                                                   (2048, 2048, 2048, 2.0, 1), (256, 180, 128, 3.0, 1),
                                                   (200, 96, 101, 2.0, 1), (256, 180, 128, 1.0, 1),
                                                   (2048, 2048, 1024, 3.0, 0), (130, 64, 64, 2.0, 1)])
def test_bst_geometry_matches_oracle(nt, nth, n, zp, supported):
    rc, h = _bst_plan(nt, nth, n, zero_pad=zp)
    assert rc == N.LPBP_OK, N.lib().lpbp_last_error()
    try:
        inf = N.BstInfo()
        assert N.lib().lpbp_bst_get_info(h, byref(inf)) == N.LPBP_OK
        ns, ds, L, dsigma, m_need = O.bst_geometry(nt, n, zp)
        assert (inf.ns, inf.L, inf.m_need, inf.nray, inf.big) == (ns, L, m_need, 2 * nth, 2 * n)
        assert inf.ds == pytest.approx(ds, rel=1e-15) and inf.dsigma == pytest.approx(dsigma, rel=1e-15)
        assert inf.out_scale == pytest.approx(O.BST_SCALE / 16.0, rel=1e-15)
        assert inf.supported == supported
    finally:
        N.lib().lpbp_bst_plan_destroy(h)


def test_bst_validation_messages_match_oracle():
    for kw, args in ((dict(n_out=1), (64, 32, 1)), (dict(n_out=8, beta=-1.0), (64, 32, 8, -1.0)),
                     (dict(n_out=8, zero_pad=0.5), (64, 32, 8, 0.0, 0.5)),
                     (dict(n_out=8, dc_mode="x"), (64, 32, 8, 0.0, 2.0, 7))):
        rc, _ = _bst_plan(*args)
        assert rc == N.LPBP_EINVAL
        with pytest.raises(ValueError) as e:
            O.bst_validate(**kw)
        assert N.lib().lpbp_last_error().decode() == str(e.value)
    rc, _ = _bst_plan(64, 32, 256)
    with pytest.raises(ValueError) as e:
        O.bst_geometry(64, 256)
    assert rc == N.LPBP_EINVAL and N.lib().lpbp_last_error().decode() == str(e.value)


# ---- the path's host-side kernel table (make_logpolar_kernel) ----

@pytest.mark.parametrize("nrho,nphi,drho", [(353, 512, 1.570872e-2), (796, 1024, 7.837091e-3), (64, 90, 0.05),
                                            (3900, 4096, 1.955031e-3)])
def test_make_logpolar_kernel_matches_oracle(nrho, nphi, drho):
    import paper_1608_03589_b200 as p
    got = p.make_logpolar_kernel(nrho, nphi, drho)
    assert np.array_equal(got, O.lp_kernel(nrho, nphi, drho))


def test_make_logpolar_kernel_against_reference(reference):
    import paper_1608_03589_b200 as p
    from fastbp.logpolar import make_logpolar_kernel, truncation_error_bound
    for args in ((353, 512, 1.570872e-2), (101, 77, 0.031)):
        assert np.array_equal(p.make_logpolar_kernel(*args), make_logpolar_kernel(*args))
    assert p.truncation_error_bound(-3.1, 0.7) == truncation_error_bound(-3.1, 0.7)
    for call, msg in ((lambda: p.make_logpolar_kernel(1, 8, 0.1), "kernel mesh must be at least 2 x 2"),
                      (lambda: p.make_logpolar_kernel(8, 8, 0.0), "drho must be positive"),
                      (lambda: p.truncation_error_bound(-1.0, -1.0), "c must be >= 0")):
        with pytest.raises(ValueError, match=msg):
            call()


def test_bst_host_helpers_against_reference(reference):
    import paper_1608_03589_b200 as p
    from fastbp.bst import kaiser_window, sigma_kernel
    for ns, beta in ((8, 3.0), (2048, 0.0), (513, 8.0)):
        np.testing.assert_allclose(p.kaiser_window(ns, beta), kaiser_window(ns, beta), rtol=1e-14, atol=0)
    assert np.array_equal(p.sigma_kernel(10, 0.3), sigma_kernel(10, 0.3))
    with pytest.raises(ValueError, match="ns must be >= 2"):
        p.kaiser_window(1, 1.0)
    with pytest.raises(ValueError, match="dsigma must be positive"):
        p.sigma_kernel(4, 0.0)


def test_synth_configs_match_oracle_phantoms():
    """bench.py's measured arm reads the package's copy of the config table; it must not drift."""
    from oracle import phantoms
    from paper_1608_03589_b200 import synth
    assert synth.CONFIGS == phantoms.CONFIGS
    assert synth.BASE_SEED == phantoms.BASE_SEED
    for seed in (phantoms.BASE_SEED, phantoms.BASE_SEED + 7919 * 3 + 11):
        e = phantoms.random_ellipses(seed, 50, 0.01, 0.3)
        ref = np.stack([e.cx, e.cy, e.a, e.b, e.tilt, e.rho], axis=1)
        assert np.array_equal(synth.ellipse_params(seed, 50, 0.01, 0.3), ref)


def test_ellipse_containers_mirror_reference():
    """Ellipse / EllipseSet (phantoms.py:36-62): same fields, same ValueError messages; the
    device entry point fails loudly without CUDA."""
    import json as _json
    import paper_1608_03589_b200 as p
    with open(os.path.join(REPO, "tests", "golden", "kat_radon.json")) as f:
        kat = _json.load(f)
    with pytest.raises(ValueError) as e:
        p.Ellipse((0.0, 0.0), (0.0, 0.1), 0.0, 1.0)
    assert str(e.value) == kat["semi_axes_message"]
    with pytest.raises(ValueError) as e:
        p.EllipseSet(())
    assert str(e.value) == kat["empty_set_message"]
    es = p.EllipseSet((p.Ellipse((0.1, -0.2), (0.3, 0.2), 0.5, 1.5), p.Ellipse((0.0, 0.0), (0.1, 0.1), 0.0, -1.0)))
    assert len(es) == 2 and [x.intensity for x in es] == [1.5, -1.0]
    assert np.array_equal(es.params(), [[0.1, -0.2, 0.3, 0.2, 0.5, 1.5], [0.0, 0.0, 0.1, 0.1, 0.0, -1.0]])
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(RuntimeError, match="no CUDA device"):
            p.radon_ellipses(es, 16, 8)


@pytest.mark.parametrize("nth,q", [(3200, 25), (768, 3), (1280, 5), (2304, 9), (3840, 15), (6144, 3), (90, 0),
                                   (2048, 0), (3600, 0)])
def test_mixed_radix_row_dft_lengths(nth, q):
    """nphi = 2 ntheta of the form Q x 2^k (Q in {3, 5, 9, 15, 25}, within the instantiated range) is
    reported as a mixed-radix plan (phi_q = Q); power-of-two nphi takes the pow2 kernels (generic = 0),
    other lengths Bluestein (phi_q = 0).  6144 angles (nphi 12288 = 3 x 4096) would need a 32768-point
    Bluestein convolution and is supported only through the mixed-radix kernels."""
    hp = HostPlan(64, nth, 64)
    assert hp.info.phi_q == q
    assert hp.info.generic == (0 if nth == 2048 else 1)


@pytest.mark.parametrize("nt,nth,n", [(256, 256, 256), (512, 512, 512), (2048, 2048, 2048), (64, 256, 64), (1024, 512, 300)])
def test_k2p_tile_tables_reproduce_the_semipolar_image(nt, nth, n):
    """K2p forms the semi-polar rows (grids.py:290-311) from two runs of <= 5 sinogram rows per tile of
    4 rows: the host tables (ptile, ploc, wab) applied in numpy give the oracle's semipolar()."""
    hp = HostPlan(nt, nth, n)
    ns = nt // 2
    assert hp.info.p_rows == 1
    ptile = hp.table("ptile", np.int32).reshape(-1, 4)
    ploc = hp.table("ploc", np.uint32)
    wab = hp.table("wab", np.float32, 4).astype(np.float64)
    assert ptile.shape[0] == ns // 4 and ploc.shape[0] == ns
    rng = np.random.default_rng(nt + n)
    g = rng.standard_normal((nt, nth))
    p = np.zeros((ns, 2 * nth))
    for j in range(ns // 4):
        a_lo, na, b_lo, nb = (int(v) for v in ptile[j])
        assert 1 <= na <= 5 and 1 <= nb <= 5 and 0 <= a_lo and a_lo + na <= nt and 0 <= b_lo and b_lo + nb <= nt
        A, B = g[a_lo:a_lo + na], g[b_lo:b_lo + nb]      # the two TMA bulk copies
        for k in range(4 * j, 4 * j + 4):
            l = [(int(ploc[k]) >> s) & 15 for s in (0, 4, 8, 12)]
            assert l[0] < na and l[1] < na and l[2] < nb and l[3] < nb
            p[k, :nth] = wab[k, 0] * A[l[0]] + wab[k, 1] * A[l[1]]
            p[k, nth:] = wab[k, 2] * B[l[2]] + wab[k, 3] * B[l[3]]
    ref = O.semipolar(g)
    assert np.abs(p - ref).max() <= 2e-7 * np.abs(ref).max()


def test_k2p_needs_four_row_tiles():
    assert HostPlan(260, 256, 128).info.p_rows == 0   # ns = 130: K2's row spectra + K3's row mix


@pytest.mark.parametrize("nt,nth,n", [(256, 256, 256), (2048, 2048, 2048), (96, 1280, 64)])
def test_fused_row_maps(nt, nth, n):
    """The fused path's row placement (plan_host build_bands): K3 writes row r of a column at rowmap[r]
    (-1: a band no pixel taps, never written) and the fused readout fetches band b at band_row[b] - 1.
    Compacted: the needed bands sit back to back in row order; identity: every needed row in place."""
    hp = HostPlan(nt, nth, n)
    i = hp.info
    if i.band_rows == 0:
        pytest.skip("no fused readout for this nphi")
    need = hp.table("band_need", np.uint32)
    cp, ident = hp.table("rowmap_cp", np.int32), hp.table("rowmap_id", np.int32)
    bcp, bid = hp.table("band_row_cp", np.uint32), hp.table("band_row_id", np.uint32)
    bits = hp.table("row_need", np.uint32)
    S, r_min = i.band_rows, i.row_min
    assert len(need) == i.nbands and len(cp) == len(ident) == r_min + S * i.nbands
    pos = 0
    for b in range(i.nbands):
        rows = np.arange(r_min + S * b, r_min + S * (b + 1))
        if need[b]:
            assert bid[b] == rows[0] + 1 and bcp[b] == pos + 1
            assert np.array_equal(ident[rows], rows) and np.array_equal(cp[rows], pos + np.arange(S))
            pos += S
        else:
            assert bid[b] == 0 and bcp[b] == 0 and (ident[rows] == -1).all() and (cp[rows] == -1).all()
    assert (cp[:r_min] == -1).all()
    nrho_pad = (i.nrho + 15) // 16 * 16
    for r in range(min(len(cp), nrho_pad)):
        assert ((int(bits[r >> 5]) >> (r & 31)) & 1) == (1 if cp[r] >= 0 else 0)
    assert 0 < pos <= len(cp) and (n < 2048 or pos < 0.75 * i.nrho)   # about a third of the rows is skipped at 2048^2
