"""CPU oracle for the log-polar backprojection / FBP path.

TEST INFRASTRUCTURE ONLY.  This module restates, in numpy/scipy (float64), the
algorithm of the fastbp reference package (arXiv 1608.03589,
/root/reference/pkg/src/fastbp) for the path this repository accelerates.  It is
imported only by tests/, by __graft_entry__.smoke() as the checker, and by
bench.py's CPU-baseline / --impl reference legs.  The product path
(paper_1608_03589_b200) never imports it.

Pinning: tests/test_oracle_pin.py checks every function here against golden
vectors produced by the reference itself (tests/golden/make_golden.py, run in a
container where /root/reference is importable) and, when the reference is
importable, directly against it.

Third-party arithmetic: the reference's FFTs are scipy.fft (pocketfft, scipy
1.18.1 in this image; next_fast_len = smallest 11-smooth length >= target).
The oracle calls the same scipy.fft entry points with the same lengths.

Conventions (grids.py:1-15): t_i = -1 + i*2/nt, theta_j = j*pi/ntheta, pixel
centres x_j = -1 + (j + 1/2)*2/n, semi-polar s_k = k/(ns-1), log-polar
rho_i = rho0 + (i+1)*drho with drho = -rho0/nrho, phi_j = j*2*pi/nphi.
"""

from __future__ import annotations

import math

import numpy as np
from scipy import fft as sfft

LOGPOLAR_SCALE = 0.5          # logpolar.py:47
FBP_SCALE = 1.0 / (2.0 * math.pi)  # filtering.py:27


# --------------------------------------------------------------------------
# interpolation primitives
# --------------------------------------------------------------------------

def lerp_rows(values: np.ndarray, fidx: np.ndarray) -> np.ndarray:
    """Per-column linear interpolation at fractional row positions; rows outside
    [0, n) contribute zero.  Restates grids.py:255-269 (_lerp_axis0)."""
    nrows = values.shape[0]
    lo = np.floor(fidx).astype(np.int64)
    frac = fidx - lo
    hi = lo + 1
    v_lo = np.take_along_axis(values, np.clip(lo, 0, nrows - 1), axis=0)
    v_hi = np.take_along_axis(values, np.clip(hi, 0, nrows - 1), axis=0)
    v_lo = np.where((lo >= 0) & (lo < nrows), v_lo, 0.0)
    v_hi = np.where((hi >= 0) & (hi < nrows), v_hi, 0.0)
    return v_lo * (1.0 - frac) + v_hi * frac


def lerp_1d(profile: np.ndarray, fidx: np.ndarray) -> np.ndarray:
    """1-D linear interpolation, zero outside.  Restates grids.py:272-282."""
    n = profile.shape[0]
    lo = np.floor(fidx).astype(np.int64)
    frac = fidx - lo
    a = np.where((lo >= 0) & (lo < n), profile[np.clip(lo, 0, n - 1)], 0.0)
    b = np.where((lo + 1 >= 0) & (lo + 1 < n), profile[np.clip(lo + 1, 0, n - 1)], 0.0)
    return a * (1.0 - frac) + b * frac


# --------------------------------------------------------------------------
# mesh sizing
# --------------------------------------------------------------------------

def adaptive_rho0(nx: int, ny: int) -> float:
    """grids.py:385-391: one octave below the finest pixel pitch."""
    if nx < 2 or ny < 2:
        raise ValueError("counts must be >= 2")
    return math.log(min(2.0 / nx, 2.0 / ny)) - math.log(2.0)


def compute_nrho(ns: int, nx: int, ny: int) -> int:
    """grids.py:372-382."""
    if ns < 2 or nx < 2 or ny < 2:
        raise ValueError("all counts must be >= 2")
    v = math.ceil(math.log(min(1.0 / nx, 1.0 / ny)) / math.log(1.0 - 2.0 / ns))
    return int(min(max(v, 2), 64 * ns))


def mesh_for(ns: int, rho0: float, nrho: int | None) -> int:
    """logpolar.py:84-97: resolution rule 1 - e^{-drho} <= 2/ns."""
    step = 2.0 / ns
    if nrho is None:
        nrho = max(2, int(math.ceil(-rho0 / -math.log1p(-step))))
    drho = -rho0 / nrho
    largest = 1.0 - math.exp(-drho)
    if largest > step * (1.0 + 1e-9):
        raise ValueError(
            "log-polar mesh too coarse: largest radial step "
            f"{largest:.3e} exceeds the sinogram step {step:.3e}"
        )
    return nrho


# --------------------------------------------------------------------------
# resampling: sinogram -> semi-polar -> log-polar
# --------------------------------------------------------------------------

def semipolar(g: np.ndarray, ns: int | None = None) -> np.ndarray:
    """Semi-polar unfolding p[ns][2*ntheta] of g[nt][ntheta] (grids.py:290-311):
    columns < ntheta read g at t = +s, the others at t = -s (the phi >= pi half)."""
    nt, ntheta = g.shape
    ns = nt // 2 if ns is None else ns
    if ns < 2:
        raise ValueError("ns must be >= 2")
    s = np.arange(ns) / (ns - 1.0)
    inv_dt = 1.0 / (2.0 / nt)
    pos = lerp_rows(g, np.broadcast_to(((s + 1.0) * inv_dt)[:, None], (ns, ntheta)).copy())
    neg = lerp_rows(g, np.broadcast_to(((1.0 - s) * inv_dt)[:, None], (ns, ntheta)).copy())
    return np.concatenate([pos, neg], axis=1)


def logpolar_resample(p: np.ndarray, rho0: float, nrho: int) -> np.ndarray:
    """Radial resampling s = e^rho onto rows rho_i = rho0 + (i+1)*drho
    (grids.py:332-347)."""
    if nrho < 2:
        raise ValueError("nrho must be >= 2")
    if not rho0 < 0:
        raise ValueError("rho0 must be negative")
    ns, nphi = p.shape
    drho = -rho0 / nrho
    rows = rho0 + (np.arange(nrho) + 1) * drho
    f = np.exp(rows) * (ns - 1.0)
    return lerp_rows(p, np.broadcast_to(f[:, None], (nrho, nphi)).copy())


# --------------------------------------------------------------------------
# kernel and convolution
# --------------------------------------------------------------------------

def lp_kernel(nrho: int, nphi: int, drho: float) -> np.ndarray:
    """Box-discretised delta kernel on the lag mesh (logpolar.py:66-81):
    1/drho where |e^{rho} cos(theta) - 1| <= drho, theta_j = -pi + j*2pi/nphi."""
    if nrho < 2 or nphi < 2:
        raise ValueError("kernel mesh must be at least 2 x 2")
    if not drho > 0:
        raise ValueError("drho must be positive")
    lag_rho = np.arange(nrho)[:, None] * drho
    lag_theta = -math.pi + np.arange(nphi)[None, :] * (2.0 * math.pi / nphi)
    hit = np.abs(np.exp(lag_rho) * np.cos(lag_theta) - 1.0) <= drho
    return hit * (1.0 / drho)


def lp_convolve(lp: np.ndarray, drho: float) -> np.ndarray:
    """FFT convolution of a log-polar image with the kernel, causal in rho
    (zero padding to next_fast_len(2*nrho)) and cyclic in phi; scaled by
    LOGPOLAR_SCALE*drho*dphi (logpolar.py:100-118)."""
    nrho, nphi = lp.shape
    kern = np.roll(lp_kernel(nrho, nphi, drho), -(nphi // 2), axis=1)
    length = sfft.next_fast_len(2 * nrho)
    spec = sfft.rfft2(lp, s=(length, nphi)) * sfft.rfft2(kern, s=(length, nphi))
    out = sfft.irfft2(spec, s=(length, nphi))[:nrho]
    return LOGPOLAR_SCALE * drho * (2.0 * math.pi / nphi) * out


def lp_readout(lp: np.ndarray, rho0: float, nx: int, ny: int) -> np.ndarray:
    """Bilinear sampling of a log-polar array at the Cartesian pixel centres
    (grids.py:399-443): zero for r > 1, r == 0 or ln r < rho0; periodic in phi;
    the sliver between rho0 and the first row clamps to row 0."""
    if nx < 2 or ny < 2:
        raise ValueError("nx and ny must be >= 2")
    nrho, nphi = lp.shape
    drho = -rho0 / nrho
    dphi = 2.0 * math.pi / nphi
    X, Y = np.meshgrid(-1.0 + (np.arange(nx) + 0.5) * (2.0 / nx), -1.0 + (np.arange(ny) + 0.5) * (2.0 / ny))
    r = np.hypot(X, Y)
    out = np.zeros((ny, nx))
    sel = (r <= 1.0) & (r > 0.0)
    if not sel.any():
        return out
    rho = np.log(r[sel])
    fi = (rho - rho0) / drho - 1.0
    fi = np.where((fi >= -1.0) & (fi < 0.0), 0.0, fi)
    fi = np.clip(fi, 0.0, nrho - 1.0)
    fj = np.mod(np.arctan2(Y[sel], X[sel]), 2.0 * math.pi) / dphi
    i0 = np.floor(fi).astype(np.int64)
    j0 = np.floor(fj).astype(np.int64)
    wi = fi - i0
    wj = fj - j0
    j0 = np.mod(j0, nphi)
    j1 = np.mod(j0 + 1, nphi)
    i1 = np.minimum(i0 + 1, nrho - 1)
    val = ((lp[i0, j0] * (1 - wi) + lp[i1, j0] * wi) * (1 - wj)
           + (lp[i0, j1] * (1 - wi) + lp[i1, j1] * wi) * wj)
    out[sel] = np.where(rho >= rho0, val, 0.0)
    return out


# --------------------------------------------------------------------------
# engines
# --------------------------------------------------------------------------

def lp_geometry(nt: int, n_out: int, rho0: float | None = None, nrho: int | None = None):
    """(ns, rho0, nrho, drho) exactly as logpolar_backproject derives them
    (logpolar.py:128-133)."""
    if n_out < 2:
        raise ValueError("n_out must be >= 2")
    if rho0 is not None and not rho0 < 0:
        raise ValueError("rho0 must be negative")
    if nrho is not None and nrho < 2:
        raise ValueError("nrho must be >= 2")
    ns = nt // 2
    r0 = rho0 if rho0 is not None else adaptive_rho0(n_out, n_out)
    nr = mesh_for(ns, r0, nrho)
    return ns, r0, nr, -r0 / nr


def logpolar_stage(g: np.ndarray, n_out: int, rho0: float | None = None, nrho: int | None = None) -> np.ndarray:
    """Convolved log-polar image: _logpolar_convolve(sinogram_to_semipolar(g))
    (logpolar.py:100-118, 134-135)."""
    g = np.asarray(g, dtype=np.float64)
    _, r0, nr, drho = lp_geometry(g.shape[0], n_out, rho0, nrho)
    return lp_convolve(logpolar_resample(semipolar(g), r0, nr), drho)


def logpolar_backproject(g: np.ndarray, n_out: int, rho0: float | None = None, nrho: int | None = None) -> np.ndarray:
    """logpolar.py:121-136."""
    g = np.asarray(g, dtype=np.float64)
    _, r0, nr, _ = lp_geometry(g.shape[0], n_out, rho0, nrho)
    return lp_readout(logpolar_stage(g, n_out, rho0, nrho), r0, n_out, n_out)


def ramp_filter(g: np.ndarray, lam: float = 0.0, cutoff: float = 1.0) -> np.ndarray:
    """filter_sinogram (filtering.py:54-70) with FilterSpec(lam, cutoff):
    per-angle FFT over t zero-padded to next_fast_len(8*nt), response
    |sigma|/(1+lam|sigma|) cut above cutoff*Nyquist, inverse, real part."""
    if lam < 0:
        raise ValueError("lambda must be >= 0")
    if not (0.0 < cutoff <= 1.0):
        raise ValueError("cutoff must lie in (0, 1]")
    g = np.asarray(g, dtype=np.float64)
    nt = g.shape[0]
    dt = 2.0 / nt
    length = sfft.next_fast_len(8 * nt)
    sigma = 2.0 * math.pi * np.fft.fftfreq(length, d=dt)
    mag = np.abs(sigma)
    resp = mag / (1.0 + lam * mag)
    resp[np.abs(sigma) > cutoff * math.pi / dt] = 0.0
    return sfft.ifft(sfft.fft(g, n=length, axis=0) * resp[:, None], axis=0).real[:nt]


def fbp_logpolar(g: np.ndarray, n: int, lam: float = 0.0, cutoff: float = 1.0,
                 rho0: float | None = None, nrho: int | None = None) -> np.ndarray:
    """fbp(g, FilterSpec(lam, cutoff), engine='logpolar', n) (filtering.py:73-98)."""
    return FBP_SCALE * logpolar_backproject(ramp_filter(g, lam, cutoff), n, rho0, nrho)


def backproject_naive(g: np.ndarray, n: int, rows: np.ndarray | None = None) -> np.ndarray:
    """Pixel-driven backprojection b(x) = dtheta * sum_k lerp_t(g[:,k], (x.xi_k + 1)/dt)
    (reference.py:21-37).  `rows` restricts the evaluation to those image rows
    (returns shape (len(rows), n)) so large cases can be sampled."""
    if n < 2:
        raise ValueError("n must be >= 2")
    g = np.asarray(g, dtype=np.float64)
    nt, ntheta = g.shape
    xs = -1.0 + (np.arange(n) + 0.5) * (2.0 / n)
    ys = xs if rows is None else xs[np.asarray(rows)]
    X, Y = np.meshgrid(xs, ys)
    acc = np.zeros(X.shape)
    inv_dt = 1.0 / (2.0 / nt)
    dtheta = math.pi / ntheta
    for k in range(ntheta):
        th = k * dtheta
        acc += lerp_1d(g[:, k], (X * math.cos(th) + Y * math.sin(th) + 1.0) * inv_dt)
    return acc * dtheta


def _as_exact(a) -> np.ndarray:
    """Widen to float64 / complex128 without dropping anything: complex inputs stay
    complex (an fp64 cast would silently discard their imaginary parts)."""
    x = np.asarray(a)
    return x.astype(np.complex128 if np.iscomplexobj(x) else np.float64, copy=False)


def relative_l2(a, b) -> float:
    """metrics.py:29-36: ||a - b|| / ||b||, b the reference.  Complex arrays are
    compared as complex (the norm of the complex difference)."""
    x = _as_exact(a)
    y = _as_exact(b)
    if x.shape != y.shape:
        raise ValueError(f"dimension mismatch: {x.shape} vs {y.shape}")
    den = np.linalg.norm(y)
    if den == 0.0:
        return 0.0 if np.linalg.norm(x) == 0.0 else float("inf")
    return float(np.linalg.norm(x - y) / den)


def max_abs(a, b) -> float:
    """Largest |a - b| (complex modulus for complex inputs)."""
    return float(np.max(np.abs(_as_exact(a) - _as_exact(b))))


# --------------------------------------------------------------------------
# sector (partial) backprojection, logpolar.py:153-299
# --------------------------------------------------------------------------

def sector_masks(ntheta: int, sectors) -> tuple[list[np.ndarray], np.ndarray]:
    """Extended angular masks of every sector and the coverage count per angle
    (logpolar.py:238-248): angle j belongs to sector (theta0, beta, a_r) when its
    distance mod pi to theta0 + beta is <= beta + 2 dtheta (+1e-12)."""
    dtheta = math.pi / ntheta
    theta = np.arange(ntheta) * dtheta
    masks = []
    for theta0, beta, _ in sectors:
        c = theta0 + beta
        dist = np.abs(np.mod(theta - c + math.pi / 2.0, math.pi) - math.pi / 2.0)  # logpolar.py:186-188
        masks.append(dist <= beta + 2.0 * dtheta + 1e-12)
    cover = np.sum(masks, axis=0).astype(np.float64)
    return masks, cover


def sector_validate(sectors, n_out: int, ntheta: int) -> None:
    """Argument checks of partial_backproject (logpolar.py:218-227, 242-246)."""
    if n_out < 2:
        raise ValueError("n_out must be >= 2")
    if not sectors:
        raise ValueError("at least one sector is required")
    for _, beta, a_r in sectors:
        if not (0.0 < beta <= math.pi / 2.0):
            raise ValueError("sector half-width beta must lie in (0, pi/2]")
        if not (0.0 < a_r < 0.5):
            raise ValueError("sector rescale a_r must lie in (0, 1/2)")
    _, cover = sector_masks(ntheta, sectors)
    if np.any(cover == 0):
        th = (np.arange(ntheta) * (math.pi / ntheta))[cover == 0][0]
        raise ValueError(f"sectors do not cover the angle range: theta = {th:.4f} uncovered")


def sector_geometry(nt: int, ntheta: int, n_out: int, theta0: float, beta: float, a_r: float):
    """(jc, theta_c, rho0_s, nrho_s) of one sector: centre snapped to the angle grid,
    mesh depth from the support of the shifted, shrunk sector (logpolar.py:254-283)."""
    dtheta = math.pi / ntheta
    jc = int(round((theta0 + beta) / dtheta))
    ext = 2.0 * dtheta
    support_min = (1.0 - a_r) * math.cos(min(beta + ext, math.pi / 2.0)) - a_r
    if support_min > 0.05:
        rho0_s = min(math.log(support_min), math.log(1.0 - 2.0 * a_r)) - 0.2
    else:
        rho0_s = math.log(a_r) + adaptive_rho0(n_out, n_out)
    nrho_s = mesh_for(nt // 2, rho0_s, None)
    return jc, jc * dtheta, rho0_s, nrho_s


def sector_sinogram(g: np.ndarray, jc: int, weights_rot: np.ndarray, a_r: float) -> np.ndarray:
    """Working-frame sinogram of one sector: angles rolled by jc with the t-flip for
    columns that wrap past pi (logpolar.py:153-172), per-angle weights, support
    shrunk by a_r (out(t) = a_r g(t/a_r), :175-179) and shifted by (1 - a_r, 0)
    (radon.py:137-158: out(t, theta) = g(t - (1 - a_r) cos theta))."""
    g = np.asarray(g, dtype=np.float64)
    nt, nth = g.shape
    shift = jc % nth
    rolled = np.empty_like(g)
    for j in range(nth):
        src = j + shift
        col = g[:, src % nth]
        if src >= nth:
            col = np.concatenate([[0.0], col[:0:-1]])  # g(-t): t_0 = -1 maps off-grid to +1
        rolled[:, j] = col
    rolled = rolled * weights_rot[None, :]
    dt = 2.0 / nt
    t = -1.0 + np.arange(nt) * dt
    scaled = a_r * lerp_rows(rolled, np.broadcast_to(((t / a_r + 1.0) / dt)[:, None], (nt, nth)).copy())
    off = (1.0 - a_r) * np.cos(np.arange(nth) * (math.pi / nth))
    return lerp_rows(scaled, (t[:, None] - off[None, :] + 1.0) / dt)


def sector_weights_rot(ntheta: int, sectors, k: int) -> np.ndarray:
    """Weights of sector k in its rotated frame: extended mask / coverage
    (logpolar.py:263-268)."""
    masks, cover = sector_masks(ntheta, sectors)
    theta0, beta, _ = sectors[k]
    jc = int(round((theta0 + beta) / (math.pi / ntheta)))
    rot = (np.arange(ntheta) + jc) % ntheta
    w = np.zeros(ntheta)
    w[masks[k][rot]] = 1.0
    return w / cover[rot]


def lp_sample(lp: np.ndarray, rho0: float, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Bilinear log-polar sample at arbitrary points with the readout's boundary rules
    (logpolar.py:191-215)."""
    nrho, nphi = lp.shape
    drho = -rho0 / nrho
    dphi = 2.0 * math.pi / nphi
    r = np.hypot(x, y)
    out = np.zeros_like(r)
    sel = (r <= 1.0) & (r > 0.0)
    if not sel.any():
        return out
    rho = np.log(r[sel])
    fi = (rho - rho0) / drho - 1.0
    fi = np.where((fi >= -1.0) & (fi < 0.0), 0.0, fi)
    fi = np.clip(fi, 0.0, nrho - 1.0)
    fj = np.mod(np.arctan2(y[sel], x[sel]), 2.0 * math.pi) / dphi
    i0 = np.floor(fi).astype(np.int64)
    wi = fi - i0
    i1 = np.minimum(i0 + 1, nrho - 1)
    j0 = np.floor(fj).astype(np.int64) % nphi
    wj = fj - np.floor(fj)
    j1 = (j0 + 1) % nphi
    val = ((lp[i0, j0] * (1 - wi) + lp[i1, j0] * wi) * (1 - wj)
           + (lp[i0, j1] * (1 - wi) + lp[i1, j1] * wi) * wj)
    out[sel] = np.where(rho >= rho0, val, 0.0)
    return out


def partial_backproject(g: np.ndarray, sectors, n_out: int, return_stages: bool = False):
    """Sector-wise log-polar backprojection (logpolar.py:210-299): every sector's
    working-frame sinogram goes through the log-polar stage on its own shallow mesh,
    is read back at x_w = (1 - a_r, 0) + a_r R(-theta_c) x and divided by a_r; the
    sector results are summed."""
    g = np.asarray(g, dtype=np.float64)
    nt, nth = g.shape
    sectors = [tuple(map(float, s)) for s in sectors]
    sector_validate(sectors, n_out, nth)
    xs = -1.0 + (np.arange(n_out) + 0.5) * (2.0 / n_out)
    X, Y = np.meshgrid(xs, xs)
    acc = np.zeros((n_out, n_out))
    stages = []
    for k, (theta0, beta, a_r) in enumerate(sectors):
        jc, theta_c, rho0_s, nrho_s = sector_geometry(nt, nth, n_out, theta0, beta, a_r)
        gs = sector_sinogram(g, jc, sector_weights_rot(nth, sectors, k), a_r)
        lp = lp_convolve(logpolar_resample(semipolar(gs), rho0_s, nrho_s), -rho0_s / nrho_s)
        ct, st = math.cos(theta_c), math.sin(theta_c)
        xw = (1.0 - a_r) + a_r * (ct * X + st * Y)
        yw = a_r * (-st * X + ct * Y)
        acc += lp_sample(lp, rho0_s, xw, yw) / a_r
        if return_stages:
            stages.append({"jc": jc, "rho0": rho0_s, "nrho": nrho_s, "sino": gs, "lp": lp})
    return (acc, stages) if return_stages else acc


# --------------------------------------------------------------------------
# BST engine (frequency-domain backprojection), bst.py:1-206
# --------------------------------------------------------------------------

BST_SCALE = 4.0 * math.pi      # bst.py:47
BST_RADIAL_OVERSAMPLE = 2      # bst.py:52
BST_DOMAIN_PAD = 2             # bst.py:58


def bst_validate(n_out: int, beta: float = 0.0, zero_pad: float = 2.0, dc_mode: str = "subtract_mean") -> None:
    """BstOptions checks (bst.py:79-87)."""
    if n_out < 2:
        raise ValueError("n_out must be >= 2")
    if beta < 0:
        raise ValueError("beta must be >= 0")
    if zero_pad < 1:
        raise ValueError("zero_pad must be >= 1")
    if dc_mode not in ("subtract_mean", "kernel_cap"):
        raise ValueError("dc_mode must be 'subtract_mean' or 'kernel_cap'")


def kaiser(ns: int, beta: float) -> np.ndarray:
    """Kaiser-Bessel taper I0(beta sqrt(1 - u^2)) / I0(beta), u = (2i - ns + 1)/(ns - 1)
    (bst.py:90-102; I0 = scipy.special.i0 as phantoms.py:184-186)."""
    from scipy import special
    if ns < 2:
        raise ValueError("ns must be >= 2")
    u = (2.0 * np.arange(ns) - ns + 1.0) / (ns - 1.0)
    return np.abs(special.i0(beta * np.sqrt(np.maximum(1.0 - u * u, 0.0)))) / abs(float(special.i0(beta)))


def bst_geometry(nt: int, n_out: int, zero_pad: float = 2.0):
    """(ns, ds, L, dsigma, m_need) of the radial spectra (bst.py:128-143)."""
    ns = BST_RADIAL_OVERSAMPLE * (nt // 2)
    ds = 1.0 / (ns - 1)
    length = sfft.next_fast_len(max(int(math.ceil(2.0 * zero_pad * (ns - 1))), ns))
    dsigma = 2.0 * math.pi / (length * ds)
    m_need = int(math.floor(math.sqrt(2.0) * math.pi * n_out / 2.0 / dsigma)) + 2
    if m_need > length // 2 + 1:
        raise ValueError(
            f"n_out = {n_out} exceeds the resolution supported by an nt = {nt} "
            f"sinogram (max ~ {int(math.sqrt(2) * (ns - 1))})"
        )
    return ns, ds, length, dsigma, m_need


def bst_radial_spectra(g: np.ndarray, n_out: int, zero_pad: float = 2.0, beta: float = 0.0):
    """Windowed, zero-padded real DFTs along s of every semi-polar ray, first m_need
    bins, times ds; the s = 0 sample carries half weight (bst.py:120-143)."""
    g = np.asarray(g, dtype=np.float64)
    ns, ds, length, dsigma, m_need = bst_geometry(g.shape[0], n_out, zero_pad)
    prof = semipolar(g, ns) * kaiser(ns, beta)[:, None]
    prof[0, :] *= 0.5
    return ds * sfft.rfft(prof, n=length, axis=0)[:m_need], dsigma


def polar_to_cartesian(P: np.ndarray, dsigma: float, nx: int, ny: int, dw: float = math.pi) -> np.ndarray:
    """Bilinear (sigma, theta) gridding onto the FFT-ordered lattice omega = dw k,
    theta periodic, then Hermitian averaging with the mirror bin (grids.py:456-508)."""
    if nx < 2 or ny < 2:
        raise ValueError("nx and ny must be >= 2")
    nsig, nray = P.shape
    nyq = math.sqrt(2.0) * dw * max(nx, ny) / 2.0
    if (nsig - 1) * dsigma < nyq * (1.0 - 1e-12):
        raise ValueError(
            f"polar spectrum reaches sigma = {(nsig - 1) * dsigma:.3f} but the cartesian "
            f"grid requires coverage up to the Nyquist radius {nyq:.3f}"
        )
    wx = math.pi * np.fft.fftfreq(nx, d=1.0 / nx) * (dw / math.pi)
    wy = math.pi * np.fft.fftfreq(ny, d=1.0 / ny) * (dw / math.pi)
    WX, WY = np.meshgrid(wx, wy)
    fi = np.minimum(np.hypot(WX, WY) / dsigma, nsig - 1.0)
    i0 = np.floor(fi).astype(np.int64)
    wi = fi - i0
    i1 = np.minimum(i0 + 1, nsig - 1)
    fj = np.mod(np.arctan2(WY, WX), 2.0 * math.pi) / (2.0 * math.pi / nray)
    j0 = np.floor(fj).astype(np.int64)
    wj = fj - j0
    j0 = np.mod(j0, nray)
    j1 = np.mod(j0 + 1, nray)
    grid = (P[i0, j0] * (1 - wi) * (1 - wj) + P[i1, j0] * wi * (1 - wj)
            + P[i0, j1] * (1 - wi) * wj + P[i1, j1] * wi * wj)
    ix = (-np.arange(nx)) % nx
    iy = (-np.arange(ny)) % ny
    return 0.5 * (grid + np.conj(grid[np.ix_(iy, ix)]))


def bst_spectrum_to_image(P: np.ndarray, dsigma: float, n_out: int) -> np.ndarray:
    """Grid on the DOMAIN_PAD-times finer lattice, zero the Nyquist row/column,
    phase-ramp so pixel p0 lands on x = -1, inverse 2-D DFT, crop (bst.py:146-170)."""
    d = BST_DOMAIN_PAD
    big = d * n_out
    dw = math.pi / d
    grid = polar_to_cartesian(P, dsigma, big, big, dw)
    if big % 2 == 0:
        grid[big // 2, :] = 0.0
        grid[:, big // 2] = 0.0
    k = np.rint(np.fft.fftfreq(big, d=1.0 / big)).astype(np.int64)
    p0 = ((d - 1) * n_out) // 2
    dx = 2.0 / n_out
    tau = np.exp(1j * dw * k * ((0.5 - p0) * dx - 1.0))
    img = sfft.ifft2(grid * tau[:, None] * tau[None, :]) * (big * big / (4.0 * d * d))
    return img.real[p0:p0 + n_out, p0:p0 + n_out]


def square_chord(t, theta) -> np.ndarray:
    """Chord length of the line x . xi_theta = t through [-1, 1]^2 (radon.py:183-209)."""
    t = np.asarray(t, dtype=np.float64)
    theta = np.asarray(theta, dtype=np.float64)
    c, s = np.cos(theta), np.sin(theta)
    big = 1e30
    with np.errstate(divide="ignore", invalid="ignore"):
        lo_x = np.where(np.abs(s) > 1e-15, (t * c - 1.0) / s, -big)
        hi_x = np.where(np.abs(s) > 1e-15, (t * c + 1.0) / s, big)
        lo_y = np.where(np.abs(c) > 1e-15, (-t * s - 1.0) / c, -big)
        hi_y = np.where(np.abs(c) > 1e-15, (-t * s + 1.0) / c, big)
    lo = np.maximum(np.minimum(lo_x, hi_x), np.minimum(lo_y, hi_y))
    hi = np.minimum(np.maximum(lo_x, hi_x), np.maximum(lo_y, hi_y))
    ok = np.where(np.abs(s) > 1e-15, True, np.abs(t * c) <= 1.0) & np.where(np.abs(c) > 1e-15, True, np.abs(t * s) <= 1.0)
    return np.where(ok, np.maximum(0.0, hi - lo), 0.0)


def mean_backprojection(g: np.ndarray) -> float:
    """Spatial mean of the backprojection over [-1, 1]^2 via <B g, 1> = <g, chord>
    (bst.py:173-180)."""
    g = np.asarray(g, dtype=np.float64)
    nt, nth = g.shape
    t = (-1.0 + np.arange(nt) * (2.0 / nt))[:, None]
    theta = (np.arange(nth) * (math.pi / nth))[None, :]
    return float(np.sum(g * square_chord(t, theta))) * (2.0 / nt) * (math.pi / nth) / 4.0


def bst_backproject(g: np.ndarray, n_out: int, beta: float = 0.0, zero_pad: float = 2.0,
                    dc_mode: str = "subtract_mean") -> np.ndarray:
    """bst.py:183-203: radial spectra, DC handling, 1/sigma kernel, gridding and
    inverse transform, BST_SCALE, exact mean restoration in subtract_mean mode."""
    bst_validate(n_out, beta, zero_pad, dc_mode)
    g = np.asarray(g, dtype=np.float64)
    H, dsigma = bst_radial_spectra(g, n_out, zero_pad, beta)
    if dc_mode == "subtract_mean":
        H = H.copy()
        H[0, :] = 0.0
    kern = np.empty(H.shape[0])
    kern[0] = 1.0 / dsigma
    kern[1:] = 1.0 / (np.arange(1, H.shape[0]) * dsigma)
    img = BST_SCALE * bst_spectrum_to_image(H * kern[:, None], dsigma, n_out)
    if dc_mode == "subtract_mean":
        img = img + (mean_backprojection(g) - float(img.mean()))
    return img


def fbp_bst(g: np.ndarray, n: int, lam: float = 0.0, cutoff: float = 1.0, beta: float = 0.0,
            zero_pad: float = 2.0, dc_mode: str = "subtract_mean") -> np.ndarray:
    """fbp(g, FilterSpec(lam, cutoff), engine='bst', n) (filtering.py:73-98)."""
    return FBP_SCALE * bst_backproject(ramp_filter(g, lam, cutoff), n, beta, zero_pad, dc_mode)
