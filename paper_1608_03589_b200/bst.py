"""BST engine — drop-in for fastbp.bst (bst.py:1-206): the reference's
frequency-domain backprojection and fbp's default engine.

bst_backproject(g, BstOptions) keeps the reference signature and options
(beta, zero_pad, dc_mode, n_out) and runs on liblpbp.so (lpbp_bst_*): a radial
kernel (semi-polar unfolding with the Kaiser window, zero-padded real DFTs along
s, 1/sigma kernel), a gridding kernel (bilinear polar -> Cartesian frequency
interpolation with Hermitian averaging, phase ramps, inverse DFT along x on the
2x padded lattice) and a column kernel (inverse DFT along y as a real
transform, crop, scale, exact mean restoration).
"""

from __future__ import annotations

import math
import threading
from collections import OrderedDict
import ctypes
from ctypes import byref, c_size_t, c_void_p
from dataclasses import dataclass

import numpy as np
import torch

from ._native import BstInfo, BstParams, check, lib
from .grids import CartesianImage, Sinogram
from .plan import _as_f32_contig, _check_out_device, _check_out_host, _require_cuda, _stream

__all__ = ["BST_SCALE", "BstOptions", "BstPlan", "bst_backproject", "bst_backproject_batch", "bst_spectrum",
           "get_bst_plan", "kaiser_window", "mean_backprojection", "sigma_kernel"]

BST_SCALE = 4.0 * math.pi  # bst.py:47


@dataclass(frozen=True)
class BstOptions:
    """Engine knobs (bst.py:61-87): beta (Kaiser shape, 0 = none), zero_pad >= 1,
    dc_mode 'subtract_mean' | 'kernel_cap', n_out."""

    n_out: int
    beta: float = 0.0
    zero_pad: float = 2.0
    dc_mode: str = "subtract_mean"

    def __post_init__(self):
        if self.n_out < 2:
            raise ValueError("n_out must be >= 2")
        if self.beta < 0:
            raise ValueError("beta must be >= 0")
        if self.zero_pad < 1:
            raise ValueError("zero_pad must be >= 1")
        if self.dc_mode not in ("subtract_mean", "kernel_cap"):
            raise ValueError("dc_mode must be 'subtract_mean' or 'kernel_cap'")


class BstPlan:
    """Tables of one BST geometry on one device; filter_spec (lam, cutoff) makes it fbp."""

    def __init__(self, nt: int, ntheta: int, opts: BstOptions, filter_spec: tuple[float, float] | None = None,
                 device: int | None = None):
        _require_cuda()
        dev = torch.cuda.current_device() if device is None else int(device)
        p = BstParams()
        p.nt, p.ntheta, p.n_out = int(nt), int(ntheta), int(opts.n_out)
        p.beta, p.zero_pad = float(opts.beta), float(opts.zero_pad)
        p.dc_mode = 0 if opts.dc_mode == "subtract_mean" else 1
        p.filter = 0 if filter_spec is None else 1
        p.lam, p.cutoff = (0.0, 1.0) if filter_spec is None else (float(filter_spec[0]), float(filter_spec[1]))
        p.device = dev
        h = c_void_p()
        torch.cuda.init()
        check(lib().lpbp_bst_plan_create(byref(p), byref(h)))
        self._h = h
        self.device = torch.device("cuda", dev)
        self.nt, self.ntheta, self.n_out = int(nt), int(ntheta), int(opts.n_out)
        inf = BstInfo()
        check(lib().lpbp_bst_get_info(self._h, byref(inf)))
        self.info = {f: getattr(inf, f) for f, _ in BstInfo._fields_}
        self.last_launches = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().lpbp_bst_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def workspace_bytes(self, chunk: int) -> int:
        v = c_size_t()
        check(lib().lpbp_bst_workspace_bytes(self._h, int(chunk), byref(v)))
        return v.value

    STAGES = ("ramp_filter", "bst_radial", "bst_grid_x", "bst_grid_y")

    def profile(self, enable: bool) -> None:
        """Record CUDA events around every stage launch (on the launching stream)."""
        check(lib().lpbp_bst_profile_enable(self._h, 1 if enable else 0))

    def profile_read(self) -> dict:
        """{stage: {"ms", "launches", "slices"}} summed since the last read (waits for the events)."""
        n = len(self.STAGES)
        ms = (ctypes.c_double * n)()
        launches = (ctypes.c_int64 * n)()
        slices = (ctypes.c_int64 * n)()
        check(lib().lpbp_bst_profile_read(self._h, ms, launches, slices, n))
        return {name: {"ms": ms[i], "launches": launches[i], "slices": slices[i]}
                for i, name in enumerate(self.STAGES) if launches[i]}

    def _check_sino(self, sino: torch.Tensor) -> torch.Tensor:
        _require_cuda(sino)
        sino = _as_f32_contig(sino, 3, "sinogram batch")
        if sino.data_ptr() % 16:
            sino = sino.clone()
        if tuple(sino.shape[1:]) != (self.nt, self.ntheta):
            raise ValueError(f"sinogram batch must have shape (B, {self.nt}, {self.ntheta}), got {tuple(sino.shape)}")
        if sino.device != self.device:
            raise ValueError(f"tensor on {sino.device}, plan on {self.device}")
        return sino

    def execute(self, sino: torch.Tensor, out: torch.Tensor | None = None, chunk: int | None = None) -> torch.Tensor:
        """[B, nt, ntheta] float32 CUDA -> [B, n_out, n_out] on the current stream."""
        sino = self._check_sino(sino)
        b = sino.shape[0]
        if out is None:
            out = torch.empty((b, self.n_out, self.n_out), dtype=torch.float32, device=self.device)
        else:
            _check_out_device(out, (b, self.n_out, self.n_out), self.device)
        c = max(1, min(b, chunk or 4))
        nbytes = self.workspace_bytes(c)
        ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            check(lib().lpbp_bst_execute(self._h, c_void_p(sino.data_ptr()), c_void_p(out.data_ptr()), b,
                                         c_void_p(ws.data_ptr()), nbytes, _stream(self.device)))
        self.last_launches = int(lib().lpbp_last_launch_count())
        return out

    def execute_host(self, sino: np.ndarray, out: np.ndarray | None = None, chunk: int = 4) -> np.ndarray:
        sino = np.ascontiguousarray(sino, dtype=np.float32)
        if sino.ndim != 3 or sino.shape[1:] != (self.nt, self.ntheta):
            raise ValueError(f"sinogram batch must have shape (B, {self.nt}, {self.ntheta})")
        b = sino.shape[0]
        if out is None:
            out = np.empty((b, self.n_out, self.n_out), dtype=np.float32)
        dst = _check_out_host(out, (b, self.n_out, self.n_out))
        check(lib().lpbp_bst_execute_host(self._h, c_void_p(sino.ctypes.data), c_void_p(dst), b,
                                          int(chunk)))
        self.last_launches = int(lib().lpbp_last_launch_count())
        return out

    def radial(self, sino: torch.Tensor) -> torch.Tensor:
        """Stage: [B, nray, m_need] complex64 = 0.5 x spectra * sigma_kernel (reference units)."""
        sino = self._check_sino(sino)
        b = sino.shape[0]
        nray, m_pad, m_need = self.info["nray"], self.info["m_pad"], self.info["m_need"]
        # ray pairs [b][ntheta + 2][m_pad][2]: pair c = (ray c, ray c + ntheta); pair row ntheta
        # repeats pair 0 swapped and row ntheta + 1 is zero (the gridding's unguarded taps)
        raw = torch.empty((b, nray // 2 + 2, m_pad, 2), dtype=torch.complex64, device=self.device)
        with torch.cuda.device(self.device):
            check(lib().lpbp_bst_radial(self._h, c_void_p(sino.data_ptr()), c_void_p(raw.data_ptr()), b,
                                        _stream(self.device)))
        out = raw[:, :nray // 2].permute(0, 3, 1, 2).reshape(b, nray, m_pad)  # rays c then c + ntheta
        return out[:, :, :m_need]


_cache: "OrderedDict[tuple, BstPlan]" = OrderedDict()
_cache_lock = threading.Lock()


def get_bst_plan(nt: int, ntheta: int, opts: BstOptions, filter_spec=None, device: int | None = None) -> BstPlan:
    dev = torch.cuda.current_device() if device is None else int(device)
    key = (nt, ntheta, opts, filter_spec, dev)
    with _cache_lock:
        p = _cache.get(key)
        if p is not None:
            _cache.move_to_end(key)
            return p
    p = BstPlan(nt, ntheta, opts, filter_spec, device=dev)
    with _cache_lock:
        _cache[key] = p
        while len(_cache) > 4:
            _cache.popitem(last=False)
    return p


def bst_backproject(g: Sinogram, opts: BstOptions) -> CartesianImage:
    """Backproject through the frequency-domain pipeline (bst.py:183-203)."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1608_03589_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    plan = get_bst_plan(g.nt, g.ntheta, opts)
    sino = torch.from_numpy(np.ascontiguousarray(g.values, dtype=np.float32)).cuda().unsqueeze(0)
    img = plan.execute(sino)
    return CartesianImage(opts.n_out, opts.n_out, img[0].double().cpu().numpy())


def bst_backproject_batch(sino: torch.Tensor, opts: BstOptions, filter_spec=None,
                          out: torch.Tensor | None = None) -> torch.Tensor:
    """Batched device entry point: [B, nt, ntheta] float32 CUDA -> [B, n_out, n_out]."""
    plan = get_bst_plan(sino.shape[1], sino.shape[2], opts, filter_spec, device=sino.device.index)
    return plan.execute(sino, out=out)


def kaiser_window(ns: int, beta: float) -> np.ndarray:
    """Kaiser-Bessel taper I0(beta sqrt(1 - u^2)) / I0(beta), u = (2i - ns + 1)/(ns - 1) (bst.py:90-102)."""
    if ns < 2:
        raise ValueError("ns must be >= 2")
    out = np.empty(int(ns), dtype=np.float64)
    check(lib().lpbp_kaiser_window(int(ns), float(beta), c_void_p(out.ctypes.data)))
    return out


def sigma_kernel(nsigma: int, dsigma: float) -> np.ndarray:
    """Radial weights 1/sigma_m, the DC bin capped at 1/dsigma (bst.py:105-117)."""
    if not dsigma > 0:
        raise ValueError("dsigma must be positive")
    out = np.empty(nsigma)
    out[0] = 1.0 / dsigma
    out[1:] = 1.0 / (np.arange(1, nsigma) * dsigma)
    return out


def mean_backprojection(g: Sinogram) -> float:
    """Spatial mean over [-1, 1]^2 of the backprojection of g through <B g, 1> = <g, chord>
    (bst.py:173-180), reduced on the device in fp64."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1608_03589_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    src = torch.from_numpy(np.ascontiguousarray(g.values, dtype=np.float32)).cuda()
    out = torch.empty(1, dtype=torch.float64, device=src.device)
    check(lib().lpbp_mean_backprojection(c_void_p(src.data_ptr()), c_void_p(out.data_ptr()), g.nt, g.ntheta, 1,
                                         _stream(src.device)))
    return float(out.item())


def bst_spectrum(g: Sinogram, opts: BstOptions):
    """The engine's native product on the omega = pi k lattice of an n_out image:
    BST_SCALE * polar_to_cartesian_frequency(spectra * sigma_kernel) (bst.py:206-226)."""
    from .resample import FrequencyImage
    plan = get_bst_plan(g.nt, g.ntheta, opts)
    sino = torch.from_numpy(np.ascontiguousarray(g.values, dtype=np.float32)).cuda().unsqueeze(0)
    radial = plan.radial(sino)  # [1, nray, m_need] = 0.5 x spectra * kernel (view with pitch m_pad)
    n, m_need, nray, m_pad = opts.n_out, plan.info["m_need"], plan.info["nray"], plan.info["m_pad"]
    out = torch.empty((n, n), dtype=torch.complex64, device=sino.device)
    check(lib().lpbp_polar_to_cartesian_frequency(c_void_p(radial.data_ptr()), c_void_p(out.data_ptr()), m_need, nray,
                                                  1, m_pad, nray * m_pad, float(plan.info["dsigma"]), n, n, math.pi,
                                                  float(2.0 * BST_SCALE), 1, _stream(sino.device)))
    return FrequencyImage(n, n, out.cpu().numpy().astype(np.complex128))