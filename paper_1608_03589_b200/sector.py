"""Sector (partial) log-polar backprojection — drop-in for
fastbp.logpolar.partial_backproject (logpolar.py:210-299).

Every sector (theta0, beta, a_r) covers the ray angles [theta0, theta0 + 2 beta]
mod pi.  Its working-frame sinogram (angles rolled to the sector centre, t-flip
for columns past pi, mask / coverage weights, support shrunk by a_r and shifted
by 1 - a_r) runs through the log-polar stage on the sector's own shallow mesh;
the sector images are read back at the rotated, scaled, shifted pixel positions,
divided by a_r and summed.  All of it runs in liblpbp.so (lpbp_sector_*): one
prep kernel per sector, the backprojection kernels of a per-sector sub-plan, and
one readout kernel that sums the sectors with fp64 coordinates.
"""

from __future__ import annotations

import ctypes
import math
import threading
import warnings
from collections import OrderedDict
from ctypes import byref, c_size_t, c_void_p

import numpy as np
import torch

from ._native import Sector, SectorInfo, check, lib
from .grids import CartesianImage, LogPolarImage, Sinogram
from .plan import _as_f32_contig, _check_out_device, _check_out_host, _require_cuda, _stream

__all__ = ["SectorPlan", "partial_backproject", "partial_backproject_batch", "get_sector_plan"]


class SectorPlan:
    """Constant tables of one (nt, ntheta, n_out, sectors) geometry on one device."""

    def __init__(self, nt: int, ntheta: int, n_out: int, sectors, device: int | None = None):
        _require_cuda()
        dev = torch.cuda.current_device() if device is None else int(device)
        self.sectors = [tuple(float(v) for v in s) for s in sectors]
        arr = (Sector * max(1, len(self.sectors)))()
        for i, (t0, b, a) in enumerate(self.sectors):
            arr[i].theta0, arr[i].beta, arr[i].a_r = t0, b, a
        handle = c_void_p()
        torch.cuda.init()
        check(lib().lpbp_sector_plan_create(int(nt), int(ntheta), int(n_out), arr, len(self.sectors), dev,
                                            byref(handle)))
        self._h = handle
        self.device = torch.device("cuda", dev)
        self.nt, self.ntheta, self.n_out = int(nt), int(ntheta), int(n_out)
        self.info = []
        for i in range(len(self.sectors)):
            inf = SectorInfo()
            check(lib().lpbp_sector_get_info(self._h, i, byref(inf)))
            self.info.append({f: getattr(inf, f) for f, _ in SectorInfo._fields_})
        self.last_launches = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().lpbp_sector_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def workspace_bytes(self, chunk: int) -> int:
        v = c_size_t()
        check(lib().lpbp_sector_workspace_bytes(self._h, int(chunk), byref(v)))
        return v.value

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
        c = max(1, min(b, chunk or 8))
        nbytes = self.workspace_bytes(c)
        ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            check(lib().lpbp_sector_execute(self._h, c_void_p(sino.data_ptr()), c_void_p(out.data_ptr()), b,
                                            c_void_p(ws.data_ptr()), nbytes, _stream(self.device)))
        self.last_launches = int(lib().lpbp_last_launch_count())
        return out

    def execute_host(self, sino: np.ndarray, out: np.ndarray | None = None, chunk: int = 4) -> np.ndarray:
        """Host -> host (numpy float32 [B, nt, ntheta] -> [B, n_out, n_out]); blocks."""
        sino = np.ascontiguousarray(sino, dtype=np.float32)
        if sino.ndim != 3 or sino.shape[1:] != (self.nt, self.ntheta):
            raise ValueError(f"sinogram batch must have shape (B, {self.nt}, {self.ntheta})")
        b = sino.shape[0]
        if out is None:
            out = np.empty((b, self.n_out, self.n_out), dtype=np.float32)
        dst = _check_out_host(out, (b, self.n_out, self.n_out))
        check(lib().lpbp_sector_execute_host(self._h, c_void_p(sino.ctypes.data), c_void_p(dst), b,
                                             int(chunk)))
        self.last_launches = int(lib().lpbp_last_launch_count())
        return out

    def prepare(self, index: int, sino: torch.Tensor) -> torch.Tensor:
        """Working-frame sinogram of sector `index` (rolled, weighted, shrunk, shifted)."""
        sino = self._check_sino(sino)
        out = torch.empty_like(sino)
        with torch.cuda.device(self.device):
            check(lib().lpbp_sector_prepare(self._h, int(index), c_void_p(sino.data_ptr()), c_void_p(out.data_ptr()),
                                            sino.shape[0], _stream(self.device)))
        return out

    def logpolar(self, index: int, work: torch.Tensor) -> torch.Tensor:
        """Convolved log-polar image [B, nrho_s, nphi] of a working-frame sinogram."""
        work = self._check_sino(work)
        inf = self.info[index]
        out = torch.empty((work.shape[0], inf["nrho"], inf["nphi"]), dtype=torch.float32, device=self.device)
        with torch.cuda.device(self.device):
            check(lib().lpbp_sector_logpolar(self._h, int(index), c_void_p(work.data_ptr()), c_void_p(out.data_ptr()),
                                             work.shape[0], _stream(self.device)))
        return out

    def clipped_mass(self, sino: torch.Tensor) -> list[float]:
        """Per sector, the fraction of the shrunk sinogram's mass that the shift pushed
        past the t range (the quantity fastbp's shift_sinogram warns about, radon.py:149-157)."""
        sino = self._check_sino(sino)
        nt, dt = self.nt, 2.0 / self.nt
        t = -1.0 + np.arange(nt) * dt
        dtheta = math.pi / self.ntheta
        ext = 2.0 * dtheta
        theta = np.arange(self.ntheta) * dtheta
        masks = [np.abs(np.mod(theta - (t0 + b) + math.pi / 2, math.pi) - math.pi / 2) <= b + ext + 1e-12
                 for t0, b, _ in self.sectors]
        cover = np.sum(masks, axis=0).astype(np.float64)
        res = []
        for k, (t0, b, a) in enumerate(self.sectors):
            jc = self.info[k]["jc"]
            rot = (np.arange(self.ntheta) + jc) % self.ntheta
            w = np.where(masks[k][rot], 1.0, 0.0) / cover[rot]
            # sum_k a * lerp(rolled, fi1_k) = sum_m coef[m] * rolled[m]
            fi = (t / a + 1.0) / dt
            lo = np.floor(fi).astype(np.int64)
            fr = fi - lo
            coef = np.zeros(nt + 2)
            for idx, wt in ((lo, 1.0 - fr), (lo + 1, fr)):
                ok = (idx >= 0) & (idx < nt)
                np.add.at(coef, idx[ok], a * wt[ok])
            coef = coef[:nt]
            shift = jc % self.ntheta
            src = (np.arange(self.ntheta) + shift)
            flip = src >= self.ntheta
            src = src % self.ntheta
            coef_flip = np.zeros(nt)
            coef_flip[1:] = coef[1:][::-1]  # rolled[m] = g[nt - m] for m >= 1, 0 at m = 0
            g = sino[0].double()
            cn = torch.from_numpy(coef).to(g.device)
            cf = torch.from_numpy(coef_flip).to(g.device)
            col_sums = torch.where(torch.from_numpy(flip).to(g.device), cf @ g, cn @ g)[torch.from_numpy(src).to(g.device)]
            mass_in = float((col_sums * torch.from_numpy(w).to(g.device)).sum())
            mass_out = float(self.prepare(k, sino[:1]).double().sum())
            res.append((mass_in - mass_out) / abs(mass_in) if abs(mass_in) > 0 else 0.0)
        return res


_cache: "OrderedDict[tuple, SectorPlan]" = OrderedDict()
_cache_lock = threading.Lock()


def get_sector_plan(nt: int, ntheta: int, n_out: int, sectors, device: int | None = None) -> SectorPlan:
    dev = torch.cuda.current_device() if device is None else int(device)
    key = (nt, ntheta, n_out, tuple(tuple(float(v) for v in s) for s in sectors), dev)
    with _cache_lock:
        p = _cache.get(key)
        if p is not None:
            _cache.move_to_end(key)
            return p
    p = SectorPlan(nt, ntheta, n_out, sectors, device=dev)
    with _cache_lock:
        _cache[key] = p
        while len(_cache) > 4:
            _cache.popitem(last=False)
    return p


def _validate(sectors, n_out: int) -> None:
    # the reference checks these before touching the sinogram (logpolar.py:218-227)
    if n_out < 2:
        raise ValueError("n_out must be >= 2")
    if not sectors:
        raise ValueError("at least one sector is required")


def partial_backproject(g: Sinogram, sectors: list[tuple[float, float, float]], n_out: int) -> CartesianImage:
    """Sector-wise backprojection (logpolar.py:210-299), same signature and errors;
    emits the reference's RuntimeWarning when a sector's shift clips more than 1e-3
    of its sinogram mass (radon.py:149-157)."""
    _validate(sectors, n_out)
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1608_03589_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    plan = get_sector_plan(g.nt, g.ntheta, n_out, sectors)
    sino = torch.from_numpy(np.ascontiguousarray(g.values, dtype=np.float32)).cuda().unsqueeze(0)
    for frac in plan.clipped_mass(sino):
        if frac > 1e-3:
            warnings.warn(f"shift_sinogram clipped {frac:.2e} of the sinogram mass at the t boundary",
                          RuntimeWarning, stacklevel=2)
    img = plan.execute(sino)
    return CartesianImage(n_out, n_out, img[0].double().cpu().numpy())


def partial_backproject_batch(sino: torch.Tensor, sectors, n_out: int, out: torch.Tensor | None = None,
                              chunk: int | None = None) -> torch.Tensor:
    """Batched device entry point: [B, nt, ntheta] float32 CUDA -> [B, n_out, n_out]."""
    _validate(sectors, n_out)
    plan = get_sector_plan(sino.shape[1], sino.shape[2], n_out, sectors, device=sino.device.index)
    return plan.execute(sino, out=out, chunk=chunk)
