"""Device-level plans: batched log-polar backprojection / FBP on torch CUDA tensors.

A LogPolarPlan owns the constant device tables of one geometry (kernel spectrum,
resampling taps, filter response, readout table) built natively in fp64 by
liblpbp.so (lpbp_plan_create).  Execution calls go straight through the C ABI on
the caller's current torch stream; torch is used only to allocate device memory
and to name the stream.
"""

from __future__ import annotations

import ctypes
import threading
from collections import OrderedDict
from ctypes import byref, c_size_t, c_void_p

import numpy as np
import torch

from . import _native
from ._native import PlanInfo, Params, check, lib


def _require_cuda(t: torch.Tensor | None = None) -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1608_03589_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    if t is not None and not t.is_cuda:
        raise ValueError("expected a CUDA tensor")


def _as_f32_contig(t: torch.Tensor, ndim: int, name: str) -> torch.Tensor:
    if t.dim() != ndim:
        raise ValueError(f"{name} must have {ndim} dimensions, got shape {tuple(t.shape)}")
    if t.dtype != torch.float32:
        raise ValueError(f"{name} must be float32, got {t.dtype}")
    return t.contiguous()


def _check_out_device(out: torch.Tensor, shape: tuple, device: torch.device) -> torch.Tensor:
    """Caller-supplied device output: the kernels write prod(shape) floats through a raw
    pointer, so anything but an exact float32, C-contiguous tensor of that shape on the
    plan's device is refused before the pointer crosses the ABI."""
    if not isinstance(out, torch.Tensor):
        raise ValueError("out must be a torch.Tensor")
    if tuple(out.shape) != tuple(shape) or out.dtype != torch.float32 or not out.is_contiguous():
        raise ValueError(f"out must be a C-contiguous float32 tensor of shape {tuple(shape)}, "
                         f"got {out.dtype} {tuple(out.shape)}")
    if out.device != device:
        raise ValueError(f"out on {out.device}, plan on {device}")
    return out


def _check_out_host(out, shape: tuple):
    """Caller-supplied host output (numpy array or CPU tensor) for the *_host entry points."""
    if isinstance(out, torch.Tensor):
        if out.is_cuda or out.dtype != torch.float32 or not out.is_contiguous() or tuple(out.shape) != tuple(shape):
            raise ValueError(f"out must be a contiguous float32 CPU tensor of shape {tuple(shape)}")
        return out.data_ptr()
    if not (isinstance(out, np.ndarray) and out.flags.c_contiguous and out.flags.writeable
            and out.dtype == np.float32 and out.shape == tuple(shape)):
        raise ValueError(f"out must be a C-contiguous writeable float32 array of shape {tuple(shape)}")
    return out.ctypes.data


def _check_workspace(ws: torch.Tensor, need: int, device: torch.device) -> int:
    if not isinstance(ws, torch.Tensor) or not ws.is_contiguous() or ws.device != device:
        raise ValueError(f"workspace must be a contiguous tensor on {device}")
    nbytes = ws.numel() * ws.element_size()
    if nbytes < need:
        raise ValueError(f"workspace holds {nbytes} bytes, the plan needs {need}")
    return nbytes


def _stream(device: torch.device) -> c_void_p:
    return c_void_p(torch.cuda.current_stream(device).cuda_stream)


class LogPolarPlan:
    """Geometry + constant tables for `nt x ntheta` sinograms -> `n_out^2` images.

    filter_spec: None for logpolar_backproject, or (lam, cutoff) for fbp
    (filter_sinogram + backprojection + 1/(2 pi)).
    """

    def __init__(self, nt: int, ntheta: int, n_out: int, rho0: float | None = None, nrho: int | None = None,
                 filter_spec: tuple[float, float] | None = None, device: int | None = None):
        _require_cuda()
        dev = torch.cuda.current_device() if device is None else int(device)
        p = Params()
        p.nt, p.ntheta, p.n_out = int(nt), int(ntheta), int(n_out)
        p.has_rho0 = 0 if rho0 is None else 1
        p.rho0 = 0.0 if rho0 is None else float(rho0)
        p.nrho = 0 if nrho is None else int(nrho)
        p.filter = 0 if filter_spec is None else 1
        p.lam, p.cutoff = (0.0, 1.0) if filter_spec is None else (float(filter_spec[0]), float(filter_spec[1]))
        p.device = dev
        handle = c_void_p()
        torch.cuda.init()
        check(lib().lpbp_plan_create(byref(p), byref(handle)))
        self._h = handle
        self.device = torch.device("cuda", dev)
        info = PlanInfo()
        check(lib().lpbp_plan_get_info(self._h, byref(info)))
        self.info = {f: getattr(info, f) for f, _ in PlanInfo._fields_}
        self.nt, self.ntheta, self.n_out = nt, ntheta, n_out
        self.nrho, self.nphi, self.rho0 = info.nrho, info.nphi, info.rho0
        self.filtered = filter_spec is not None
        self.last_launches = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().lpbp_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    # ------------------------------------------------------------------
    def workspace_bytes(self, chunk: int) -> int:
        v = c_size_t()
        check(lib().lpbp_workspace_bytes(self._h, int(chunk), byref(v)))
        return v.value

    def _check_sino(self, sino: torch.Tensor) -> torch.Tensor:
        _require_cuda(sino)
        sino = _as_f32_contig(sino, 3, "sinogram batch")
        if sino.data_ptr() % 16:  # the kernels stream rows with 16-byte TMA bulk copies
            sino = sino.clone()
        if tuple(sino.shape[1:]) != (self.nt, self.ntheta):
            raise ValueError(f"sinogram batch must have shape (B, {self.nt}, {self.ntheta}), got {tuple(sino.shape)}")
        if sino.device != self.device:
            raise ValueError(f"tensor on {sino.device}, plan on {self.device}")
        return sino

    def _workspace(self, batch: int, chunk: int | None) -> tuple[torch.Tensor, int]:
        c = max(1, min(batch, chunk or 8))
        nbytes = self.workspace_bytes(c)
        return torch.empty(nbytes, dtype=torch.uint8, device=self.device), nbytes

    def execute(self, sino: torch.Tensor, out: torch.Tensor | None = None, chunk: int | None = None,
                workspace: torch.Tensor | None = None) -> torch.Tensor:
        """[B, nt, ntheta] float32 -> [B, n_out, n_out] float32 on the current stream."""
        sino = self._check_sino(sino)
        b = sino.shape[0]
        if out is None:
            out = torch.empty((b, self.n_out, self.n_out), dtype=torch.float32, device=self.device)
        else:
            _check_out_device(out, (b, self.n_out, self.n_out), self.device)
        if workspace is None:
            workspace, nbytes = self._workspace(b, chunk)
        else:
            nbytes = _check_workspace(workspace, self.workspace_bytes(1), self.device)
        with torch.cuda.device(self.device):
            check(lib().lpbp_execute(self._h, c_void_p(sino.data_ptr()), c_void_p(out.data_ptr()), b,
                                     c_void_p(workspace.data_ptr()), nbytes, _stream(self.device)))
        self.last_launches = int(lib().lpbp_last_launch_count())
        return out

    def logpolar(self, sino: torch.Tensor, chunk: int | None = None) -> torch.Tensor:
        """Convolved log-polar image [B, nrho, nphi] (no filter, no readout)."""
        sino = self._check_sino(sino)
        b = sino.shape[0]
        out = torch.empty((b, self.nrho, self.nphi), dtype=torch.float32, device=self.device)
        ws, nbytes = self._workspace(b, chunk)
        with torch.cuda.device(self.device):
            check(lib().lpbp_logpolar(self._h, c_void_p(sino.data_ptr()), c_void_p(out.data_ptr()), b,
                                      c_void_p(ws.data_ptr()), nbytes, _stream(self.device)))
        return out

    def filter(self, sino: torch.Tensor) -> torch.Tensor:
        """filter_sinogram on a batch (plan must be an FBP plan)."""
        sino = self._check_sino(sino)
        out = torch.empty_like(sino)
        with torch.cuda.device(self.device):
            check(lib().lpbp_filter(self._h, c_void_p(sino.data_ptr()), c_void_p(out.data_ptr()), sino.shape[0],
                                    _stream(self.device)))
        return out

    def readout(self, lp: torch.Tensor) -> torch.Tensor:
        """logpolar_to_cartesian (times the plan's output scale) on a batch."""
        _require_cuda(lp)
        lp = _as_f32_contig(lp, 3, "log-polar batch")
        if tuple(lp.shape[1:]) != (self.nrho, self.nphi):
            raise ValueError(f"log-polar batch must have shape (B, {self.nrho}, {self.nphi})")
        out = torch.empty((lp.shape[0], self.n_out, self.n_out), dtype=torch.float32, device=self.device)
        with torch.cuda.device(self.device):
            check(lib().lpbp_readout(self._h, c_void_p(lp.data_ptr()), c_void_p(out.data_ptr()), lp.shape[0],
                                     _stream(self.device)))
        return out

    def execute_host(self, sino: np.ndarray | torch.Tensor, out: np.ndarray | torch.Tensor | None = None,
                     chunk: int = 4):
        """Host -> host: chunked H2D / compute / D2H overlapped inside liblpbp.
        Accepts numpy arrays or (preferably pinned) CPU torch tensors; blocks."""
        is_torch = isinstance(sino, torch.Tensor)
        if is_torch:
            if sino.is_cuda or sino.dtype != torch.float32 or not sino.is_contiguous():
                raise ValueError("execute_host expects a contiguous float32 CPU tensor")
            b = sino.shape[0]
            src_ptr = sino.data_ptr()
            if out is None:
                out = torch.empty((b, self.n_out, self.n_out), dtype=torch.float32, pin_memory=sino.is_pinned())
        else:
            sino = np.ascontiguousarray(sino, dtype=np.float32)
            b = sino.shape[0]
            src_ptr = sino.ctypes.data
            if out is None:
                out = np.empty((b, self.n_out, self.n_out), dtype=np.float32)
        if sino.dim() != 3 if is_torch else sino.ndim != 3:
            raise ValueError(f"sinogram batch must have shape (B, {self.nt}, {self.ntheta})")
        dst_ptr = _check_out_host(out, (b, self.n_out, self.n_out))
        if tuple(sino.shape[1:]) != (self.nt, self.ntheta):
            raise ValueError(f"sinogram batch must have shape (B, {self.nt}, {self.ntheta})")
        check(lib().lpbp_execute_host(self._h, c_void_p(src_ptr), c_void_p(dst_ptr), b, int(chunk)))
        self.last_launches = int(lib().lpbp_last_launch_count())
        return out

    STAGES = ("ramp_filter", "row_rdft", "rho_conv", "row_irdft", "readout", "irdft_readout")

    def profile(self, enable: bool) -> None:
        """Record CUDA events around every stage launch (on the launching stream)."""
        check(lib().lpbp_profile_enable(self._h, 1 if enable else 0))

    def profile_read(self) -> dict:
        """{stage: {"ms", "launches", "slices"}} summed since the last read (waits for the events)."""
        n = len(self.STAGES)
        ms = (ctypes.c_double * n)()
        launches = (ctypes.c_int64 * n)()
        slices = (ctypes.c_int64 * n)()
        check(lib().lpbp_profile_read(self._h, ms, launches, slices, n))
        return {name: {"ms": ms[i], "launches": launches[i], "slices": slices[i]}
                for i, name in enumerate(self.STAGES) if launches[i]}

    def table(self, which: str) -> np.ndarray:
        n = c_size_t()
        check(lib().lpbp_plan_table(self._h, which.encode(), None, 0, byref(n)))
        if which == "kernel_cells":
            a = np.empty((n.value, 2), dtype=np.int32)
        elif which == "ramp":
            a = np.empty(n.value, dtype=np.float32)
        elif which == "khat":
            a = np.empty(n.value, dtype=np.complex64)
        elif which in ("row_need", "ploc", "band_need"):
            a = np.empty(n.value, dtype=np.uint32)
        else:
            raise ValueError(which)
        check(lib().lpbp_plan_table(self._h, which.encode(), c_void_p(a.ctypes.data), n.value, byref(n)))
        return a


def naive_backproject(sino: torch.Tensor, n: int) -> torch.Tensor:
    """Direct pixel-driven backprojection of a batch [B, nt, ntheta] -> [B, n, n]."""
    _require_cuda(sino)
    sino = _as_f32_contig(sino, 3, "sinogram batch")
    b, nt, ntheta = sino.shape
    out = torch.empty((b, n, n), dtype=torch.float32, device=sino.device)
    nbytes = c_size_t()
    check(lib().lpbp_naive_workspace_bytes(nt, ntheta, b, byref(nbytes)))
    ws = torch.empty(max(1, nbytes.value // 4), dtype=torch.float32, device=sino.device)
    with torch.cuda.device(sino.device):
        check(lib().lpbp_naive_backproject(c_void_p(sino.data_ptr()), c_void_p(out.data_ptr()), nt, ntheta, int(n), b,
                                           c_void_p(ws.data_ptr()), _stream(sino.device)))
    return out


_cache: "OrderedDict[tuple, LogPolarPlan]" = OrderedDict()
_cache_lock = threading.Lock()
_CACHE_SIZE = 4


def get_plan(nt: int, ntheta: int, n_out: int, rho0: float | None, nrho: int | None,
             filter_spec: tuple[float, float] | None, device: int | None = None) -> LogPolarPlan:
    """Plans are immutable; cache the most recent few per geometry."""
    dev = torch.cuda.current_device() if device is None else int(device)
    key = (nt, ntheta, n_out, rho0, nrho, filter_spec, dev)
    with _cache_lock:
        plan = _cache.get(key)
        if plan is not None:
            _cache.move_to_end(key)
            return plan
    plan = LogPolarPlan(nt, ntheta, n_out, rho0=rho0, nrho=nrho, filter_spec=filter_spec, device=dev)
    with _cache_lock:
        _cache[key] = plan
        while len(_cache) > _CACHE_SIZE:
            _cache.popitem(last=False)
    return plan
