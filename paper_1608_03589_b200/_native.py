"""ctypes binding of liblpbp.so (include/lpbp.h).

The library is built in-tree by __graft_entry__.build() / `make`.  There is no
fallback: if the shared object is missing or fails to load, every entry point
raises ImportError / RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_char_p, c_double, c_int32, c_int64, c_size_t, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblpbp.so")

LPBP_OK = 0
LPBP_EINVAL = 1
LPBP_ECUDA = 2
LPBP_EUNSUPPORTED = 3
LPBP_ENOMEM = 4


class Params(ctypes.Structure):
    _fields_ = [
        ("nt", c_int32),
        ("ntheta", c_int32),
        ("n_out", c_int32),
        ("has_rho0", c_int32),
        ("rho0", c_double),
        ("nrho", c_int32),
        ("filter", c_int32),
        ("lam", c_double),
        ("cutoff", c_double),
        ("device", c_int32),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("nt", c_int32), ("ntheta", c_int32), ("n_out", c_int32), ("ns", c_int32), ("nphi", c_int32),
        ("nrho", c_int32), ("L", c_int32), ("M", c_int32), ("kernel_nnz", c_int32), ("kmax", c_int32),
        ("filter", c_int32), ("device", c_int32),
        ("rho0", c_double), ("drho", c_double), ("dphi", c_double), ("out_scale", c_double),
        ("table_bytes", c_size_t), ("workspace_per_slice", c_size_t), ("readout_sector_bytes", c_size_t),
        ("band_rows", c_int32), ("row_min", c_int32), ("nbands", c_int32), ("generic", c_int32), ("MB", c_int32),
        ("phi_q", c_int32), ("p_rows", c_int32),
    ]


class Sector(ctypes.Structure):
    _fields_ = [("theta0", c_double), ("beta", c_double), ("a_r", c_double)]


class SectorInfo(ctypes.Structure):
    _fields_ = [
        ("jc", c_int32), ("nrho", c_int32), ("L", c_int32), ("nphi", c_int32),
        ("theta_c", c_double), ("rho0", c_double), ("drho", c_double), ("support_min", c_double),
        ("a_r", c_double), ("table_bytes", c_size_t),
    ]


class BstParams(ctypes.Structure):
    _fields_ = [
        ("nt", c_int32), ("ntheta", c_int32), ("n_out", c_int32),
        ("beta", c_double), ("zero_pad", c_double), ("dc_mode", c_int32), ("filter", c_int32),
        ("lam", c_double), ("cutoff", c_double), ("device", c_int32),
    ]


class BstInfo(ctypes.Structure):
    _fields_ = [
        ("ns", c_int32), ("nray", c_int32), ("L", c_int32), ("m_need", c_int32), ("m_pad", c_int32),
        ("big", c_int32), ("p0", c_int32), ("supported", c_int32),
        ("ds", c_double), ("dsigma", c_double), ("out_scale", c_double),
        ("table_bytes", c_size_t), ("workspace_per_slice", c_size_t),
    ]


# symbol -> (restype, argtypes); exactly the functions declared in include/lpbp.h
SIGNATURES = {
    "lpbp_plan_create": (c_int32, [POINTER(Params), POINTER(c_void_p)]),
    "lpbp_plan_destroy": (None, [c_void_p]),
    "lpbp_plan_get_info": (c_int32, [c_void_p, POINTER(PlanInfo)]),
    "lpbp_workspace_bytes": (c_int32, [c_void_p, c_int32, POINTER(c_size_t)]),
    "lpbp_execute": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_size_t, c_void_p]),
    "lpbp_execute_host": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32]),
    "lpbp_filter": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p]),
    "lpbp_logpolar": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_size_t, c_void_p]),
    "lpbp_readout": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p]),
    "lpbp_naive_workspace_bytes": (c_int32, [c_int32, c_int32, c_int32, POINTER(c_size_t)]),
    "lpbp_naive_backproject": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p]),
    "lpbp_plan_table": (c_int32, [c_void_p, c_char_p, c_void_p, c_size_t, POINTER(c_size_t)]),
    "lpbp_profile_enable": (c_int32, [c_void_p, c_int32]),
    "lpbp_bst_profile_enable": (c_int32, [c_void_p, c_int32]),
    "lpbp_bst_profile_read": (c_int32, [c_void_p, POINTER(ctypes.c_double), POINTER(c_int64), POINTER(c_int64),
                                        c_int32]),
    "lpbp_profile_read": (c_int32, [c_void_p, POINTER(ctypes.c_double), POINTER(c_int64), POINTER(c_int64), c_int32]),
    "lpbp_radon_ellipses": (c_int32, [c_void_p, c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p]),
    "lpbp_radon_ellipses_f64": (c_int32, [c_void_p, c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p]),
    "lpbp_radon_ellipses_host": (c_int32, [c_void_p, c_int32, c_int32, c_int32, c_int32, c_void_p, c_int32]),
    "lpbp_sector_plan_create": (c_int32, [c_int32, c_int32, c_int32, POINTER(Sector), c_int32, c_int32,
                                          POINTER(c_void_p)]),
    "lpbp_sector_plan_destroy": (None, [c_void_p]),
    "lpbp_sector_get_info": (c_int32, [c_void_p, c_int32, POINTER(SectorInfo)]),
    "lpbp_sector_workspace_bytes": (c_int32, [c_void_p, c_int32, POINTER(c_size_t)]),
    "lpbp_sector_execute": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_size_t, c_void_p]),
    "lpbp_sector_execute_host": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32]),
    "lpbp_sector_prepare": (c_int32, [c_void_p, c_int32, c_void_p, c_void_p, c_int32, c_void_p]),
    "lpbp_sector_logpolar": (c_int32, [c_void_p, c_int32, c_void_p, c_void_p, c_int32, c_void_p]),
    "lpbp_bst_plan_create": (c_int32, [POINTER(BstParams), POINTER(c_void_p)]),
    "lpbp_bst_plan_destroy": (None, [c_void_p]),
    "lpbp_bst_get_info": (c_int32, [c_void_p, POINTER(BstInfo)]),
    "lpbp_bst_workspace_bytes": (c_int32, [c_void_p, c_int32, POINTER(c_size_t)]),
    "lpbp_bst_execute": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_size_t, c_void_p]),
    "lpbp_bst_execute_host": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32]),
    "lpbp_bst_radial": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p]),
    "lpbp_sinogram_to_semipolar": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_int32, c_int32, c_void_p]),
    "lpbp_semipolar_to_logpolar": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_double, c_int32, c_int32,
                                             c_void_p]),
    "lpbp_logpolar_to_cartesian": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_double, c_int32, c_int32,
                                             c_int32, c_void_p]),
    "lpbp_logpolar_kernel": (c_int32, [c_int32, c_int32, c_double, c_void_p]),
    "lpbp_polar_to_cartesian_frequency": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_int64, c_int64, c_int64,
                                                    c_double, c_int32, c_int32, c_double, ctypes.c_float, c_int32,
                                                    c_void_p]),
    "lpbp_mean_backprojection": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_int32, c_void_p]),
    "lpbp_kaiser_window": (c_int32, [c_int32, c_double, c_void_p]),
    "lpbp_last_launch_count": (c_int64, []),
    "lpbp_last_error": (c_char_p, []),
    "lpbp_version": (c_int32, []),
}

_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Load liblpbp.so (once).  Raises ImportError if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build() "
                    "(there is no CPU fallback)"
                )
            handle = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


class LpbpError(RuntimeError):
    pass


def check(rc: int) -> None:
    """Map an LPBP_* status to the reference's exception types."""
    if rc == LPBP_OK:
        return
    msg = lib().lpbp_last_error().decode()
    if rc == LPBP_EINVAL:
        raise ValueError(msg)
    if rc == LPBP_EUNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == LPBP_ENOMEM:
        raise MemoryError(msg)
    raise LpbpError(msg)
