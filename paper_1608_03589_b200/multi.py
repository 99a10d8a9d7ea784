"""Multi-GPU volume reconstruction by slice sharding.

Slices are independent, so a volume [S, nt, ntheta] is split into contiguous
slice-index blocks, one per device; each device has its own plan (constant
tables) and runs its block host -> host through liblpbp's chunked pipeline
(H2D / compute / D2H overlapped on the device's own streams).  One host thread
per device drives it (ctypes releases the GIL for the duration of the C call).
There is no collective: results land directly in the caller's output array.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from .plan import LogPolarPlan


def shard_bounds(total: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous, balanced [lo, hi) slice ranges (same rule as bench.shard)."""
    return [(total * r // parts, total * (r + 1) // parts) for r in range(parts)]


class VolumeReconstructor:
    """Log-polar BP / FBP of whole volumes over several GPUs of one node.

    filter_spec: None for backprojection, (lam, cutoff) for FBP.
    devices: CUDA ordinals (default: all visible).  A device may appear more than
    once (several plans/streams on one GPU).
    """

    def __init__(self, nt: int, ntheta: int, n_out: int, filter_spec=None, rho0=None, nrho=None,
                 devices: list[int] | None = None, chunk: int = 8):
        if not torch.cuda.is_available():
            raise RuntimeError("VolumeReconstructor needs CUDA devices; there is no CPU fallback")
        self.devices = list(range(torch.cuda.device_count())) if devices is None else list(devices)
        if not self.devices:
            raise ValueError("no devices")
        self.nt, self.ntheta, self.n_out, self.chunk = nt, ntheta, n_out, chunk
        self.plans = [LogPolarPlan(nt, ntheta, n_out, rho0=rho0, nrho=nrho, filter_spec=filter_spec, device=d)
                      for d in self.devices]

    def run(self, volume, out=None):
        """volume: [S, nt, ntheta] float32 (numpy or pinned CPU tensor) -> [S, n, n] float32."""
        is_torch = isinstance(volume, torch.Tensor)
        s = volume.shape[0]
        if tuple(volume.shape[1:]) != (self.nt, self.ntheta):
            raise ValueError(f"volume must have shape (S, {self.nt}, {self.ntheta})")
        if out is None:
            out = (torch.empty((s, self.n_out, self.n_out), dtype=torch.float32, pin_memory=volume.is_pinned())
                   if is_torch else np.empty((s, self.n_out, self.n_out), dtype=np.float32))
        if not is_torch:
            volume = np.ascontiguousarray(volume, dtype=np.float32)
        errors: list[BaseException] = []

        def work(plan, lo, hi):
            try:
                if hi > lo:
                    plan.execute_host(volume[lo:hi], out[lo:hi], chunk=self.chunk)
            except BaseException as e:  # surfaced to the caller below
                errors.append(e)

        threads = [threading.Thread(target=work, args=(p, lo, hi))
                   for p, (lo, hi) in zip(self.plans, shard_bounds(s, len(self.plans)))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        return out
