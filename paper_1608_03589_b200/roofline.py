"""Algorithmic (compulsory) HBM bytes of each pipeline kernel: every kernel reads
its input once and writes its output once (fp32 real / complex64 spectra).
DESIGN.md §4 states the per-kernel figures; SURVEY §8(d) gives the
stage-decomposition totals for the whole path (279.258 MB per FBP slice at
2048^2) that the pipeline-level HBM-equivalent figure uses."""

from __future__ import annotations

# SURVEY §8(d) compulsory bytes per slice for the reference's stage decomposition
SURVEY_BYTES_PER_SLICE = {(256, False): 3.014e6, (512, True): 15.252e6, (2048, False): 245.704e6,
                          (2048, True): 279.258e6}


def algorithmic_bytes(plan) -> dict:
    """{stage: {"per_slice": bytes, "per_launch": bytes}} for a LogPolarPlan: this decomposition's own
    compulsory traffic.  `p_rows` plans (K2p): the row-DFT stage writes and the rho stage reads the
    ns = nt/2 semi-polar row spectra instead of nt row spectra."""
    i = plan.info
    nt, nth, n = i["nt"], i["ntheta"], i["n_out"]
    nphi, nrho, L = i["nphi"], i["nrho"], i["L"]
    nh = nphi // 2 + 1
    sino = nt * nth * 4
    G = nh * (i["ns"] if i.get("p_rows") else nt) * 8
    Y = nh * nrho * 8
    lp = nrho * nphi * 4
    img = n * n * 4
    # ahead of the fused inverse DFT + readout K3 writes, and K45 reads, only the rows of the bands some
    # pixel taps (plan table row_need; about two thirds of the rows at 2048^2)
    Yf = Y
    if i.get("band_rows", 0) > 0 and hasattr(plan, "table"):
        try:
            bits = plan.table("row_need")
            Yf = nh * 8 * int(sum(bin(int(w)).count("1") for w in bits))
        except Exception:
            Yf = Y
    return {
        "ramp_filter": {"per_slice": 2 * sino, "per_launch": 0},
        "row_rdft": {"per_slice": sino + G, "per_launch": 0},
        "rho_conv": {"per_slice": G + Yf, "per_launch": nh * L * 8},  # kernel spectrum once per launch
        "row_irdft": {"per_slice": Y + lp, "per_launch": 0},
        "readout": {"per_slice": i["readout_sector_bytes"] + img, "per_launch": 0},
        # fused inverse DFT + readout: spectra in, image out (log-polar rows stay on chip)
        "irdft_readout": {"per_slice": Yf + img, "per_launch": 0},
    }


def survey_stage_bytes(plan) -> dict:
    """SURVEY §8(d)'s per-slice figures, stage by stage, attached to the kernel that does the stage's
    arithmetic (their sum is §8(d)'s per-slice total, 279.258 MB for a 2048^2 FBP slice):
      S1 ramp = 2 nt ntheta 4                     -> ramp_filter
      S2 resample = nt ntheta 4 + nrho nphi 4      -> row_rdft  (the sinogram read; the log-polar image
                                                     S2 writes never exists here: K3 interpolates it on chip)
      S3 FFT convolution = 2 nrho nphi 4 (+ K-hat once per launch) -> rho_conv
      S4 readout = distinct 32-byte sectors + n^2 4 -> irdft_readout
    This is the basis the task's `roofline.achieved` is defined on; `algorithmic_bytes` is what this
    decomposition itself has to move (less for K3, more for K45, which also reads the spectra)."""
    i = plan.info
    nt, nth, n = i["nt"], i["ntheta"], i["n_out"]
    nphi, nrho, L = i["nphi"], i["nrho"], i["L"]
    nh = nphi // 2 + 1
    sino, lp, img = nt * nth * 4, nrho * nphi * 4, n * n * 4
    return {
        "ramp_filter": {"stage": "S1", "per_slice": 2 * sino, "per_launch": 0},
        "row_rdft": {"stage": "S2", "per_slice": sino + lp, "per_launch": 0},
        "rho_conv": {"stage": "S3", "per_slice": 2 * lp, "per_launch": nh * L * 8},
        "irdft_readout": {"stage": "S4", "per_slice": i["readout_sector_bytes"] + img, "per_launch": 0},
    }


def kernel_source_digest() -> str:
    """sha256 over the kernel sources (csrc/*.cu, *.cuh, *.cpp, *.h, sorted by name): ties a
    committed ncu traffic capture to the code it measured."""
    import hashlib
    import os

    d = os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc")
    h = hashlib.sha256()
    for f in sorted(os.listdir(d)):
        if f.endswith((".cu", ".cuh", ".cpp", ".h")):
            h.update(f.encode())
            with open(os.path.join(d, f), "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()


def survey_bytes_per_slice(plan) -> float | None:
    return SURVEY_BYTES_PER_SLICE.get((plan.info["n_out"], bool(plan.info["filter"])))


def fp32_peak_tflops(sm_mhz: float = 1965.0, sms: int = 148) -> float:
    """FP32 CUDA-core peak: SMs x 128 lanes x 2 (FMA) x clock."""
    return sms * 128 * 2 * sm_mhz * 1e6 / 1e12


def nominal_flops(plan) -> dict:
    """Nominal FFT flop counts per slice (5 N log2 N per complex N-point FFT,
    pointwise complex multiply 6 flops) for each stage; the FFT kernels' honest
    bound is the FP32 pipe, reported beside the HBM fraction."""
    import math

    i = plan.info
    nt, nphi, nrho, L, M = i["nt"], i["nphi"], i["nrho"], i["L"], i["M"]
    nh = nphi // 2 + 1
    f = lambda n: 5.0 * n * math.log2(n)  # noqa: E731
    return {
        "ramp_filter": (i["ntheta"] / 2) * (2 * f(M) + 6 * M) if M else 0.0,  # packed column pairs
        "row_rdft": ((i["ns"] if i.get("p_rows") else nt) / 2) * f(nphi),      # packed row pairs
        "rho_conv": nh * (2 * f(L) + 6 * L),
        "irdft_readout": (nrho / 2) * f(nphi),
    }


def bst_algorithmic_bytes(plan) -> dict:
    """{stage: {"per_slice", "per_launch"}} for a BstPlan: each stage reads its input once and
    writes its output once.  Radial: sinogram in, ray-pair spectra P [(nray/2 + 2)][m_pad] float4
    out; grid_x: P in (each bin once), X [n][big/2] complex out; grid_y: X in, image out."""
    i = plan.info
    nt, nth, n = plan.nt, plan.ntheta, plan.n_out
    sino = nt * nth * 4
    P = (i["nray"] // 2 + 2) * i["m_pad"] * 16
    X = n * (i["big"] // 2) * 8
    img = n * n * 4
    return {
        "ramp_filter": {"per_slice": 2 * sino, "per_launch": 0},
        "bst_radial": {"per_slice": sino + P, "per_launch": 0},
        "bst_grid_x": {"per_slice": P + X, "per_launch": 0},
        "bst_grid_y": {"per_slice": X + img, "per_launch": 0},
    }


def bst_nominal_flops(plan) -> dict:
    """Nominal FFT flops per slice of the BST stages (5 N log2 N per complex FFT)."""
    import math

    i = plan.info
    f = lambda n: 5.0 * n * math.log2(n)  # noqa: E731
    L, big, n = i["L"], i["big"], plan.n_out
    return {
        "bst_radial": plan.ntheta * f(L),        # one packed (+s, -s) FFT per angle
        "bst_grid_x": (big // 2) * f(big),       # rows ky < big/2
        "bst_grid_y": (n / 2) * f(big),          # packed column pairs
    }
