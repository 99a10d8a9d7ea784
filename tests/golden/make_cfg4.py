"""Config-4 golden values from the REFERENCE (fastbp, /root/reference/pkg/src):
its direct backprojector and its log-polar backprojector on the config-2 slice 0
sinogram (the same inputs configs[4] names), at the full 2048^2 size.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cfg4.py      (~10 min, one core)

Writes tests/golden/cfg4.npz: sampled rows of the reference's direct image and the
LP-vs-direct relative L2 gap (unit disk and full image), which the GPU tests pin.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import fastbp as fb  # noqa: E402  (the reference)

from oracle import phantoms  # noqa: E402

ROWS = np.arange(3, 2048, 97)


def main() -> None:
    g = phantoms.config_sinogram(4, 0).astype(np.float64)
    s = fb.Sinogram(*g.shape, g)
    t = time.time()
    lp = fb.logpolar_backproject(s, 2048).values
    t_lp = time.time() - t
    t = time.time()
    nv = fb.backproject_naive(s, 2048).values
    t_nv = time.time() - t
    xs = -1.0 + (np.arange(2048) + 0.5) * (2.0 / 2048)
    X, Y = np.meshgrid(xs, xs)
    disk = np.hypot(X, Y) <= 1.0
    gap_disk = float(np.linalg.norm(lp[disk] - nv[disk]) / np.linalg.norm(nv[disk]))
    gap_full = float(np.linalg.norm(lp - nv) / np.linalg.norm(nv))
    np.savez_compressed(os.path.join(HERE, "cfg4.npz"), rows=ROWS, naive_rows=nv[ROWS], lp_rows=lp[ROWS],
                        gap_disk=gap_disk, gap_full=gap_full)
    info = {"gap_disk": gap_disk, "gap_full": gap_full, "seconds_logpolar": t_lp, "seconds_naive": t_nv,
            "input": "phantoms.config_sinogram(4, 0) == config 2 slice 0"}
    with open(os.path.join(HERE, "kat_cfg4.json"), "w") as f:
        json.dump(info, f, indent=1)
    print(json.dumps(info))


if __name__ == "__main__":
    main()
