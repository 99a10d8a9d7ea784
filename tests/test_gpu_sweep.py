"""Whole-config parity sweep: every slice of configs[1] (16) and configs[2] (64), and 32 slices
spread over configs[3]'s 2048-slice volume, generated on the device exactly as bench.py generates
them (synth.config_batch: fp64 ellipse line integrals + seeded device noise), reconstructed by the
CUDA path, downloaded, and compared slice by slice with the CPU oracle on the same inputs (oracle
runs in one spawned process per host core).  Bar: relative L2 <= 1e-4 (BASELINE.json north_star),
max-abs reported.  With LPBP_SWEEP_OUT set, the per-slice table is written there as JSON."""

import json
import multiprocessing as mp
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

RTOL = 1e-4

# (label, config, slice ids, fbp, n)
CASES = [
    ("config1", 1, list(range(16)), True, 512),
    ("config2", 2, list(range(64)), False, 2048),
    ("config3", 3, list(range(0, 2048, 64)), True, 2048),
]


def _workers() -> int:
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    try:
        avail_gb = int(open("/proc/meminfo").read().split("MemAvailable:")[1].split()[0]) / 1e6
    except Exception:
        avail_gb = 16.0
    return max(1, min(ncpu, int(avail_gb / 3.0), 32))


def test_whole_config_parity_sweep(tmp_path):
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    import paper_1608_03589_b200 as p
    from paper_1608_03589_b200 import synth

    dev = torch.device("cuda")
    jobs = []
    for label, cfg, ids, fbp, n in CASES:
        for lo in range(0, len(ids), 16):
            part = ids[lo:lo + 16]
            x = synth.config_batch(cfg, part, dev)
            img = p.fbp_batch(x, p.FilterSpec(), n) if fbp else p.logpolar_backproject_batch(x, n)
            xs, ims = x.cpu().numpy(), img.cpu().numpy()
            for j, sid in enumerate(part):
                sp, ip = tmp_path / f"{label}_{sid}_g.npy", tmp_path / f"{label}_{sid}_img.npy"
                np.save(sp, xs[j])
                np.save(ip, ims[j])
                jobs.append((label, sid, fbp, n, str(sp), str(ip)))
            del x, img
    torch.cuda.empty_cache()

    import sweep_worker

    with mp.get_context("spawn").Pool(_workers()) as pool:
        rows = pool.map(sweep_worker.oracle_compare, jobs, chunksize=1)

    summary = {}
    for label, _, ids, _, _ in CASES:
        r = [x for x in rows if x[0] == label]
        rel = np.array([x[2] for x in r])
        mab = np.array([x[3] for x in r])
        summary[label] = dict(slices=len(r), rel_l2_max=float(rel.max()), rel_l2_median=float(np.median(rel)),
                              max_abs_max=float(mab.max()), worst_slice=int(r[int(rel.argmax())][1]))
        print(f"{label}: {len(r)} slices, rel_l2 max {rel.max():.3e} median {np.median(rel):.3e}, "
              f"max_abs max {mab.max():.3e} (worst slice {summary[label]['worst_slice']})")
    out = os.environ.get("LPBP_SWEEP_OUT")
    if out:
        with open(out, "w") as f:
            json.dump(dict(bar=RTOL, summary=summary,
                           slices=[dict(config=x[0], slice=x[1], rel_l2=x[2], max_abs=x[3], ref_max_abs=x[4])
                                   for x in rows]), f, indent=1)
    bad = [x for x in rows if not x[2] <= RTOL]
    assert not bad, bad
