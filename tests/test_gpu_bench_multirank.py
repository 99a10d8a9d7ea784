"""The N > 1 bench path end to end (what the driver's scaling run launches), as a functional check.

Two ranks under torch.distributed.run on the box's GPU(s): on a one-GPU box both ranks share cuda:0
(bench.py flags `run.shared_device`; no scaling number is taken from such a run).  The ranks never
wait on each other's kernels — the only cross-rank traffic is the gloo barrier and the max/sum of
timings — so sharing a device cannot deadlock.  Checks that every collective is reached by every rank
(a rank-0-only reduction once hung the line's assembly), that the strong-scaling shards cover the
volume's slice ids exactly once, and that the line carries the contract's keys.
"""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_two_ranks_strong_shards():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--gpus", "2", "--steps", "1",
           "--warmup", "3", "--slices", "32", "--no-cpu-baseline", "--e2e-slices", "8", "--e2e-steps", "1"]
    r = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    c = d["config"]
    assert c["slices_total"] == 32 and c["slices_per_rank"] == 16
    ids = [i for lo, hi in c["rank_slice_ranges"] for i in range(lo, hi)]
    assert sorted(ids) == list(range(32))
    # what the ranks actually took (gathered) is what `config` states from the arguments
    assert [list(v) for v in d["run"]["rank_slice_ranges_gathered"]] == c["rank_slice_ranges"]
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    for k in ("roofline", "pipeline", "clocks", "ms_per_step"):
        assert k in d
