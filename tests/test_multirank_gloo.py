"""World-size-2 gloo run of bench.py's multi-rank plumbing on CPU: the slice
ranks run_ours reconstructs (bench.rank_slices, strong and weak scaling) cover the
volume exactly once, the gathered shard table every rank reports agrees, and the
max/sum reductions the bench uses for timing and throughput agree across ranks.
(The data path has no collective: slices are independent.)"""

import os
import socket

import pytest
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, total, scaling, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench

    d = bench.Dist()
    ids = bench.rank_slices(total, world, rank, scaling)
    shards = d.gather([ids[0], ids[-1] + 1] if ids else [0, 0])
    t_max = d.max(float(rank + 1))
    n_sum = d.sum(float(len(ids)))
    d.barrier()
    q.put((rank, ids, shards, t_max, n_sum))
    d.close()


def _run(world, total, scaling):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, total, scaling, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("total", [2048, 7])
def test_two_rank_strong_shards_and_reductions(total):
    res = _run(2, total, "strong")
    all_ids = res[0][1] + res[1][1]
    assert all_ids == list(range(total))                 # every slice exactly once, in order
    assert res[0][2] == res[1][2] == [[r[1][0], r[1][-1] + 1] for r in res]
    assert all(r[3] == 2.0 for r in res)                  # max over ranks
    assert all(r[4] == float(total) for r in res)         # total slices


def test_two_rank_weak_slices():
    res = _run(2, 5, "weak")
    assert res[0][1] == list(range(0, 5)) and res[1][1] == list(range(5, 10))
    assert all(r[4] == 10.0 for r in res)


def test_rank_slices_config3_at_1_2_4_8():
    import bench

    for world in (1, 2, 4, 8):
        ids = [i for r in range(world) for i in bench.rank_slices(2048, world, r, "strong")]
        assert ids == list(range(2048))
        assert {len(bench.rank_slices(2048, world, r, "strong")) for r in range(world)} == {2048 // world}


def test_both_arms_state_the_same_config():
    """The reference arm's `config` (built without a GPU from the oracle's mesh rule) is the dict our arm
    prints for the same command line: same keys, same values, at every world size of the scaling run."""
    import argparse

    import bench

    from oracle import fastbp_oracle as fo, phantoms

    for world in (1, 2, 4, 8):
        a = argparse.Namespace(slices=0, scaling="strong", config=3, chunk=0, streams=0, geometry=None, gpus=world)
        c = dict(phantoms.CONFIGS[3])
        _, _, nr, _ = fo.lp_geometry(c["nt"], c["n"])
        geom = {"nrho": nr, "L": 8192, "nphi": 4096}
        cfg = bench.workload_config(a, c, world, geom, *bench.default_schedule(a, False, False))
        assert cfg["slices_total"] == 2048 and cfg["slices_per_rank"] == 2048 // world
        assert [i for lo, hi in cfg["rank_slice_ranges"] for i in range(lo, hi)] == list(range(2048))
        assert (cfg["nrho"], cfg["L"], cfg["nphi"], cfg["chunk"], cfg["streams"]) == (3900, 8192, 4096, min(256, 2048 // world), 1)
        assert cfg["workload"] == "config3: FBP 2048 bins x 2048 angles -> 2048^2"


def test_reference_arm_line_config_matches(tmp_path):
    """`bench.py --impl reference` on a tiny sample: one JSON line whose config is workload_config's."""
    import json
    import subprocess
    import sys

    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1", "--steps", "1",
                        "--warmup", "0", "--cpu-workers", "2"], cwd=REPO, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["impl"] == "reference" and d["config"]["nphi"] == 1024 and d["config"]["L"] == 2048
    assert set(d["config"]) == {"workload", "slices_total", "slices_per_rank", "rank_slice_ranges", "chunk",
                                "streams", "parallelism", "l2", "nrho", "L", "nphi"}
    assert d["e2e"]["value"] == d["value"] and d["cpu_baseline"]["kind"] == "port"
