"""World-size-2 gloo run of bench.py's multi-rank plumbing on CPU: contiguous
slice sharding covers every slice exactly once, and the max/sum reductions the
bench uses for timing and throughput agree across ranks.  (The data path has no
collective: slices are independent.)"""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench

    d = bench.Dist()
    ids = list(bench.shard(total, world, rank))
    t_max = d.max(float(rank + 1))
    n_sum = d.sum(float(len(ids)))
    d.barrier()
    q.put((rank, ids, t_max, n_sum))
    d.close()


@pytest.mark.parametrize("total", [2048, 7])
def test_two_rank_shard_and_reductions(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    all_ids = res[0][1] + res[1][1]
    assert all_ids == list(range(total))
    assert all(r[2] == 2.0 for r in res)          # max over ranks
    assert all(r[3] == float(total) for r in res)  # total slices
