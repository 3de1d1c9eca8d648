"""CPU, world_size 2 over gloo (127.0.0.1): the multi-rank plumbing of bench.py — max-over-ranks
aggregation and the striped mode's barrier protocol (rank 0 drives the pool, the others only join
its barriers) — without a GPU."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    agg = bench.max_over_ranks({"p50": 1.0 + rank, "wall_s": 10.0 - rank}, world)
    # the striped mode: non-zero ranks wait on exactly the three barriers rank 0 passes
    if rank != 0:
        bench.striped_follower()
    else:
        for _ in range(bench.STRIPED_BARRIERS):
            dist.barrier()
    q.put((rank, agg))
    dist.destroy_process_group()


def test_max_over_ranks_and_barriers_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        assert out[r] == {"p50": 2.0, "wall_s": 10.0}


def test_max_over_ranks_single_rank_is_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks({"a": 3.0}, 1) == {"a": 3.0}
