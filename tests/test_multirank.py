"""Multi-rank host logic on CPU (gloo, world_size 2): bench.py runs N
independent replicas ("replicas only"); the whole-job value sums
solves over ranks and divides by the max rank time."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    solves = 10 + rank * 5
    t_ms = 1000.0 + 250.0 * rank
    e2e_ms = 1100.0 + 100.0 * rank
    out = bench.aggregate_replicas(dist, "cpu", solves, t_ms, e2e_ms)
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_replica_aggregation_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=100) for _ in procs)
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    for r in (0, 1):
        solves_all, t_max, te = res[r]
        assert solves_all == 25
        assert t_max == 1250.0
        assert te == 1200.0
