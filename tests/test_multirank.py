"""N > 1 host logic of bench.py on CPU: world_size-2 gloo process group (replicas only; the
north star keeps the path on one GPU, so the only cross-rank operation is the max-over-ranks
timing reduction)."""
import os
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms = [40.0, 55.5][rank]
    ms_max = bench.max_over_ranks(ms, world, torch.device("cpu"))
    val = bench.job_throughput(world, 64, ms_max)
    q.put((rank, ms_max, val))
    dist.destroy_process_group()


def test_bench_max_over_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ms_max, val in res:
        assert ms_max == pytest.approx(55.5)
        assert val == pytest.approx(2 * 64 / 0.0555)


def test_bench_single_rank_passthrough():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks(12.5, 1, torch.device("cpu")) == 12.5
    assert bench.job_throughput(1, 64, 40.0) == pytest.approx(1600.0)
