"""The N>1 path on CPU: gloo world_size 2 -- replicas with a barrier and a MAX-reduce of times."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_13224_b200.replicas import max_over_ranks, replica_seed, whole_job_rate
    local_ms = 10.0 + 5.0 * rank
    dist.barrier()
    m = max_over_ranks(local_ms)
    rate = whole_job_rate(1e9, m, world)
    # each replica runs its own seeded instance: seeds differ, shapes agree
    g = torch.Generator().manual_seed(replica_seed(0, rank))
    x = torch.randn(4, generator=g)
    xs = [torch.zeros(4) for _ in range(world)]
    dist.all_gather(xs, x)
    q.put((rank, m, rate, not torch.equal(xs[0], xs[1])))
    dist.destroy_process_group()


def test_two_replicas_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, m, rate, distinct in out:
        assert m == 15.0                       # slowest rank sets the job time
        assert abs(rate - 2e9 / 0.015) < 1e-3  # whole-job aggregate over both replicas
        assert distinct


def test_single_process_identity():
    from paper_2509_13224_b200.replicas import max_over_ranks, whole_job_rate
    assert max_over_ranks(3.5) == 3.5
    assert whole_job_rate(2.0, 1000.0, 1) == 2.0
