"""Multi-GPU policy: replicas only.

One TT-IGA solve (and one matvec+round of the benchmark) is a sequential chain of
small dependent factorizations; nothing in the reference partitions it. With N
GPUs, bench.py runs N independent seeded instances, one process per GPU; the only
collectives are a barrier around the timed region and a MAX-reduce of the device
times (the job is as slow as its slowest rank). These helpers are shared by
bench.py and the gloo tests (tests/test_replicas.py).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def max_over_ranks(x: float, device=None) -> float:
    """MAX of a per-rank scalar over the process group (identity without one)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(work_per_rank: float, ms_max: float, world: int) -> float:
    """Aggregate throughput (work units / s) of `world` replicas timed by the slowest one."""
    return work_per_rank * world / (ms_max / 1e3)


def replica_seed(base: int, rank: int) -> int:
    return int(base) + int(rank)
