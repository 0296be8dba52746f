"""Replica bookkeeping for ``bench.py --gpus N`` (replicas only).

Every rank runs the same hot-path workload on its own GPU; there is no
collective on the data path.  The only cross-rank communication is the
timing reduction: the job's time is the MAX over ranks of the device-timed
region, and its throughput is the work of ALL ranks divided by that time.
Works with any ``torch.distributed`` backend (NCCL on the GPU box, gloo in
the CPU tests).
"""

from __future__ import annotations

import os


def rank_info():
    """(rank, world_size, local_rank) from the torchrun environment."""
    def _i(name, default):
        try:
            return int(os.environ.get(name, default))
        except ValueError:
            return default
    return _i("RANK", 0), _i("WORLD_SIZE", 1), _i("LOCAL_RANK", 0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (no-op without an initialised process group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(units_per_rank: float, ms_this_rank: float, device=None) -> tuple:
    """(whole-job units/s, job ms) with the job time = max over ranks."""
    import torch.distributed as dist
    world = dist.get_world_size() if (dist.is_available() and dist.is_initialized()) else 1
    ms = max_over_ranks(ms_this_rank, device)
    return world * units_per_rank / (ms * 1e-3), ms
