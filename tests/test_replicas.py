"""N > 1 path of bench.py (replicas only), world_size 2 over gloo on CPU."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2409_14222_b200.replicas import job_throughput, max_over_ranks, rank_info
    r, w, lr = rank_info()
    assert (r, w, lr) == (rank, world, rank)
    # rank-dependent timings: the job time is the slowest rank's
    ms = 10.0 + 5.0 * rank
    value, job_ms = job_throughput(units_per_rank=66049 * 20, ms_this_rank=ms)
    q.put((rank, value, job_ms, max_over_ranks(float(rank))))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_throughput_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, value, job_ms, mx in out:
        assert job_ms == pytest.approx(15.0)               # max over ranks
        assert value == pytest.approx(2 * 66049 * 20 / 15e-3)   # all ranks' work
        assert mx == 1.0


def test_single_process_defaults():
    from paper_2409_14222_b200.replicas import job_throughput, max_over_ranks
    assert max_over_ranks(3.5) == 3.5
    v, ms = job_throughput(100.0, 2.0)
    assert ms == 2.0 and v == pytest.approx(100.0 / 2e-3)
