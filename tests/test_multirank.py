"""N>1 host logic on CPU with a world_size-2 gloo group (no GPU): contiguous
even-aligned shards cover the batch exactly, per-rank results concatenate to
the single-rank result bit for bit (the per-record arithmetic is the product
math built for the CPU, tests/hostmath), and the max-over-ranks timing
reduction bench.py uses picks the slowest rank."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_00292_b200.shard import shard_bounds


@pytest.mark.parametrize("n", [0, 1, 2, 3, 7, 1000, 1001, 2 ** 20 + 3])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_bounds_partition(n, world):
    bounds = [shard_bounds(n, world, r) for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == n
    for (lo, hi), (lo2, _) in zip(bounds, bounds[1:]):
        assert hi == lo2 and lo <= hi
    assert all(lo % 2 == 0 for lo, _ in bounds)


def test_strong_shards_of_the_bench_job():
    """bench.py's N-rank job: 2^28 records cut like eig33_multi_eigvals cuts a batch."""
    for world in (1, 2, 4, 8):
        b = [shard_bounds(1 << 28, world, r) for r in range(world)]
        assert [hi - lo for lo, hi in b] == [(1 << 28) // world] * world


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    from tests import _util as U

    a = U.mixed_corpus(40001, 21)
    lo, hi = shard_bounds(a.shape[0], world, rank)
    part = np.ascontiguousarray(a[lo:hi])
    lam = np.empty((hi - lo, 3))
    U.hostmath().hm_eigvals(U.ptr(part), U.S(hi - lo), U.ptr(lam), None)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)  # stand-in per-rank time
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    gathered = [None] * world
    dist.all_gather_object(gathered, lam)
    if rank == 0:
        out.put((np.concatenate(gathered), float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shards_match_single_rank():
    from tests import _util as U

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    lam_multi, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = U.mixed_corpus(40001, 21)
    lam = np.empty((a.shape[0], 3))
    U.hostmath().hm_eigvals(U.ptr(a), U.S(a.shape[0]), U.ptr(lam), None)
    assert U.bit_equal(lam_multi, lam).all()
    assert tmax == 2.0
