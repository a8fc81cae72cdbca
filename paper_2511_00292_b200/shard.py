"""Batch partitioning for multi-GPU runs (no inter-GPU communication).

The path shards with no exchange step: every record is independent,
so a batch is cut into contiguous shards and each GPU (one process per GPU, or
one host thread per GPU in eig33_multi_eigvals) evaluates its own shard.

shard_bounds: strong sharding of one given batch -- the formula the C++ host
driver uses (paper_2511_00292_b200/csrc/eig33_host.cpp eig33_multi_eigvals)
and bench.py's N-rank job: lo_g = 2*floor(g*n/(2G)), even so every shard's
device copy stays 16-B aligned for the TMA loads; the last shard takes the
remainder.
"""


def shard_bounds(n: int, world: int, rank: int):
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    lo = 2 * (rank * n // (2 * world))
    hi = n if rank + 1 == world else 2 * ((rank + 1) * n // (2 * world))
    return lo, hi
