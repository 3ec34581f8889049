"""Cofactor sharding over GPUs.

P = 2^p ranks, one process per GPU.  Rank r owns the cofactor in which the
top p variable ids (n-1 .. n-p, the paper's b_1..b_p) spell r, i.e. the
contiguous valuation range [r 2^(n-p), (r+1) 2^(n-p)).  Every rank runs the
same code (one kernel, compiled once on rank 0 and loaded by the others from
the JIT cache; no rank specialisation), so the work per rank is the same
number of valuations.  This is the default partition (north_star: "the 2^n
space is split by the top log2(P) variables into cofactor ranges").

count: the only exchange is ONE all-reduce(SUM) of the 8-byte count, issued
after the stream that produced it (NCCL over NVLink/NVSwitch on the GPU
box).  Counts are summed as int64; two's-complement addition is addition mod
2^64, so the bit pattern equals the uint64 sum even at n = 63.
eval: no collective; each rank writes its own slice of the vector.

balanced=True is the alternative partition (bfa_count_shard): an LPT
assignment of the pieces of a deterministic Shannon decomposition (for
programs whose top-variable cofactors differ wildly in work after the
Reduction); measured against the default in DESIGN.md §6.
"""
from __future__ import annotations


def rank_range(n: int, rank: int, world: int):
    """Valuation range [lo, hi) owned by `rank` of `world` (a power of two)."""
    if world < 1 or world & (world - 1):
        raise ValueError(f"world size {world} is not a power of two")
    p = world.bit_length() - 1
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside [0, {world})")
    if n - p < 5:
        raise ValueError(f"n={n} too small to shard over {world} ranks (need n - log2(P) >= 5)")
    span = 1 << (n - p)
    return rank * span, (rank + 1) * span


def _world_rank(group):
    import torch.distributed as dist
    if dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def prepare_sharded(prog, n: int, group=None):
    """Compile this rank's count kernel once for the whole job: rank 0 runs
    the role search + NVRTC (host only) and writes the persistent JIT cache,
    the other ranks wait on a barrier and then load its results.  Every rank
    needs the same kernel (the ranges are congruent sub-cubes)."""
    import torch.distributed as dist
    world, rank = _world_rank(group)
    k_free = n - (world.bit_length() - 1)
    if rank == 0:
        prog.prepare_range(n, k_free)
    if world > 1:
        dist.barrier(group)
        if rank != 0:
            prog.prepare_range(n, k_free)


def count_sharded(prog, n: int, group=None, count_range=None, stream=None, balanced: bool = False,
                  count_shard=None):
    """Model count over all 2^n valuations, sharded over the process group.

    Returns a 1-element int64 tensor holding the global count on every rank.
    Default: rank r counts its contiguous range rank_range(n, r, P) with
    `count_range(n, lo, hi)` (default: prog.count_range on `stream`).
    balanced=True: rank r counts the decomposition pieces bfa_count_shard
    assigns it, with `count_shard(n, rank, world)` (default prog.count_shard).
    The CPU multi-process tests inject oracle-backed counters to exercise the
    partition and the reduction with gloo."""
    import torch.distributed as dist
    world, rank = _world_rank(group)
    if balanced:
        t = count_shard(n, rank, world) if count_shard else prog.count_shard(n, rank, world, stream=stream)
    else:
        lo, hi = rank_range(n, rank, world)
        t = count_range(n, lo, hi) if count_range else prog.count_range(n, lo, hi, stream=stream)
    if world > 1:
        if t.is_cuda:
            # NCCL orders the collective after torch's CURRENT stream; the
            # count was produced on `stream`, so make the current stream wait
            import torch
            cur = torch.cuda.current_stream(t.device)
            if stream is not None and stream != cur:
                cur.wait_stream(stream if not isinstance(stream, int) else torch.cuda.ExternalStream(stream))
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def eval_sharded(prog, n: int, group=None, out=None, count_out=None, stream=None):
    """This rank's slice of the DNF vector (no collective).  Returns
    (slice tensor, lo, hi).  Needs n - log2(P) >= 6 (whole u64 words)."""
    world, rank = _world_rank(group)
    lo, hi = rank_range(n, rank, world)
    if world > 1 and (hi - lo) % 64:
        raise ValueError("sharded eval needs n - log2(P) >= 6")
    return prog.eval_range(n, lo, hi, out=out, count_out=count_out, stream=stream), lo, hi
