"""Multi-process (world_size 2 and 4, gloo, CPU) test of the cofactor
sharding host logic (paper_1310_6978_b200/dist.py): the rank ranges tile
[0, 2^n) in order, and the single all-reduce of the per-rank counts gives the
full count.  The per-rank range counter here is the CPU oracle (tests only);
on the GPU box it is bfa_count_range and the backend is NCCL."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1310_6978_b200.dist import rank_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, text, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1310_6978_b200.dist import count_sharded

    def oracle_range(n_, lo, hi):
        return torch.tensor([oracle.count(text, n_, lo, hi, threads=2)], dtype=torch.int64)

    t = count_sharded(None, n, count_range=oracle_range)
    q.put((rank, int(t.item()), rank_range(n, rank, world)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_count_sharded_gloo(world):
    import oracle
    import workloads as W
    text, n = W.posets(4), 16
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, text, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = oracle.count(text, n)
    assert full == 219
    assert all(c == full for _, c, _ in res)
    ranges = [r for _, _, r in res]
    assert ranges[0][0] == 0 and ranges[-1][1] == 1 << n
    assert all(ranges[k][1] == ranges[k + 1][0] for k in range(world - 1))


def test_rank_range_rules():
    assert rank_range(36, 0, 8) == (0, 1 << 33)
    assert rank_range(36, 7, 8) == (7 << 33, 1 << 36)
    with pytest.raises(ValueError):
        rank_range(36, 0, 6)
    with pytest.raises(ValueError):
        rank_range(7, 0, 8)
    with pytest.raises(ValueError):
        rank_range(36, 8, 8)


def _plan_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1310_6978_b200 as bfa
    import workloads as W
    out = []
    for cfg in ("c4", "c5"):
        text, n, _ = W.config(cfg)
        plan = bfa.Program(text).shard_plan(n, world)      # host only: no GPU, no communication
        flat = torch.tensor([x for piece in plan for x in piece], dtype=torch.int64)
        gathered = [torch.zeros_like(flat) for _ in range(world)]
        dist.all_gather(gathered, flat)
        out.append((cfg, n, plan, all(torch.equal(g, flat) for g in gathered)))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_shard_plan_identical_on_all_ranks(world):
    """Work-balanced cofactor sharding (bfa_count_shard) needs no exchange to
    agree on who counts what: every rank derives the same plan on its own.
    The pieces tile the 2^n cube, each non-constant piece has one owner, and
    the estimated loads are balanced."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, out in res:
        for cfg, n, plan, same in out:
            assert same, cfg
            assert sum(1 << nv for _, nv, _ in plan) == 1 << n
            assert {o for o, _, w in plan if w} == set(range(world))
            load = [sum(w for o, _, w in plan if o == r) for r in range(world)]
            assert max(load) <= 1.5 * sum(load) / world
