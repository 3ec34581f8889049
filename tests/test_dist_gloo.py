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


def _balanced_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_1310_6978_b200 as bfa
    import workloads as W
    from paper_1310_6978_b200.dist import count_sharded
    out = []
    for name, text, n in (("posets5", W.posets(5), 25), ("equiv5", W.equivalences(5), 25),
                          ("bounded5", W.bounded_posets(5), 25)):
        prog = bfa.Program(text).set_option("split_min_vars", 10)

        def oracle_pieces(n_, r, w):
            # this rank's LPT pieces, each counted by the oracle from its text
            plan = prog.shard_plan(n_, w)
            c = sum(oracle.count(prog.shard_piece_text(n_, w, i), nv, threads=2)
                    for i, (own, nv, wk) in enumerate(plan) if own == r and wk > 0)
            return torch.tensor([c], dtype=torch.int64)

        t = count_sharded(prog, n, balanced=True, count_shard=oracle_pieces)
        own = sum(1 for o, _, w in prog.shard_plan(n, world) if o == rank and w)
        out.append((name, int(t.item()), own))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_balanced_shards_oracle_gloo(world):
    """The work-balanced partition (bfa_count_shard's LPT plan): every rank
    counts ITS pieces with the CPU oracle (piece programs exported as text by
    bfa_shard_piece_text), one all-reduce sums them, and the total is the
    closed form (A001035(5) = 4231, Bell(5) = 52, bounded posets 5*4*19 = 380)
    on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_balanced_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = {"posets5": 4231, "equiv5": 52, "bounded5": 380}
    for _, out in res:
        for name, total, own in out:
            assert total == expect[name], (name, total)
            assert own >= 1


def _prepare_worker(rank, world, port, cache, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["BFA_JIT_CACHE"] = cache
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import time

    import paper_1310_6978_b200 as bfa
    import workloads as W
    from paper_1310_6978_b200 import presets
    from paper_1310_6978_b200.dist import prepare_sharded
    text, n, _ = W.config("c4")
    prog = presets.apply(bfa.Program(text), presets.EXHAUSTIVE)
    t0 = time.perf_counter()
    prepare_sharded(prog, n)
    dt = time.perf_counter() - t0
    perm = prog.roles(n, n - (world.bit_length() - 1), sms=148)
    q.put((rank, dt, perm))
    dist.barrier()
    dist.destroy_process_group()


def test_prepare_sharded_rank0_first(tmp_path):
    """Multi-GPU preparation: rank 0 searches the roles and compiles the one
    kernel every rank runs (its cofactor range is a congruent sub-cube);
    rank 1 waits and loads both from the shared JIT cache -- same roles."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_prepare_worker, args=(r, world, port, str(tmp_path), q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][2] == res[1][2]
    assert any(f.startswith("k_") for f in os.listdir(tmp_path))
    assert any(f.startswith("r_") for f in os.listdir(tmp_path))
