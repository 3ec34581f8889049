"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit
for bit.  Vectors and counts are integer results, so the bar is exact
equality (BASELINE.json north star: "bit-exact")."""
import re

import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

bfa = pytest.importorskip("paper_1310_6978_b200")
from paper_1310_6978_b200 import presets  # noqa: E402


def host(words_t):
    return words_t.cpu().numpy().view(np.uint64)


def check_full(text, n, prog=None):
    prog = prog or bfa.Program(text)
    ow, oc = oracle.evaluate(text, n)
    gw = host(prog.eval(n))
    assert np.array_equal(gw, ow), (text[:200], n)
    assert prog.count(n) == oc
    return oc


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.set_device(0)


# ------------------------------------------------------------ paper fixtures
def test_c1_posets3(golden):
    g = golden("c1_posets3.json")
    p = bfa.Program(W.posets(3))
    w = host(p.eval(9))
    assert [int(x) for x in w] == [int(x, 16) for x in g["words_u64"]]
    assert p.count(9) == 19


def test_generators_and_baequ(golden):
    g = golden("generators_n3.json")
    for var, bits in g["vectors"].items():
        w = host(bfa.Program(var).eval(3))
        assert "".join(str((int(w[0]) >> mu) & 1) for mu in range(8)) == bits
    b = golden("baequ.json")
    w = host(bfa.Program(b["program"]).eval(4))
    assert int(w[0]) == int(b["word0"], 16)


@pytest.mark.parametrize("family", ["posets", "equivalences", "linear_orders", "bounded_posets",
                                    "special_posets"])
def test_closed_forms_gpu(golden, family):
    g = golden("closed_forms.json")[family]
    gen = getattr(W, family)
    for k, expect in zip(g["k"], g["count"]):
        if k > 5:
            continue
        p = bfa.Program(gen(k))
        assert p.count(k * k) == expect, (family, k)


def test_c3_vectors():
    """Config C3: equivalences (52) and posets (4231) on 5 points, full
    2^25-bit vectors against the oracle."""
    for name in ("c3_equiv", "c3_posets"):
        text, n, expect = W.config(name)
        assert check_full(text, n) == expect


# ------------------------------------------------------------ random suite
@pytest.mark.parametrize("block", range(10))
def test_random_terms(block):
    """500 random terms: n = seed mod 21 in [0, 20]."""
    for seed in range(block * 50, block * 50 + 50):
        p = W.random_program(seed, max_n=20)
        check_full(p.text, p.n)


GEOMETRIES = [dict(slot_bits=0, thread_bits=5, inner_bits=0), dict(slot_bits=1, thread_bits=6, inner_bits=2),
              dict(slot_bits=3, thread_bits=7, inner_bits=3), dict(slot_bits=2, thread_bits=8, inner_bits=4),
              dict(force_generic=1), dict(imad_cost_pct=20), dict(imad_cost_pct=20, force_generic=1),
              dict(dual_pipe=0), dict(slot_bits=5, imad_cost_pct=50), dict(slot_bits=4, inner_bits=2, min_blocks=2),
              dict(engine=1), dict(segment_cells=40), dict(segment_cells=16, segment_remat=0)]


@pytest.mark.parametrize("geo", range(len(GEOMETRIES)))
def test_launch_geometries(geo):
    """Results independent of the launch geometry."""
    for seed in list(range(12, 21)) + [100, 120, 140]:
        p = W.random_program(seed, max_n=20)
        prog = bfa.Program(p.text)
        for k, v in GEOMETRIES[geo].items():
            prog.set_option(k, v)
        check_full(p.text, p.n, prog)
    for text, n in ((W.posets(4), 16), (W.random_dag(20, 300, seed=9), 20)):
        prog = bfa.Program(text)
        for k, v in GEOMETRIES[geo].items():
            prog.set_option(k, v)
        check_full(text, n, prog)


def test_ranges_concatenate():
    """P-11: range slices concatenate to the vector; range counts sum."""
    text, n = W.random_dag(22, 400, seed=2), 22
    p = bfa.Program(text)
    full = host(p.eval(n))
    total = 0
    parts = []
    bounds = [0, 64 * 7, 1 << 12, (1 << 20) + 64 * 3, 3 << 20, 1 << 22]
    for lo, hi in zip(bounds, bounds[1:]):
        parts.append(host(p.eval_range(n, lo, hi)))
        total += int(p.count_range(n, lo, hi).item())
    assert np.array_equal(np.concatenate(parts), full)
    assert total == p.count(n) == oracle.count(text, n)
    # count ranges at 32-granularity
    lo, hi = 32 * 5, 32 * 1001
    assert int(p.count_range(n, lo, hi).item()) == oracle.count(text, n, lo, hi)


def test_edge_cases():
    for n in range(0, 7):
        check_full("1", n)
        check_full("0", n)
    for n in range(1, 8):
        check_full(f"x{n - 1}", n)
        check_full(" ^ ".join(f"x{v}" for v in range(n)), n)
    check_full("", 5)
    assert bfa.Program("x0 | ~x0").count(40) == 1 << 40
    assert bfa.Program("x0 & ~x0").count(40) == 0
    p = bfa.Program("x62 & x61 | x0")
    lo = (1 << 63) - (1 << 20)
    assert int(p.count_range(63, lo, 1 << 63).item()) == oracle.count("x62 & x61 | x0", 63, lo, 1 << 63)
    with pytest.raises(bfa.BfaError) as e:
        bfa.Program("x5").count(5)
    assert e.value.code == bfa.BFA_E_RANGE
    with pytest.raises(bfa.BfaError):
        bfa.Program("x0").count(64)
    with pytest.raises(bfa.BfaError):
        bfa.Program("x0").count_range(20, 3, 64)


def test_invariants_large():
    """P-11 at sizes beyond the oracle: count(f) + count(~f) = 2^n,
    count(f ^ x_fresh) = 2^(n-1), Shannon on one variable."""
    text = W.random_dag(34, 500, seed=4)
    body = "\n".join(text.splitlines()[:-1])
    out = text.splitlines()[-1]
    n = 34
    c = bfa.Program(text).count(n)
    assert c + bfa.Program(f"{body}\n~{out}").count(n) == 1 << n
    assert bfa.Program(f"{body}\n{out} ^ x34").count(n + 1) == 1 << n
    assert (bfa.Program(f"{body}\n{out} & x20").count(n) + bfa.Program(f"{body}\n{out} & ~x20").count(n)) == c


# ------------------------------------------------------------ configs at full size
def test_c4_posets6_count_and_subcubes():
    """Config C4 at full size (n=36) with the default options:
    count = A001035(6) = 130023; sampled cofactor sub-cubes of the vector
    equal the oracle's."""
    text, n, expect = W.config("c4")
    p = bfa.Program(text)
    assert p.count(n) == expect
    rng = np.random.default_rng(7)
    refl = sum(1 << (35 - 7 * i) for i in range(6))   # all p(i,i) set
    for _ in range(3):
        lo = (int(rng.integers(0, 1 << 36)) | refl) & ~((1 << 24) - 1)
        hi = lo + (1 << 24)
        ow, oc = oracle.evaluate(text, n, lo, hi)
        gw = host(p.eval_range(n, lo, hi))
        assert np.array_equal(gw, ow) and int(p.count_range(n, lo, hi).item()) == oc


def test_c4_full_set_bits():
    """P-14: the full 2^36-bit vector's set-bit list equals the oracle's
    (full oracle run in 2^30-valuation chunks; short-circuit on the
    reflexivity conjuncts keeps it cheap)."""
    text, n, expect = W.config("c4")
    p = bfa.Program(text)
    gw = p.eval(n)                               # 8 GiB on the device
    nz = torch.nonzero(gw).flatten()
    words = gw[nz].cpu().numpy().view(np.uint64)
    idx = nz.cpu().numpy()
    del gw
    torch.cuda.empty_cache()
    bits = np.unpackbits(words.view(np.uint8), bitorder="little").reshape(-1, 64)
    r, c = np.nonzero(bits)
    gbits = np.sort(idx[r].astype(np.int64) * 64 + c)
    chunk = 1 << 30
    obits = []
    for k in range(1 << (n - 30)):
        ow, _ = oracle.evaluate(text, n, k * chunk, (k + 1) * chunk)
        obits.append(oracle.set_bits(ow, k * chunk))
    obits = np.concatenate(obits)
    assert len(obits) == expect == len(gbits)
    assert np.array_equal(gbits, obits)


def renamed(text, perm):
    """f'(x) = f(x with x_v renamed x_perm[v]) -- input transformation only
    (the oracle's arithmetic is untouched): the models of f' at position q are
    the models of f at the valuation the permuted kernel enumerates at q."""
    return re.sub(r"\bx(\d+)\b", lambda m: f"x{perm[int(m.group(1))]}", text)


@pytest.mark.parametrize("cfg,plan", [("c5", "exhaustive"), ("c5", "cold"), ("c4", "exhaustive")])
def test_exhaustive_bench_kernel_vs_oracle(cfg, plan):
    """The headline kernel bench.py times (presets.exhaustive(cfg) over the whole
    2^n cube: same variant, same searched roles, same cubin) against the
    oracle on 4 random sub-ranges of its enumeration order, 2^24 valuations
    each for C5, 2^26 (one outer-iteration unit) for C4 (P-13; C5 cannot be
    oracle-checked whole).  bfa_count_positions runs
    exactly that kernel; the oracle counts the renamed program f' on the same
    position range."""
    text, n, expect = W.config(cfg)
    preset = getattr(presets, plan)(cfg)     # bench.py's value (exhaustive) and e2e (cold) kernels
    p = presets.apply(bfa.Program(text), preset)
    perm = p.roles(n)
    assert sorted(perm) == list(range(64)) and perm != list(range(64))
    text2 = renamed(text, perm)
    rng = np.random.default_rng(13106978)
    span = 1 << (26 if cfg == "c4" else 24)   # >= one outer-iteration unit of the kernel
    for _ in range(4):
        if cfg == "c4":          # sub-ranges where every reflexivity letter is 1 (else no models)
            lo = (int(rng.integers(0, 1 << 36)) | sum(1 << perm[35 - 7 * i] for i in range(6))) & ~(span - 1)
        else:
            lo = int(rng.integers(0, 1 << (n - 24))) << 24
        got = int(p.count_positions(n, n, lo, lo + span).item())
        assert got == oracle.count(text2, n, lo, lo + span), (cfg, lo)
    # the same compiled kernel over the whole cube: the count bench.py reports
    c = p.count(n)
    ll = bfa.last_launch()
    seg = ll["segments"][0]
    assert ll["kernels"] == 1 and seg["roles"] == "searched" and seg["s"] == preset["slot_bits"]
    if expect is not None:
        assert c == expect
    else:                          # C5: complement invariant (P-11) with the same preset
        body, out = "\n".join(text.splitlines()[:-1]), text.splitlines()[-1]
        pc = presets.apply(bfa.Program(f"{body}\n~{out}"), preset)
        assert c + pc.count(n) == 1 << n


def test_decomposed_work_queue_vs_oracle():
    """The decomposed path (presets.DECOMPOSED: Shannon leaves in persistent
    work-queue kernels, queue_inner 2, role budget 400, slot 5, IMAD 50),
    scaled down so it runs on oracle-checkable sub-cubes: decomposition of
    aligned 2^24 C5 sub-cubes (decompose_min_k 24) into leaves of >= 18
    variables (split_min_vars 18), one module and many modules, direct /
    graph-captured / replayed calls, each against the oracle."""
    text, n, _ = W.config("c5")
    rng = np.random.default_rng(42)
    base = bfa.Program(text)

    def nontrivial_subcube():
        # a sub-cube whose cofactor (top 18 variables fixed) the Reduction
        # does not fold to a constant, so it really decomposes
        while True:
            lo = int(rng.integers(0, 1 << (n - 24))) << 24
            q, _, _ = base.assume(n, {v: (lo >> v) & 1 for v in range(24, n)})
            if q.info["const_value"] == -1 and q.info["gates"] >= 100:
                return lo

    for qb in (512, 4, 512, 4):
        p = presets.apply(bfa.Program(text), presets.DECOMPOSED, split_pieces=64, queue_bodies=qb,
                          decompose_min_k=24, split_min_vars=18, queue_slot_bits=5)
        lo = nontrivial_subcube()
        expect = oracle.count(text, n, lo, lo + (1 << 24))
        out = torch.zeros(1, dtype=torch.int64, device="cuda")
        for _ in range(3):                       # direct, capture, replay
            p.count_range(n, lo, lo + (1 << 24), out=out)
            assert int(out.item()) == expect, (qb, lo)
        ll = bfa.last_launch()
        assert ll["variant"] == "decomposed" and ll["queue"]["bodies"] > 1, ll


def test_role_search_subcubes():
    """Count mode over an aligned sub-cube of >= 2^24 valuations enumerates it
    in a searched variable order (DESIGN.md §5 role search): counts equal the
    oracle's on such sub-cubes, and a program and its complement (searched
    independently) sum to the sub-cube size."""
    text, n, _ = W.config("c4")
    p = bfa.Program(text)
    refl = sum(1 << (35 - 7 * i) for i in range(6))
    rng = np.random.default_rng(5)
    for _ in range(3):
        lo = (int(rng.integers(0, 1 << 36)) | refl) & ~((1 << 26) - 1)
        assert int(p.count_range(n, lo, lo + (1 << 26)).item()) == oracle.count(text, n, lo, lo + (1 << 26))
        assert bfa.last_launch()["segments"][0].get("roles") == "searched"
    text, n, _ = W.config("c5")
    p = bfa.Program(text)
    body, out = "\n".join(text.splitlines()[:-1]), text.splitlines()[-1]
    pc = bfa.Program(f"{body}\n~{out}")
    for lo in ((123 << 24), (1 << 42) - (1 << 24)):
        c = int(p.count_range(n, lo, lo + (1 << 24)).item())
        assert c == oracle.count(text, n, lo, lo + (1 << 24))
        assert c + int(pc.count_range(n, lo, lo + (1 << 24)).item()) == 1 << 24
    for k in (30, 36):
        lo = (5 << 36) & ~((1 << k) - 1)
        a = int(p.count_range(n, lo, lo + (1 << k)).item())
        b = int(pc.count_range(n, lo, lo + (1 << k)).item())
        assert a + b == 1 << k


@pytest.mark.gpu
@pytest.mark.parametrize("pairs", [1, 2])
def test_imad_pair_cells_vs_oracle(pairs):
    """Option imad_pairs (kind-2 IMAD cells x * K(u1, u2) + C(u1, u2), K and C
    hoisted LOP3 cells): the whole-cube C5 kernel built with it, run by
    bfa_count_positions on 2 ranges of 2^24 positions of its enumeration
    order, against the oracle on the renamed program (PAPER.md:341-354 Prop
    2.2); C4's full cube gives the closed form 130023 (OEIS A001035)."""
    text, n, _ = W.config("c5")
    p = presets.apply(bfa.Program(text), presets.exhaustive("c5"), role_seeds=1, imad_pairs=pairs)
    text2 = renamed(text, p.roles(n))
    for lo in ((77 << 24), (1 << 42) - (1 << 24)):
        got = int(p.count_positions(n, n, lo, lo + (1 << 24)).item())
        assert got == oracle.count(text2, n, lo, lo + (1 << 24)), (pairs, lo)
    t4, n4, e4 = W.config("c4")
    q = presets.apply(bfa.Program(t4), presets.exhaustive("c4"), imad_pairs=pairs)
    assert q.count(n4) == e4


@pytest.mark.gpu
def test_kernel_cofactoring():
    """Kernel-level cofactoring (2^j cofactor programs via bfa_assume, each
    with its own role search and kernel, constant-0 cofactors decided at
    compile time) leaves every count unchanged: full cubes, oracle
    sub-cubes, and f / ~f summing to the cube."""
    text, n, expect = W.config("c4")
    for j in (1, 3, 5):
        p = bfa.Program(text).set_option("kernel_cofactor_bits", j)
        assert p.count(n) == expect
        assert bfa.last_launch()["variant"] == "kernel-cofactored"
    refl = sum(1 << (35 - 7 * i) for i in range(6))
    lo = refl & ~((1 << 28) - 1)
    p = bfa.Program(text).set_option("kernel_cofactor_bits", 3)
    assert int(p.count_range(n, lo, lo + (1 << 28)).item()) == oracle.count(text, n, lo, lo + (1 << 28))
    text, n, _ = W.config("c5")
    body, out = "\n".join(text.splitlines()[:-1]), text.splitlines()[-1]
    for j in (2, 5):
        p = bfa.Program(text).set_option("kernel_cofactor_bits", j)
        pc = bfa.Program(f"{body}\n~{out}").set_option("kernel_cofactor_bits", j)
        lo = 9 << 30
        a = int(p.count_range(n, lo, lo + (1 << 30)).item())
        assert a == int(bfa.Program(text).count_range(n, lo, lo + (1 << 30)).item())
        assert a + int(pc.count_range(n, lo, lo + (1 << 30)).item()) == 1 << 30
    lo = 77 << 24
    p = bfa.Program(text).set_option("kernel_cofactor_bits", 0)
    assert int(p.count_range(n, lo, lo + (1 << 24)).item()) == oracle.count(text, n, lo, lo + (1 << 24))


def test_multi_body_kernels():
    """Cofactor children fused into one multi-body launch per split give the
    same counts as separate launches."""
    for cfg in ("c4", "c5"):
        text, n, _ = W.config(cfg)
        full = bfa.Program(text).count(n)
        p = bfa.Program(text).set_option("kernel_cofactor_bits", 4).set_option("multi_body", 1)
        assert p.count(n) == full
        ll = bfa.last_launch()
        assert ll["constant_zero"] <= ll["cofactors"]
        if cfg == "c5":                      # C4 keeps a single live child: separate launch
            assert ll.get("multi_body") == 1
        p = bfa.Program(text).set_option("split_pieces", 8).set_option("kernel_cofactor_bits", 3)
        p.set_option("multi_body", 1)
        for _ in range(3):
            assert p.count(n) == full


def test_split_pieces():
    """Shannon decomposition into pieces (each with kernel-level
    cofactoring) leaves counts unchanged, on the full cube and on an aligned
    sub-cube."""
    for cfg in ("c4", "c5"):
        text, n, _ = W.config(cfg)
        full = bfa.Program(text).count(n)
        for sp, j in ((8, 0), (8, 4), (16, 2)):
            p = bfa.Program(text).set_option("split_pieces", sp).set_option("kernel_cofactor_bits", j)
            assert p.count(n) == full, (cfg, sp, j)              # bfa_count (host result)
            assert int(p.count_range(n, 0, 1 << n).item()) == full
            assert bfa.last_launch()["variant"] == "decomposed"
    text, n, _ = W.config("c5")
    lo = 5 << 32
    p = bfa.Program(text).set_option("split_pieces", 8).set_option("kernel_cofactor_bits", 2)
    assert int(p.count_range(n, lo, lo + (1 << 32)).item()) == \
        int(bfa.Program(text).count_range(n, lo, lo + (1 << 32)).item())


def test_work_queue_kernels():
    """Decomposition leaves run as persistent work-queue kernels (blocks take
    equal-work chunks of many noinline bodies with an atomic counter that the
    last block resets): counts equal the plain kernel's on the full cube, on
    an aligned sub-cube, over direct / captured / replayed calls, for one body
    per module up to 512, and f + ~f fills the cube."""
    for cfg in ("c4", "c5"):
        text, n, _ = W.config(cfg)
        full = bfa.Program(text).count(n)
        for sp, qb in ((64, 1), (256, 16), (1024, 512)):
            p = bfa.Program(text).set_option("split_pieces", sp).set_option("queue_bodies", qb)
            out = torch.zeros(1, dtype=torch.int64, device="cuda")
            for _ in range(4):                   # direct, graph capture, replays
                p.count_range(n, 0, 1 << n, out=out)
                assert int(out.item()) == full, (cfg, sp, qb)
            ll = bfa.last_launch()
            q = ll["queue"]
            assert ll["variant"] == "decomposed" and q["bodies"] > 0
            assert q["unique"] <= q["bodies"] and q["modules"] >= -(-q["bodies"] // qb)
            assert p.count(n) == full
    text, n, _ = W.config("c5")
    body, out = "\n".join(text.splitlines()[:-1]), text.splitlines()[-1]
    lo = 5 << 32
    ref = int(bfa.Program(text).count_range(n, lo, lo + (1 << 32)).item())
    p = bfa.Program(text).set_option("split_pieces", 512).set_option("queue_bodies", 64)
    pc = bfa.Program(f"{body}\n~{out}").set_option("split_pieces", 512).set_option("queue_bodies", 64)
    a = int(p.count_range(n, lo, lo + (1 << 32)).item())
    assert a == ref
    assert a + int(pc.count_range(n, lo, lo + (1 << 32)).item()) == 1 << 32
    full = bfa.Program(text).count(n)
    for sup in (0, 1):                   # support reduction: counts scaled by 2^(dropped variables)
        p = bfa.Program(text).set_option("split_pieces", 1024).set_option("queue_bodies", 64)
        p.set_option("queue_support", sup)
        assert p.count(n) == full
        assert (bfa.last_launch()["queue"]["support_reduced"] > 0) == bool(sup)
    p = bfa.Program(text).set_option("split_pieces", 256).set_option("queue_bodies", 32)
    for world in (2, 4):
        shares = [int(p.count_shard(n, r, world).item()) for r in range(world)]
        assert sum(shares) == full


def test_graph_replay():
    """Multi-launch counts replay as CUDA graphs from the third call on:
    results and the launch counter stay exact across direct, captured and
    replayed calls and across option changes."""
    text, n, expect = W.config("c4")
    p = bfa.Program(text).set_option("split_pieces", 8).set_option("kernel_cofactor_bits", 2)
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    counters = []
    for _ in range(5):
        p.count_range(n, 0, 1 << n, out=out)
        torch.cuda.synchronize()
        assert int(out.item()) == expect
        counters.append(bfa.last_launch()["launch_counter"])
    steps = [b - a for a, b in zip(counters, counters[1:])]
    assert len(set(steps)) == 1 and steps[0] > 0
    p.set_option("kernel_cofactor_bits", 3)
    for _ in range(3):
        p.count_range(n, 0, 1 << n, out=out)
        assert int(out.item()) == expect


def test_count_shard_sums_to_count():
    """Work-balanced cofactor sharding (bfa_count_shard): the ranks' shares,
    computed here one after another in one process, sum to the closed form
    A001035(6) = 130023 on C4, and on C5 the shares of f and of ~f sum to
    2^42 (P-11) for P = 2, 4, 8; the LPT loads are balanced."""
    text, n, expect = W.config("c4")
    p = bfa.Program(text)
    for world in (2, 4, 8):
        out = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(world)]
        for rep in range(3):          # direct, graph capture, graph replay
            shares = [int(p.count_shard(n, r, world, out=out[r]).item()) for r in range(world)]
            assert sum(shares) == expect, (world, rep, shares)
        load = bfa.last_launch()["load"]
        assert len(load) == world and max(load) <= 1.6 * sum(load) / world, (world, load)
    text, n, _ = W.config("c5")
    body, outl = "\n".join(text.splitlines()[:-1]), text.splitlines()[-1]
    p, pc = bfa.Program(text), bfa.Program(f"{body}\n~{outl}")
    for world in (2, 4, 8):
        a = sum(int(p.count_shard(n, r, world).item()) for r in range(world))
        b = sum(int(pc.count_shard(n, r, world).item()) for r in range(world))
        assert a + b == 1 << n, world


def test_decomposed_body_options_vs_oracle():
    """Work-queue body variants (more slot bits, one inner bit, the light
    tail's smaller bodies, ptxas -O1) on a 2^24 C5 sub-cube vs the oracle."""
    text, n, _ = W.config("c5")
    base = bfa.Program(text)
    rng = np.random.default_rng(99)
    while True:
        lo = int(rng.integers(0, 1 << (n - 24))) << 24
        q, _, _ = base.assume(n, {v: (lo >> v) & 1 for v in range(24, n)})
        if q.info["const_value"] == -1 and q.info["gates"] >= 150:
            break
    expect = oracle.count(text, n, lo, lo + (1 << 24))
    for extra in ({"queue_slot_bits": 6, "queue_inner": 1},
                  {"queue_slot_bits": 5, "queue_light_pct": 40, "queue_opt_level": 1}):
        p = presets.apply(bfa.Program(text), presets.DECOMPOSED, split_pieces=64, decompose_min_k=24,
                          split_min_vars=19, **extra)
        assert int(p.count_range(n, lo, lo + (1 << 24)).item()) == expect, extra
        assert bfa.last_launch()["queue"]["bodies"] > 1


def test_decomposed_large_modules_vs_oracle():
    """Work-queue modules of up to 512 bodies each (the bench preset's module
    size) on an oracle-checkable sub-cube: a 2^26 C5 sub-cube decomposed into
    leaves of >= 15 variables, bodies of 32 threads, counted against the
    oracle over direct / captured / replayed calls."""
    text, n, _ = W.config("c5")
    base = bfa.Program(text)
    rng = np.random.default_rng(7)
    while True:
        lo = int(rng.integers(0, 1 << (n - 26))) << 26
        q, _, _ = base.assume(n, {v: (lo >> v) & 1 for v in range(26, n)})
        if q.info["const_value"] == -1 and q.info["gates"] >= 300:
            break
    p = presets.apply(bfa.Program(text), presets.DECOMPOSED, thread_bits=5, split_pieces=2048, split_min_vars=15,
                      decompose_min_k=24, queue_inner=0, queue_slot_bits=5)
    expect = oracle.count(text, n, lo, lo + (1 << 26))
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(4):
        p.count_range(n, lo, lo + (1 << 26), out=out)
        assert int(out.item()) == expect
    q = bfa.last_launch()["queue"]
    assert q["bodies"] >= 512 and q["modules"] <= -(-q["bodies"] // 16), q


def test_decomposed_bench_preset_full_cube():
    """The bench's replay configuration itself (presets.DECOMPOSED: 16384
    Shannon leaves with slot-7 bodies in work-queue modules of <= 256 bodies) over the whole C5
    cube equals the oracle-checked exhaustive kernel's count, replay after
    replay, and f + ~f covers the cube on the exhaustive side (P-11)."""
    text, n, _ = W.config("c5")
    ref = presets.apply(bfa.Program(text), presets.EXHAUSTIVE).count(n)
    p = presets.apply(bfa.Program(text), presets.DECOMPOSED)
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(5):
        p.count_range(n, 0, 1 << n, out=out)
        assert int(out.item()) == ref
    assert bfa.last_launch()["queue"]["bodies"] == presets.DECOMPOSED["split_pieces"]


def test_concurrent_counts_on_two_streams():
    """One prepared decomposed C5 program counted on two streams at once
    (work-queue chunk counters are per caller stream and zeroed by every
    call): every result is exact, over direct, captured and replayed calls."""
    text, n, _ = W.config("c5")
    p = presets.apply(bfa.Program(text), presets.DECOMPOSED, split_pieces=1024, queue_bodies=64)
    ref = torch.zeros(1, dtype=torch.int64, device="cuda")
    p.count_range(n, 0, 1 << n, out=ref)
    expect = int(ref.item())
    assert expect == presets.apply(bfa.Program(text), presets.EXHAUSTIVE).count(n)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    o1 = torch.zeros(4, dtype=torch.int64, device="cuda")
    o2 = torch.zeros(4, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    for i in range(4):
        p.count_range(n, 0, 1 << n, out=o1[i:i + 1], stream=s1)
        p.count_range(n, 0, 1 << n, out=o2[i:i + 1], stream=s2)
    torch.cuda.synchronize()
    assert o1.tolist() == [expect] * 4 and o2.tolist() == [expect] * 4


def test_queue_options_change_rebuilds():
    """Changing a launch option after a work-queue count rebuilds the
    modules (the queue key covers every option): thread_bits 8 -> 7 keeps
    the count exact."""
    text, n, expect = W.config("c4")
    p = bfa.Program(text).set_option("split_pieces", 256).set_option("queue_bodies", 32)
    assert p.count(n) == expect
    p.set_option("thread_bits", 7)
    assert p.count(n) == expect
    assert p.count(n) == expect


def test_autotune_keeps_results():
    """bfa_autotune only changes speed: C4 still counts 130023 and a
    sub-cube vector still equals the oracle's after tuning."""
    text, n, expect = W.config("c4")
    p = bfa.Program(text).set_option("tune_counts", 100000)   # many counts: every stage is worth trying
    rep = p.autotune(n)
    assert rep["best"] and len(rep["candidates"]) >= 6
    assert all("skipped" not in x for x in rep["plans"][:2])
    assert p.count(n) == expect
    lo = (1 << 36) - (1 << 22)
    ow, oc = oracle.evaluate(text, n, lo, 1 << 36)
    assert np.array_equal(host(p.eval_range(n, lo, 1 << 36)), ow)


def test_autotune_total_cost_objective():
    """bfa_autotune minimises preparation + tune_counts x count time: for ONE
    count of C5 the plan with minutes of preparation is never chosen (its
    predicted preparation alone exceeds the best total), and the choice is
    the plan of least total among those tried."""
    text, n, _ = W.config("c5")
    p = presets.apply(bfa.Program(text), presets.EXHAUSTIVE, tune_counts=1)
    rep = p.autotune(n)
    tried = [x for x in rep["plans"] if "skipped" not in x]
    assert tried and rep["best"]["total_s"] == min(x["total_s"] for x in tried)
    assert any("skipped" in x and x["split_pieces"] == 32768 for x in rep["plans"])
    assert rep["best"]["total_s"] < 10
    assert p.count(n) == presets.apply(bfa.Program(text), presets.EXHAUSTIVE).count(n)


# ------------------------------------------------------------ NEXT-4
def test_batch_counts(golden):
    """Batched counting: many programs in one launch give the same counts as
    the closed forms, the oracle, and one launch per program."""
    progs, ns, expect = [], [], []
    cf = golden("closed_forms.json")
    for fam in ("posets", "equivalences", "linear_orders"):
        for k, c in zip(cf[fam]["k"], cf[fam]["count"]):
            if k <= 5:
                progs.append(bfa.Program(getattr(W, fam)(k))); ns.append(k * k); expect.append(c)
    for seed in range(60):
        rp = W.random_program(seed, max_n=20)
        progs.append(bfa.Program(rp.text)); ns.append(rp.n); expect.append(oracle.count(rp.text, rp.n))
    b = bfa.Batch(progs)
    got = b.count(ns).cpu().tolist()
    assert got == expect
    assert bfa.last_launch()["kernels"] == 1


def test_batch_cofactors_of_c4():
    """The 64 cofactors of C4 over its top 6 letters (bfa_assume), counted
    as one batch, sum to 130023 and each equals the count of its sub-cube."""
    text, n, expect = W.config("c4")
    p = bfa.Program(text)
    cof = []
    for r in range(64):
        a = {30 + b: (r >> b) & 1 for b in range(6)}
        q, nf, _ = p.assume(n, a)
        cof.append(q)
    got = bfa.Batch(cof).count([30] * 64).cpu().tolist()
    assert sum(got) == expect
    for r in (0, 37, 63):
        assert got[r] == int(p.count_range(n, r << 30, (r + 1) << 30).item())


# ------------------------------------------------------------ NEXT-3
def test_paper_scale_term_segmented():
    """SURVEY §8(f) NEXT-3, the paper's timed experiment shape (PAPER.md:
    374-380): a 30-variable term with 2^17 tree nodes runs as segmented
    kernels.  Oracle sub-cube counts and vectors agree; count(f) + count(~f)
    = 2^30 over the full cube."""
    text, n, _ = W.config("paper_2p17")
    p = bfa.Program(text)
    c = p.count(n)
    ll = bfa.last_launch()
    assert ll["variant"] == "segmented" and ll["segments"] > 8
    body, out = "\n".join(text.splitlines()[:-1]), text.splitlines()[-1]
    assert c + bfa.Program(f"{body}\n~{out}").count(n) == 1 << n
    lo = 3 << 24
    ow, oc = oracle.evaluate(text, n, lo, lo + (1 << 14))
    assert int(p.count_range(n, lo, lo + (1 << 14)).item()) == oc
    assert np.array_equal(host(p.eval_range(n, lo, lo + (1 << 14))), ow)


# ------------------------------------------------------------ NEXT-1 / NEXT-2
def test_bounded_posets_n8_paper():
    """PAPER.md:1193-1204 (§5.2): bounded posets on 8 points; killing 34
    letters (Eq. conspa) leaves v = 30, whose models are the partial orders
    of the 6 middle elements: |K| = A001035(6) = 130023, and
    l_{T,8} = 8 * 7 * |K| = 7,281,288.  Enumerated models, reinstated,
    satisfy the unreduced theory (checked by the oracle for k = 7)."""
    k = 8
    a = W.bounded_poset_kills(k)
    q, nf, ids = bfa.Program(W.posets(k)).assume(64, a)
    assert nf == 30
    c = q.count(nf)
    assert c == 130023 and k * (k - 1) * c == 7281288
    mus, total = q.enumerate(nf, capacity=1 << 18)
    assert total == 130023 and len(mus) == total
    m = mus.cpu().numpy()
    assert (np.diff(m) > 0).all()
    k = 7
    text = W.posets(k)
    a = W.bounded_poset_kills(k)
    q, nf, ids = bfa.Program(text).assume(49, a)
    mus, total = q.enumerate(nf, capacity=1 << 16)
    assert total == 4231                       # A001035(5)
    full = bfa.reinstate(mus.cpu().numpy()[::97], ids, a)
    for mu in full:
        assert oracle.count(text, 49, mu, mu + 1) == 1


def test_special_posets_assumptions():
    """SO.txt with assumptions p(i,i) = 1: k = 5 gives
    the closed form 1840 (SURVEY P-9) on 20 free letters; k = 6 is the paper's
    run with 30 unknowns, checked against the oracle on
    the reduced program's text."""
    import re
    for k, expect in ((5, 1840), (6, None)):
        text = W.special_posets(k)
        a = {W.letter_id(k, i, i): 1 for i in range(k)}
        q, nf, ids = bfa.Program(text).assume(k * k, a)
        assert nf == k * k - k
        c = q.count(nf)
        if expect is not None:
            assert c == expect
        else:
            # the reduced program as text (test-side substitution + renumbering)
            new = {old: i for i, old in enumerate(ids)}
            red = re.sub(r"\bx(\d+)\b", lambda mm: str(a[int(mm.group(1))]) if int(mm.group(1)) in a
                         else f"x{new[int(mm.group(1))]}", text)
            assert c == oracle.count(red, nf)


def test_rows_out_txt(golden):
    """out.txt rows: one row per model, one character per
    letter with id n-1 (the paper's b_1) first, so a row read as a binary
    number is its valuation mu.  C1 rows equal the golden model list; for
    bounded posets on 7 points the rows of the killed program (34 letters
    fixed) carry the killed letters reinstated and each
    row satisfies the unreduced theory (oracle)."""
    g = golden("c1_posets3.json")
    mus, total = bfa.Program(W.posets(3)).enumerate(9)
    lines = bfa.rows(mus, 9).decode().split("\n")
    assert lines[-1] == "" and all(len(x) == 9 for x in lines[:-1])
    assert [int(x, 2) for x in lines[:-1]] == g["set_bits"]
    k = 7
    text = W.posets(k)
    a = W.bounded_poset_kills(k)
    q, nf, ids = bfa.Program(text).assume(k * k, a)
    mus, total = q.enumerate(nf, capacity=1 << 16)
    assert total == 4231
    lines = bfa.rows(mus, k * k, ids, a).decode().splitlines()
    assert len(lines) == 4231
    want = bfa.reinstate(mus.cpu().numpy(), ids, a)
    assert [int(x, 2) for x in lines] == want
    for x in lines[::211]:
        mu = int(x, 2)
        assert oracle.count(text, k * k, mu, mu + 1) == 1


def test_enumerate_matches_oracle(golden):
    g = golden("c1_posets3.json")
    mus, total = bfa.Program(W.posets(3)).enumerate(9)
    assert total == 19 and mus.cpu().tolist() == g["set_bits"]
    mus, total = bfa.Program(W.BAEQU).enumerate(4)
    assert mus.cpu().tolist() == [0, 9, 15]
    text, n, _ = W.config("c3_posets")
    ow, oc = oracle.evaluate(text, n)
    mus, total = bfa.Program(text).enumerate(n, capacity=8192)
    assert total == oc == 4231 and np.array_equal(mus.cpu().numpy(), oracle.set_bits(ow))
    for seed in (7, 17, 27, 37):
        p = W.random_program(seed, max_n=20)
        ow, oc = oracle.evaluate(p.text, p.n)
        mus, total = bfa.Program(p.text).enumerate(p.n, capacity=1 << 21)
        assert total == oc and np.array_equal(mus.cpu().numpy(), oracle.set_bits(ow))
    # a sub-range of C4 and a too-small capacity (count still exact)
    text, n, _ = W.config("c4")
    refl = sum(1 << (35 - 7 * i) for i in range(6))
    lo = refl & ~((1 << 24) - 1)
    ow, oc = oracle.evaluate(text, n, lo, lo + (1 << 24))
    mus, total = bfa.Program(text).enumerate(n, lo, lo + (1 << 24), capacity=1 << 16)
    assert total == oc and np.array_equal(mus.cpu().numpy(), oracle.set_bits(ow, lo))
    first, total = bfa.Program(text).enumerate(n, capacity=4)
    assert total == 130023
    ow, _ = oracle.evaluate(text, n, (1 << 36) - (1 << 30), 1 << 36)   # the models are in mu order:
    top = oracle.set_bits(ow, (1 << 36) - (1 << 30))                 # the first four are the smallest
    allm, _ = bfa.Program(text).enumerate(n, capacity=1 << 18)
    assert len(allm) == 130023 and (np.diff(allm.cpu().numpy()) > 0).all()
    assert first.cpu().tolist() == allm[:4].cpu().tolist()
    assert np.array_equal(allm.cpu().numpy()[-len(top):], top)


# ------------------------------------------------------------ materialised mode
def test_fill_generators_and_popcount():
    n = 12
    tab = host(bfa.fill_generators(n)).reshape(n, -1)
    for v in range(n):
        ow, _ = oracle.evaluate(f"x{v}", n)
        assert np.array_equal(tab[v], ow)
    x = torch.randint(-(1 << 62), 1 << 62, (1001,), dtype=torch.int64, device="cuda")
    ref = int(np.unpackbits(x.cpu().numpy().view(np.uint8)).sum())
    assert int(bfa.popcount(x).item()) == ref


@pytest.mark.parametrize("variant", [0, 1])
def test_materialised_modes(variant):
    for text, n in ((W.cnf3(14, 30, seed=3), 14), (W.posets(4), 16), (W.random_dag(12, 150, seed=8), 12),
                    ("x3", 9), ("~x3", 9), ("x0 & ~x0", 9)):
        p = bfa.Program(text)
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        gw = host(p.eval_materialised(n, variant, count_out=cnt))
        ow, oc = oracle.evaluate(text, n)
        assert np.array_equal(gw, ow), (text[:80], variant)
        assert int(cnt.item()) == oc


def test_c2_materialised():
    """Config C2 (3-CNF, n=28): m=2000 gives 0 models; the m=100 variant's
    full 2^28-bit vector equals the oracle's, in both materialised variants."""
    text, n, expect = W.config("c2")
    p = bfa.Program(text)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for variant in (0, 1):
        p.eval_materialised(n, variant, count_out=cnt)
        assert int(cnt.item()) == expect == 0
    text, n, _ = W.config("c2_m100")
    ow, oc = oracle.evaluate(text, n)
    p = bfa.Program(text)
    for variant in (0, 1):
        gw = host(p.eval_materialised(n, variant, count_out=cnt))
        assert np.array_equal(gw, ow) and int(cnt.item()) == oc
    assert p.count(n) == oc


def test_programs_release_device_memory():
    """Freeing a program unloads its JIT modules: compiling, running and
    dropping many programs does not drift the device's free memory."""
    import gc

    def churn(k):
        for s in range(k):
            p = bfa.Program(W.random_dag(14, 60, seed=1000 + s))
            p.set_option("graphs", 0)
            p.count(14)
            del p
        gc.collect()
        torch.cuda.synchronize()

    churn(20)                                   # warm the allocators
    free0 = torch.cuda.mem_get_info()[0]
    churn(200)
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < 64 << 20, (free0 - free1) >> 20


def test_bench_multi_rank_functional():
    """The bench's N > 1 path end to end on the one GPU this pool gives:
    torchrun with 2 ranks sharing cuda:0 over gloo (a functional run, not a
    scaling measurement): rank-0-first preparation, per-rank cofactor ranges
    with the same kernel, the count all-reduce, max-over-ranks timing and the
    cold e2e -- the reported count is the closed form."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--e2e-steps", "1", "--no-extras", "--no-cpu-baseline", "--config", "c4",
           "--backend", "gloo", "--share-device"]
    p = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [x for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["count"] == 130023 and d["value"] > 0 and d["e2e"]["value"] > 0
