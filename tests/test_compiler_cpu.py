"""CPU tests of the product's host side: the C ABI loads and exports every
symbol include/bfa.h declares, the compiler's LUT3 cover is sound (its IR,
interpreted here with numpy, equals the oracle's truth table), the generated
kernels compile for sm_100a through NVRTC, and compute calls fail loudly
without a GPU (no CPU fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import paper_1310_6978_b200 as bfa
import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "bfa.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bfa_[a-z_0-9]+)\s*\(", text)))


def test_abi_exports_every_declared_symbol():
    import ctypes
    names = header_functions()
    assert "bfa_compile" in names and "bfa_count" in names and "bfa_eval" in names
    lib = ctypes.CDLL(bfa.lib_path())
    for name in names:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", bfa.lib_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (bfa_\w+)", out))
    assert set(names) <= exported
    # nothing but the C ABI is exported
    assert all(s.startswith("bfa_") for s in re.findall(r" T (\S+)", out)), out


# ----------------------------------------------------------- IR interpreter
PAT = None


def eval_ir(ir: str, n: int) -> np.ndarray:
    """Interpret the LUT3 IR (bfa_dump what=0) over all 2^n valuations with
    numpy bool arrays: lop3(a,b,c,imm) bit = imm[4a+2b+c] (PTX immLut)."""
    mu = np.arange(1 << n, dtype=np.uint64)
    vals = {}

    def operand(tok):
        tok = tok.strip()
        if tok.startswith("x"):
            return ((mu >> np.uint64(int(tok[1:]))) & np.uint64(1)).astype(bool)
        if tok.startswith("L"):
            return vals[tok]
        w = int(tok, 16)
        return np.full(1 << n, bool(w & 1))   # only 0/~0 constants can reach the IR
    out = None
    for line in ir.strip().splitlines():
        lhs, rhs = [s.strip() for s in line.split("=", 1)]
        if lhs == "out":
            neg = rhs.startswith("~")
            v = operand(rhs.lstrip("~"))
            out = ~v if neg else v
            continue
        m = re.match(r"lop3\((.*), (.*), (.*), (0x[0-9a-f]+)\)", rhs)
        a, b, c = (operand(m.group(k)) for k in (1, 2, 3))
        imm = int(m.group(4), 16)
        idx = (a.astype(np.uint8) << 2) | (b.astype(np.uint8) << 1) | c.astype(np.uint8)
        vals[lhs] = ((imm >> idx) & 1).astype(bool)
    return out


@pytest.mark.parametrize("block", range(4))
def test_lut_cover_matches_oracle_random(block):
    for seed in range(block * 50, block * 50 + 50):
        p = W.random_program(seed, max_n=12)
        prog = bfa.Program(p.text)
        info = prog.info
        tt = eval_ir(prog.dump(0), p.n)
        words, c = oracle.evaluate(p.text, p.n)
        assert np.array_equal(oracle.pack_bool(tt), words), (seed, p.text)
        if info["const_value"] >= 0:
            assert c in (0, 1 << p.n) and c == info["const_value"] << p.n


def test_lut_cover_matches_oracle_relations():
    for gen, k in ((W.posets, 3), (W.posets, 4), (W.equivalences, 4), (W.linear_orders, 3),
                   (W.bounded_posets, 4), (W.special_posets, 4)):
        text = gen(k)
        prog = bfa.Program(text)
        tt = eval_ir(prog.dump(0), k * k)
        words, _ = oracle.evaluate(text, k * k)
        assert np.array_equal(oracle.pack_bool(tt), words)
    text = W.random_dag(14, 300, seed=5)
    tt = eval_ir(bfa.Program(text).dump(0), 14)
    assert np.array_equal(oracle.pack_bool(tt), oracle.evaluate(text, 14)[0])


def test_reduction_and_info():
    """Reduction: constants propagate to 0/1."""
    assert bfa.Program("x0 & ~x0").info["const_value"] == 0
    assert bfa.Program("x3 | ~x3").info["const_value"] == 1
    assert bfa.Program("(x1 -> 1) & (0 | 1)").info["const_value"] == 1
    assert bfa.Program("").info["const_value"] == 1
    i = bfa.Program("x0 & x1 | x2").info
    assert i["const_value"] == -1 and i["gates"] == 2 and i["luts"] == 1 and i["support"] == 3
    assert i["tree_nodes"] == 5 and i["max_var_id"] == 2
    # hash-consing: the two antisymmetry clauses (i,j),(j,i) are one gate
    i = bfa.Program("~x1 | ~x2\n~x2 | ~x1").info
    assert i["gates"] == 1
    c4 = bfa.Program(W.posets(6)).info
    assert c4["support"] == 36 and c4["luts"] <= c4["gates"]


@pytest.mark.parametrize("bad", ["x0 &", "(x0", "x0 x1", "2", "x64", "y", "let a = x0\nlet a = x1",
                                 "x0 $ x1", "let = x0", "a = x0\na = x1"])
def test_parse_errors_agree_with_oracle(bad):
    with pytest.raises(bfa.BfaError) as e:
        bfa.Program(bad)
    assert e.value.code == bfa.BFA_E_PARSE
    assert re.match(r"bfa error -1: \d+:\d+: ", str(e.value))


def test_generated_kernels_compile_sm100a(tmp_path):
    """Every kernel variant of a few programs JIT-compiles for sm_100a
    (NVRTC needs no GPU); the SASS of the specialised count kernel is LOP3
    code with no local-memory spills."""
    for text in (W.posets(4), W.random_dag(20, 200, seed=1), "x0", "x40 ^ x7"):
        p = bfa.Program(text)
        for what in (1, 2, 3, 4):
            assert len(p.jit_cubin(what)) > 1000
    cub = tmp_path / "k.cubin"
    cub.write_bytes(bfa.Program(W.posets(5)).jit_cubin(1))
    sass = subprocess.run(["cuobjdump", "-sass", str(cub)], capture_output=True, text=True).stdout
    assert "LOP3" in sass and "STL" not in sass and "LDL" not in sass


def test_options_validation():
    p = bfa.Program("x0")
    with pytest.raises(bfa.BfaError):
        p.set_option("slot_bits", 15)
    with pytest.raises(bfa.BfaError):
        p.set_option("nonsense", 1)
    p.set_option("thread_bits", 7).set_option("inner_bits", 2)


def test_no_cpu_fallback():
    """Without a CUDA device every compute call fails loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = bfa.Program(W.posets(3))
    with pytest.raises(bfa.BfaError) as e:
        p.count(9)
    assert e.value.code == bfa.BFA_E_CUDA


# ----------------------------------------------------------- killing variables
def test_bounded_poset_kill_counts():
    """PAPER.md:1193-1203 (§5.2, Eq. conspa, reading C-13): 5k-6 letters are
    killed, leaving v = k^2 - 5k + 6 (v = 30 at k = 8); the kills never
    assign one letter two values."""
    for k in range(2, 11):
        a = W.bounded_poset_kills(k)
        assert len(a) == 5 * k - 6
        assert k * k - len(a) == k * k - 5 * k + 6
    assert 64 - len(W.bounded_poset_kills(8)) == 30


def test_assume_matches_oracle():
    """bfa_assume = substitute + Reduction + dense renumbering: the reduced
    program's LUT cover, evaluated here over the free letters, equals the
    oracle's models of the original program with the kills as conjuncts
    (each mapped to its free bits)."""
    for gen, k in ((W.posets, 4), (W.posets, 5), (W.equivalences, 4)):
        text = gen(k)
        a = W.bounded_poset_kills(k)
        q, nf, ids = bfa.Program(text).assume(k * k, a)
        assert nf == k * k - len(a) and ids == sorted(set(range(k * k)) - set(a))
        lits = "\n".join(("" if b else "~") + f"x{v}" for v, b in a.items())
        ow, oc = oracle.evaluate(text + lits + "\n", k * k)
        full = oracle.set_bits(ow)
        reduced = sorted(sum(((int(m) >> old) & 1) << new for new, old in enumerate(ids)) for m in full)
        tt = eval_ir(q.dump(0), nf)
        assert [int(x) for x in np.nonzero(tt)[0]] == reduced
        assert q.info["max_var_id"] < nf


def test_assume_to_constant():
    q, nf, ids = bfa.Program("x0 & x5 | x3").assume(6, {0: 1, 5: 1})
    assert q.info["const_value"] == 1 and nf == 4 and ids == [1, 2, 3, 4]
    q, nf, _ = bfa.Program("x63 & x1").assume(64, {63: 0})
    assert q.info["const_value"] == 0 and nf == 63


def test_prepare_host_only():
    """bfa_prepare runs every host-side step of a count without a GPU: the
    Shannon decomposition, role searches, emission and NVRTC of the
    work-queue modules (sm_100a) -- and reports them; bad n is rejected."""
    text, n, _ = W.config("c5")
    p = bfa.Program(text).set_option("split_pieces", 48).set_option("queue_bodies", 8)
    p.set_option("slot_bits", 3)
    p.prepare(n, 148)
    ll = bfa.last_launch()
    assert ll["variant"] == "prepare" and ll["pieces"] >= 48
    q = ll["queue"]
    assert 0 < q["unique"] <= q["bodies"] <= 48 and q["modules"] >= -(-q["bodies"] // 8)
    assert q["chunks"] >= q["bodies"]
    p.prepare(n, 148)                     # cached: a second call is free
    with pytest.raises(bfa.BfaError):
        p.prepare(40)                     # the program uses x41
    bfa.Program(W.posets(4)).prepare(16)  # plain kernel path


def test_decomposition_tiles_the_cube():
    """The Shannon decomposition (host only) tiles the 2^n cube for both split
    policies and with the light-sibling merge: sum of 2^vars over the pieces
    is 2^n, the requested number of non-constant pieces is reached (merge
    only removes pieces), and the plan is reproducible."""
    text, n, _ = W.config("c5")
    sizes = {}
    for policy, merge in ((0, 0), (1, 0), (1, 16)):
        p = bfa.Program(text).set_option("split_pieces", 512).set_option("split_policy", policy)
        p.set_option("split_merge", merge)
        plan = p.shard_plan(n, 1)
        assert sum(1 << nv for _, nv, _ in plan) == 1 << n
        live = sum(1 for _, _, w in plan if w)
        sizes[(policy, merge)] = live
        assert plan == bfa.Program(text).set_option("split_pieces", 512).set_option(
            "split_policy", policy).set_option("split_merge", merge).shard_plan(n, 1)
    assert sizes[(0, 0)] >= 512 and sizes[(1, 0)] >= 512
    assert sizes[(1, 16)] <= sizes[(1, 0)]


def test_cache_key_is_sha256():
    """The persistent JIT cache key is SHA-256 over salt, NVRTC version,
    options and source (no 64-bit hash collisions can load a wrong cubin)."""
    import hashlib
    src = bfa.Program(W.posets(3)).dump(3, 9)          # generic kernel: CUDA C++ through NVRTC
    key = bfa.cache_key(src)
    assert re.fullmatch(r"[0-9a-f]{64}", key)
    opts = "--gpu-architecture=sm_100a|-lineinfo|--std=c++17|"
    expect = hashlib.sha256(("bfa-cubin-v2|12.9|" + opts + src).encode()).hexdigest()
    assert key == expect
    assert bfa.cache_key(src + " ") != key
    ptx = bfa.Program(W.posets(3)).dump(1, 9)          # specialised count kernel: generated PTX
    assert ptx.startswith("// generated by libbfa (PTX)")
    expect = hashlib.sha256(("bfa-ptx-v1|12.9|--gpu-name=sm_100a|-O3|" + ptx).encode()).hexdigest()
    assert bfa.cache_key(ptx) == expect


def test_last_error_code():
    """bfa_last_error_code classifies failures (no message parsing)."""
    with pytest.raises(bfa.BfaError) as e:
        bfa.Program("x0 &")
    assert e.value.code == bfa.BFA_E_PARSE == bfa._load().bfa_last_error_code()
    with pytest.raises(bfa.BfaError):
        bfa.Program("x0").set_option("slot_bits", 15)
    assert bfa._load().bfa_last_error_code() == bfa.BFA_E_ARG


def test_roles_are_a_permutation_of_the_free_variables():
    """bfa_roles (host only): the count kernel of an aligned 2^k sub-cube
    enumerates it in a permuted variable order that fixes every variable
    >= k; the same program object reports the same order again."""
    text, n, _ = W.config("c4")
    p = bfa.Program(text).set_option("slot_bits", 5).set_option("imad_cost_pct", 50)
    for k in (36, 30):
        perm = p.roles(n, k, sms=148)
        assert sorted(perm) == list(range(64))
        assert all(perm[v] == v for v in range(k, 64))
        assert p.roles(n, k, sms=148) == perm
    with pytest.raises(bfa.BfaError):
        bfa.Program(text).set_option("force_generic", 1).roles(n, n, sms=148)


def test_role_seed_is_deterministic_and_selects_the_search():
    """Option role_seed: the role search of one seed gives the same
    permutation on every new program object (it is pinned in presets), and
    another seed searches from another start."""
    text, n, _ = W.config("c4")

    def perm(seed):
        p = bfa.Program(text).set_option("slot_bits", 5).set_option("imad_cost_pct", 50)
        p.set_option("jit_cache", 0).set_option("role_budget", 40).set_option("role_seed", seed)
        return p.roles(n, n, sms=148)

    a = perm(3)
    assert sorted(a) == list(range(64))
    assert perm(3) == a
    assert any(perm(s) != a for s in (0, 1, 2))
    with pytest.raises(bfa.BfaError):
        bfa.Program(text).set_option("role_seed", -1)
