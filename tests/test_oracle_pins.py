"""Pins for the CPU oracle (oracle/bfa_oracle.c), independent of the oracle.

Each test checks the oracle against something the paper or mathematics
fixes: printed worked examples, closed forms
(OEIS A001035, Bell, k!, l = n(n-1)|K|), a second brute force that uses
Python's own parser over numpy bool arrays (Python-AE is
Python), hand-written truth tables for the grammar's precedence and
associativity, and Boolean-algebra invariants (complement, Shannon expansion,
a fresh XOR variable).  A plausible oracle bug -- a dropped term, a wrong
sign/index, a transposed operand, a wrong precedence -- fails one of these.
"""
import hashlib

import numpy as np
import pytest

import oracle
import workloads as W


def bitstring(words, nbits):
    return "".join(str(int(b)) for b in
                   np.unpackbits(np.asarray(words, "<u8").view(np.uint8), bitorder="little")[:nbits])


# ---------------------------------------------------------------- paper
def test_free_generators_n3(golden):
    """b1=00001111, b2=00110011, b3=01010101 (C-1)."""
    g = golden("generators_n3.json")
    for var, bits in g["vectors"].items():
        words, c = oracle.evaluate(var, 3)
        assert bitstring(words, 8) == bits
        assert c == 4


def test_free_generators_independent():
    """§2.2 / SPEC.md:170-178: every signed meet of the generators is nonzero
    (exactly one valuation), for n <= 4."""
    import itertools
    for n in range(1, 5):
        for signs in itertools.product([0, 1], repeat=n):
            expr = " & ".join(("" if s else "~") + f"x{v}" for v, s in enumerate(signs))
            words, c = oracle.evaluate(expr, n)
            assert c == 1
            mu = int(oracle.set_bits(words)[0])
            assert mu == sum(s << v for v, s in enumerate(signs))


def test_spec_examples():
    """SPEC.md:149-151, 158-159 rewritten in ids (paper x1 = MSB = id v-1)."""
    assert bitstring(oracle.evaluate("x1 & ~x0", 2)[0], 4) == "0010"
    w, _ = oracle.evaluate("x2", 3, 4, 8)          # chunk 1 of k=2 blocks
    assert bitstring(w, 4) == "1111"
    w, c = oracle.evaluate("x1 | x0", 2)
    assert bitstring(w, 4) == "0111" and c == 3
    w, c = oracle.evaluate("x0 & ~x0", 1)
    assert bitstring(w, 2) == "00" and c == 0


def test_baequ(golden):
    """PAPER.md:1154-1165 (§5.1): solutions xyzu in {0000, 1001, 1111}."""
    g = golden("baequ.json")
    assert g["program"] == W.BAEQU
    words, c = oracle.evaluate(g["program"], 4)
    assert c == 3
    assert oracle.set_bits(words).tolist() == g["mu"]
    assert int(words[0]) == int(g["word0"], 16)


def test_c1_posets3_vector(golden):
    """Config C1: exact vector (SURVEY P-4) and count 19 = A001035(3)."""
    g = golden("c1_posets3.json")
    words, c = oracle.evaluate(W.posets(3), 9)
    assert c == g["count"] == 19
    assert oracle.set_bits(words).tolist() == g["set_bits"]
    assert [int(x) for x in words] == [int(x, 16) for x in g["words_u64"]]
    assert hashlib.sha256(np.asarray(words, "<u8").tobytes()).hexdigest() == g["sha256_packed_le"]


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("family,gen", [("posets", W.posets), ("equivalences", W.equivalences),
                                        ("linear_orders", W.linear_orders),
                                        ("bounded_posets", W.bounded_posets),
                                        ("special_posets", W.special_posets)])
def test_closed_forms(golden, family, gen):
    g = golden("closed_forms.json")[family]
    for k, expect in zip(g["k"], g["count"]):
        if k > 5:
            continue          # k=6 (n=36) is checked on the GPU box (test_gpu_configs)
        assert oracle.count(gen(k), k * k) == expect, (family, k)


def test_relation_families_vs_numpy():
    """Second brute force: the same relation programs evaluated by Python's
    parser on numpy arrays (their text only uses ~ & ^ |, which Python reads
    with the same precedence -- PAPER.md:1043-1046)."""
    for gen in (W.posets, W.equivalences, W.linear_orders, W.special_posets, W.bounded_posets):
        for k in (2, 3, 4):
            text = gen(k)
            lines = [ln for ln in text.splitlines() if ln.strip()]
            tt = oracle.numpy_truth_table(k * k, [], lines)
            words, c = oracle.evaluate(text, k * k)
            assert c == int(tt.sum())
            assert np.array_equal(words, oracle.pack_bool(tt))


# ---------------------------------------------------------------- grammar
def tt_bits(n, fn):
    return "".join(str(int(bool(fn(*[(mu >> v) & 1 for v in range(n)])))) for mu in range(1 << n))


HAND = [
    # (expr, n, expected truth table mu = 0..2^n-1), written by hand
    ("x0 | x1 & x2", 3, "01010111"),        # & binds tighter than |  (x v yz)
    ("(x0 | x1) & x2", 3, "00000111"),
    ("x0 ^ x1 & x2", 3, "01010110"),        # & tighter than ^
    ("x0 | x1 ^ x2", 3, "01111101"),        # ^ tighter than |
    ("x0 -> x1 -> x2", 3, "11101111"),      # right-assoc: x0 -> (x1 -> x2)
    ("(x0 -> x1) -> x2", 3, "01001111"),
    ("x0 | x1 -> x2", 3, "10001111"),       # | tighter than ->
    ("x0 <-> x1 -> x2", 3, "01100101"),     # -> tighter than <->  : x0 <-> (x1 -> x2)
    ("~x0 & x1", 2, "0010"),                # ~ binds tightest
    ("~(x0 & x1)", 2, "1110"),
    ("x0 ^ x1", 2, "0110"),                 # x+y = x~y v ~xy
    ("x0 <-> x1", 2, "1001"),
    ("x0 -> x1", 2, "1011"),
    ("1", 2, "1111"),
    ("0 | x1", 2, "0011"),
    ("", 2, "1111"),                        # no constraints: constant 1
    ("x0; x1", 2, "0001"),                  # constraints are conjoined
    ("let a = x0 ^ x1\na & ~x1", 2, "0100"),
    ("e1 = x0 | x1\ne1 -> x0", 2, "0101"),  # named constraint is also a binding
]


@pytest.mark.parametrize("expr,n,bits", HAND)
def test_grammar_hand_tables(expr, n, bits):
    assert bitstring(oracle.evaluate(expr, n)[0], 1 << n) == bits


def test_hand_tables_are_what_they_say():
    """The hand tables above agree with Python lambdas of the intended
    parse (guards against typos in the hand tables themselves)."""
    assert tt_bits(3, lambda a, b, c: a | (b & c)) == HAND[0][2]
    assert tt_bits(3, lambda a, b, c: (not a) or ((not b) or c)) == HAND[4][2]
    assert tt_bits(3, lambda a, b, c: (not ((not a) or b)) or c) == HAND[5][2]
    assert tt_bits(3, lambda a, b, c: (not (a or b)) or c) == HAND[6][2]
    assert tt_bits(3, lambda a, b, c: a == ((not b) or c)) == HAND[7][2]


@pytest.mark.parametrize("bad", ["x0 &", "(x0", "x0 x1", "2", "x64", "y", "let a = x0\nlet a = x1",
                                 "x0 $ x1", "let = x0", "a = x0\na = x1"])
def test_parse_errors(bad):
    with pytest.raises(oracle.OracleError) as e:
        oracle.evaluate(bad, 5)
    assert e.value.code == -1


def test_range_errors():
    with pytest.raises(oracle.OracleError) as e:
        oracle.evaluate("x5", 5)
    assert e.value.code == -3
    with pytest.raises(oracle.OracleError):
        oracle.evaluate("x0", 64)


# ---------------------------------------------------------------- random terms
@pytest.mark.parametrize("block", range(4))
def test_random_terms_vs_numpy(block):
    """SPEC acceptance 1: 200 random terms, n <= 12, every bit
    of the oracle equals Python's evaluation of an independently rendered,
    fully parenthesised expression."""
    for seed in range(block * 50, block * 50 + 50):
        p = W.random_program(seed, max_n=12)
        tt = oracle.numpy_truth_table(p.n, p.py_lets, p.py_constraints)
        words, c = oracle.evaluate(p.text, p.n)
        assert c == int(tt.sum()), (seed, p.text)
        assert np.array_equal(words, oracle.pack_bool(tt)), (seed, p.text)


def test_random_cnf_vs_numpy():
    for seed in range(10):
        text = W.cnf3(12, 40, seed)
        lines = [ln for ln in text.splitlines() if ln.strip()]
        tt = oracle.numpy_truth_table(12, [], lines)
        words, c = oracle.evaluate(text, 12)
        assert c == int(tt.sum())
        assert np.array_equal(words, oracle.pack_bool(tt))


# ---------------------------------------------------------------- invariants
def test_invariants_random():
    """count(f)+count(~f) = 2^n; count(f ^ x_fresh) = 2^(n-1);
    Shannon: count(f) = count(f & xv) + count(f & ~xv)."""
    for seed in range(1, 60):
        p = W.random_program(seed, max_n=14)
        if p.n < 2 or p.py_lets:
            continue
        body = " & ".join(f"({ln})" for ln in p.text.splitlines() if ln.strip())
        n = p.n
        c = oracle.count(body, n)
        assert c + oracle.count(f"~({body})", n) == 1 << n
        assert oracle.count(f"({body}) ^ x{n}", n + 1) == 1 << n
        v = seed % n
        assert oracle.count(f"({body}) & x{v}", n) + oracle.count(f"({body}) & ~x{v}", n) == c


def test_range_additivity_and_threads():
    text = W.random_dag(16, 200, seed=3)
    full_w, full_c = oracle.evaluate(text, 16, threads=1)
    parts = [oracle.evaluate(text, 16, r << 12, (r + 1) << 12, threads=3) for r in range(16)]
    assert sum(c for _, c in parts) == full_c
    assert np.array_equal(np.concatenate([w for w, _ in parts]), full_w)
    w8, c8 = oracle.evaluate(text, 16, threads=8)
    assert c8 == full_c and np.array_equal(w8, full_w)


def test_tautology_contradiction():
    for n in (1, 5, 7, 12):
        assert oracle.count(f"x0 | ~x0", n) == 1 << n
        assert oracle.count(f"x0 & ~x0", n) == 0


def test_small_n_padding():
    """n < 6: the vector occupies the low 2^n bits of word 0; padding is 0."""
    for n in range(0, 6):
        w, c = oracle.evaluate("1", n)
        assert c == 1 << n and int(w[0]) == (1 << (1 << n)) - 1


def test_c2_cnf_zero_models():
    """SURVEY P-10: 2000 random 3-clauses on 28 vars: E[#models] = 2^28 (7/8)^2000
    ~ 1e-108, and the oracle finds 0 (short-circuit makes this cheap)."""
    text, n, expect = W.config("c2")
    assert oracle.count(text, n) == expect == 0


def test_c5_density():
    """The C5 random DAG seed has sampled density within [0.01, 0.99] on 2^20
    valuations (SURVEY.md §8(d) C5 reseed rule)."""
    text, n, _ = W.config("c5")
    c = oracle.count(text, n, 0, 1 << 20)
    assert 0.01 < c / (1 << 20) < 0.99
