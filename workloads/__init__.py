"""Seeded synthetic input generators for the free-Boolean-vector hot path.

This module is shared by the oracle tests, the GPU parity tests and bench.py.
It holds NONE of the method's arithmetic: it only emits expression TEXT in the
grammar of include/bfa.h (and, for the random-term suite, an equivalent
fully-parenthesised Python rendering used by the numpy cross-check in tests).
Nothing here evaluates a Boolean function.

Workload shapes follow the paper's examples (§4.2 SO.txt;
PAPER.md:1141-1165, §5.1 BAequ; §5.2 bounded posets) and
the concrete configs of SURVEY.md §8(d):

  C1  posets k=3      (9 vars)   -> posets(3)
  C2  random 3-CNF    (n=28, m=2000) -> cnf3(28, 2000)
  C3  equivalence k=5 / posets k=5 (25 vars)
  C4  posets k=6      (36 vars)
  C5  random 1000-gate DAG over n=42 -> random_dag(42, 1000)

Letter convention (reading C-3): for a k x k
relation the letter p(i,j) has variable id  k*k - 1 - (i*k + j), so the
canonically-first letter p(0,0) is the most significant bit of the valuation
index mu, as the paper's b_1 is the MSB row of matrix M.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

SEED = 13106978  # one seed everywhere


# --------------------------------------------------------------------------
# relation letters
# --------------------------------------------------------------------------
def letter_id(k: int, i: int, j: int) -> int:
    """Variable id of p(i,j) on a k-element domain (reading C-3)."""
    return k * k - 1 - (i * k + j)


def _p(k: int, i: int, j: int) -> str:
    return f"x{letter_id(k, i, j)}"


def _refl(k):
    return [_p(k, i, i) for i in range(k)]


def _antisym(k):
    # PAPER.md:1024 f1 = A[i,j:S2] (~p(i,j) | ~p(j,i))
    return [f"~{_p(k, i, j)} | ~{_p(k, j, i)}" for i, j in itertools.permutations(range(k), 2)]


def _trans(k):
    # PAPER.md:1026 f2 = A[i,j,k:S3] (~(p(i,j) & p(j,k)) | p(i,k))
    return [f"~({_p(k, i, j)} & {_p(k, j, l)}) | {_p(k, i, l)}"
            for i, j, l in itertools.permutations(range(k), 3)]


def _sym(k):
    return [f"~{_p(k, i, j)} | {_p(k, j, i)}" for i, j in itertools.permutations(range(k), 2)]


def _total(k):
    return [f"{_p(k, i, j)} | {_p(k, j, i)}" for i, j in itertools.permutations(range(k), 2)]


def _program(lines) -> str:
    return "\n".join(lines) + "\n"


def posets(k: int) -> str:
    """Labeled partial orders on k points: refl & antisym(S2) & trans(S3).

    All k*k letters free, reflexivity as a conjunct (reading C-9); expected
    counts 1, 3, 19, 219, 4231, 130023 (OEIS A001035)."""
    return _program(_refl(k) + _antisym(k) + _trans(k))


def equivalences(k: int) -> str:
    """Equivalence relations: refl & sym(S2) & trans(S3); Bell numbers."""
    return _program(_refl(k) + _sym(k) + _trans(k))


def linear_orders(k: int) -> str:
    """Linear orders: posets & totality over S2; k! models."""
    return _program(_refl(k) + _antisym(k) + _trans(k) + _total(k))


def special_posets(k: int) -> str:
    """SO.txt: posets with an element comparable to all.

    f3 = E[i:S].A[j:S] (p(i,j) | p(j,i)); reflexivity as a conjunct (C-9)."""
    f3 = " | ".join(
        "(" + " & ".join(f"({_p(k, i, j)} | {_p(k, j, i)})" for j in range(k)) + ")"
        for i in range(k))
    return _program(_refl(k) + _antisym(k) + _trans(k) + [f3])


def bounded_posets(k: int) -> str:
    """Posets with a least and a greatest element."""
    least = " | ".join("(" + " & ".join(_p(k, a, j) for j in range(k)) + ")" for a in range(k))
    great = " | ".join("(" + " & ".join(_p(k, j, b) for j in range(k)) + ")" for b in range(k))
    return _program(_refl(k) + _antisym(k) + _trans(k) + [least, great])


def bounded_poset_kills(k: int) -> dict:
    """Eq. (conspa) of PAPER.md:1194-1198 (reading C-13: p_{0i} = 1,
    p_{j0} = 0, p_{i,k-1} = 1, p_{k-1,j} = 0, p_{ii} = 1): the assumptions
    that make 0 the least and k-1 the greatest element.  5k-6 letters are
    killed, leaving v = k^2 - 5k + 6."""
    a = {}
    for i in range(k):
        a[letter_id(k, 0, i)] = 1
        a[letter_id(k, i, k - 1)] = 1
        a[letter_id(k, i, i)] = 1
    for j in range(1, k):
        a[letter_id(k, j, 0)] = 0
    for j in range(0, k - 1):
        a[letter_id(k, k - 1, j)] = 0
    return a


# BAequ (§5.1) with x=id3, y=id2, z=id1, u=id0 (reading C-1)
BAEQU = "e1 = x3 ^ x2 ^ ~x1 ^ x0\ne2 = ~((x3 | x2 & x1) ^ x0)\n"


# --------------------------------------------------------------------------
# random 3-CNF (config C2)
# --------------------------------------------------------------------------
def cnf3(n: int, m: int, seed: int = SEED) -> str:
    """m clauses; each takes 3 distinct ids uniformly and negates each
    literal with p=1/2. One clause per line."""
    rng = np.random.default_rng(seed)
    lines = []
    for _ in range(m):
        ids = rng.choice(n, 3, replace=False)
        neg = rng.integers(0, 2, size=3)
        lines.append(" | ".join(("~" if s else "") + f"x{int(v)}" for v, s in zip(ids, neg)))
    return _program(lines)


# --------------------------------------------------------------------------
# random DAG (config C5)
# --------------------------------------------------------------------------
_DAG_OPS = ("&", "|", "^", "->")
_DAG_P = (0.3, 0.3, 0.2, 0.2)


def random_dag(n: int, gates: int, seed: int = SEED, window: int = 32) -> str:
    """Random Boolean DAG, emitted as `let gK = ...` lines.

    Gate g: op in {AND .3, OR .3, XOR .2, IMP .2}; input a is one of the last
    `window` nodes (variables first, then gates); input b is variable
    (17 g mod n) for g < n (guarantees full support when gcd(17, n) = 1),
    else with p=.5 a uniform variable, else one of the last `window` nodes.
    Each input is negated with p=.25.  The program's value is the last gate."""
    rng = np.random.default_rng(seed)
    nodes = [f"x{v}" for v in range(n)]
    lines = []
    for g in range(gates):
        op = _DAG_OPS[int(rng.choice(4, p=_DAG_P))]
        a = nodes[len(nodes) - 1 - int(rng.integers(0, min(window, len(nodes))))]
        if g < n:
            b = f"x{(17 * g) % n}"
        elif rng.random() < 0.5:
            b = f"x{int(rng.integers(0, n))}"
        else:
            b = nodes[len(nodes) - 1 - int(rng.integers(0, min(window, len(nodes))))]
        na = "~" if rng.random() < 0.25 else ""
        nb = "~" if rng.random() < 0.25 else ""
        name = f"g{g}"
        lines.append(f"let {name} = {na}{a} {op} {nb}{b}")
        nodes.append(name)
    lines.append(nodes[-1])
    return _program(lines)


# --------------------------------------------------------------------------
# paper-scale term (NEXT-3): 30 variables, 2^17 expression-tree nodes
# --------------------------------------------------------------------------
def paper_scale_tree(n: int = 30, nodes: int = 1 << 17, seed: int = SEED) -> str:
    """A random binary expression TREE with `nodes` nodes (2^16 literal leaves
    and 2^16 - 1 binary operators for the default), the shape of the paper's
    timed experiment "a Boolean term t with 30 variables and 2^17 nodes"
    (PAPER.md:374-380).  Leaves are variables (uniform, negated p=1/2);
    operators are paired level by level (a balanced tree of depth 16) with op
    AND/OR/XOR/IFF uniform so the term neither collapses to a constant nor
    loses its dependence on the leaves.  Emitted as one `let` per level-16
    subtree of 64 leaves so the text stays parseable by line."""
    rng = np.random.default_rng(seed)
    leaves = (nodes + 1) // 2
    ops = ("&", "|", "^", "<->")
    level = []
    for _ in range(leaves):
        v = int(rng.integers(0, n))
        level.append(("~" if rng.random() < 0.5 else "") + f"x{v}")
    lines = []
    group = 64
    names = []
    for g in range(0, leaves, group):
        cur = level[g:g + group]
        while len(cur) > 1:
            nxt = []
            for i in range(0, len(cur) - 1, 2):
                nxt.append(f"({cur[i]} {ops[int(rng.integers(0, 4))]} {cur[i + 1]})")
            if len(cur) & 1:
                nxt.append(cur[-1])
            cur = nxt
        name = f"t{len(names)}"
        lines.append(f"let {name} = {cur[0]}")
        names.append(name)
    cur = names
    while len(cur) > 1:
        nxt = []
        for i in range(0, len(cur) - 1, 2):
            name = f"u{len(lines)}"
            lines.append(f"let {name} = {cur[i]} {ops[int(rng.integers(0, 4))]} {cur[i + 1]}")
            nxt.append(name)
        if len(cur) & 1:
            nxt.append(cur[-1])
        cur = nxt
    lines.append(cur[0])
    return _program(lines)


# --------------------------------------------------------------------------
# random terms for the parity suite (SPEC acceptance 1)
# --------------------------------------------------------------------------
# term = ('var', i) | ('const', b) | ('not', t) | (op, a, b), op in
# {'and','or','xor','imp','iff'}
_PREC = {"iff": 1, "imp": 2, "or": 3, "xor": 4, "and": 5, "not": 6, "var": 7, "const": 7, "ref": 7}
_SYM = {"iff": "<->", "imp": "->", "or": "|", "xor": "^", "and": "&"}


def _rand_term(rng, n: int, depth: int, max_depth: int, refs):
    leaf = depth >= max_depth or (depth > 0 and rng.random() < depth / max_depth)
    if leaf:
        if refs and rng.random() < 0.3:
            return ("ref", refs[int(rng.integers(0, len(refs)))])
        if n > 0 and rng.random() < 0.85:
            return ("var", int(rng.integers(0, n)))
        return ("const", int(rng.integers(0, 2)))
    op = ("not", "and", "or", "xor", "imp", "iff")[int(rng.integers(0, 6))]
    if op == "not":
        return ("not", _rand_term(rng, n, depth + 1, max_depth, refs))
    return (op, _rand_term(rng, n, depth + 1, max_depth, refs),
            _rand_term(rng, n, depth + 1, max_depth, refs))


def render_text(t, rng=None) -> str:
    """Render in the bfa grammar with MINIMAL parentheses (so the parsers'
    precedence and associativity are exercised); rng adds redundant ones."""
    kind = t[0]
    if kind == "var":
        return f"x{t[1]}"
    if kind == "const":
        return str(t[1])
    if kind == "ref":
        return t[1]
    if kind == "not":
        inner = render_text(t[1], rng)
        if _PREC[t[1][0]] < _PREC["not"]:
            inner = f"({inner})"
        return f"~{inner}"
    p = _PREC[kind]
    a, b = render_text(t[1], rng), render_text(t[2], rng)
    pa, pb = _PREC[t[1][0]], _PREC[t[2][0]]
    # '->' is right-associative, the others left-associative (include/bfa.h)
    if pa < p or (pa == p and kind == "imp"):
        a = f"({a})"
    if pb < p or (pb == p and kind != "imp"):
        b = f"({b})"
    s = f"{a} {_SYM[kind]} {b}"
    if rng is not None and rng.random() < 0.1:
        s = f"({s})"
    return s


def render_python(t) -> str:
    """Fully parenthesised Python/numpy rendering (bool arrays; T/F constants).
    IMP -> (~a | b), IFF -> ~(a ^ b): the paper's Python-AE operator meanings
    (PAPER.md:1043-1046)."""
    kind = t[0]
    if kind == "var":
        return f"x{t[1]}"
    if kind == "const":
        return "T" if t[1] else "F"
    if kind == "ref":
        return t[1]
    if kind == "not":
        return f"(~{render_python(t[1])})"
    a, b = render_python(t[1]), render_python(t[2])
    if kind == "imp":
        return f"((~{a}) | {b})"
    if kind == "iff":
        return f"(~({a} ^ {b}))"
    return f"({a} {_SYM[kind]} {b})"


@dataclass
class RandomProgram:
    seed: int
    n: int
    text: str                                  # bfa grammar
    py_lets: list = field(default_factory=list)  # [(name, python expr)]
    py_constraints: list = field(default_factory=list)


def random_program(seed: int, max_n: int = 20, max_depth: int = 8) -> RandomProgram:
    """Parity-suite term `seed`: n = seed mod (max_n+1); every 5th term is
    wrapped in 3-5 `let` definitions to exercise sharing."""
    rng = np.random.default_rng(SEED + seed)
    n = seed % (max_n + 1)
    prog = RandomProgram(seed=seed, n=n, text="")
    lines, refs = [], []
    if seed % 5 == 0:
        for i in range(int(rng.integers(3, 6))):
            t = _rand_term(rng, n, 2, max_depth, refs)
            name = f"g{i}"
            lines.append(f"let {name} = {render_text(t, rng)}")
            prog.py_lets.append((name, render_python(t)))
            refs.append(name)
    n_constraints = 1 + int(rng.integers(0, 2))
    for _ in range(n_constraints):
        t = _rand_term(rng, n, 0, max_depth, refs)
        lines.append(render_text(t, rng))
        prog.py_constraints.append(render_python(t))
    prog.text = _program(lines)
    return prog


# --------------------------------------------------------------------------
# named configs (BASELINE.json configs[0..4])
# --------------------------------------------------------------------------
C5_SEED = SEED


def config(name: str):
    """Return (text, n, expected_count_or_None) for a named config."""
    if name == "c1":
        return posets(3), 9, 19
    if name == "c2":
        return cnf3(28, 2000), 28, 0
    if name == "c2_m100":
        return cnf3(28, 100), 28, None
    if name == "c2_n32":
        return cnf3(32, 2000), 32, 0
    if name == "c3_equiv":
        return equivalences(5), 25, 52
    if name == "c3_posets":
        return posets(5), 25, 4231
    if name == "c4":
        return posets(6), 36, 130023
    if name == "c5":
        return random_dag(42, 1000, C5_SEED), 42, None
    if name == "paper_2p17":
        return paper_scale_tree(30, 1 << 17), 30, None
    raise KeyError(name)
