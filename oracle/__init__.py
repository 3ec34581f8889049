"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package.  The product path
(paper_1310_6978_b200) never imports it, and it imports nothing from the
product.  The evaluator is the plain C program oracle/bfa_oracle.c: one
valuation at a time, recursive descent (Prop 2.2).

`numpy_truth_table` is a second, independent brute force used only to pin
the C oracle: Python's own parser evaluates a fully parenthesised rendering
over numpy bool truth-table arrays (Python-AE syntax is Python,
PAPER.md:1001, 1043).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bfa_oracle.c")
_LIB = os.path.join(_HERE, "libbfa_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc; no tuning flags beyond -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-pthread", _SRC, "-o", _LIB])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.bfa_oracle_eval.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_uint64,
                                        ctypes.c_uint64, ctypes.c_void_p,
                                        ctypes.POINTER(ctypes.c_uint64), ctypes.c_int,
                                        ctypes.c_char_p, ctypes.c_size_t]
        lib.bfa_oracle_eval.restype = ctypes.c_int
        lib.bfa_oracle_parse.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int),
                                         ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                         ctypes.c_char_p, ctypes.c_size_t]
        lib.bfa_oracle_parse.restype = ctypes.c_int
        _lib = lib
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def default_threads() -> int:
    return len(os.sched_getaffinity(0))


def parse(text: str):
    """Return (max_var_id, n_lets, n_constraints) or raise OracleError."""
    lib = _load()
    mv, nl, nc = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    err = ctypes.create_string_buffer(512)
    rc = lib.bfa_oracle_parse(text.encode(), ctypes.byref(mv), ctypes.byref(nl),
                              ctypes.byref(nc), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return mv.value, nl.value, nc.value


def evaluate(text: str, n: int, lo: int = 0, hi: int | None = None, *,
             vector: bool = True, threads: int | None = None):
    """Oracle truth table of `text` over valuations [lo, hi) of n variables.

    Returns (words, count): words is a uint64 array of ceil((hi-lo)/64)
    little-endian words with bit (mu-lo) at word (mu-lo)>>6 (or None when
    vector=False); count is the number of models in the range."""
    lib = _load()
    if not 0 <= n <= 63:       # let the C side report the range error
        lo, hi, vector = 0, 0, False
    if hi is None:
        hi = 1 << n
    nwords = (hi - lo + 63) // 64
    words = np.zeros(max(nwords, 1), dtype=np.uint64) if vector else None
    cnt = ctypes.c_uint64()
    err = ctypes.create_string_buffer(512)
    rc = lib.bfa_oracle_eval(text.encode(), n, lo, hi,
                             words.ctypes.data if vector else None, ctypes.byref(cnt),
                             threads or default_threads(), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    if vector:
        words = words[:nwords]
    return words, cnt.value


def count(text: str, n: int, lo: int = 0, hi: int | None = None, threads: int | None = None) -> int:
    return evaluate(text, n, lo, hi, vector=False, threads=threads)[1]


def set_bits(words: np.ndarray, offset: int = 0) -> np.ndarray:
    """Sorted indices of the set bits of a packed little-endian u64 vector."""
    bits = np.unpackbits(np.asarray(words, dtype="<u8").view(np.uint8), bitorder="little")
    return np.nonzero(bits)[0].astype(np.int64) + offset


def numpy_truth_table(n: int, py_lets, py_constraints) -> np.ndarray:
    """Independent brute force for pinning the oracle (small n only):
    Python evaluates each rendered expression over bool arrays of length 2^n
    in which variable v is ((mu >> v) & 1).  Returns a bool array."""
    mu = np.arange(1 << n, dtype=np.uint64)
    env = {f"x{v}": ((mu >> np.uint64(v)) & np.uint64(1)).astype(bool) for v in range(n)}
    env["T"] = np.ones(1 << n, dtype=bool)
    env["F"] = np.zeros(1 << n, dtype=bool)
    for name, expr in py_lets:
        env[name] = eval(expr, {"__builtins__": {}}, env)
    out = np.ones(1 << n, dtype=bool)
    for expr in py_constraints:
        out &= eval(expr, {"__builtins__": {}}, env)
    return out


def pack_bool(bits: np.ndarray) -> np.ndarray:
    """Pack a bool array (index = mu) into little-endian u64 words."""
    nbytes = (len(bits) + 63) // 64 * 8
    packed = np.packbits(bits.astype(np.uint8), bitorder="little")
    buf = np.zeros(nbytes, dtype=np.uint8)
    buf[:len(packed)] = packed
    return buf.view("<u8").astype(np.uint64)
