"""paper_1310_6978_b200 -- B200-native evaluation of Boolean terms on the free
generators of the free Boolean algebra (arXiv 1310.6978, §2.3).

Thin ctypes binding over the C ABI of libbfa.so (include/bfa.h): argument
marshalling only; every step of the hot path runs in the library's sm_100a
kernels.  PyTorch provides device memory and streams.  There is no CPU
fallback: if libbfa.so is missing, importing the binding's entry points
raises, and without a CUDA device every compute call raises BfaError.
"""
from __future__ import annotations

import ctypes
import json
import os

__all__ = ["Program", "Batch", "BfaError", "words_for", "reinstate", "last_launch", "fill_generators", "popcount",
           "peak_int", "lib_path", "version", "cache_key", "rows"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libbfa.so")
_lib = None

BFA_OK, BFA_E_PARSE, BFA_E_ARG, BFA_E_RANGE, BFA_E_CUDA, BFA_E_JIT, BFA_E_NOMEM = 0, -1, -2, -3, -4, -5, -6
UINT64_MAX = (1 << 64) - 1

_c = ctypes
_SIGS = {
    "bfa_compile": (_c.c_int, [_c.c_char_p, _c.POINTER(_c.c_void_p)]),
    "bfa_free": (None, [_c.c_void_p]),
    "bfa_info_get": (_c.c_int, [_c.c_void_p, _c.c_void_p]),
    "bfa_set_option": (_c.c_int, [_c.c_void_p, _c.c_char_p, _c.c_int64]),
    "bfa_count": (_c.c_uint64, [_c.c_void_p, _c.c_int]),
    "bfa_eval": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_void_p]),
    "bfa_count_range": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_uint64, _c.c_uint64, _c.c_void_p, _c.c_void_p]),
    "bfa_eval_range": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_uint64, _c.c_uint64, _c.c_void_p, _c.c_void_p,
                                  _c.c_void_p]),
    "bfa_fill_generators": (_c.c_int, [_c.c_int, _c.c_int, _c.c_void_p, _c.c_void_p]),
    "bfa_eval_materialised": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_int, _c.c_void_p, _c.c_void_p, _c.c_void_p]),
    "bfa_popcount": (_c.c_int, [_c.c_void_p, _c.c_uint64, _c.c_void_p, _c.c_void_p]),
    "bfa_peak_int": (_c.c_int, [_c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_void_p, _c.c_void_p]),
    "bfa_last_launch_json": (_c.c_int, [_c.c_char_p, _c.c_size_t]),
    "bfa_dump": (_c.c_int64, [_c.c_void_p, _c.c_int, _c.c_int, _c.c_char_p, _c.c_size_t]),
    "bfa_jit_cubin": (_c.c_int64, [_c.c_void_p, _c.c_int, _c.c_int, _c.c_void_p, _c.c_size_t]),
    "bfa_autotune": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_void_p, _c.c_char_p, _c.c_size_t]),
    "bfa_autotune_range": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_int, _c.c_void_p, _c.c_char_p, _c.c_size_t]),
    "bfa_assume": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_uint64, _c.c_uint64, _c.POINTER(_c.c_void_p),
                              _c.POINTER(_c.c_int), _c.POINTER(_c.c_int)]),
    "bfa_enumerate": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_uint64, _c.c_uint64, _c.c_void_p, _c.c_uint64,
                                 _c.c_void_p, _c.c_void_p]),
    "bfa_rows": (_c.c_int, [_c.c_void_p, _c.c_uint64, _c.c_int, _c.POINTER(_c.c_int), _c.c_int, _c.c_uint64,
                             _c.c_void_p, _c.c_void_p]),
    "bfa_batch_create": (_c.c_int, [_c.POINTER(_c.c_void_p), _c.c_int, _c.POINTER(_c.c_void_p)]),
    "bfa_batch_count": (_c.c_int, [_c.c_void_p, _c.POINTER(_c.c_int), _c.c_void_p, _c.c_void_p]),
    "bfa_batch_free": (None, [_c.c_void_p]),
    "bfa_count_shard": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_int, _c.c_int, _c.c_void_p, _c.c_void_p]),
    "bfa_shard_plan": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_int, _c.POINTER(_c.c_int), _c.POINTER(_c.c_int),
                                  _c.POINTER(_c.c_uint64), _c.c_int, _c.POINTER(_c.c_int)]),
    "bfa_prepare": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_int]),
    "bfa_prepare_range": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_int, _c.c_int]),
    "bfa_shard_piece_text": (_c.c_int64, [_c.c_void_p, _c.c_int, _c.c_int, _c.c_int, _c.c_char_p, _c.c_size_t]),
    "bfa_roles": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_int, _c.c_int, _c.POINTER(_c.c_int8)]),
    "bfa_count_positions": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_int, _c.c_uint64, _c.c_uint64, _c.c_void_p,
                                       _c.c_void_p]),
    "bfa_last_error": (_c.c_char_p, []),
    "bfa_last_error_code": (_c.c_int, []),
    "bfa_cache_key": (_c.c_int, [_c.c_char_p, _c.c_char_p, _c.c_size_t]),
    "bfa_version": (_c.c_char_p, []),
}


class _Info(ctypes.Structure):
    _fields_ = [("max_var_id", ctypes.c_int32), ("const_value", ctypes.c_int32),
                ("tree_nodes", ctypes.c_uint64), ("gates", ctypes.c_uint32), ("luts", ctypes.c_uint32),
                ("support", ctypes.c_uint32), ("lets", ctypes.c_uint32)]


class BfaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"bfa error {code}: {msg}")
        self.code = code


def lib_path() -> str:
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(libbfa has no CPU fallback)")
        lib = ctypes.CDLL(_LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def _check(rc: int):
    if rc < 0:
        raise BfaError(rc, _load().bfa_last_error().decode(errors="replace"))
    return rc


def version() -> str:
    return _load().bfa_version().decode()


def words_for(n: int) -> int:
    """u64 words of a full DNF vector of n variables (include/bfa.h)."""
    return max(1, 1 << max(n - 6, 0))


def _stream(stream):
    import torch
    if stream is None:
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _u64_out(out, numel):
    import torch
    if out is None:
        return torch.empty(numel, dtype=torch.int64, device="cuda")
    if out.dtype not in (torch.int64, torch.uint64) or not out.is_cuda or out.numel() < numel or not out.is_contiguous():
        raise BfaError(BFA_E_ARG, f"output must be a contiguous CUDA int64 tensor of >= {numel} elements")
    return out


def last_launch() -> dict:
    buf = ctypes.create_string_buffer(1 << 16)
    _check(_load().bfa_last_launch_json(buf, len(buf)))
    return json.loads(buf.value.decode())


class Program:
    """A compiled Boolean program (bfa_compile).  Grammar: include/bfa.h."""

    def __init__(self, text: str):
        lib = _load()
        h = ctypes.c_void_p()
        _check(lib.bfa_compile(text.encode(), ctypes.byref(h)))
        self._h = h
        self.text = text

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.bfa_free(self._h)
            self._h = None

    @property
    def info(self) -> dict:
        i = _Info()
        _check(_load().bfa_info_get(self._h, ctypes.byref(i)))
        return {f: getattr(i, f) for f, _ in _Info._fields_}

    def set_option(self, key: str, value: int) -> "Program":
        _check(_load().bfa_set_option(self._h, key.encode(), int(value)))
        return self

    def autotune(self, n: int, k_free: int | None = None, stream=None) -> dict:
        """bfa_autotune(_range): pick the fastest kernel variant for counting
        over 2^n (or aligned 2^k_free sub-cubes); sets the options."""
        buf = ctypes.create_string_buffer(1 << 16)
        if k_free is None:
            _check(_load().bfa_autotune(self._h, n, _stream(stream), buf, len(buf)))
        else:
            _check(_load().bfa_autotune_range(self._h, n, k_free, _stream(stream), buf, len(buf)))
        return json.loads(buf.value.decode())

    # ---- register-synthesised mode
    def count(self, n: int) -> int:
        """bfa_count: number of models over all 2^n valuations (synchronous)."""
        c = _load().bfa_count(self._h, n)
        if c == UINT64_MAX:
            raise BfaError(_err_code(), _load().bfa_last_error().decode(errors="replace"))
        return int(c)

    def count_range(self, n: int, lo: int, hi: int, out=None, stream=None):
        """bfa_count_range: models in [lo, hi) into a 1-element device tensor (async)."""
        out = _u64_out(out, 1)
        _check(_load().bfa_count_range(self._h, n, lo, hi, ctypes.c_void_p(out.data_ptr()), _stream(stream)))
        return out

    def roles(self, n: int, k_free: int | None = None, sms: int = 0) -> list:
        """bfa_roles: perm[v] = bit position of variable v in the enumeration
        order of the count kernel for an aligned 2^k_free sub-cube (host only)."""
        perm = (ctypes.c_int8 * 64)()
        _check(_load().bfa_roles(self._h, n, n if k_free is None else k_free, sms, perm))
        return list(perm)

    def count_positions(self, n: int, k_free: int, lo: int, hi: int, out=None, stream=None):
        """bfa_count_positions: models among positions [lo, hi) of the exact
        kernel a 2^k_free sub-cube count launches (async, device tensor)."""
        out = _u64_out(out, 1)
        _check(_load().bfa_count_positions(self._h, n, k_free, lo, hi, ctypes.c_void_p(out.data_ptr()),
                                           _stream(stream)))
        return out

    def prepare(self, n: int, sms: int = 0):
        """bfa_prepare (host only, no GPU needed): compile everything count(n)
        needs before its first launch; returns self."""
        _check(_load().bfa_prepare(self._h, n, sms))
        return self

    def prepare_range(self, n: int, k_free: int, sms: int = 0):
        """bfa_prepare_range (host only): compile the count kernel for aligned
        2^k_free sub-cubes (a rank's cofactor range); returns self."""
        _check(_load().bfa_prepare_range(self._h, n, k_free, sms))
        return self

    def count_shard(self, n: int, rank: int, world: int, out=None, stream=None):
        """bfa_count_shard: this rank's share of the count under work-balanced
        cofactor sharding (sum over ranks = count(n))."""
        out = _u64_out(out, 1)
        _check(_load().bfa_count_shard(self._h, n, rank, world, ctypes.c_void_p(out.data_ptr()), _stream(stream)))
        return out

    def shard_plan(self, n: int, world: int):
        """bfa_shard_plan (host only): [(owner rank, free variables, work)] per piece."""
        lib = _load()
        np_ = ctypes.c_int()
        _check(lib.bfa_shard_plan(self._h, n, world, None, None, None, 0, ctypes.byref(np_)))
        k = np_.value
        own, nv, wk = (ctypes.c_int * k)(), (ctypes.c_int * k)(), (ctypes.c_uint64 * k)()
        _check(lib.bfa_shard_plan(self._h, n, world, own, nv, wk, k, ctypes.byref(np_)))
        return [(own[i], nv[i], wk[i]) for i in range(k)]

    def shard_piece_text(self, n: int, world: int, index: int) -> str:
        """bfa_shard_piece_text (host only): piece `index` of the shard plan
        as program text over its free variables."""
        lib = _load()
        size = _check(lib.bfa_shard_piece_text(self._h, n, world, index, None, 0))
        buf = ctypes.create_string_buffer(size + 1)
        _check(lib.bfa_shard_piece_text(self._h, n, world, index, buf, size + 1))
        return buf.value.decode()

    def eval(self, n: int, out=None):
        """bfa_eval: the full-DNF vector as words_for(n) device int64 words (synchronous)."""
        out = _u64_out(out, words_for(n))
        _check(_load().bfa_eval(self._h, n, ctypes.c_void_p(out.data_ptr())))
        return out

    def eval_range(self, n: int, lo: int, hi: int, out=None, count_out=None, stream=None):
        """bfa_eval_range: slice [lo, hi) of the vector (async); optional fused count."""
        out = _u64_out(out, max(1, (hi - lo + 63) // 64))
        cp = ctypes.c_void_p(count_out.data_ptr()) if count_out is not None else None
        _check(_load().bfa_eval_range(self._h, n, lo, hi, ctypes.c_void_p(out.data_ptr()), cp, _stream(stream)))
        return out

    # ---- killing variables / enumeration
    def assume(self, n: int, assignment: dict):
        """bfa_assume: fix variables (id -> 0/1), re-run the Reduction and
        renumber the free variables densely.  Returns (program, n_free,
        free_ids) with free_ids[new id] = original id."""
        mask = values = 0
        for v, b in assignment.items():
            mask |= 1 << v
            values |= (1 << v) if b else 0
        h = ctypes.c_void_p()
        nf = ctypes.c_int()
        ids = (ctypes.c_int * 64)()
        _check(_load().bfa_assume(self._h, n, mask, values, ctypes.byref(h), ctypes.byref(nf), ids))
        q = Program.__new__(Program)
        q._h = h
        q.text = None
        return q, nf.value, list(ids[:nf.value])

    def enumerate(self, n: int, lo: int = 0, hi: int | None = None, capacity: int = 1 << 20, stream=None):
        """bfa_enumerate: ascending models in [lo, hi) as a device int64 tensor
        (at most `capacity`), and the total number of models."""
        import torch
        hi = (1 << n) if hi is None else hi
        out = torch.empty(max(capacity, 1), dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        _check(_load().bfa_enumerate(self._h, n, lo, hi, ctypes.c_void_p(out.data_ptr()), capacity,
                                     ctypes.c_void_p(cnt.data_ptr()), _stream(stream)))
        total = int(cnt.item())
        return out[:min(total, capacity)], total

    # ---- materialised mode
    def eval_materialised(self, n: int, variant: int = 0, out=None, count_out=None, stream=None):
        out = _u64_out(out, words_for(n))
        cp = ctypes.c_void_p(count_out.data_ptr()) if count_out is not None else None
        _check(_load().bfa_eval_materialised(self._h, n, variant, ctypes.c_void_p(out.data_ptr()), cp,
                                             _stream(stream)))
        return out

    # ---- introspection (no GPU needed)
    def dump(self, what: int = 0, n: int = 0) -> str:
        lib = _load()
        size = _check(lib.bfa_dump(self._h, what, n, None, 0))
        buf = ctypes.create_string_buffer(size + 1)
        _check(lib.bfa_dump(self._h, what, n, buf, size + 1))
        return buf.value.decode()

    def jit_cubin(self, what: int = 1, n: int = 0) -> bytes:
        lib = _load()
        size = _check(lib.bfa_jit_cubin(self._h, what, n, None, 0))
        buf = ctypes.create_string_buffer(size)
        _check(lib.bfa_jit_cubin(self._h, what, n, buf, size))
        return buf.raw


class Batch:
    """bfa_batch_*: count many programs in one launch (NEXT-4)."""

    def __init__(self, programs):
        self.programs = list(programs)              # keep them alive
        arr = (ctypes.c_void_p * len(self.programs))(*[p._h.value for p in self.programs])
        h = ctypes.c_void_p()
        _check(_load().bfa_batch_create(arr, len(self.programs), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.bfa_batch_free(self._h)
            self._h = None

    def count(self, ns, out=None, stream=None):
        out = _u64_out(out, len(self.programs))
        arr = (ctypes.c_int * len(self.programs))(*ns)
        _check(_load().bfa_batch_count(self._h, arr, ctypes.c_void_p(out.data_ptr()), _stream(stream)))
        return out


def reinstate(mu_free, free_ids, assignment: dict) -> list:
    """Map models of an assumed program back to valuations of the original
    (killed letters reinstated)."""
    fixed = sum((1 << v) for v, b in assignment.items() if b)
    out = []
    for m in mu_free:
        m = int(m)
        full = fixed
        for new, old in enumerate(free_ids):
            full |= ((m >> new) & 1) << old
        out.append(full)
    return out


def rows(mu, n_all: int, free_ids=None, assignment: dict | None = None, stream=None) -> bytes:
    """bfa_rows: out.txt rows (one '0'/'1' character per letter, id n_all-1
    first, then a newline) of the models `mu` (device int64 tensor) of a
    program over len(free_ids) letters; killed letters from `assignment`."""
    import torch
    count = mu.numel()
    free_ids = list(range(n_all)) if free_ids is None else list(free_ids)
    fixed = sum((1 << v) for v, b in (assignment or {}).items() if b)
    out = torch.empty(max(1, count * (n_all + 1)), dtype=torch.uint8, device=mu.device if count else "cuda")
    ids = (ctypes.c_int * max(1, len(free_ids)))(*free_ids)
    _check(_load().bfa_rows(ctypes.c_void_p(mu.data_ptr()) if count else None, count, len(free_ids), ids, n_all,
                            fixed, ctypes.c_void_p(out.data_ptr()), _stream(stream)))
    return bytes(out[:count * (n_all + 1)].cpu().numpy())


def _err_code() -> int:
    return int(_load().bfa_last_error_code())


def cache_key(source: str) -> str:
    """bfa_cache_key: SHA-256 key of a generated kernel source in the JIT cache."""
    buf = ctypes.create_string_buffer(65)
    _check(_load().bfa_cache_key(source.encode(), buf, 65))
    return buf.value.decode()


def fill_generators(n: int, rows: int | None = None, out=None, stream=None):
    """bfa_fill_generators: the table S of free generators (rows x words_for(n))."""
    rows = n if rows is None else rows
    out = _u64_out(out, rows * words_for(n))
    _check(_load().bfa_fill_generators(n, rows, ctypes.c_void_p(out.data_ptr()), _stream(stream)))
    return out


def popcount(vec, count_out=None, stream=None):
    count_out = _u64_out(count_out, 1)
    _check(_load().bfa_popcount(ctypes.c_void_p(vec.data_ptr()), vec.numel(),
                                ctypes.c_void_p(count_out.data_ptr()), _stream(stream)))
    return count_out


def peak_int(op: int, blocks: int, threads: int, iters: int, sink, stream=None):
    """bfa_peak_int: op 0 LOP3, 1 IMAD, 2 LOP3+IMAD 1:1; 256 ops/thread/iter."""
    _check(_load().bfa_peak_int(op, blocks, threads, iters, ctypes.c_void_p(sink.data_ptr()), _stream(stream)))
