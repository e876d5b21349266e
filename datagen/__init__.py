"""Seeded synthetic inputs for the oracle tests, the GPU parity tests and bench.py.

Holds none of the sorting method's arithmetic: only key generation (SplitMix64,
see ``datagen.cpp``) and the layouts BASELINE.json names.  Both the oracle and
the CUDA path consume the arrays produced here; neither produces them.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
_SO = os.path.join(_HERE, "libdatagen.so")
_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    src = os.path.join(_HERE, "datagen.cpp")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _ROOT, "datagen/libdatagen.so"], check=True,
                       stdout=subprocess.DEVNULL)
    lib = ctypes.CDLL(_SO)
    u64, sz, p, cs, i32, dbl = (ctypes.c_uint64, ctypes.c_size_t, ctypes.c_void_p,
                                ctypes.c_char_p, ctypes.c_int, ctypes.c_double)
    sig = {
        "dg_mix": ([u64], u64),
        "dg_stream_key": ([u64, cs], u64),
        "dg_draw": ([u64, u64], u64),
        "dg_uniform_u64": ([p, sz, u64, cs], None),
        "dg_uniform_u32": ([p, sz, u64, cs], None),
        "dg_lowbits_u64": ([p, sz, u64, cs, i32], None),
        "dg_normal_u64": ([p, sz, u64, cs, u64, dbl], None),
        "dg_exponential_u64": ([p, sz, u64, cs, dbl], None),
        "dg_zipf_u64": ([p, sz, u64, cs, dbl, sz], None),
        "dg_few_unique_u32": ([p, sz, u64, cs, ctypes.c_uint32], None),
        "dg_const_u32": ([p, sz, u64, cs], None),
        "dg_iota_u32": ([p, sz], None),
        "dg_sort_asc_u64": ([p, sz], None),
        "dg_reverse_u64": ([p, sz], None),
        "dg_transpose_u64": ([p, sz, u64, cs, sz], None),
        "dg_sort_runs_u64": ([p, sz, sz], None),
        "dg_fingerprint": ([p, sz, i32, p], None),
        "dg_is_sorted_u64": ([p, sz], i32),
        "dg_is_sorted_u32": ([p, sz], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def mix(z: int) -> int:
    return _load().dg_mix(z)


def stream_key(seed: int, name: str) -> int:
    return _load().dg_stream_key(seed, name.encode())


def draw(key: int, i: int) -> int:
    return _load().dg_draw(key, i)


def uniform_u64(n, seed, stream="base"):
    a = np.empty(n, np.uint64)
    _load().dg_uniform_u64(_ptr(a), n, seed, stream.encode())
    return a


def uniform_u32(n, seed, stream="base"):
    a = np.empty(n, np.uint32)
    _load().dg_uniform_u32(_ptr(a), n, seed, stream.encode())
    return a


def lowbits_u64(n, seed, bits, stream="base"):
    a = np.empty(n, np.uint64)
    _load().dg_lowbits_u64(_ptr(a), n, seed, stream.encode(), bits)
    return a


def normal_u64(n, seed, mean, sd, stream="normal"):
    a = np.empty(n, np.uint64)
    _load().dg_normal_u64(_ptr(a), n, seed, stream.encode(), int(mean), float(sd))
    return a


def exponential_u64(n, seed, scale, stream="exp"):
    a = np.empty(n, np.uint64)
    _load().dg_exponential_u64(_ptr(a), n, seed, stream.encode(), float(scale))
    return a


def zipf_u64(n, seed, s=1.1, universe=1 << 20, stream="zipf"):
    a = np.empty(n, np.uint64)
    _load().dg_zipf_u64(_ptr(a), n, seed, stream.encode(), float(s), universe)
    return a


def few_unique_u32(n, seed, distinct=256, stream="few"):
    a = np.empty(n, np.uint32)
    _load().dg_few_unique_u32(_ptr(a), n, seed, stream.encode(), distinct)
    return a


def const_u32(n, seed, stream="equal"):
    a = np.empty(n, np.uint32)
    _load().dg_const_u32(_ptr(a), n, seed, stream.encode())
    return a


def iota_u32(n):
    a = np.empty(n, np.uint32)
    _load().dg_iota_u32(_ptr(a), n)
    return a


def sort_asc_u64(a):
    _load().dg_sort_asc_u64(_ptr(a), a.size)
    return a


def reverse_u64(a):
    _load().dg_reverse_u64(_ptr(a), a.size)
    return a


def transpose_u64(a, seed, swaps, stream="swaps"):
    _load().dg_transpose_u64(_ptr(a), a.size, seed, stream.encode(), swaps)
    return a


def sort_runs_u64(a, run):
    _load().dg_sort_runs_u64(_ptr(a), a.size, run)
    return a


def fingerprint(a: np.ndarray):
    out = np.zeros(2, np.uint64)
    _load().dg_fingerprint(_ptr(a), a.size, a.dtype.itemsize, _ptr(out))
    return int(out[0]), int(out[1])


def is_sorted(a: np.ndarray) -> bool:
    f = _load().dg_is_sorted_u64 if a.dtype == np.uint64 else _load().dg_is_sorted_u32
    return bool(f(_ptr(a), a.size))


# --------------------------------------------------------------------------
# BASELINE.json configs c1..c5 (recipes: DESIGN.md "Input recipe")
# --------------------------------------------------------------------------
@dataclass
class Case:
    name: str          # e.g. "c5-uniform"
    config: str        # "c1".."c5"
    n: int
    key_dtype: str     # "u32" | "u64"
    pairs: bool
    seed: int


CASES = {
    "c1": Case("c1", "c1", 1 << 16, "u32", False, 1),
    "c2": Case("c2", "c2", 1 << 24, "u64", False, 2),
    "c3-normal": Case("c3-normal", "c3", 1 << 26, "u64", False, 3),
    "c3-exp": Case("c3-exp", "c3", 1 << 26, "u64", False, 3),
    "c3-zipf": Case("c3-zipf", "c3", 1 << 26, "u64", False, 3),
    "c4-few": Case("c4-few", "c4", 1 << 27, "u32", True, 4),
    "c4-equal": Case("c4-equal", "c4", 1 << 27, "u32", True, 4),
    "c5-uniform": Case("c5-uniform", "c5", 1 << 28, "u64", False, 5),
    "c5-sorted": Case("c5-sorted", "c5", 1 << 28, "u64", False, 5),
    "c5-reverse": Case("c5-reverse", "c5", 1 << 28, "u64", False, 5),
    "c5-nearly": Case("c5-nearly", "c5", 1 << 28, "u64", False, 5),
    "c5-runs": Case("c5-runs", "c5", 1 << 28, "u64", False, 5),
    "c5-low20": Case("c5-low20", "c5", 1 << 28, "u64", False, 5),
    # the paper's own workloads: 64-bit keys at
    # N = 256^3 .. 256^3.75, uniform (Fig. 1), wide normal
    # (mean ~2^63, sd ~2^61; Fig. 2), narrow normal (mean ~2^32, sd
    # ~2^30; Fig. 3); n is chosen per run (default 256^3.5 = 2^28)
    "paper-uniform": Case("paper-uniform", "paper", 1 << 28, "u64", False, 6),
    "paper-wide-normal": Case("paper-wide-normal", "paper", 1 << 28, "u64", False, 6),
    "paper-narrow-normal": Case("paper-narrow-normal", "paper", 1 << 28, "u64", False, 6),
    # 16-byte records (SPEC's key + tag): uniform u64 keys, u64 tags
    "paper-records": Case("paper-records", "paper", 1 << 27, "u64", True, 6),
}


def make_case(name: str, n: int | None = None):
    """Return (keys, vals_or_None) for a named case; ``n`` overrides the size
    (same recipe, smaller/larger) for the oracle-sized parity tests."""
    c = CASES[name]
    n = c.n if n is None else n
    s = c.seed
    vals = iota_u32(n) if c.pairs else None
    if name == "c1":
        return uniform_u32(n, s), None
    if name == "c2":
        return uniform_u64(n, s), None
    if name == "c3-normal":
        return normal_u64(n, s, 1 << 63, 2.0 ** 40), None
    if name == "c3-exp":
        return exponential_u64(n, s, 2.0 ** 32), None
    if name == "c3-zipf":
        return zipf_u64(n, s, 1.1, 1 << 20), None
    if name == "c4-few":
        return few_unique_u32(n, s, 256), vals
    if name == "c4-equal":
        return const_u32(n, s), vals
    if name == "paper-uniform":
        return uniform_u64(n, s, "paper-uniform"), None
    if name == "paper-wide-normal":
        return normal_u64(n, s, 1 << 63, 2.0 ** 61, "paper-wide"), None
    if name == "paper-narrow-normal":
        return normal_u64(n, s, 1 << 32, 2.0 ** 30, "paper-narrow"), None
    if name == "paper-records":
        return uniform_u64(n, s, "paper-records"), uniform_u64(n, s, "paper-tags")
    base = uniform_u64(n, s, "base")
    if name == "c5-uniform":
        return base, None
    if name == "c5-sorted":
        return sort_asc_u64(base), None
    if name == "c5-reverse":
        return reverse_u64(sort_asc_u64(base)), None
    if name == "c5-nearly":
        return transpose_u64(sort_asc_u64(base), s, n // 200), None
    if name == "c5-runs":
        return sort_runs_u64(base, 4096), None
    if name == "c5-low20":
        return lowbits_u64(n, s, 20), None
    raise KeyError(name)
