"""CPU oracle for DFR (arXiv 2207.14334) — TEST INFRASTRUCTURE ONLY.

Plain, single-threaded C++ (``oracle.cpp``) following PAPER.md Alg. 4
 step by step; see that file's header for every citation.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2207_14334_b200``) never imports it and shares no code
with it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

STAT_FIELDS = ("passes", "skippable_passes", "diversions", "diverted_records",
               "large_buckets", "max_depth", "level0_p", "level0_large",
               "count_ops", "deal_ops")


class _Stats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint64) for f in STAT_FIELDS]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f in STAT_FIELDS}


def _load():
    global _lib
    if _lib is not None:
        return _lib
    src = os.path.join(_HERE, "oracle.cpp")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _ROOT, "oracle/liboracle.so"], check=True,
                       stdout=subprocess.DEVNULL)
    lib = ctypes.CDLL(_SO)
    u64, p, i32 = ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int
    sp = ctypes.POINTER(_Stats)
    sig = {
        "oracle_est_top_passes": ([u64, i32, u64], i32),
        "oracle_extract_digit_u64": ([u64, i32, i32], u64),
        "oracle_prefix_sum_exclusive": ([p, p, u64], None),
        "oracle_dfr_u32": ([p, u64, i32, u64, sp], i32),
        "oracle_dfr_u64": ([p, u64, i32, u64, sp], i32),
        "oracle_dfr_pairs_u32": ([p, p, u64, i32, u64, sp], i32),
        "oracle_dfr_pairs_u64": ([p, p, u64, i32, u64, sp], i32),
        "oracle_insertion_sort_pairs_u64": ([p, p, u64], None),
        "oracle_hist_u32": ([p, u64, i32, i32, p], None),
        "oracle_hist_u64": ([p, u64, i32, i32, p], None),
        "oracle_group_u32": ([p, p, u64, u64, sp], i32),
        "oracle_group_u64": ([p, u64, u64, sp], i32),
        "oracle_pass_u64": ([p, u64, i32], i32),
        "oracle_pass_pairs_u32": ([p, p, u64, i32], i32),
        "oracle_level_buckets_u64": ([p, u64, i32, u64, u64, p], None),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _ptr(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def est_top_passes(n: int, radix_bits: int = 8, n_d: int = 64) -> int:
    """Alg. 4 l.4 under SPEC's reading S:284: least p with n <= N_d*M^p."""
    return _load().oracle_est_top_passes(n, radix_bits, n_d)


def extract_digit(key: int, d: int, radix_bits: int = 8) -> int:
    return int(_load().oracle_extract_digit_u64(key, d, radix_bits))


def prefix_sum_exclusive(counts):
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
    out = np.zeros_like(c)
    _load().oracle_prefix_sum_exclusive(_ptr(c), _ptr(out), c.size)
    return out


def dfr_sort(keys: np.ndarray, vals: np.ndarray | None = None, *, radix_bits: int = 8,
             n_d: int = 64, copy: bool = True):
    """DFR (Alg. 4) on a copy of ``keys`` (and ``vals``); returns (keys, vals, stats)."""
    lib = _load()
    k = np.array(keys, copy=True) if copy else keys
    v = None if vals is None else (np.array(vals, copy=True) if copy else vals)
    st = _Stats()
    n = k.size
    if k.dtype == np.uint32 and v is None:
        rc = lib.oracle_dfr_u32(_ptr(k), n, radix_bits, n_d, ctypes.byref(st))
    elif k.dtype == np.uint64 and v is None:
        rc = lib.oracle_dfr_u64(_ptr(k), n, radix_bits, n_d, ctypes.byref(st))
    elif k.dtype == np.uint32 and v is not None and v.dtype == np.uint32:
        rc = lib.oracle_dfr_pairs_u32(_ptr(k), _ptr(v), n, radix_bits, n_d, ctypes.byref(st))
    elif k.dtype == np.uint64 and v is not None and v.dtype == np.uint64:
        rc = lib.oracle_dfr_pairs_u64(_ptr(k), _ptr(v), n, radix_bits, n_d, ctypes.byref(st))
    else:
        raise TypeError(f"unsupported dtypes {k.dtype} / {None if v is None else v.dtype}")
    if rc != 0:
        raise ValueError(f"oracle_dfr failed rc={rc}")
    return k, v, st.as_dict()


def insertion_sort_pairs_u64(keys, vals):
    k = np.array(keys, dtype=np.uint64, copy=True)
    v = np.array(vals, dtype=np.uint64, copy=True)
    _load().oracle_insertion_sort_pairs_u64(_ptr(k), _ptr(v), k.size)
    return k, v


def hist(keys: np.ndarray, digit_lo: int, p: int) -> np.ndarray:
    """Counts of digits digit_lo..digit_lo+p-1 (radix 256); shape (p, 256)."""
    out = np.zeros((p, 256), np.uint32)
    f = _load().oracle_hist_u64 if keys.dtype == np.uint64 else _load().oracle_hist_u32
    f(_ptr(np.ascontiguousarray(keys)), keys.size, digit_lo, p, _ptr(out))
    return out


def group(keys: np.ndarray, vals: np.ndarray | None = None, n_d: int = 64):
    """Level-0 top-group LSD passes only (Alg. 4 l.4-6); returns (keys, vals, p)."""
    k = np.array(keys, copy=True)
    v = None if vals is None else np.array(vals, copy=True)
    st = _Stats()
    if k.dtype == np.uint64:
        assert v is None
        p = _load().oracle_group_u64(_ptr(k), k.size, n_d, ctypes.byref(st))
    else:
        p = _load().oracle_group_u32(_ptr(k), _ptr(v), k.size, n_d, ctypes.byref(st))
    return k, v, p


def counting_pass(keys: np.ndarray, d: int, vals: np.ndarray | None = None):
    """One stable counting-sort pass on digit d."""
    k = np.array(keys, copy=True)
    v = None if vals is None else np.array(vals, copy=True)
    if k.dtype == np.uint64:
        _load().oracle_pass_u64(_ptr(k), k.size, d)
    else:
        _load().oracle_pass_pairs_u32(_ptr(k), _ptr(v if v is not None else np.zeros(k.size, np.uint32)), k.size, d)
    return k, v


def level_buckets(keys_grouped: np.ndarray, p: int, n_d: int = 64, cap: int = 4096):
    out = np.zeros(6, np.uint64)
    _load().oracle_level_buckets_u64(_ptr(keys_grouped), keys_grouped.size, p, n_d, cap, _ptr(out))
    return dict(zip(("buckets", "small", "mid", "large", "mid_records", "large_records"),
                    (int(x) for x in out)))
