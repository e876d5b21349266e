"""B200-native Diverting Fast Radix (DFR) sort — thin Python binding.

The sort runs entirely in the hand-written sm_100a kernels of ``libdfr.so``
(C ABI declared in ``include/dfr.h``); this module only marshals arguments:
device pointers, element counts and the current CUDA stream of PyTorch
tensors.  There is no CPU fallback: without the built library or a CUDA
device every call raises.

Method: PAPER.md §3 Alg. 4 — see include/dfr.h and DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os

__all__ = [
    "DfrError", "lib", "sort", "sort_u32", "sort_u64", "sort_pairs_u32", "sort_pairs_u64", "histogram",
    "partition_pass", "top_passes", "workspace_bytes", "status_string", "EXPORTS", "overflow_mc",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DFR_LIB") or os.path.join(_HERE, "libdfr.so")

# every symbol include/dfr.h declares
EXPORTS = (
    "dfr_sort_u32", "dfr_sort_u64", "dfr_sort_pairs_u32", "dfr_sort_pairs_u64",
    "dfr_sort_u32_ex", "dfr_sort_u64_ex", "dfr_sort_pairs_u32_ex", "dfr_sort_pairs_u64_ex",
    "dfr_histogram_u32", "dfr_histogram_u64",
    "dfr_partition_pass_u64", "dfr_partition_pass_pairs_u32",
    "dfr_top_passes", "dfr_workspace_bytes", "dfr_launch_counter", "dfr_status_string",
    "dfr_overflow_mc",
)

PHASES = ("hist", "plan", "scatter0", "scatter1", "scatter2", "scatter3", "divert", "levels", "mid")

DFR_OK, DFR_ERR_INVALID, DFR_ERR_ALLOC, DFR_ERR_CUDA, DFR_ERR_TOO_LARGE = 0, -1, -2, -3, -4


class DfrError(RuntimeError):
    pass


class Config(ctypes.Structure):
    _fields_ = [("n_d", ctypes.c_uint32), ("skip_trivial_passes", ctypes.c_uint32),
                ("phase_events", ctypes.POINTER(ctypes.c_void_p)),
                ("fused_last_pass", ctypes.c_uint32), ("full_lsd", ctypes.c_uint32),
                ("fast_radix", ctypes.c_uint32), ("stable_deals", ctypes.c_uint32)]


class Stats(ctypes.Structure):
    _fields_ = [("level0_p", ctypes.c_uint32), ("level0_passes_run", ctypes.c_uint32),
                ("level0_large", ctypes.c_uint64), ("mid_buckets", ctypes.c_uint64),
                ("global_segments", ctypes.c_uint64), ("levels", ctypes.c_uint32),
                ("overflow", ctypes.c_uint32), ("fused", ctypes.c_uint32),
                ("fr_overflow", ctypes.c_uint32)]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


_lib = None


def lib() -> ctypes.CDLL:
    """Load libdfr.so (built in-tree by ``make`` / ``__graft_entry__.build()``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DfrError(f"{LIB_PATH} is missing: build it with `make` (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    p, sz, i32, u32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint32
    cfgp, stp = ctypes.POINTER(Config), ctypes.POINTER(Stats)
    sig = {
        "dfr_sort_u32": [p, sz, p],
        "dfr_sort_u64": [p, sz, p],
        "dfr_sort_pairs_u32": [p, p, sz, p],
        "dfr_sort_pairs_u64": [p, p, sz, p],
        "dfr_sort_pairs_u64_ex": [p, p, sz, p, cfgp, stp],
        "dfr_sort_u32_ex": [p, sz, p, cfgp, stp],
        "dfr_sort_u64_ex": [p, sz, p, cfgp, stp],
        "dfr_sort_pairs_u32_ex": [p, p, sz, p, cfgp, stp],
        "dfr_histogram_u32": [p, sz, i32, i32, p, p],
        "dfr_histogram_u64": [p, sz, i32, i32, p, p],
        "dfr_partition_pass_u64": [p, p, sz, i32, p],
        "dfr_partition_pass_pairs_u32": [p, p, p, p, sz, i32, p],
        "dfr_top_passes": [sz, i32, u32],
        "dfr_workspace_bytes": [sz, i32, i32],
        "dfr_status_string": [i32],
        "dfr_launch_counter": [],
        "dfr_overflow_mc": [ctypes.c_uint64, u32, u32, ctypes.c_uint64, p, p],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = i32
    L.dfr_workspace_bytes.restype = ctypes.c_size_t
    L.dfr_status_string.restype = ctypes.c_char_p
    L.dfr_launch_counter.restype = ctypes.c_uint64
    _lib = L
    return L


def status_string(code: int) -> str:
    return lib().dfr_status_string(code).decode()


def _check(rc: int, what: str):
    if rc != DFR_OK:
        raise DfrError(f"{what} failed: {status_string(rc)} ({rc})")


def _stream(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def _dev_tensor(t, widths):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise DfrError("expected a CUDA tensor (no CPU path exists)")
    if not t.is_contiguous():
        raise DfrError("tensor must be contiguous")
    if t.element_size() not in widths:
        raise DfrError(f"unsupported element size {t.element_size()}")
    return t


def _cfg(n_d, skip_trivial, events=None, fused=None, full_lsd=False, fast_radix=False,
         stable_deals=False):
    """events: None or a sequence of 2*len(PHASES) torch.cuda.Event(enable_timing=True)
    (None entries: that phase is not timed).
    fused: None (default: the fused last deal + diversion where eligible, dfr.h),
    True (same, explicit) or False (always the separate deal and diversion)."""
    mode = 0 if fused is None else (1 if fused else 2)
    c = Config(int(n_d), 1 if skip_trivial else 0, None, mode, 1 if full_lsd else 0,
               1 if fast_radix else 0, 1 if stable_deals else 0)
    if events is not None:
        arr = (ctypes.c_void_p * len(events))(*[int(e.cuda_event) if e is not None else 0
                                                  for e in events])
        c._keep = arr
        c.phase_events = ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p))
    return c


def launch_counter() -> int:
    return int(lib().dfr_launch_counter())


def sort_u32(keys, *, n_d=64, skip_trivial=True, stream=None, stats=False, events=None,
             fused=None, full_lsd=False, fast_radix=False, stable_deals=False):
    """In-place ascending sort of a contiguous CUDA tensor of 32-bit keys (bit
    patterns read as uint32)."""
    _dev_tensor(keys, (4,))
    st = Stats() if stats else None
    rc = lib().dfr_sort_u32_ex(keys.data_ptr(), keys.numel(), _stream(stream),
                               ctypes.byref(_cfg(n_d, skip_trivial, events, fused, full_lsd,
                                                 fast_radix, stable_deals)),
                               ctypes.byref(st) if st is not None else None)
    _check(rc, "dfr_sort_u32")
    return st.as_dict() if st is not None else None


def sort_u64(keys, *, n_d=64, skip_trivial=True, stream=None, stats=False, events=None,
             fused=None, fast_radix=False, stable_deals=False):
    """In-place ascending sort of a contiguous CUDA tensor of 64-bit keys (bit
    patterns read as uint64; int64 tensors are accepted as raw storage)."""
    _dev_tensor(keys, (8,))
    st = Stats() if stats else None
    rc = lib().dfr_sort_u64_ex(keys.data_ptr(), keys.numel(), _stream(stream),
                               ctypes.byref(_cfg(n_d, skip_trivial, events, fused,
                                                 fast_radix=fast_radix,
                                                 stable_deals=stable_deals)),
                               ctypes.byref(st) if st is not None else None)
    _check(rc, "dfr_sort_u64")
    return st.as_dict() if st is not None else None


def sort_pairs_u32(keys, vals, *, n_d=64, skip_trivial=True, stream=None, stats=False,
                   events=None, fused=None, full_lsd=False):
    """Stable in-place sort of (uint32 key, uint32 value) pairs held in two
    contiguous CUDA tensors of equal length."""
    _dev_tensor(keys, (4,))
    _dev_tensor(vals, (4,))
    if keys.numel() != vals.numel():
        raise DfrError("keys and vals differ in length")
    st = Stats() if stats else None
    rc = lib().dfr_sort_pairs_u32_ex(keys.data_ptr(), vals.data_ptr(), keys.numel(),
                                     _stream(stream),
                                     ctypes.byref(_cfg(n_d, skip_trivial, events, fused, full_lsd)),
                                     ctypes.byref(st) if st is not None else None)
    _check(rc, "dfr_sort_pairs_u32")
    return st.as_dict() if st is not None else None


def sort_pairs_u64(keys, vals, *, n_d=64, skip_trivial=True, stream=None, stats=False,
                   events=None, fused=None):
    """Stable in-place sort of (uint64 key, uint64 value) records held in two
    contiguous CUDA tensors of 8-byte elements and equal length."""
    _dev_tensor(keys, (8,))
    _dev_tensor(vals, (8,))
    if keys.numel() != vals.numel():
        raise DfrError("keys and vals differ in length")
    st = Stats() if stats else None
    rc = lib().dfr_sort_pairs_u64_ex(keys.data_ptr(), vals.data_ptr(), keys.numel(),
                                     _stream(stream), ctypes.byref(_cfg(n_d, skip_trivial, events, fused)),
                                     ctypes.byref(st) if st is not None else None)
    _check(rc, "dfr_sort_pairs_u64")
    return st.as_dict() if st is not None else None


def sort(keys, vals=None, **kw):
    """Dispatch on widths: 4-byte keys -> u32 (pairs if ``vals``), 8-byte keys
    -> u64 (pairs with 8-byte ``vals``)."""
    if vals is not None:
        if keys.element_size() == 8:
            return sort_pairs_u64(keys, vals, **kw)
        return sort_pairs_u32(keys, vals, **kw)
    if keys.element_size() == 8:
        return sort_u64(keys, **kw)
    return sort_u32(keys, **kw)


def histogram(keys, digit_lo: int, p: int, *, stream=None):
    """Counts of digits digit_lo..digit_lo+p-1 (radix 256) -> int32 CUDA tensor (p, 256)."""
    import torch
    _dev_tensor(keys, (4, 8))
    out = torch.empty((p, 256), dtype=torch.int32, device=keys.device)
    f = lib().dfr_histogram_u64 if keys.element_size() == 8 else lib().dfr_histogram_u32
    _check(f(keys.data_ptr(), keys.numel(), digit_lo, p, out.data_ptr(), _stream(stream)),
           "dfr_histogram")
    return out


def partition_pass(keys, d: int, vals=None, *, stream=None):
    """One stable counting-sort pass on digit d (out of place); returns (keys, vals)."""
    import torch
    _dev_tensor(keys, (4, 8))
    ko = torch.empty_like(keys)
    if keys.element_size() == 8:
        if vals is not None:
            raise DfrError("pairs pass is u32 only")
        _check(lib().dfr_partition_pass_u64(keys.data_ptr(), ko.data_ptr(), keys.numel(), d,
                                            _stream(stream)), "dfr_partition_pass_u64")
        return ko, None
    vo = torch.empty_like(vals) if vals is not None else None
    _check(lib().dfr_partition_pass_pairs_u32(
        keys.data_ptr(), vals.data_ptr() if vals is not None else None, ko.data_ptr(),
        vo.data_ptr() if vo is not None else None, keys.numel(), d, _stream(stream)),
        "dfr_partition_pass_pairs_u32")
    return ko, vo


def overflow_mc(n: int, m: int, trials: int, key: int, *, stream=None):
    """Fast Radix overflow Monte Carlo (dfr_overflow_mc): int64 CUDA tensor of
    the per-trial overflow sum_i max(0, count_i - ceil(n/m))."""
    import torch
    out = torch.empty(trials, dtype=torch.int64, device="cuda")
    _check(lib().dfr_overflow_mc(n, m, trials, key & ((1 << 64) - 1), out.data_ptr(), _stream(stream)),
           "dfr_overflow_mc")
    return out


def top_passes(n: int, key_bytes: int = 8, n_d: int = 64) -> int:
    return lib().dfr_top_passes(n, key_bytes, n_d)


def workspace_bytes(n: int, key_bytes: int = 8, val_bytes: int = 0) -> int:
    return lib().dfr_workspace_bytes(n, key_bytes, val_bytes)
