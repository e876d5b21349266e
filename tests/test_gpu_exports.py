"""GPU parity of every required export in the configurations the level-0 kernels
reach only at larger sizes, each compared element by element with the CPU
oracle on the same seeded input:

* u32 keys and (u32 key, u32 index) pairs with distinct keys at n = 2^23 and
  2^27: p = 3 (Alg. 4 l.4), so the diversion sees R = 8 remaining
  bits -- the exact-composite mode of the stand-alone k_divert, for keys and
  for pairs (stability);
* N_d = 100 on u32 keys above 100 * 2^16: p = 3 with an 8-bit bucket index, the
  lossy composite with R = 8;
* the three plain entry points (no _ex) on device data;
* two sorts running at once on two distinct streams (dfr.h: reentrant)."""
import ctypes

import numpy as np
import pytest

import datagen
import oracle
import paper_2207_14334_b200 as dfr
from gpu_util import gpu_sort, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _same(a, b, what):
    bad = np.flatnonzero(a != b)
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first at {bad[:5]}"


@pytest.mark.parametrize("n", [1 << 23, (1 << 23) + 12345, 1 << 27])
def test_u32_keys_distinct_p3(n):
    k = datagen.uniform_u32(n, 201)
    assert dfr.top_passes(n, 4, 64) == 3
    gk, _, st = gpu_sort(k, stats=True)
    rk, _, ost = oracle.dfr_sort(k)
    assert st["level0_p"] == ost["level0_p"] == 3 and st["overflow"] == 0
    _same(gk, rk, "keys")
    if n >= 1 << 27:  # the separate stand-alone deal + diversion as well
        gk, _, st = gpu_sort(k, stats=True, fused=False)
        assert st["fused"] == 0
        _same(gk, rk, "keys (separate last pass)")


@pytest.mark.parametrize("n", [1 << 23, (1 << 23) + 777, 1 << 27])
def test_u32_pairs_distinct_p3(n):
    k = datagen.uniform_u32(n, 202)
    v = np.arange(n, dtype=np.uint32)
    gk, gv, st = gpu_sort(k, v, stats=True)
    rk, rv, ost = oracle.dfr_sort(k, v)
    assert st["level0_p"] == ost["level0_p"] == 3 and st["overflow"] == 0
    _same(gk, rk, "keys")
    _same(gv, rv, "values (stability)")


@pytest.mark.parametrize("pairs", [False, True])
def test_u32_nd100_lossy_r8(pairs):
    n = 100 * (1 << 16) + 4321
    k = datagen.uniform_u32(n, 203)
    v = np.arange(n, dtype=np.uint32) if pairs else None
    assert dfr.top_passes(n, 4, 100) == 3
    gk, gv, st = gpu_sort(k, v, stats=True, n_d=100)
    rk, rv, ost = oracle.dfr_sort(k, v, n_d=100)
    assert st["level0_p"] == ost["level0_p"] == 3
    _same(gk, rk, "keys")
    if pairs:
        _same(gv, rv, "values")


def test_plain_exports_on_device_data():
    """dfr_sort_u32 / dfr_sort_u64 / dfr_sort_pairs_u32 (no config, no stats)
    called through ctypes on torch device memory, on the legacy stream 0 and on
    a created stream."""
    import torch
    L = dfr.lib()
    n = (1 << 22) + 9
    k64 = datagen.uniform_u64(n, 204)
    k32 = datagen.uniform_u32(n, 205)
    kp, vp = datagen.make_case("c4-few", n)
    t64, t32 = to_dev(k64), to_dev(k32)
    tk, tv = to_dev(kp), to_dev(vp)
    torch.cuda.synchronize()
    assert L.dfr_sort_u64(t64.data_ptr(), n, None) == 0
    s = torch.cuda.Stream()
    assert L.dfr_sort_u32(t32.data_ptr(), n, s.cuda_stream) == 0
    assert L.dfr_sort_pairs_u32(tk.data_ptr(), tv.data_ptr(), n, s.cuda_stream) == 0
    torch.cuda.synchronize()
    _same(to_host(t64, np.uint64), oracle.dfr_sort(k64)[0], "u64")
    _same(to_host(t32, np.uint32), oracle.dfr_sort(k32)[0], "u32")
    rk, rv, _ = oracle.dfr_sort(kp, vp)
    _same(to_host(tk, np.uint32), rk, "pairs keys")
    _same(to_host(tv, np.uint32), rv, "pairs values")


def test_concurrent_streams():
    """Two sorts in flight at once on two distinct streams (each call owns its
    workspace and control block; dfr.h: reentrant)."""
    import torch
    n = (1 << 24) + 5
    ka = datagen.uniform_u64(n, 206)
    kb, vb = datagen.make_case("c4-few", n)
    ta, tb, tvb = to_dev(ka), to_dev(kb), to_dev(vb)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):  # several rounds so that the two streams overlap
        a, b, bv = ta.clone(), tb.clone(), tvb.clone()
        torch.cuda.synchronize()
        dfr.sort(a, stream=s1)
        dfr.sort(b, bv, stream=s2)
        torch.cuda.synchronize()
        _same(to_host(a, np.uint64), np.sort(ka), "stream 1 (u64)")
        rk, rv, _ = oracle.dfr_sort(kb, vb)
        _same(to_host(b, np.uint32), rk, "stream 2 keys")
        _same(to_host(bv, np.uint32), rv, "stream 2 values")


@pytest.mark.parametrize("case,n", [("uniform", 1000), ("uniform", 300007), ("uniform", (1 << 21) + 3),
                                    ("uniform", (1 << 22) + 5), ("uniform", 1 << 24),
                                    ("few", (1 << 22) + 1), ("zipf", 1 << 22), ("equal", 100003)])
def test_u64_pairs(case, n):
    """dfr_sort_pairs_u64: (u64 key, u64 tag) records (SPEC's Record),
    stable: equal keys keep input order; keys and tags bit-exact vs the
    oracle's pairs sort."""
    if case == "uniform":
        k = datagen.uniform_u64(n, 211)
    elif case == "few":
        k = datagen.uniform_u64(256, 212)[datagen.uniform_u64(n, 213) >> np.uint64(56)]
    elif case == "zipf":
        k = datagen.zipf_u64(n, 214)
    else:
        k = np.full(n, 0x0123456789ABCDEF, np.uint64)
    v = datagen.uniform_u64(n, 215, "tags")
    gk, gv, st = gpu_sort(k, v, stats=True)
    rk, rv, _ = oracle.dfr_sort(k, v)
    assert st["overflow"] == 0
    _same(gk, rk, "keys")
    _same(gv, rv, "values (stability)")


@pytest.mark.parametrize("n", [(1 << 20) + 7, (1 << 23) + 3])
def test_full_lsd_ablation_u32(n):
    """dfr_config.full_lsd (SPEC AC7): the top call is a plain LSD sort
    over all four digits -- the same output as DFR (keys and stable pairs)."""
    k = datagen.uniform_u32(n, 221)
    gk, _, st = gpu_sort(k, stats=True, full_lsd=True)
    assert st["level0_p"] == 4
    _same(gk, oracle.dfr_sort(k)[0], "keys")
    kp, vp = datagen.make_case("c4-few", n)
    gk, gv, st = gpu_sort(kp, vp, stats=True, full_lsd=True)
    rk, rv, _ = oracle.dfr_sort(kp, vp)
    _same(gk, rk, "pair keys")
    _same(gv, rv, "pair values")
