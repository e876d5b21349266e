"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element
by element, bit-exact (integer work: SURVEY §8(c)/(d))."""
import numpy as np
import pytest

import datagen
import oracle
from gpu_util import gpu_sort, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


# ------------------------------------------------------------------ stages
@pytest.mark.parametrize("n", [1, 100, 4096, 4097, 3 * 4096 + 17, 1 << 20, (1 << 20) + 3])
def test_histogram_u64(n):
    import paper_2207_14334_b200 as dfr
    k = datagen.uniform_u64(n, 21)
    for lo, p in ((5, 3), (0, 4), (4, 4), (7, 1)):
        h = dfr.histogram(to_dev(k), lo, p).cpu().numpy().astype(np.uint32)
        assert (h == oracle.hist(k, lo, p)).all(), (lo, p)


@pytest.mark.parametrize("n", [100, 4097, (1 << 18) + 5])
def test_histogram_u32_skewed(n):
    import paper_2207_14334_b200 as dfr
    for k in (datagen.uniform_u32(n, 22), datagen.const_u32(n, 22), datagen.few_unique_u32(n, 22, 3)):
        h = dfr.histogram(to_dev(k), 0, 4).cpu().numpy().astype(np.uint32)
        assert (h == oracle.hist(k, 0, 4)).all()


@pytest.mark.parametrize("n", [1, 33, 4096, 4097, 5 * 4096 + 1000, (1 << 20) + 7])
def test_partition_pass(n):
    import paper_2207_14334_b200 as dfr
    k = datagen.uniform_u64(n, 23)
    for d in (0, 5, 7):
        out, _ = dfr.partition_pass(to_dev(k), d)
        ref, _ = oracle.counting_pass(k, d)
        assert (to_host(out, np.uint64) == ref).all(), d
    k32 = datagen.few_unique_u32(n, 24, 5)
    v = np.arange(n, dtype=np.uint32)
    for d in (0, 3):
        ko, vo = dfr.partition_pass(to_dev(k32), d, to_dev(v))
        rk, rv = oracle.counting_pass(k32, d, v)
        assert (to_host(ko, np.uint32) == rk).all() and (to_host(vo, np.uint32) == rv).all()


# ------------------------------------------------------------------ end to end
SIZES = [0, 1, 2, 3, 63, 64, 65, 200, 4095, 4096, 4097, 12345, 65536, 100003, (1 << 20) + 11]


@pytest.mark.parametrize("n", SIZES)
def test_sort_u64_uniform(n):
    k = datagen.uniform_u64(n, 31 + n)
    out, _, _ = gpu_sort(k)
    ref, _, _ = oracle.dfr_sort(k)
    assert (out == ref).all()


@pytest.mark.parametrize("n", SIZES)
def test_sort_u32_uniform(n):
    k = datagen.uniform_u32(n, 41 + n)
    out, _, _ = gpu_sort(k)
    ref, _, _ = oracle.dfr_sort(k)
    assert (out == ref).all()


@pytest.mark.parametrize("n", SIZES)
def test_sort_pairs_few_unique(n):
    k = datagen.few_unique_u32(n, 51 + n, 16)
    v = np.arange(n, dtype=np.uint32)
    ok, ov, _ = gpu_sort(k, v)
    rk, rv, _ = oracle.dfr_sort(k, v)
    assert (ok == rk).all() and (ov == rv).all()


@pytest.mark.parametrize("case", sorted(datagen.CASES))
@pytest.mark.parametrize("n", [50000, (1 << 21) + 999])
def test_config_recipes_small(case, n):
    """Every BASELINE config recipe at oracle-friendly sizes (several tiles + ragged tail)."""
    k, v = datagen.make_case(case, n)
    ok, ov, _ = gpu_sort(k, v)
    rk, rv, _ = oracle.dfr_sort(k, v)
    assert (ok == rk).all()
    if v is not None:
        assert (ov == rv).all()


@pytest.mark.parametrize("n_d", [8, 16, 64, 100, 256])
def test_nd_sweep(n_d):
    for name in ("c3-normal", "c3-zipf", "c5-uniform", "c4-few"):
        k, v = datagen.make_case(name, 300001)
        ok, ov, _ = gpu_sort(k, v, n_d=n_d)
        rk, rv, _ = oracle.dfr_sort(k, v, n_d=n_d)
        assert (ok == rk).all(), name
        if v is not None:
            assert (ov == rv).all(), name


def test_no_pass_skipping_same_bytes():
    for name in ("c4-equal", "c5-low20", "c3-exp"):
        k, v = datagen.make_case(name, 200000)
        a = gpu_sort(k, v, skip_trivial=False)
        b = gpu_sort(k, v, skip_trivial=True)
        rk, rv, _ = oracle.dfr_sort(k, v)
        assert (a[0] == rk).all() and (b[0] == rk).all(), name


def test_degenerate_inputs():
    n = 1 << 20
    base = datagen.uniform_u64(n, 61)
    for k in (np.sort(base), np.sort(base)[::-1].copy(), np.full(n, 7, np.uint64),
              np.zeros(n, np.uint64), np.full(n, 2 ** 64 - 1, np.uint64),
              (base & np.uint64(0xFF00000000000000)).copy(), (base & np.uint64(0xFF)).copy()):
        out, _, _ = gpu_sort(k)
        assert (out == np.sort(k)).all()
    v = np.arange(n, dtype=np.uint32)
    k32 = np.full(n, 123, np.uint32)
    ok, ov, _ = gpu_sort(k32, v)
    assert (ov == v).all()


def test_unaligned_views():
    """Caller pointers with only natural alignment (scalar load path)."""
    import torch
    import paper_2207_14334_b200 as dfr
    n = 100001
    k = datagen.uniform_u64(n + 1, 71)
    t = to_dev(k)
    view = t[1:]
    dfr.sort(view)
    torch.cuda.synchronize()
    out = to_host(t, np.uint64)
    assert out[0] == k[0] and (out[1:] == np.sort(k[1:])).all()
    k32 = datagen.few_unique_u32(n + 3, 72, 9)
    v = np.arange(n + 3, dtype=np.uint32)
    tk, tv = to_dev(k32), to_dev(v)
    dfr.sort(tk[3:], tv[1:n + 1])
    torch.cuda.synchronize()
    rk, rv, _ = oracle.dfr_sort(k32[3:].copy(), v[1:n + 1].copy())
    assert (to_host(tk, np.uint32)[3:] == rk).all() and (to_host(tv, np.uint32)[1:n + 1] == rv).all()


def test_stats_level0_structure():
    k, _ = datagen.make_case("c1")
    _, _, st = gpu_sort(k, stats=True)
    _, _, ost = oracle.dfr_sort(k)
    assert st["level0_p"] == ost["level0_p"] == 2
    assert st["level0_large"] == ost["level0_large"] == 0
    assert st["overflow"] == 0  # no queue overflow
    k, _ = datagen.make_case("c3-zipf", 1 << 20)
    _, _, st = gpu_sort(k, stats=True)
    _, _, ost = oracle.dfr_sort(k)
    assert st["level0_p"] == ost["level0_p"]
    assert st["level0_large"] == ost["level0_large"]
    assert st["overflow"] == 0


def test_stream_and_repeat():
    """Two calls on a side stream; results identical (deterministic)."""
    import torch
    import paper_2207_14334_b200 as dfr
    k = datagen.uniform_u64(1 << 20, 81)
    s = torch.cuda.Stream()
    a, b = to_dev(k), to_dev(k)
    with torch.cuda.stream(s):
        dfr.sort(a)
        dfr.sort(b, stream=s)
    s.synchronize()
    assert (to_host(a, np.uint64) == to_host(b, np.uint64)).all()
    assert (to_host(a, np.uint64) == np.sort(k)).all()


def test_divert_tie_fallback():
    """u64 buckets whose keys share the top 24 of their remaining 40 bits and
    differ only below: the 16-bit lossy rank composites tie, and the exact
    re-rank of the diversion (full keys, index tie-break) must restore the order."""
    rng = np.random.default_rng(5)
    n = 300000
    prefix = rng.integers(0, 6000, n, dtype=np.uint64) << np.uint64(40)      # ~50 per bucket
    mid = rng.integers(0, 3, n, dtype=np.uint64) << np.uint64(16)            # few top-24 values
    low = rng.integers(0, 1 << 16, n, dtype=np.uint64)
    k = prefix | mid | low
    out, _, st = gpu_sort(k, stats=True)
    ref, _, ost = oracle.dfr_sort(k)
    assert (out == ref).all()
    assert st["overflow"] == 0
