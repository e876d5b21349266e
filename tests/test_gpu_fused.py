"""GPU parity of the fused last pass (the deal on the top group digit and the
diversion of the resulting small buckets in one kernel over run-aligned
tiles; Alg. 4 l.6 + l.7-14) against the CPU oracle,
element by element, on inputs built to reach each of its branches:

* uniform u64 / u32 keys at 2^27 (lossy 16-bit composites / exact composites);
* buckets whose keys tie in the 16-bit lossy composite (the exact re-rank);
* level-0 buckets larger than N_d inside a tile (queued for recursion, mid
  and global queue) next to small ones;
* an s-run longer than a tile (the device-side fallback to the separate deal
  and diversion through the third buffer);
* other N_d values (8-bit bucket index; small N_d);
* every bucket's keys in ONE sub-bucket (the work list of sub-buckets of > 4
  keys: several 8-word groups per sub-bucket, distinct and tied top words)."""
import numpy as np
import pytest

import datagen
import oracle
from gpu_util import gpu_sort

pytestmark = pytest.mark.gpu

N = 1 << 27


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _check(k, fused_expected, **kw):
    gk, _, st = gpu_sort(k, stats=True, **kw)
    rk, _, ost = oracle.dfr_sort(k, n_d=kw.get("n_d", 64))
    assert st["overflow"] == 0, st
    assert st["level0_p"] == ost["level0_p"], (st, ost)
    assert st["level0_large"] == ost["level0_large"], (st, ost)
    assert st["fused"] == fused_expected, st
    bad = np.flatnonzero(gk != rk)
    assert bad.size == 0, f"{bad.size} key mismatches, first at {bad[:5]}"
    return st


def test_fused_uniform_u64():
    _check(datagen.uniform_u64(N, 301), 1)


def test_fused_uniform_u32_exact_composites():
    _check(datagen.uniform_u32(N, 302), 1)


def test_fused_ragged_size():
    _check(datagen.uniform_u64(N + 4097, 303), 1)


def test_fused_composite_ties():
    """Within each top-24-bit bucket the next 16 bits take one of three
    values, so the lossy 16-bit composites tie constantly and the ranks come
    from the exact re-rank on the full keys."""
    r = datagen.uniform_u64(N, 304)
    top = r & np.uint64(0xFFFFFF0000000000)
    mid = (r % np.uint64(3)) << np.uint64(24)
    low = (r >> np.uint64(7)) & np.uint64(0xFFFFFF)
    _check(top | mid | low, 1)


def test_fused_large_buckets_in_tiles():
    """Level-0 buckets of 65 .. 2000 keys (> N_d) at distinct (mid, lo) digit
    pairs among uniform keys: the fused kernel writes them and queues them
    (mid buckets on-chip, the rest through the global queue)."""
    k = datagen.uniform_u64(N, 305)
    sizes = [65, 100, 300, 1000, 2000]  # + ~2048 uniform keys per run: <= 4608
    r = datagen.uniform_u64(sum(sizes), 306)
    off = 0
    for i, sz in enumerate(sizes):
        d7, d6, d5 = (0x13 * (i + 1)) & 255, (0x2b * (i + 3)) & 255, (0x31 * (i + 5)) & 255
        pre = np.uint64(d7 << 16 | d6 << 8 | d5)
        k[off * 7:off * 7 + sz] = (pre << np.uint64(40)) | (r[off:off + sz] & np.uint64((1 << 40) - 1))
        off += sz
    st = _check(k, 1)
    assert st["level0_large"] >= len(sizes)


def test_fused_fallback_long_run():
    """One (mid, lo) digit pair holds 6000 keys (> 4608, the longest run a
    fused tile holds): the plan kernel falls back to the separate last deal
    and diversion (B -> C -> A with the second scratch buffer)."""
    k = datagen.uniform_u64(N, 307)
    r = datagen.uniform_u64(6000, 308)
    # top digit random, the two lower group digits fixed, low 40 bits random
    k[:6000] = ((r >> np.uint64(56)) << np.uint64(56)) | (np.uint64(0x4242) << np.uint64(40)) | \
        (r & np.uint64((1 << 40) - 1))
    _check(k, 0)


@pytest.mark.parametrize("n_d", [16, 100, 256])
def test_fused_other_nd(n_d):
    k = datagen.uniform_u64(N, 309)
    _check(k, 1, n_d=n_d)


def test_fused_u32_nd100():
    """u32 keys with an 8-bit bucket index: lossy composites of R = 8 bits."""
    _check(datagen.uniform_u32(N, 310), 1, n_d=100)


@pytest.mark.parametrize("n_d", [64, 256])
def test_fused_long_sub_buckets(n_d):
    """The 3 bits below the group digits are cleared, so the ~16 keys of every
    bucket share one sub-bucket: all ranks come from the work list of
    sub-buckets of > 4 keys (two or more 8-word groups each)."""
    k = datagen.uniform_u64(N, 311) & ~np.uint64(7 << 37)
    _check(k, 1, n_d=n_d)


def test_fused_long_sub_buckets_ties():
    """As above with only 2 distinct values of the composite's top word per
    bucket and random low bits: the rank-sum check of the work list raises the
    tie flag and the tile is re-ranked on the full composites."""
    r = datagen.uniform_u64(N, 312)
    k = (r & np.uint64(0xFFFFFF0000000000)) | ((r >> np.uint64(3)) & np.uint64(1)) << np.uint64(30) | (r & np.uint64(31))
    _check(k, 1)


def test_fused_mixed_sub_bucket_sizes_u32():
    """u32 keys (exact, unique composites) with a skewed sub-bucket split:
    half of the keys of a bucket in one sub-bucket."""
    r = datagen.uniform_u32(N, 313)
    k = np.where(r & np.uint32(1), r & ~np.uint32(7 << 5), r)
    _check(k.astype(np.uint32), 1)
