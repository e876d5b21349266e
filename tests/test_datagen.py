"""Input generator checks: published SplitMix64 vectors, determinism, and the
distribution shapes BASELINE.json asks for."""
import math

import numpy as np

import datagen

GAMMA = 0x9E3779B97F4A7C15


def test_splitmix64_reference_vectors():
    # SplitMix64 reference outputs (Steele/Lea/Flood; the xoshiro seeding
    # generator): state 0 -> first output 0xE220A8397B1DCDAF; state 1234567 ->
    # 6457827717110365317, 3203168211198807973.
    k0 = 0
    assert datagen.draw(k0, 0) == 0xE220A8397B1DCDAF
    assert datagen.draw(1234567, 0) == 6457827717110365317
    assert datagen.draw(1234567, 1) == 3203168211198807973


def test_determinism_and_streams():
    a = datagen.uniform_u64(1000, 5)
    b = datagen.uniform_u64(1000, 5)
    c = datagen.uniform_u64(1000, 6)
    assert (a == b).all() and not (a == c).all()
    key = datagen.stream_key(5, "base")
    assert int(a[17]) == datagen.draw(key, 17)


def test_uniform_bytes_chi_squared():
    k = datagen.uniform_u64(1 << 20, 2)
    for d in range(8):
        h = np.bincount(((k >> np.uint64(8 * d)) & np.uint64(255)).astype(np.int64), minlength=256)
        e = k.size / 256
        chi = ((h - e) ** 2 / e).sum()
        assert chi < 400, (d, chi)  # 255 dof; p ~ 1e-8 at 400


def test_normal_moments_and_clamp():
    n = 1 << 20
    k = datagen.normal_u64(n, 3, 1 << 63, 2.0 ** 40)
    z = (k.astype(np.float64) - 2.0 ** 63) / 2.0 ** 40
    assert abs(z.mean()) < 5 / math.sqrt(n)
    assert abs(z.std() - 1) < 0.01
    # keys are integers, not quantised to ulp(2^63) = 2048
    assert (k % np.uint64(2048) != 0).mean() > 0.9
    # clamping at the edges with a huge sd
    w = datagen.normal_u64(4096, 3, 1 << 63, 2.0 ** 66)
    assert (w == np.uint64(0)).any() and (w == np.uint64(2 ** 64 - 1)).any()


def test_exponential_mean():
    n = 1 << 20
    k = datagen.exponential_u64(n, 3, 2.0 ** 32)
    m = k.astype(np.float64).mean() / 2.0 ** 32
    assert abs(m - 1) < 5 / math.sqrt(n)


def test_zipf_rank1_frequency():
    n = 1 << 20
    k = datagen.zipf_u64(n, 3, 1.1, 1 << 20)
    H = sum(r ** -1.1 for r in range(1, (1 << 20) + 1))
    vals, cnt = np.unique(k, return_counts=True)
    p1 = cnt.max() / n
    se = math.sqrt((1 / H) * (1 - 1 / H) / n)
    assert abs(p1 - 1 / H) < 4 * se
    assert vals.size <= 1 << 20


def test_few_unique_and_equal():
    k = datagen.few_unique_u32(1 << 18, 4, 256)
    assert np.unique(k).size == 256
    e = datagen.const_u32(1000, 4)
    assert (e == e[0]).all()


def test_layouts():
    n = 1 << 16
    base = datagen.uniform_u64(n, 5)
    s = datagen.sort_asc_u64(base.copy())
    assert (s == np.sort(base)).all()
    r = datagen.reverse_u64(s.copy())
    assert (r == s[::-1]).all()
    nearly = datagen.transpose_u64(s.copy(), 5, n // 200)
    moved = (nearly != s).mean()
    assert 0.002 < moved < 0.02  # ~1% of positions displaced
    runs = datagen.sort_runs_u64(base.copy(), 4096)
    for b in range(0, n, 4096):
        assert (np.diff(runs[b:b + 4096].astype(np.float64)) >= 0).all()
    assert datagen.fingerprint(runs) == datagen.fingerprint(base)
    assert datagen.is_sorted(s) and not datagen.is_sorted(base)


def test_make_case_small():
    for name in datagen.CASES:
        k, v = datagen.make_case(name, 4096)
        assert k.size == 4096
        c = datagen.CASES[name]
        assert k.dtype == (np.uint64 if c.key_dtype == "u64" else np.uint32)
        assert (v is not None) == c.pairs
