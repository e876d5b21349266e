"""The Fast Radix overflow model (§3.1 Eq. 1 / Eq. 2, P:292-306;
SURVEY §8(f) NEXT-4): the oracle (oracle/overflow.py) pinned against brute
force, closed forms and an independent generator implementation, and the GPU
Monte Carlo (dfr_overflow_mc) checked trial by trial against the oracle's."""
import math

import numpy as np
import pytest

import datagen
from oracle import overflow as ov


# ------------------------------------------------------------------ CPU pins
def test_eq2_worked_example_and_zero():
    # (N=4, M=2, k=1) -> 1 * 0.5 * 4 * 0.5 * 0.125 = 0.125
    assert ov.eq2_term(4, 2, 1) == pytest.approx(0.125, rel=1e-12)
    # the leading factor (N/M - k) vanishes at k = N/M
    for n, m in [(512, 256), (1024, 256), (96, 3)]:
        assert ov.eq2_term(n, m, n // m) == 0.0
    # sign of the leading factor (SPEC property)
    assert ov.eq2_term(1000, 256, 2) > 0 and ov.eq2_term(1000, 256, 6) < 0
    with pytest.raises(ValueError):
        ov.eq2_term(10, 1, 3)


@pytest.mark.parametrize("n,m", [(1, 2), (2, 2), (3, 2), (4, 2), (5, 2), (4, 3), (6, 3), (4, 4),
                                 (5, 4), (7, 2), (3, 5)])
def test_expected_overflow_equals_bruteforce(n, m):
    """Exact expectation vs enumeration of all m^n assignments."""
    assert ov.expected_overflow(n, m) == pytest.approx(float(ov.expected_overflow_bruteforce(n, m)),
                                                       rel=1e-12, abs=1e-15)


def test_expected_overflow_special_cases():
    assert ov.expected_overflow(0, 256) == 0.0
    assert ov.expected_overflow(1, 256) == 0.0      # capacity 1, at most one record per bucket
    assert ov.expected_overflow(1000, 1) == 0.0     # one bucket holds everything
    # n = m: capacity 1, the excess of a bucket is X - 1 when X >= 1
    n = m = 64
    p0 = (1 - 1 / m) ** n
    assert ov.expected_overflow(n, m) == pytest.approx(m * (1.0 - (1 - p0)) / n, rel=1e-12)


@pytest.mark.parametrize("n,m", [(1 << 20, 256), (1 << 22, 256), (1 << 24, 64)])
def test_expected_overflow_normal_limit(n, m):
    """Large N: X ~ Normal(mu, sigma^2); E[max(0, X - c)] = sigma*phi(z) - (c - mu)*(1 - Phi(z))."""
    mu, c = n / m, -(-n // m)
    sigma = math.sqrt(n / m * (1 - 1 / m))
    z = (c - mu) / sigma
    e = sigma * math.exp(-z * z / 2) / math.sqrt(2 * math.pi) - (c - mu) * 0.5 * math.erfc(z / math.sqrt(2))
    assert ov.expected_overflow(n, m) == pytest.approx(m * e / n, rel=2e-3)


def test_expected_overflow_monotone_and_small():
    vals = [ov.expected_overflow(n, 256) for n in (1000, 1 << 12, 1 << 16, 1 << 20)]
    assert all(a > b for a, b in zip(vals, vals[1:]))
    assert vals[-1] < 0.01


def test_generator_matches_datagen():
    """The oracle's numpy SplitMix64 equals datagen's C implementation."""
    key = datagen.stream_key(7, "overflow-mc")
    with np.errstate(over="ignore"):
        i = np.arange(1000, dtype=np.uint64)
        mine = ov._mix(np.uint64(key) + (i + np.uint64(1)) * np.uint64(ov.GAMMA))
    ref = np.array([datagen.draw(key, int(x)) for x in i], dtype=np.uint64)
    assert (mine == ref).all()


def test_mc_oracle_agrees_with_expectation():
    n, m, trials = 1000, 256, 3000
    o = ov.overflow_mc(n, m, trials, datagen.stream_key(8, "overflow-mc")).astype(np.float64)
    mean, se = o.mean() / n, o.std(ddof=1) / math.sqrt(trials) / n
    assert abs(mean - ov.expected_overflow(n, m)) < 4 * se


def test_eq1_as_printed():
    """Eq. 1 has no base case: with g(1) = 0 (SPEC's reading) it
    is negative at once; with g(1) = 1 it decreases monotonically (P:302
    "clearly monotonically decreasing").  Its value is parity unpinned."""
    assert ov.eq1_fraction(2, 2, base=0.0) < 0
    g = [ov.eq1_fraction(n, 256, base=1.0) for n in range(2, 600, 37)]
    assert all(a >= b for a, b in zip(g, g[1:]))


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("n,m,trials", [(1000, 256, 64), (4096, 16, 40), (10007, 7, 9),
                                        (50000, 16384, 5), (1, 3, 4), (300000, 256, 3)])
def test_gpu_mc_trials_bit_exact(n, m, trials):
    import torch
    import paper_2207_14334_b200 as dfr
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    key = datagen.stream_key(9, f"overflow-mc-{n}-{m}")
    g = dfr.overflow_mc(n, m, trials, key).cpu().numpy().view(np.uint64)
    r = ov.overflow_mc(n, m, trials, key)
    assert (g == r).all(), (g[:8], r[:8])


@pytest.mark.gpu
def test_gpu_mc_headline_pass_overflow():
    """The overflow an estimated 256-way pass of 2^20 uniform records sees:
    the GPU Monte Carlo mean within 4 standard errors of the exact expectation."""
    import torch
    import paper_2207_14334_b200 as dfr
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    n, m, trials = 1 << 20, 256, 2048
    o = dfr.overflow_mc(n, m, trials, datagen.stream_key(10, "overflow-mc")).double().cpu().numpy()
    mean, se = o.mean() / n, o.std(ddof=1) / math.sqrt(trials) / n
    assert abs(mean - ov.expected_overflow(n, m)) < 4 * se


@pytest.mark.gpu
def test_gpu_mc_rejects_bad_arguments():
    import torch
    import paper_2207_14334_b200 as dfr
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    L = dfr.lib()
    out = torch.empty(4, dtype=torch.int64, device="cuda")
    assert L.dfr_overflow_mc(100, 0, 4, 1, out.data_ptr(), None) == dfr.DFR_ERR_INVALID
    assert L.dfr_overflow_mc(100, 16385, 4, 1, out.data_ptr(), None) == dfr.DFR_ERR_INVALID
    assert L.dfr_overflow_mc(100, 16, 4, 1, None, None) == dfr.DFR_ERR_INVALID
    assert L.dfr_overflow_mc(100, 16, 0, 1, None, None) == dfr.DFR_OK
