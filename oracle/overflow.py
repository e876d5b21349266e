"""Overflow model of Fast Radix estimation (§3.1) — TEST
INFRASTRUCTURE ONLY (the oracle package's rules apply: only tests/,
__graft_entry__.smoke() and bench.py may import it).

Fast Radix deals a pass into buckets whose size is ESTIMATED as ceil(N/M)
("each bucket gets capacity ceil(n/m)") instead of counted; a record
whose bucket is full goes to overflow space (Alg. 3).  The paper
models the overflow fraction for uniform inputs with Eq. 1 (a recursion,
P:296) and Eq. 2 (its term).  Eq. 1 has no base case and is
garbled: with g_o(1, M) = 0 (SPEC's reading) it goes
negative; with g_o(1, M) = 1 it is monotone but is not the expectation.

What this module computes, all in float64 / exact integers:
  eq2_term(N, M, k)           Eq. 2 as printed, binomial in log space
  eq1_fraction(N, M, base)    Eq. 1 as printed with an explicit base case
                              -- "parity unpinned" (no independent truth)
  expected_overflow(N, M)     the exact expected overflow fraction of
                              balls-into-bins: E[sum_i max(0, X_i - c)] / N,
                              X_i ~ Binomial(N, 1/M), c = ceil(N/M) -- the
                              quantity Eq. 1 models (reading E6, pinned)
  overflow_mc(N, M, T, key)   T Monte-Carlo trials of that experiment with
                              the SplitMix64 counter-based generator; the
                              GPU kernel (dfr_overflow_mc) implements the
                              same generator independently (parity test)
"""
from __future__ import annotations

import math
from fractions import Fraction
from itertools import product

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def eq2_term(N: int, M: int, k: int) -> float:
    """Eq. 2: (N/M - k) * (M/N) * C(N,k) * (1/M)^k * (1 - 1/M)^(N-k)."""
    if M < 2:
        raise ValueError("Eq. 2 needs M >= 2 (the (1 - 1/M) factor)")
    if not 0 <= k <= N:
        return 0.0
    logp = (math.lgamma(N + 1) - math.lgamma(k + 1) - math.lgamma(N - k + 1)
            - k * math.log(M) + (N - k) * math.log1p(-1.0 / M))
    return (N / M - k) * (M / N) * math.exp(logp)


def eq1_fraction(N: int, M: int, base: float = 1.0) -> float:
    """Eq. 1 evaluated as printed: g(n) = g(n-1) - (1/M) g_o(n-1, M,
    ceil(n/M) - 1), g(1) = base (the paper gives no base case).  PARITY
    UNPINNED: nothing independent fixes the recursion's value."""
    g = base
    for n in range(2, N + 1):
        g = g - eq2_term(n - 1, M, -(-n // M) - 1) / M
    return g


def _binom_pmf(N: int, M: int) -> np.ndarray:
    x = np.arange(N + 1, dtype=np.float64)
    lg = np.array([math.lgamma(v + 1) for v in range(N + 1)])
    logp = lg[N] - lg - lg[::-1] + x * math.log(1.0 / M) + (N - x) * math.log1p(-1.0 / M)
    return np.exp(logp)


def expected_overflow(N: int, M: int) -> float:
    """E[sum over the M buckets of max(0, X_i - ceil(N/M))] / N with the
    bucket occupancies X_i ~ Binomial(N, 1/M) (linearity of expectation:
    M times one bucket's expected excess)."""
    if N <= 0 or M == 1:
        return 0.0
    c = -(-N // M)
    pmf = _binom_pmf(N, M)
    x = np.arange(N + 1, dtype=np.float64)
    excess = np.clip(x - c, 0.0, None)
    return float(M * np.dot(excess, pmf) / N)


def expected_overflow_bruteforce(N: int, M: int) -> Fraction:
    """The same expectation by enumerating all M^N assignments (tiny N, M)."""
    c = -(-N // M)
    total = Fraction(0)
    for a in product(range(M), repeat=N):
        cnt = [0] * M
        for b in a:
            cnt[b] += 1
        total += sum(max(0, x - c) for x in cnt)
    return total / (M ** N) / N


def _mix(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(0xBF58476D1CE4E5B9)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def overflow_mc(N: int, M: int, trials: int, key: int) -> np.ndarray:
    """Per-trial total overflow sum_i max(0, count_i - ceil(N/M)): trial t draws
    stream key k_t = mix(key + (t+1)*GAMMA); ball b goes to bucket
    floor(hi32(mix(k_t + (b+1)*GAMMA)) * M / 2^32)."""
    c = -(-N // M)
    out = np.empty(trials, np.uint64)
    with np.errstate(over="ignore"):
        g = np.uint64(GAMMA)
        tk = _mix(np.uint64(key) + (np.arange(trials, dtype=np.uint64) + np.uint64(1)) * g)
        b = np.arange(N, dtype=np.uint64) + np.uint64(1)
        for t in range(trials):
            r = _mix(tk[t] + b * g)
            bins = ((r >> np.uint64(32)) * np.uint64(M)) >> np.uint64(32)
            cnt = np.bincount(bins.astype(np.int64), minlength=M)
            out[t] = np.clip(cnt - c, 0, None).sum()
    return out
