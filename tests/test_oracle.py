"""Pins for the CPU oracle (oracle/), independent of the oracle itself.

Every check compares the oracle with something other than its own code:
worked examples (tests/golden/spec_examples.txt, each cited), numpy's stable
sort / bincount (library routines that define the result DFR must reach, since
DFR is stable end to end — SURVEY §8(c)), brute-force enumeration on tiny
inputs, and control-flow counts derived by hand from Alg. 4.
"""
import itertools
import os
import re

import numpy as np
import pytest

import datagen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.txt")


def _stable_ref(keys, vals=None):
    idx = np.argsort(keys, kind="stable")
    return keys[idx], (None if vals is None else vals[idx])


# ---------------------------------------------------------------- golden pins
def _golden():
    for line in open(GOLDEN):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        lhs, rhs = line.split("->")
        op, *args = lhs.split()
        yield op, args, rhs.strip()


def test_golden_examples():
    n = 0
    for op, args, rhs in _golden():
        n += 1
        if op == "extract_digit":
            assert oracle.extract_digit(int(args[0], 16), int(args[1]), int(args[2])) == int(rhs, 16)
        elif op == "prefix_sum_exclusive":
            counts = [int(x) for x in args[0].split(",")]
            assert list(oracle.prefix_sum_exclusive(counts)) == [int(x) for x in rhs.split(",")]
        elif op == "est_top_passes":
            assert oracle.est_top_passes(int(args[0]), int(args[1]), int(args[2])) == int(rhs)
        elif op == "insertion_sort":
            pairs = [a.split(":") for a in args[0].split(",")]
            k = np.array([int(a) for a, _ in pairs], np.uint64)
            v = np.array([ord(b) for _, b in pairs], np.uint64)
            ok, ov = oracle.insertion_sort_pairs_u64(k, v)
            exp = [a.split(":") for a in rhs.split(",")]
            assert list(ok) == [int(a) for a, _ in exp]
            assert list(ov) == [ord(b) for _, b in exp]
        elif op == "lsd_sort":
            k = np.array([int(x, 16) for x in args[0].split(",")], np.uint64)
            out, _, _ = oracle.dfr_sort(k, n_d=1)  # N_d=1 forces the radix passes
            assert list(out) == [int(x, 16) for x in rhs.split(",")]
        elif op == "dfr_stats_n50":
            nn, nd = int(args[0]), int(args[1])
            k = datagen.uniform_u64(nn, 7)
            _, _, st = oracle.dfr_sort(k, n_d=nd)
            exp = dict(kv.split("=") for kv in rhs.split(","))
            for key, val in exp.items():
                assert st[key] == int(val), (key, st)
        else:
            raise AssertionError(op)
    assert n >= 13


# ------------------------------------------------------------ pass estimate
def test_est_top_passes_definition_and_configs():
    # defining property: least p >= 0 with n <= N_d * M^p
    rng = np.random.default_rng(0)
    for n in list(range(0, 300)) + [int(x) for x in rng.integers(1, 1 << 40, 500)]:
        for nd in (2, 16, 64, 1024):
            p = oracle.est_top_passes(n, 8, nd)
            assert n <= nd * 256 ** p
            assert p == 0 or n > nd * 256 ** (p - 1)
    # p per BASELINE config
    assert oracle.est_top_passes(1 << 16) == 2
    for lg in (24, 26, 27, 28):
        assert oracle.est_top_passes(1 << lg) == 3
    # boundaries: p = 1 for 64 < n <= 2^14, 2 for <= 2^22, 3 for <= 2^30
    assert oracle.est_top_passes(64) == 0 and oracle.est_top_passes(65) == 1
    assert oracle.est_top_passes(1 << 14) == 1 and oracle.est_top_passes((1 << 14) + 1) == 2
    assert oracle.est_top_passes(1 << 30) == 3 and oracle.est_top_passes((1 << 30) + 1) == 4


# ------------------------------------------------------------------ stages
@pytest.mark.parametrize("dtype", [np.uint32, np.uint64])
def test_hist_matches_bincount(dtype):
    k = datagen.uniform_u64(5000, 11).astype(dtype) if dtype == np.uint64 else datagen.uniform_u32(5000, 11)
    D = k.dtype.itemsize
    h = oracle.hist(k, 0, D)
    assert h.sum() == k.size * D
    for d in range(D):
        ref = np.bincount(((k >> np.array(8 * d, k.dtype)) & np.array(255, k.dtype)).astype(np.int64),
                          minlength=256)
        assert (h[d] == ref).all()


def test_counting_pass_is_stable_sort_by_digit():
    k = datagen.uniform_u64(4097, 12)
    for d in range(8):
        out, _ = oracle.counting_pass(k, d)
        dig = (k >> np.uint64(8 * d)) & np.uint64(255)
        assert (out == k[np.argsort(dig, kind="stable")]).all()
    k32 = datagen.few_unique_u32(3000, 4, 7)
    v = np.arange(3000, dtype=np.uint32)
    ok, ov = oracle.counting_pass(k32, 1, v)
    idx = np.argsort((k32 >> 8) & 255, kind="stable")
    assert (ok == k32[idx]).all() and (ov == v[idx]).all()


def test_group_is_stable_sort_by_top_prefix():
    k = datagen.uniform_u64(1 << 16, 13)
    out, _, p = oracle.group(k)
    assert p == 2
    idx = np.argsort(k >> np.uint64(48), kind="stable")
    assert (out == k[idx]).all()
    k32 = datagen.uniform_u32(1 << 15, 14)
    v = np.arange(k32.size, dtype=np.uint32)
    ok, ov, p = oracle.group(k32, v)
    assert p == 2
    idx = np.argsort(k32 >> 16, kind="stable")
    assert (ok == k32[idx]).all() and (ov == v[idx]).all()


# ----------------------------------------------------- end-to-end vs stable
def _inputs(n, seed):
    yield "uniform64", datagen.uniform_u64(n, seed)
    yield "uniform32", datagen.uniform_u32(n, seed)
    yield "few32", datagen.few_unique_u32(n, seed, 16)
    yield "equal32", datagen.const_u32(n, seed)
    yield "normal64", datagen.normal_u64(n, seed, 1 << 63, 2.0 ** 40)
    yield "exp64", datagen.exponential_u64(n, seed, 2.0 ** 32)
    yield "zipf64", datagen.zipf_u64(n, seed, 1.1, 1 << 12)
    yield "low20", datagen.lowbits_u64(n, seed, 20)


@pytest.mark.parametrize("n", [0, 1, 2, 10, 63, 64, 65, 1000, 20000, 100003])
@pytest.mark.parametrize("n_d", [2, 16, 64, 256])
def test_dfr_equals_stable_sort(n, n_d):
    for name, k in _inputs(n, 100 + n):
        out, _, st = oracle.dfr_sort(k, n_d=n_d)
        assert (out == np.sort(k, kind="stable")).all(), name
        assert st["max_depth"] <= k.itemsize * 8 // 8, name  # digit budget
        # with pairs (payload = index) the result must be THE stable sort
        if k.dtype == np.uint32:
            v = np.arange(n, dtype=np.uint32)
            ok, ov, _ = oracle.dfr_sort(k, v, n_d=n_d)
            rk, rv = _stable_ref(k, v)
            assert (ok == rk).all() and (ov == rv).all(), name
        else:
            v = np.arange(n, dtype=np.uint64)
            ok, ov, _ = oracle.dfr_sort(k, v, n_d=n_d)
            rk, rv = _stable_ref(k, v)
            assert (ok == rk).all() and (ov == rv).all(), name


@pytest.mark.parametrize("radix_bits", [4, 16])
def test_dfr_other_radix(radix_bits):
    for name, k in _inputs(30000, 5):
        v = np.arange(k.size, dtype=np.uint64 if k.dtype == np.uint64 else np.uint32)
        ok, ov, _ = oracle.dfr_sort(k, v, n_d=16, radix_bits=radix_bits)
        rk, rv = _stable_ref(k, v)
        assert (ok == rk).all() and (ov == rv).all(), name


def test_exhaustive_tiny_sequences():
    """Every sequence of length <= 5 over a 7-key alphabet built to share
    prefixes, with N_d in {2,3}, radix in {4,8}: forces multi-level recursion,
    bulk runs and exhausted-digit buckets (SURVEY §8(c) 'Recursion / scan logic')."""
    alpha = [0, 1, 1 << 8, (1 << 8) + 1, 1 << 56, 1 << 63, (1 << 64) - 1]
    count = 0
    for L in range(0, 6):
        for seq in itertools.product(range(7), repeat=L):
            k = np.array([alpha[i] for i in seq], np.uint64)
            v = np.arange(L, dtype=np.uint64)
            rk, rv = _stable_ref(k, v)
            for nd, r in ((2, 4), (3, 8), (2, 8)):
                ok, ov, _ = oracle.dfr_sort(k, v, n_d=nd, radix_bits=r)
                assert (ok == rk).all() and (ov == rv).all(), (seq, nd, r)
                count += 1
    assert count == 3 * sum(7 ** L for L in range(6))


# ------------------------------------------------------------ control flow
def _buckets_input(sizes, seed=0):
    """Keys whose top byte (digit 7 of u64) is the bucket index, lower bytes random."""
    rng = np.random.default_rng(seed)
    parts = []
    for b, s in enumerate(sizes):
        low = rng.integers(0, 1 << 56, s, dtype=np.uint64)
        parts.append((np.uint64(b) << np.uint64(56)) | low)
    k = np.concatenate(parts) if parts else np.zeros(0, np.uint64)
    rng.shuffle(k)
    return k


def test_scan_and_divert_counts():
    # S:307 all groups small -> exactly 1 diversion over the whole region.
    # 200 buckets of <= 64 (n = 12800 -> p = 1 at N_d = 64, digit 7 only).
    k = _buckets_input([64] * 200)
    _, _, st = oracle.dfr_sort(k, n_d=64)
    assert st["level0_p"] == 1 and st["diversions"] == 1 and st["large_buckets"] == 0
    assert st["passes"] == 1
    # S:308 alternating small/large groups: diversions = #maximal small runs
    # (+ those inside recursions), large = #large groups at level 0.
    sizes = [10, 10, 500, 3, 700, 700, 5]  # runs of small: [10,10], [3], [5] -> 3
    k = _buckets_input(sizes, 1)
    out, _, st = oracle.dfr_sort(k, n_d=64)
    assert (out == np.sort(k)).all()
    assert st["level0_p"] == 1 and st["level0_large"] == 3
    # each large bucket (500 / 700 / 700 random low bits) -> p' = 1 (digit 6):
    # ~256 sub-buckets of ~2-3 keys -> one bulk diversion each.
    assert st["large_buckets"] == 3
    assert st["diversions"] == 3 + 3
    # S:309 empty region -> no calls
    _, _, st = oracle.dfr_sort(np.zeros(0, np.uint64))
    assert st["diversions"] == 0 and st["passes"] == 0


def test_degenerate_inputs():
    n = 100000
    # all-equal: output = input order (stability), recursion bounded by D
    k = np.full(n, 0xDEADBEEF, np.uint32)
    v = np.arange(n, dtype=np.uint32)
    ok, ov, st = oracle.dfr_sort(k, v)
    assert (ov == v).all() and st["max_depth"] <= 4
    assert st["skippable_passes"] == st["passes"]
    # sorted input: idempotent; reverse sorted
    k = np.sort(datagen.uniform_u64(n, 3))
    out, _, _ = oracle.dfr_sort(k)
    assert (out == k).all()
    out, _, _ = oracle.dfr_sort(k[::-1].copy())
    assert (out == k).all()


def test_level0_structure_uniform():
    # c1 at its real size: p = 2, all 2^16 buckets (mean 1) diverted in one run
    k, _ = datagen.make_case("c1")
    _, _, st = oracle.dfr_sort(k)
    assert st["level0_p"] == 2 and st["level0_large"] == 0 and st["diversions"] == 1
    # level-bucket classifier on a grouped array
    g, _, p = oracle.group(datagen.uniform_u64(1 << 20, 9))
    assert p == 2
    b = oracle.level_buckets(g, p, 64, 4096)
    assert b["small"] + b["mid"] + b["large"] == b["buckets"] <= 1 << 16
    assert b["large"] == 0


def test_level_buckets_constructed_sizes():
    """oracle_level_buckets_u64 pinned on buckets of constructed sizes around
    both thresholds (Alg. 4 l.8-9; reading E2: size <= N_d is small,
    S:293/S:304; <= C goes on-chip): a '<' vs '<=' slip at N_d = 64 or at
    C = 4096, or a prefix of the wrong width, changes one of the counts."""
    sizes = [1, 64, 65, 3, 4096, 4097, 100, 2]
    rng = np.random.default_rng(11)
    for p in (1, 3, 8):
        shift = 8 * (8 - p)
        parts = []
        for b, s in enumerate(sizes):
            pre = np.uint64(b + 1) << np.uint64(shift) if shift < 64 else np.uint64(0)
            if p == 8:  # the whole key is the prefix: a bucket is a run of equal keys
                low = np.full(s, b + 1, np.uint64)
            else:       # random bits below the prefix, the prefix itself constant
                low = rng.integers(0, 1 << min(shift, 62), s, dtype=np.uint64)
            parts.append(pre | low if p < 8 else low)
        g = np.concatenate(parts)
        b = oracle.level_buckets(g, p, 64, 4096)
        assert b == {"buckets": 8, "small": 4, "mid": 3, "large": 1,
                     "mid_records": 65 + 4096 + 100, "large_records": 4097}, (p, b)
    # N_d and C move the boundaries by exactly one record
    g = np.concatenate([np.full(s, i, np.uint64) for i, s in enumerate(sizes)])
    assert oracle.level_buckets(g, 8, 65, 4097)["small"] == 5
    assert oracle.level_buckets(g, 8, 65, 4097)["large"] == 0
    assert oracle.level_buckets(g, 8, 63, 4095)["small"] == 3
    assert oracle.level_buckets(g, 8, 63, 4095)["large"] == 2
