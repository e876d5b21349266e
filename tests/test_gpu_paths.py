"""GPU parity on the boundaries between the sort's execution paths (DESIGN.md
§7): the small-input cooperative path (n <= 2^21) vs the stand-alone kernels,
mid buckets around the 1024-key (k_mid_s) and 4096-key (k_mid) capacities and
just above them (global queue), recursion levels whose passes reach digit 0
(SEG_SORTED), and several sorts queued back to back on one stream (programmatic
dependent launch between the kernels).  Every output is compared element by
element with the CPU oracle on the same input."""
import numpy as np
import pytest

import datagen
import oracle
from gpu_util import gpu_sort, to_dev, to_host

pytestmark = pytest.mark.gpu

SMALL_N = 1 << 21  # DFR_SMALL_N (dfr_device.cuh)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _check(k, v=None, **kw):
    ok, ov, st = gpu_sort(k, v, stats=True, **kw)
    rk, rv, _ = oracle.dfr_sort(k, v, **kw)
    assert st["overflow"] == 0
    bad = np.flatnonzero(ok != rk)
    assert bad.size == 0, f"{bad.size} key mismatches, first at {bad[:5]}"
    if v is not None:
        badv = np.flatnonzero(ov != rv)
        assert badv.size == 0, f"{badv.size} value mismatches, first at {badv[:5]}"
    return st


@pytest.mark.parametrize("n", [SMALL_N - 1, SMALL_N, SMALL_N + 1])
def test_small_input_boundary(n):
    _check(datagen.uniform_u64(n, 61))
    _check(datagen.uniform_u32(n, 62))
    _check(datagen.few_unique_u32(n, 63, 40), np.arange(n, dtype=np.uint32))


def _prefix_buckets(sizes, bits, seed, n_fill):
    """Keys of `bits` bits whose top 16 bits form one prefix per entry of
    `sizes` (that many keys, random low bits) plus n_fill uniform keys, shuffled."""
    dt = np.uint64 if bits == 64 else np.uint32
    low_bits = bits - 16
    parts = []
    r = datagen.uniform_u64(sum(sizes) + n_fill, seed)
    off = 0
    for i, s in enumerate(sizes):
        pre = np.uint64(0x8000 | (0x111 * (i + 1)))  # top bit set: no filler key shares it
        low = r[off:off + s] & np.uint64((1 << low_bits) - 1)
        parts.append(((pre << np.uint64(low_bits)) | low).astype(dt))
        off += s
    fill = r[off:] >> np.uint64(1)  # top bit clear
    parts.append((fill >> np.uint64(64 - bits)).astype(dt) if bits == 32 else fill)
    k = np.concatenate(parts)
    perm = np.argsort(datagen.uniform_u64(k.size, seed + 1), kind="stable")
    return k[perm]


SIZES_MID = [65, 1023, 1024, 1025, 2048, 4095, 4096, 4097, 9000]


@pytest.mark.parametrize("bits", [64, 32])
def test_mid_bucket_capacities(bits):
    """Level-0 buckets of exactly the mid capacities (N_d < s <= 1024: k_mid_s;
    <= 4096: k_mid; above: the global queue) among uniform filler."""
    k = _prefix_buckets(SIZES_MID, bits, 71 + bits, (1 << 20) - sum(SIZES_MID))
    st = _check(k)
    assert st["level0_large"] == len(SIZES_MID)
    assert st["mid_buckets"] >= sum(1 for s in SIZES_MID if s <= 4096)
    assert st["global_segments"] >= sum(1 for s in SIZES_MID if s > 4096)
    if bits == 32:
        _check(k, np.arange(k.size, dtype=np.uint32))


@pytest.mark.parametrize("n", [SMALL_N + 5, (1 << 22) + 3])
def test_levels_reaching_digit_zero(n):
    """Keys with only their low 12 (u32) / 20 (u64) bits set: level 0 skips its
    constant digits and re-queues the whole input; level 1's passes end on
    digit 0, so its buckets are constant keys and the diversion only copies."""
    k32 = (datagen.uniform_u32(n, 81) & np.uint32(0xFFF)).astype(np.uint32)
    _check(k32)
    _check(k32, np.arange(n, dtype=np.uint32))
    k64 = datagen.uniform_u64(n, 82) & np.uint64((1 << 20) - 1)
    _check(k64)


def test_back_to_back_on_one_stream():
    """Several sorts of different sizes and paths queued on one stream without
    a host synchronisation in between, then checked."""
    import torch
    import paper_2207_14334_b200 as dfr
    inputs = [datagen.uniform_u64((1 << 20) + 5, 91), datagen.uniform_u64(5000, 92),
              datagen.uniform_u64(SMALL_N - 3, 93), datagen.make_case("c3-exp", 1 << 19)[0],
              datagen.uniform_u64((1 << 21) + 1, 94)]
    devs = [to_dev(k) for k in inputs]
    torch.cuda.synchronize()
    for d in devs:
        dfr.sort(d)
    torch.cuda.synchronize()
    for k, d in zip(inputs, devs):
        ref, _, _ = oracle.dfr_sort(k)
        assert (to_host(d, np.uint64) == ref).all()
