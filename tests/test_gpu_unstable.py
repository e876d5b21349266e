"""GPU parity of the keys-only deals that rank keys of equal digit in any order
(R5; dfr_config.stable_deals = 0, the default for keys-only sorts)
against the CPU oracle, element by element.

A deal on the lowest digit of a group, or on a higher one inside a tile that
is constant in the group digits below it, may order keys of equal digit
arbitrarily: equal keys are indistinguishable, the group's later passes are
stable and every resulting bucket is then sorted on all lower digits
(Alg. 4 l.6-14).  The output must therefore still be byte for byte
the oracle's.  The inputs mix tiles that take the atomic ranks with tiles
that straddle a run of the lower digit (the stable ballot ranks), on every
route: the plain three-deal route (2^22, 2^24), the fused level 0 (2^27),
recursion levels (normal, Zipf-like duplicates), u32 keys, and the same
inputs with stable_deals = 1."""
import numpy as np
import pytest

import datagen
import oracle
from gpu_util import gpu_sort

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _check(k, **kw):
    gk, _, st = gpu_sort(k, stats=True, **kw)
    rk, _, ost = oracle.dfr_sort(k)
    assert st["overflow"] == 0, st
    assert st["level0_p"] == ost["level0_p"], (st, ost)
    bad = np.flatnonzero(gk != rk)
    assert bad.size == 0, f"{bad.size} key mismatches, first at {bad[:5]}"
    return st


@pytest.mark.parametrize("stable", [False, True])
@pytest.mark.parametrize("n", [(1 << 22) + 333, (1 << 24) + 4097])
def test_uniform_u64_plain_route(n, stable):
    # lo runs of ~n/256 keys: about one mid-pass tile in four (2^22) or
    # sixteen (2^24) straddles a lo boundary and takes the stable ranks
    _check(datagen.uniform_u64(n, 401), stable_deals=stable)


@pytest.mark.parametrize("stable", [False, True])
def test_uniform_u64_fused(stable):
    st = _check(datagen.uniform_u64((1 << 27) + 5, 402), stable_deals=stable)
    assert st["fused"] == 1


@pytest.mark.parametrize("stable", [False, True])
def test_uniform_u32(stable):
    _check(datagen.uniform_u32((1 << 24) + 77, 403), stable_deals=stable)


@pytest.mark.parametrize("n", [(1 << 20) + 3, 3_000_001])
def test_short_lo_runs(n):
    """p = 2 (group digits 7 and 6): runs of the lo digit of ~n/256 keys, one
    to three tiles long, so most mid-pass tiles straddle a boundary (stable
    ranks) next to constant ones; 2^20 + 3 runs every level in the cooperative
    kernel, 3M through the stand-alone kernels."""
    st = _check(datagen.uniform_u64(n, 404))
    assert st["level0_p"] == 2


def test_recursion_normal_and_duplicates():
    """Large buckets recursed through the segment queue (narrow normal) and
    many equal keys (few-unique u64): the unstable deals at recursion levels."""
    z = datagen.uniform_u64(1 << 23, 405)
    normal = (np.uint64(1) << np.uint64(63)) + (z >> np.uint64(40))  # 24-bit spread
    _check(normal)
    vals = datagen.uniform_u64(300, 406)
    few = vals[(datagen.uniform_u64(1 << 22, 407) % np.uint64(300)).astype(np.int64)]
    _check(few)


@pytest.mark.parametrize("layout", ["sorted", "reverse"])
def test_presorted_layouts(layout):
    k = np.sort(datagen.uniform_u64((1 << 23) + 9, 408))
    if layout == "reverse":
        k = k[::-1].copy()
    _check(k)
