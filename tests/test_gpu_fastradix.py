"""GPU parity of Fast Radix estimation (dfr_config.fast_radix; §3
Alg. 3): the pass on the lowest group digit
deals into estimated buckets of ceil(n/256) keys with overflow chunks, the
middle pass reads them bucket by bucket and counts the top digit.  The output
must equal the oracle's element by element (estimation changes the
mechanism, not the result), on uniform inputs (little overflow, compared with
the exact expectation of oracle/overflow.py) and on inputs that overflow
massively (the estimate is wrong: "a glorified counting pass")."""
import numpy as np
import pytest

import datagen
import oracle
from oracle import overflow as ov
from gpu_util import gpu_sort

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _check(k, **kw):
    gk, _, st = gpu_sort(k, stats=True, fast_radix=True, **kw)
    rk, _, ost = oracle.dfr_sort(k)
    assert st["overflow"] == 0 and st["level0_p"] == ost["level0_p"], st
    bad = np.flatnonzero(gk != rk)
    assert bad.size == 0, f"{bad.size} key mismatches, first at {bad[:5]}"
    return st


@pytest.mark.parametrize("n", [1 << 27, (1 << 27) + 333, 1 << 28])
def test_fast_radix_uniform(n):
    st = _check(datagen.uniform_u64(n, 401))
    assert st["fused"] == 1
    # the estimated 256-way pass overflows about E[overflow] records (exact
    # balls-into-bins expectation; one sample, sd ~ 1/3 of the mean here)
    e = ov.expected_overflow(n, 256) * n
    assert 0.5 * e < st["fr_overflow"] < 1.5 * e, (st["fr_overflow"], e)


def test_fast_radix_u32():
    st = _check(datagen.uniform_u32(1 << 27, 402))
    assert st["fused"] == 1


@pytest.mark.parametrize("name", ["c5-sorted", "c5-nearly", "c5-runs"])
def test_fast_radix_layouts(name):
    k, _ = datagen.make_case(name, 1 << 27)
    _check(k)


@pytest.mark.parametrize("name", ["c5-low20", "c3-normal", "c3-zipf"])
def test_fast_radix_heavy_overflow(name):
    """Estimation badly wrong: every key of c5-low20 falls in one bucket of the
    first pass (the overflow chunks hold all but ceil(n/256) of them)."""
    k, _ = datagen.make_case(name, 1 << 27)
    st = _check(k)
    if name == "c5-low20":
        assert st["fr_overflow"] == k.size - ((k.size + 255) // 256)
