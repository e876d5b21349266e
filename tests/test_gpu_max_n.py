"""The paper's largest size, N = 256^3.75 = 2^30 64-bit keys (Fig. 1-3
axes), through the public C ABI.

At 2^30 a look-back inclusive prefix can reach 2^30, one past the 30-bit count
field of a status word: the kernels sum the counts mod 2^30, which is exact for
every non-empty bucket (its start is < n <= 2^30).  The oracle would need ~40 s
and ~24 GB of host memory per input here, so parity is checked through
properties that fix the output uniquely for keys-only sorts: the output is
non-decreasing and is a permutation of the input (two independent 64-bit
multiset fingerprints, datagen.fingerprint).  A sorted permutation of a
multiset is unique, so these two properties equal element-by-element parity
with any correct sort.  The plan (level-0 passes p) is checked against the
oracle's estimate (Alg. 4 l.4)."""
import numpy as np
import pytest

import datagen
import oracle
from gpu_util import gpu_sort

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N_MAX = 1 << 30


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    free, _ = torch.cuda.mem_get_info()
    if free < 40 * (1 << 30):
        pytest.skip("needs ~40 GiB of free device memory")


@pytest.mark.parametrize("name", ["paper-uniform", "paper-narrow-normal"])
def test_sort_u64_at_2_30(name):
    keys, _ = datagen.make_case(name, N_MAX)
    fp_in = datagen.fingerprint(keys)
    gk, _, st = gpu_sort(keys, None, stats=True)
    del keys
    assert st["overflow"] == 0, st
    assert st["level0_p"] == oracle.est_top_passes(N_MAX, 8, 64) == 3, st
    assert gk.size == N_MAX
    assert datagen.is_sorted(gk), f"{name}: output not sorted"
    assert datagen.fingerprint(gk) == fp_in, f"{name}: output is not a permutation of the input"
