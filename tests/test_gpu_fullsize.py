"""Full-size parity: every input of BASELINE.json's five configs (13 inputs, up
to 2^28 keys) sorted on the GPU through the C ABI and compared element by
element with the CPU oracle's output on the same seeded input (keys, and
values for the c4 pairs).  The oracle is plain single-threaded DFR; several
oracle runs go in parallel threads (ctypes releases the GIL) while the GPU
works through the cases in order."""
import concurrent.futures as cf
import os

import numpy as np
import pytest

import datagen
import oracle
from gpu_util import gpu_sort

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CONFIGS = {
    "c1": ["c1"],
    "c2": ["c2"],
    "c3": ["c3-normal", "c3-exp", "c3-zipf"],
    "c4": ["c4-few", "c4-equal"],
    "c5": ["c5-uniform", "c5-sorted", "c5-reverse", "c5-nearly", "c5-runs", "c5-low20"],
}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _oracle_job(keys, vals):
    k, v, st = oracle.dfr_sort(keys, vals)
    return k, v, st


@pytest.mark.parametrize("config", sorted(CONFIGS))
def test_fullsize_config(config):
    cases = CONFIGS[config]
    workers = max(1, min(len(cases), (os.cpu_count() or 2) // 2, 4))
    with cf.ThreadPoolExecutor(workers) as pool:
        jobs = []
        for name in cases:
            keys, vals = datagen.make_case(name)
            assert keys.size == datagen.CASES[name].n
            fut = pool.submit(_oracle_job, keys, vals)
            gk, gv, st = gpu_sort(keys, vals, stats=True)
            jobs.append((name, keys, fut, gk, gv, st))
        for name, keys, fut, gk, gv, st in jobs:
            rk, rv, ost = fut.result()
            assert st["overflow"] == 0, name
            # the fused last pass runs on the large keys-only top calls whose
            # three group passes all execute (c5 except c5-low20)
            assert st["fused"] == int(config == "c5" and name != "c5-low20"), (name, st)
            assert st["level0_p"] == ost["level0_p"], (name, st, ost)
            assert gk.size == rk.size
            bad = np.flatnonzero(gk != rk)
            assert bad.size == 0, f"{name}: {bad.size} key mismatches, first at {bad[:5]}"
            if rv is not None:
                badv = np.flatnonzero(gv != rv)
                assert badv.size == 0, f"{name}: {badv.size} value mismatches, first at {badv[:5]}"


@pytest.mark.parametrize("name", ["c5-uniform", "c5-runs", "c5-reverse"])
def test_fullsize_separate_last_pass(name):
    """The separate last deal + diversion kernels (dfr_config.fused_last_pass =
    2) on 2^28 u64 inputs, which the default fused path otherwise replaces:
    bit-exact vs the oracle."""
    keys, _ = datagen.make_case(name)
    with cf.ThreadPoolExecutor(1) as pool:
        fut = pool.submit(_oracle_job, keys, None)
        gk, _, st = gpu_sort(keys, None, stats=True, fused=False)
        rk, _, ost = fut.result()
    assert st["overflow"] == 0 and st["level0_p"] == ost["level0_p"]
    assert st["fused"] == 0, st
    bad = np.flatnonzero(gk != rk)
    assert bad.size == 0, f"{name}: {bad.size} key mismatches, first at {bad[:5]}"
