"""Host-side checks of the C-ABI library (no GPU needed): it loads, it exports
every symbol include/dfr.h declares, and its host-only entry points answer."""
import ctypes
import os
import re

import pytest

import paper_2207_14334_b200 as dfr
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dfr.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|uint64_t|const char\*)\s+(dfr_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    L = dfr.lib()
    decl = _declared()
    assert len(decl) == 17
    assert sorted(dfr.EXPORTS) == decl
    for name in decl:
        assert hasattr(L, name), name


def test_host_entry_points():
    assert dfr.status_string(0) == "DFR_OK"
    assert dfr.status_string(-4) == "DFR_ERR_TOO_LARGE"
    # planner's top passes == the oracle's (Alg. 4 l.4), capped at D
    for n in [2, 64, 65, 1 << 14, (1 << 14) + 1, 1 << 16, 1 << 22, (1 << 22) + 1, 1 << 24,
              1 << 26, 1 << 27, 1 << 28]:
        for kb in (4, 8):
            assert dfr.top_passes(n, kb, 64) == min(oracle.est_top_passes(n, 8, 64), kb)
    # the workspace holds at least the input-sized buffer (Alg. 4 l.2)
    n = 1 << 20
    assert dfr.workspace_bytes(n, 8, 0) >= 8 * n
    assert dfr.workspace_bytes(n, 4, 4) >= 8 * n


def test_trivial_calls_need_no_device():
    L = dfr.lib()
    # n <= 1 returns DFR_OK without launching anything
    assert L.dfr_sort_u64(None, 0, None) == 0
    assert L.dfr_sort_u32(None, 1, None) == 0
    assert L.dfr_sort_pairs_u32(None, None, 0, None) == 0
    assert L.dfr_sort_pairs_u64(None, None, 1, None) == 0
    assert L.dfr_sort_pairs_u64(None, None, 10, None) == dfr.DFR_ERR_INVALID
    # bad configuration is rejected up front
    bad = dfr.Config(3, 1)
    assert L.dfr_sort_u64_ex(None, 10, None, ctypes.byref(bad), None) == dfr.DFR_ERR_INVALID
    bad = dfr.Config(64, 1, None, 3)  # fused_last_pass out of range
    assert L.dfr_sort_u64_ex(None, 10, None, ctypes.byref(bad), None) == dfr.DFR_ERR_INVALID
    bad = dfr.Config(64, 1, None, 0, 0, 0, 2)  # stable_deals out of range
    assert L.dfr_sort_u64_ex(None, 10, None, ctypes.byref(bad), None) == dfr.DFR_ERR_INVALID
    lsd = dfr.Config(64, 1, None, 0, 1)  # the full-LSD ablation holds 4 digits: not u64
    assert L.dfr_sort_u64_ex(ctypes.c_void_p(0x1000), 10, None, ctypes.byref(lsd), None) == dfr.DFR_ERR_INVALID
    # null pointer with n > 1
    assert L.dfr_sort_u64(None, 10, None) == dfr.DFR_ERR_INVALID
    # misaligned element pointer
    assert L.dfr_sort_u64(ctypes.c_void_p(0x1004), 10, None) == dfr.DFR_ERR_INVALID
    # size bound: n <= 2^30 = 256^3.75 (the paper's largest N) is accepted
    # by the checks; one more key is DFR_ERR_TOO_LARGE before any device work
    assert L.dfr_sort_u64(ctypes.c_void_p(0x1000), (1 << 30) + 1, None) == dfr.DFR_ERR_TOO_LARGE
    assert L.dfr_sort_u32(ctypes.c_void_p(0x1000), (1 << 30) + 1, None) == dfr.DFR_ERR_TOO_LARGE
    assert L.dfr_sort_pairs_u64(ctypes.c_void_p(0x1000), ctypes.c_void_p(0x10000000000),
                                (1 << 30) + 1, None) == dfr.DFR_ERR_TOO_LARGE


def test_product_has_no_oracle_dependency():
    """The product path never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2207_14334_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "liboracle" not in txt, f
                assert "from oracle" not in txt, f
