"""The C-ABI library loads on a CPU-only host and exports every entry point include/hetermoe.h
declares (no compute call is made here)."""

import os
import re

from paper_2504_03871_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "hetermoe.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(hm_\w+)\s*\(", src, re.M)))


def test_header_and_binding_agree():
    assert _header_functions() == sorted(_native.SIGNATURES)


def test_library_exports_all_symbols():
    assert os.path.exists(_native.LIB_PATH), "build first: python -c 'import __graft_entry__ as g; g.build()'"
    assert sorted(_native.exported_symbols()) == _header_functions()


def test_pure_host_entry_points():
    lib = _native.load()
    assert lib.hm_abi_version() == 3
    # per-chunk table + the fused router's completion counter
    assert lib.hm_router_chunk_elems(4096, 8) == 64 * 8 + 1
    assert lib.hm_router_chunk_elems(1, 64) == 64 + 1
    assert lib.hm_router_launches(16384, 4096, 8) == 1  # logits + top-k + histogram + scan fused
    assert lib.hm_router_launches(16384, 2048, 64) == 3  # 8 expert groups: logits, top-k, scan
    assert lib.hm_router_launches(16384, 768, 8) == 1  # any d % 256 == 0 up to 16384
    assert lib.hm_router_launches(16384, 6144, 8) == 3  # 4-expert register groups: two groups
    assert lib.hm_router_launches(16384, 300, 8) == 0
    # dlogit (T*k), dense dlogit rows (T*8), then at least 16 splits of dWg partials
    assert lib.hm_router_bwd_part_elems(16384, 4096, 8, 2) >= 16384 * 2 + 16384 * 8 + 16 * 8 * 4096
