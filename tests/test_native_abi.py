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


def test_error_contract_without_a_device():
    """Shape, alignment and argument errors are reported before any CUDA call, as HM_E_* codes
    with a thread-local message (include/hetermoe.h), so they hold on a CPU-only host too."""
    lib = _native.load()
    HM_E_SHAPE, HM_E_ALIGN, HM_E_ARG = 1001, 1002, 1004
    A = 1 << 20  # a 16-byte aligned fake device address (never dereferenced on these paths)

    def msg():
        m = lib.hm_last_error()
        return m.decode() if m else ""

    assert lib.hm_router_topk(A, A, None, -1, 4096, 8, 2, A, A, A, A, A, A, None) == HM_E_SHAPE
    assert "router" in msg()
    assert lib.hm_router_topk(A, A, None, 64, 300, 8, 2, A, A, A, A, A, A, None) == HM_E_SHAPE  # d % 256
    assert lib.hm_router_topk(A, A, None, 64, 4096, 8, 9, A, A, A, A, A, A, None) == HM_E_SHAPE  # k > E
    assert lib.hm_router_topk(A + 2, A, None, 64, 4096, 8, 2, A, A, A, A, A, A, None) == HM_E_ALIGN
    assert lib.hm_dispatch_permute(A, A, A, 64, 4096, 8, 0, A, A, A, None) == HM_E_SHAPE  # k = 0
    assert lib.hm_dispatch_permute(A, A, A, 64, 4100, 8, 2, A, A, A, None) == HM_E_SHAPE  # d % 8
    assert lib.hm_dispatch_permute(A, A, A, 64, 4096, 8, 2, A + 8, A, A, None) == HM_E_ALIGN
    assert lib.hm_combine(A, A, A, -5, 4096, 2, A, None) == HM_E_SHAPE
    assert lib.hm_combine(A + 4, A, A, 64, 4096, 2, A, None) == HM_E_ALIGN
    assert "combine" in msg()
    gemm = lambda mode, E, N, ldo=4096: lib.hm_grouped_gemm(  # noqa: E731
        mode, A, A, A, E, 128, 0, N, 4096, A, ldo, None, 0, None, 0, None, 0, None)
    assert gemm(99, 8, 4096) == HM_E_ARG and "mode" in msg()
    assert gemm(_native.GEMM_FWD_DOWN, 0, 4096) == HM_E_SHAPE
    assert gemm(_native.GEMM_FWD_DOWN, 8, 4100) == HM_E_SHAPE
    assert gemm(_native.GEMM_FWD_DOWN, 8, 4096, ldo=4100) == HM_E_ALIGN
    assert gemm(_native.GEMM_WGRAD, 8, 4096) == HM_E_ARG  # weight gradients need the workspace
