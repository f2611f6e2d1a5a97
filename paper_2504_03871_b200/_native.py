"""ctypes binding of libhetermoe_kernels.so (the C ABI declared in include/hetermoe.h).

The shared library is built in-tree (``paper_2504_03871_b200/libhetermoe_kernels.so``) by
``paper_2504_03871_b200.build.build_native()``. There is no fallback: if the library is
missing, every op raises :class:`NativeLibraryError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

LIB_NAME = "libhetermoe_kernels.so"
LIB_PATH = os.environ.get("HM_KERNELS_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

# GEMM modes (include/hetermoe.h)
GEMM_FWD_UPGATE = 0
GEMM_FWD_DOWN = 1
GEMM_BWD_DACT = 2
GEMM_BWD_DX = 3
GEMM_WGRAD = 4
GEMM_WGRAD_ACC = 5

_P = ctypes.c_void_p
_I = ctypes.c_int
_F = ctypes.c_void_p  # float* passed as raw address

# name -> (restype, argtypes)
SIGNATURES = {
    "hm_abi_version": (_I, []),
    "hm_last_error": (ctypes.c_char_p, []),
    "hm_num_sms": (_I, []),
    "hm_gemm_stats": (_I, [_P]),
    "hm_router_chunk_elems": (ctypes.c_size_t, [_I, _I]),
    "hm_router_launches": (_I, [_I, _I, _I]),
    "hm_router_topk": (_I, [_P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "hm_dispatch_permute": (_I, [_P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P]),
    "hm_unpermute_sum": (_I, [_P, _P, _I, _I, _I, _P, _P]),
    "hm_combine": (_I, [_P, _P, _P, _I, _I, _I, _P, _P]),
    "hm_combine_bwd": (_I, [_P, _P, _P, _P, _I, _I, _I, _P, _P, _P]),
    "hm_router_bwd": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P]),
    "hm_router_bwd_part_elems": (ctypes.c_size_t, [_I, _I, _I, _I]),
    "hm_transpose_bf16": (_I, [_P, _I, _I, _P, _P]),
    "hm_grouped_gemm": (_I, [_I, _P, _P, _P, _I, _I, _I, _I, _I, _P, _I, _P, _I, _P, _I, _P, _I, _P]),
    "hm_grouped_gemm_workspace_bytes": (ctypes.c_size_t, [_I, _I]),
    "hm_grouped_gemm_rows": (_I, [_I, _P, _P, _P, _I, _I, _I, _I, _I, _P, _I, _P, _I, _P, _I, _P, _P, _I, _P]),
    "hm_dispatch_permute_p2p": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    "hm_combine_bwd_p2p": (_I, [_P, _P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P]),
    "hm_signal_peers": (_I, [_P, _I, _P]),
    "hm_wait_flags": (_I, [_P, _I, _P, _I, _P]),
    "hm_grouped_wgrad_multi": (_I, [_I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _I, _P, _I, _P]),
    "hm_grouped_wgrad_multi_workspace_bytes": (ctypes.c_size_t, [_I, _I]),
    "hm_grouped_gemm_shifted": (_I, [_I, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _I, _P, _I, _P, _I, _P, _P, _P,
                                     _I, _P]),
    "hm_grouped_wgrad_multi_shifted": (_I, [_I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _I, _P, _P, _I, _P, _I, _P]),
    "hm_zp_layout": (_I, [_P, _I, _I, _P, _I, _I, _I, _P, ctypes.c_longlong, _I, _P, _P, _P, _P, _P, _P, _I, _I,
                          _P, _P]),
    "hm_grouped_ffn_fwd": (_I, [_P, _I, _P, _I, _P, _P, _I, _I, _P, _P, _P, _I, _P]),
    "hm_grouped_ffn_bwd": (_I, [_P, _P, _P, _P, _I, _P, _I, _P, _P, _I, _I, _P, _P, _P, _P, _P, _I, _P]),
}


class NativeLibraryError(RuntimeError):
    """The CUDA extension is missing or a kernel call failed."""


_lib = None
_lock = threading.Lock()


def load(path: str | None = None):
    """Load (once) and return the ctypes handle; raises NativeLibraryError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise NativeLibraryError(
                f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(p)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def exported_symbols(path: str | None = None):
    """Names from SIGNATURES that the library exports (no CUDA call is made)."""
    lib = ctypes.CDLL(path or LIB_PATH)
    return [n for n in SIGNATURES if hasattr(lib, n)]


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().hm_last_error()
        raise NativeLibraryError(f"{what} failed (rc={rc}): {msg.decode() if msg else ''}")
