"""ctypes binding of libfea_gpu.so (the C ABI declared in include/fea_gpu.h).

The library is the product: there is no CPU fallback. If libfea_gpu.so is missing this
module raises instead of degrading (build it with ``python -m paper_2012_00585_b200.build``).
"""
from __future__ import annotations

import ctypes
from ctypes import POINTER, c_char_p, c_int, c_int32, c_int64, c_uint32, c_uint64, c_void_p
from pathlib import Path

import os

LIB_PATH = Path(os.environ.get("FEA_LIB_PATH") or Path(__file__).resolve().with_name("libfea_gpu.so"))

FEA_OK = 0
FEA_ERR_INVALID = 1
FEA_ERR_MISSING_ENTRY = 2
FEA_ERR_OOM = 3
FEA_ERR_CUDA = 4
FEA_ERR_INVALID_COLOURING = 5

FEA_ATOMIC = 0
FEA_DET_SORTED = 1
FEA_DET_COLOUR = 2

FEA_ACCUMULATE = 0
FEA_OVERWRITE = 1
FEA_COLOUR_PASSES = 2
FEA_PLAN_K_COMPACT = 1
FEA_FORMAT_CSR = 0
FEA_FORMAT_CRAC = 1

_P64 = POINTER(c_int64)
_P32 = POINTER(c_int32)

# name -> (restype, argtypes); mirrors include/fea_gpu.h one to one
SIGNATURES = {
    "fea_last_error": (c_char_p, []),
    "fea_version": (c_int, []),
    "fea_plan_create": (c_int, [c_int, c_void_p, c_int64, c_int32, c_int64, c_int32, c_int64,
                                c_int64, c_uint32, POINTER(c_void_p)]),
    "fea_plan_create_with_pattern": (c_int, [c_int, c_void_p, c_int64, c_int32, c_int64, c_int32,
                                             c_void_p, c_void_p, POINTER(c_void_p)]),
    "fea_plan_destroy": (None, [c_void_p]),
    "fea_plan_sizes": (c_int, [c_void_p, _P64, _P64, _P64, _P64]),
    "fea_plan_info": (c_int, [c_void_p, _P32, _P32, _P64]),
    "fea_plan_copy_csr": (c_int, [c_void_p, c_void_p, c_void_p]),
    "fea_plan_copy_crac": (c_int, [c_void_p, c_void_p, c_void_p]),
    "fea_plan_copy_elements": (c_int, [c_void_p, c_void_p]),
    "fea_plan_greedy_colouring": (c_int, [c_void_p, c_void_p, _P32]),
    "fea_plan_set_colouring": (c_int, [c_void_p, c_void_p]),
    "fea_plan_jp_colouring": (c_int, [c_void_p, c_uint64, c_void_p, _P32]),
    "fea_assemble": (c_int, [c_void_p, c_void_p, c_int32, c_void_p, c_uint32, c_void_p]),
    "fea_assemble_host": (c_int, [c_void_p, c_void_p, c_int32, c_void_p, c_uint32, c_void_p]),
    "fea_plan_set_host_windows": (c_int, [c_void_p, c_int32]),
    "fea_assemble_host_batch": (c_int, [c_void_p, POINTER(c_void_p), c_int32, POINTER(c_void_p),
                                        c_int32, c_uint32, c_void_p]),
    "fea_plan_missing_entry": (c_int, [c_void_p, _P64, _P64, _P64]),
    "fea_plan_last_launches": (c_int32, [c_void_p]),
    "fea_assemble_seeded": (c_int, [c_void_p, c_uint64, c_int32, c_void_p, c_uint32, c_void_p]),
    "fea_fill_seeded_k": (c_int, [c_void_p, c_int64, c_int32, c_uint64, c_void_p, c_void_p]),
    "fea_spmv_csr": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "fea_spmv_crac": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "fea_plan_spmv": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "fea_exclusive_sum_i64": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "fea_sort_pairs_u32": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_int32, c_void_p]),
    "fea_ipc_export": (c_int, [c_void_p, c_void_p, _P64]),
    "fea_ipc_open": (c_int, [c_void_p, c_int, POINTER(c_void_p)]),
    "fea_ipc_close": (c_int, [c_void_p]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load libfea_gpu.so once and declare every ABI signature."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: the CUDA library is required (no CPU fallback). "
                "Build it with `python -m paper_2012_00585_b200.build`.")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    return (lib().fea_last_error() or b"").decode()
