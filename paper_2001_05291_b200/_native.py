"""Loads the in-tree native library and declares the C ABI signatures.

There is no CPU fallback: if the library or a CUDA device is missing, the
product API raises instead of computing anything.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import _abi as A

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libfleetplace_b200.so"

# Every symbol include/fleetplace_b200.h declares (checked by the CPU tests).
EXPORTS = (
    "fp_abi_version", "fp_last_error", "fp_ctx_create", "fp_ctx_destroy",
    "fp_ctx_kernel_launches", "fp_ctx_last_kernel_ms", "fp_ctx_last_copy_ms", "fp_ctx_set_row_copy", "fp_validate_instance", "fp_generate_instance",
    "fp_build_distance_table", "fp_table_upload", "fp_table_download",
    "fp_column_totals", "fp_rank_bases", "fp_initial_pool", "fp_search",
    "fp_search_batch", "fp_search_batch_configs", "fp_neighbourhood_sweep", "fp_enumerate_moves", "fp_objective_km", "fp_haversine_batch",
    "fp_permutations", "fp_column_totals_chain", "fp_rank_from_totals",
)

_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        if os.environ.get("FLEETPLACE_B200_NO_BUILD"):
            raise RuntimeError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
        from ._build import build
        build()
    l = C.CDLL(str(LIB_PATH))
    i32, u64, f64, p = C.c_int32, C.c_uint64, C.c_double, C.c_void_p
    i32p, u8p, f64p = C.POINTER(C.c_int32), C.POINTER(C.c_uint8), C.POINTER(C.c_double)
    inst_p = C.POINTER(A.fp_instance)
    l.fp_abi_version.restype = i32
    l.fp_last_error.restype = C.c_char_p
    l.fp_ctx_create.argtypes = [i32, C.POINTER(p)]
    l.fp_ctx_create.restype = i32
    l.fp_ctx_destroy.argtypes = [p]
    l.fp_ctx_destroy.restype = None
    l.fp_ctx_kernel_launches.argtypes = [p]
    l.fp_ctx_kernel_launches.restype = u64
    l.fp_ctx_last_kernel_ms.argtypes = [p]
    l.fp_ctx_last_kernel_ms.restype = f64
    l.fp_ctx_last_copy_ms.argtypes = [p]
    l.fp_ctx_last_copy_ms.restype = f64
    l.fp_ctx_set_row_copy.argtypes = [p, i32]
    l.fp_ctx_set_row_copy.restype = i32
    l.fp_permutations.argtypes = [p, u64, i32, i32, i32p]
    l.fp_permutations.restype = i32
    l.fp_validate_instance.argtypes = [inst_p]
    l.fp_validate_instance.restype = i32
    l.fp_generate_instance.argtypes = [u64, f64p, i32, i32, i32, i32, f64, u64, i32, i32,
                                       i32p, u8p, f64p, f64p, i32p, u8p, i32p, f64p, f64p,
                                       f64p, f64p, u8p]
    l.fp_generate_instance.restype = i32
    l.fp_build_distance_table.argtypes = [p, inst_p, f64, f64p]
    l.fp_build_distance_table.restype = i32
    l.fp_table_upload.argtypes = [p, i32, i32, f64p]
    l.fp_table_upload.restype = i32
    l.fp_table_download.argtypes = [p, f64p]
    l.fp_table_download.restype = i32
    l.fp_column_totals.argtypes = [p, f64p]
    l.fp_column_totals.restype = i32
    l.fp_rank_bases.argtypes = [p, inst_p, C.POINTER(A.fp_ranked_start)]
    l.fp_rank_bases.restype = i32
    l.fp_column_totals_chain.argtypes = [p, i32, i32, p, p, i32]
    l.fp_column_totals_chain.restype = i32
    l.fp_rank_from_totals.argtypes = [p, inst_p, f64p, C.POINTER(A.fp_ranked_start)]
    l.fp_rank_from_totals.restype = i32
    l.fp_initial_pool.argtypes = [inst_p, i32p, i32p, i32p, i32, i32p, i32p, i32p]
    l.fp_initial_pool.restype = i32
    l.fp_search.argtypes = [p, inst_p, C.POINTER(A.fp_search_config),
                            C.POINTER(A.fp_search_start), C.POINTER(A.fp_search_result)]
    l.fp_search.restype = i32
    l.fp_search_batch.argtypes = [p, i32, inst_p, C.POINTER(f64p), C.POINTER(A.fp_search_config),
                                  C.POINTER(A.fp_search_start), C.POINTER(A.fp_search_result)]
    l.fp_search_batch.restype = i32
    l.fp_search_batch_configs.argtypes = [p, i32, inst_p, C.POINTER(f64p), f64,
                                          C.POINTER(A.fp_search_config),
                                          C.POINTER(A.fp_search_start),
                                          C.POINTER(A.fp_search_result)]
    l.fp_search_batch_configs.restype = i32
    l.fp_neighbourhood_sweep.argtypes = [p, inst_p, C.POINTER(A.fp_search_start),
                                         C.POINTER(A.fp_sweep_result)]
    l.fp_neighbourhood_sweep.restype = i32
    l.fp_enumerate_moves.argtypes = [p, inst_p, C.POINTER(A.fp_search_start), i32, i32, i32p,
                                     f64p, i32p]
    l.fp_enumerate_moves.restype = i32
    l.fp_objective_km.argtypes = [p, i32, i32p, i32p, f64p]
    l.fp_haversine_batch.argtypes = [p, i32, f64p, f64p, f64p, f64p, f64p, f64p, f64, f64p]
    l.fp_haversine_batch.restype = i32
    l.fp_objective_km.restype = i32
    _lib = l
    return l


def last_error() -> str:
    return lib().fp_last_error().decode(errors="replace")
