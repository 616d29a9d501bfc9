"""ctypes mirror of include/fleetplace_b200.h (the C ABI of the hot path).

Shared by the product binding (``_native.py``) and by the test harness that
drives the reference (``oracle/_ref``) through the same struct layouts.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

FP_OK = 0
FP_ERR_INVALID_ARGUMENT = 1
FP_ERR_VALIDATION = 2
FP_ERR_INFEASIBLE = 3
FP_ERR_NO_COMPATIBLE = 4
FP_ERR_POOL_TOO_SMALL = 5
FP_ERR_LOGIC = 6
FP_ERR_ERROR = 7
FP_ERR_CUDA = 8
FP_ERR_OUT_OF_MEMORY = 9

FP_AERODROME, FP_HELIPAD = 0, 1
FP_ROTARY, FP_FIXED = 0, 1
FP_POOL_EMPTY_BASE, FP_POOL_IDLE_VEHICLE = 0, 1
FP_MODE_LOCAL, FP_MODE_TABU = 0, 1
FP_MOVE_TAKEOVER, FP_MOVE_RELOCATE, FP_MOVE_REASSIGN = 0, 1, 2

_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)
_f64p = C.POINTER(C.c_double)


class fp_instance(C.Structure):
    _fields_ = [
        ("n_bases", C.c_int32), ("base_id", _i32p), ("base_kind", _u8p),
        ("base_lat", _f64p), ("base_lon", _f64p),
        ("n_vehicles", C.c_int32), ("vehicle_id", _i32p), ("vehicle_kind", _u8p),
        ("n_missions", C.c_int32), ("mission_id", _i32p),
        ("pickup_lat", _f64p), ("pickup_lon", _f64p),
        ("delivery_lat", _f64p), ("delivery_lon", _f64p), ("rotary_only", _u8p),
    ]


class fp_search_config(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("mode", C.c_int32), ("tabu_tenure", C.c_int32),
                ("max_passes", C.c_int32), ("debug_check_deltas", C.c_int32)]


class fp_search_stats(C.Structure):
    _fields_ = [("passes", C.c_uint64), ("evaluations", C.c_uint64),
                ("applied_moves", C.c_uint64), ("committed_moves", C.c_uint64),
                ("tabu_skips_outer", C.c_uint64), ("tabu_skips_inner", C.c_uint64),
                ("final_objective_km", C.c_double)]


class fp_search_start(C.Structure):
    _fields_ = [("vehicle_base", _i32p), ("mission_vehicle", _i32p),
                ("pool_size", C.c_int32), ("pool_kind", _i32p), ("pool_index", _i32p)]


class fp_search_result(C.Structure):
    _fields_ = [("vehicle_base", _i32p), ("mission_vehicle", _i32p),
                ("stats", fp_search_stats), ("device_ms", C.c_double),
                ("kernel_launches", C.c_uint64), ("exact_fallbacks", C.c_uint64),
                ("phase_cycles", C.c_uint64 * 16), ("init_ms", C.c_double),
                ("sweep_ms", C.c_double), ("event_counts", C.c_uint64 * 5),
                ("init_part_ms", C.c_double * 4), ("pass_ms", C.c_double),
                ("pass_launches", C.c_uint64)]


class fp_ranked_start(C.Structure):
    _fields_ = [("base_totals", _f64p), ("vehicle_base", _i32p),
                ("mission_vehicle", _i32p), ("unused_bases", _i32p),
                ("n_unused", C.c_int32)]


def ptr(a: np.ndarray | None, ctype):
    """Pointer to a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return C.cast(None, C.POINTER(ctype))
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))


STATS_FIELDS = ("passes", "evaluations", "applied_moves", "committed_moves",
                "tabu_skips_outer", "tabu_skips_inner", "final_objective_km")


class fp_sweep_result(C.Structure):
    _fields_ = [("reloc_sum", C.c_void_p), ("reloc_err", C.c_void_p), ("reloc_abs", C.c_void_p),
                ("improve_rows", C.c_void_p), ("mission_cost", C.c_void_p),
                ("device_ptrs", C.c_int32), ("sweep_ms", C.c_double), ("total_ms", C.c_double)]
