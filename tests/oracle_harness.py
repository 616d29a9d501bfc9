"""Test-only bindings to the oracles (never imported by the product).

* ``REF``: the UNMODIFIED reference compiled from /root/reference/proj/src by
  oracle/Makefile (oracle/_ref/libfleetplace_ref.so + our C wrapper).
* ``ORC``: our C restatement (oracle/_ref/libfleetplace_oracle.so), pinned
  against REF in tests/test_oracle.py; it also emits move logs.

Both take the index-array structs of include/fleetplace_b200.h.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from paper_2001_05291_b200 import _abi as A
from paper_2001_05291_b200.fleetplace import Instance

ROOT = Path(__file__).resolve().parents[1]
REF_SO = ROOT / "oracle" / "_ref" / "libfleetplace_ref.so"
ORC_SO = ROOT / "oracle" / "_ref" / "libfleetplace_oracle.so"

_i32p, _u8p, _f64p = C.POINTER(C.c_int32), C.POINTER(C.c_uint8), C.POINTER(C.c_double)
_inst_p = C.POINTER(A.fp_instance)


def _load_ref():
    l = C.CDLL(str(REF_SO))
    l.ref_last_error.restype = C.c_char_p
    l.ref_haversine_km.restype = C.c_double
    l.ref_haversine_km.argtypes = [C.c_double] * 5
    l.ref_mission_cost_km.restype = C.c_double
    l.ref_mission_cost_km.argtypes = [C.c_double] * 7
    l.ref_generate_instance.argtypes = [C.c_uint64, _f64p, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_double, C.c_uint64, C.c_int32, C.c_int32,
                                        _i32p, _u8p, _f64p, _f64p, _i32p, _u8p, _i32p, _f64p,
                                        _f64p, _f64p, _f64p, _u8p]
    l.ref_validate_instance.argtypes = [_inst_p]
    l.ref_build_distance_table.argtypes = [_inst_p, C.c_double, _f64p, _f64p]
    l.ref_column_totals.argtypes = [C.c_int32, C.c_int32, _f64p, C.c_int32, _f64p]
    l.ref_rank_bases.argtypes = [_inst_p, _f64p, C.POINTER(A.fp_ranked_start), _f64p]
    l.ref_search.argtypes = [_inst_p, _f64p, C.POINTER(A.fp_search_config),
                             C.POINTER(A.fp_search_start), C.c_int32,
                             C.POINTER(A.fp_search_result), _f64p]
    l.ref_search_entry.argtypes = [_inst_p, _f64p, C.POINTER(A.fp_search_config),
                                   C.POINTER(A.fp_search_start), C.c_int32,
                                   C.POINTER(A.fp_search_result)]
    l.ref_enumerate_moves.argtypes = [_inst_p, _f64p, C.POINTER(A.fp_search_start), C.c_int32,
                                      C.c_int32, _i32p, _f64p, _i32p]
    l.ref_objective_km.argtypes = [_inst_p, _f64p, _i32p, _i32p, _f64p]
    l.ref_check_feasible_count.argtypes = [_inst_p, _i32p, _i32p, _i32p]
    l.ref_brute_force_optimal_km.argtypes = [_inst_p, _f64p]
    return l


class OrMove(C.Structure):
    _fields_ = [("tick", C.c_int64), ("pass_", C.c_int32), ("kind", C.c_int32), ("i", C.c_int32),
                ("j", C.c_int32), ("gain", C.c_int32), ("target", C.c_int32)]


def _load_orc():
    l = C.CDLL(str(ORC_SO))
    l.or_haversine_km.restype = C.c_double
    l.or_haversine_km.argtypes = [C.c_double] * 5
    l.or_build_table.argtypes = [_inst_p, C.c_double, _f64p]
    l.or_column_totals.argtypes = [C.c_int32, C.c_int32, _f64p, _f64p]
    l.or_rank_bases.argtypes = [_inst_p, _f64p, C.POINTER(A.fp_ranked_start)]
    l.or_search.argtypes = [_inst_p, _f64p, C.POINTER(A.fp_search_config),
                            C.POINTER(A.fp_search_start), C.POINTER(A.fp_search_result),
                            C.POINTER(OrMove), C.c_int64, C.POINTER(C.c_int64)]
    l.or_mt19937_64.argtypes = [C.c_uint64, C.c_int32, C.POINTER(C.c_uint64)]
    l.or_permutations.argtypes = [C.c_uint64, C.c_int32, C.c_int32, _i32p]
    l.or_objective_km.restype = C.c_double
    l.or_objective_km.argtypes = [C.c_int32, _f64p, _i32p, _i32p]
    return l


REF = _load_ref() if REF_SO.exists() else None
ORC = _load_orc() if ORC_SO.exists() else None

_EXC = {}


def _err(lib, rc):
    if rc != 0:
        from paper_2001_05291_b200 import fleetplace as F
        msg = lib.ref_last_error().decode() if hasattr(lib, "ref_last_error") else "oracle error"
        raise F._STATUS.get(rc, F.Error)(msg)


P = A.ptr


def ref_generate(pool_seed, aerodromes, helipads, health_sites, missions, frac, seed, rotary,
                 fixed, bbox=None) -> Instance:
    B, V, M = aerodromes + helipads, rotary + fixed, missions
    a = dict(base_id=np.empty(B, np.int32), base_kind=np.empty(B, np.uint8), base_lat=np.empty(B),
             base_lon=np.empty(B), vehicle_id=np.empty(V, np.int32),
             vehicle_kind=np.empty(V, np.uint8), mission_id=np.empty(M, np.int32),
             pickup_lat=np.empty(M), pickup_lon=np.empty(M), delivery_lat=np.empty(M),
             delivery_lon=np.empty(M), rotary_only=np.empty(M, np.uint8))
    bb = None if bbox is None else np.asarray(bbox, np.float64)
    _err(REF, REF.ref_generate_instance(
        pool_seed, P(bb, C.c_double), aerodromes, helipads, health_sites, missions, frac, seed,
        rotary, fixed, P(a["base_id"], C.c_int32), P(a["base_kind"], C.c_uint8),
        P(a["base_lat"], C.c_double), P(a["base_lon"], C.c_double), P(a["vehicle_id"], C.c_int32),
        P(a["vehicle_kind"], C.c_uint8), P(a["mission_id"], C.c_int32),
        P(a["pickup_lat"], C.c_double), P(a["pickup_lon"], C.c_double),
        P(a["delivery_lat"], C.c_double), P(a["delivery_lon"], C.c_double),
        P(a["rotary_only"], C.c_uint8)))
    return Instance.from_arrays(**a)


def ref_small_generated(seed, missions=10, aerodromes=12, helipads=8, rotary=3, fixed=2):
    return ref_generate(seed, aerodromes, helipads, 30, missions, 0.3, seed, rotary, fixed,
                        bbox=(43.0, 49.0, -82.0, -74.0))


def ref_survey_instance(n_bases, n_missions, n_vehicles, seed=1):
    a = (274 * n_bases + 189) // 378
    r = (2 * n_vehicles + 1) // 3
    return ref_generate(seed, a, n_bases - a, max(200, n_missions // 50), n_missions, 0.3, seed,
                        r, n_vehicles - r)


def ref_table(inst: Instance, radius=6371.0088) -> np.ndarray:
    """Flat column-major (b*M + m) fp64 table from the reference."""
    out = np.empty(inst.n_missions * inst.n_bases, np.float64)
    _err(REF, REF.ref_build_distance_table(C.byref(inst.c()), radius, P(out, C.c_double), None))
    return out


def orc_table(inst: Instance, radius=6371.0088) -> np.ndarray:
    out = np.empty(inst.n_missions * inst.n_bases, np.float64)
    ORC.or_build_table(C.byref(inst.c()), radius, P(out, C.c_double))
    return out


@dataclass
class Ranked:
    totals: np.ndarray
    vehicle_base: np.ndarray
    mission_vehicle: np.ndarray
    unused: np.ndarray


def _ranked_buffers(inst):
    B, V, M = inst.n_bases, inst.n_vehicles, inst.n_missions
    r = Ranked(np.empty(B), np.empty(V, np.int32), np.empty(M, np.int32), np.empty(B, np.int32))
    s = A.fp_ranked_start(P(r.totals, C.c_double), P(r.vehicle_base, C.c_int32),
                          P(r.mission_vehicle, C.c_int32), P(r.unused, C.c_int32), 0)
    return r, s


def ref_rank(inst, cost) -> Ranked:
    r, s = _ranked_buffers(inst)
    _err(REF, REF.ref_rank_bases(C.byref(inst.c()), P(cost, C.c_double), C.byref(s), None))
    r.unused = r.unused[:s.n_unused].copy()
    return r


def orc_rank(inst, cost) -> Ranked:
    r, s = _ranked_buffers(inst)
    rc = ORC.or_rank_bases(C.byref(inst.c()), P(cost, C.c_double), C.byref(s))
    _err(ORC, rc)
    r.unused = r.unused[:s.n_unused].copy()
    return r


def initial_pool_idx(inst, vehicle_base, mission_vehicle, unused):
    """initial_pool in index form (proj/src/search.cpp:364-377)."""
    kinds = [A.FP_POOL_EMPTY_BASE] * len(unused)
    idx = list(int(u) for u in unused)
    served = np.zeros(inst.n_vehicles, bool)
    served[mission_vehicle[mission_vehicle >= 0]] = True
    placed = [v for v in range(inst.n_vehicles) if vehicle_base[v] >= 0]
    for v in sorted(placed, key=lambda v: int(inst.vehicle_id[v])):
        if not served[v]:
            kinds.append(A.FP_POOL_IDLE_VEHICLE)
            idx.append(v)
    return np.array(kinds, np.int32), np.array(idx, np.int32)


@dataclass
class Searched:
    vehicle_base: np.ndarray
    mission_vehicle: np.ndarray
    stats: tuple
    seconds: float = 0.0
    moves: list = None


def _cfg(mode, seed, tenure=0, max_passes=None, debug=False):
    return A.fp_search_config(seed, mode, tenure, -1 if max_passes is None else max_passes, int(debug))


def _start(vb, mv, pk, px):
    return A.fp_search_start(P(vb, C.c_int32), P(mv, C.c_int32), len(pk), P(pk, C.c_int32),
                             P(px, C.c_int32))


def _stats_tuple(s):
    return tuple(getattr(s, f) for f in A.STATS_FIELDS)


def ref_search(inst, cost, mode, seed, vb, mv, pk, px, tenure=0, max_passes=None, workers=0,
               debug=False) -> Searched:
    cfg = _cfg(mode, seed, tenure, max_passes, debug)
    st = _start(vb, mv, pk, px)
    ovb = np.empty(inst.n_vehicles, np.int32)
    omv = np.empty(inst.n_missions, np.int32)
    res = A.fp_search_result()
    res.vehicle_base, res.mission_vehicle = P(ovb, C.c_int32), P(omv, C.c_int32)
    secs = C.c_double(0)
    _err(REF, REF.ref_search(C.byref(inst.c()), P(cost, C.c_double), C.byref(cfg), C.byref(st),
                             workers, C.byref(res), C.byref(secs)))
    return Searched(ovb, omv, _stats_tuple(res.stats), secs.value)


def orc_search(inst, cost, mode, seed, vb, mv, pk, px, tenure=0, max_passes=None,
               log_cap=0) -> Searched:
    cfg = _cfg(mode, seed, tenure, max_passes)
    st = _start(vb, mv, pk, px)
    ovb = np.empty(inst.n_vehicles, np.int32)
    omv = np.empty(inst.n_missions, np.int32)
    res = A.fp_search_result()
    res.vehicle_base, res.mission_vehicle = P(ovb, C.c_int32), P(omv, C.c_int32)
    log = (OrMove * max(log_cap, 1))()
    n = C.c_int64(0)
    ORC.or_search(C.byref(inst.c()), P(cost, C.c_double), C.byref(cfg), C.byref(st), C.byref(res),
                  log, log_cap, C.byref(n))
    moves = [(m.tick, m.pass_, m.kind, m.i, m.j, m.gain, m.target)
             for m in log[:min(n.value, log_cap)]] if log_cap else None
    return Searched(ovb, omv, _stats_tuple(res.stats), 0.0, moves)
