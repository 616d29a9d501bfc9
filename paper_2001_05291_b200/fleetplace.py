"""Python mirror of the reference solver interface, backed by the B200 path.

Same names, argument meaning and error behaviour as the reference's public
C++ API (/root/reference/proj/include/fleetplace/{geo,model,rank,search,
parallel,errors}.hpp), so tests read like the reference's own tests:

    inst = Instance(bases=[...], fleet=[...], missions=[...])
    t = build_distance_table(inst)               # kernel (1), model.cpp:76-90
    start = rank_bases(inst, t)                  # kernel (2), rank.cpp:25-124
    a = tabu_search(start, inst, t, SearchConfig(seed=7, mode=SearchMode.Tabu))
                                                  # kernels (3)+(4), search.cpp:446-460

Every call goes through the C ABI in include/fleetplace_b200.h
(paper_2001_05291_b200/_lib/libfleetplace_b200.so). There is no CPU
fallback: without the library or a CUDA device the calls raise.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Iterable, NamedTuple, Optional, Sequence

import numpy as np

from . import _abi as A
from ._native import last_error, lib

kEarthRadiusKm = 6371.0088  # proj/include/fleetplace/geo.hpp:7


# ---------------------------------------------------------------- errors ----
# proj/include/fleetplace/errors.hpp:8-62 plus the std:: types the
# reference throws on the hot path.
class Error(RuntimeError):
    pass


class ParseError(Error):
    pass


class ValidationError(Error):
    pass


class InfeasibleError(Error):
    pass


class BudgetExceededError(Error):
    pass


class NoCompatibleVehicleError(Error):
    pass


class PoolTooSmallError(Error):
    pass


class InvalidArgument(ValueError):
    """std::invalid_argument."""


class LogicError(RuntimeError):
    """std::logic_error (debug_check_deltas drift)."""


class CudaError(RuntimeError):
    """CUDA failure or no device: the B200 path has no CPU fallback."""


_STATUS = {
    A.FP_ERR_INVALID_ARGUMENT: InvalidArgument,
    A.FP_ERR_VALIDATION: ValidationError,
    A.FP_ERR_INFEASIBLE: InfeasibleError,
    A.FP_ERR_NO_COMPATIBLE: NoCompatibleVehicleError,
    A.FP_ERR_POOL_TOO_SMALL: PoolTooSmallError,
    A.FP_ERR_LOGIC: LogicError,
    A.FP_ERR_ERROR: Error,
    A.FP_ERR_CUDA: CudaError,
    A.FP_ERR_OUT_OF_MEMORY: MemoryError,
}


def _check(rc: int) -> None:
    if rc != A.FP_OK:
        raise _STATUS.get(rc, Error)(last_error())


# ----------------------------------------------------------------- model ----
class BaseKind(IntEnum):
    Aerodrome = 0
    Helipad = 1


class VehicleKind(IntEnum):
    RotaryWing = 0
    FixedWing = 1


class GeoPoint(NamedTuple):
    lat_deg: float = 0.0
    lon_deg: float = 0.0


@dataclass
class Base:
    id: int = 0
    kind: BaseKind = BaseKind.Aerodrome
    location: GeoPoint = GeoPoint()


@dataclass
class Vehicle:
    id: int = 0
    kind: VehicleKind = VehicleKind.RotaryWing


@dataclass
class Mission:
    id: int = 0
    pickup: GeoPoint = GeoPoint()
    delivery: GeoPoint = GeoPoint()
    rotary_only: bool = False


def _tup(x):
    return tuple(x) if not isinstance(x, tuple) else x


class Instance:
    """proj/include/fleetplace/model.hpp:41-54, stored structure-of-arrays.

    Entity order is load order; it fixes every index downstream. Construct
    from Base/Vehicle/Mission lists (or (id, kind, (lat, lon)) tuples) or
    with from_arrays() for large generated instances.
    """

    def __init__(self, bases: Iterable = (), fleet: Iterable = (), missions: Iterable = ()):
        bl = [b if isinstance(b, Base) else Base(b[0], BaseKind(b[1]), GeoPoint(*b[2])) for b in bases]
        vl = [v if isinstance(v, Vehicle) else Vehicle(v[0], VehicleKind(v[1])) for v in fleet]
        ml = [m if isinstance(m, Mission) else Mission(m[0], GeoPoint(*m[1]), GeoPoint(*m[2]), bool(m[3]))
              for m in missions]
        self._set(
            np.array([b.id for b in bl], np.int32), np.array([int(b.kind) for b in bl], np.uint8),
            np.array([b.location[0] for b in bl], np.float64), np.array([b.location[1] for b in bl], np.float64),
            np.array([v.id for v in vl], np.int32), np.array([int(v.kind) for v in vl], np.uint8),
            np.array([m.id for m in ml], np.int32),
            np.array([m.pickup[0] for m in ml], np.float64), np.array([m.pickup[1] for m in ml], np.float64),
            np.array([m.delivery[0] for m in ml], np.float64), np.array([m.delivery[1] for m in ml], np.float64),
            np.array([bool(m.rotary_only) for m in ml], np.uint8))

    @classmethod
    def from_arrays(cls, base_id, base_kind, base_lat, base_lon, vehicle_id, vehicle_kind,
                    mission_id, pickup_lat, pickup_lon, delivery_lat, delivery_lon, rotary_only):
        self = cls.__new__(cls)
        self._set(np.ascontiguousarray(base_id, np.int32), np.ascontiguousarray(base_kind, np.uint8),
                  np.ascontiguousarray(base_lat, np.float64), np.ascontiguousarray(base_lon, np.float64),
                  np.ascontiguousarray(vehicle_id, np.int32), np.ascontiguousarray(vehicle_kind, np.uint8),
                  np.ascontiguousarray(mission_id, np.int32),
                  np.ascontiguousarray(pickup_lat, np.float64), np.ascontiguousarray(pickup_lon, np.float64),
                  np.ascontiguousarray(delivery_lat, np.float64),
                  np.ascontiguousarray(delivery_lon, np.float64),
                  np.ascontiguousarray(rotary_only, np.uint8))
        return self

    def _set(self, base_id, base_kind, base_lat, base_lon, vehicle_id, vehicle_kind, mission_id,
             pickup_lat, pickup_lon, delivery_lat, delivery_lon, rotary_only):
        self.base_id, self.base_kind, self.base_lat, self.base_lon = base_id, base_kind, base_lat, base_lon
        self.vehicle_id, self.vehicle_kind = vehicle_id, vehicle_kind
        self.mission_id = mission_id
        self.pickup_lat, self.pickup_lon = pickup_lat, pickup_lon
        self.delivery_lat, self.delivery_lon = delivery_lat, delivery_lon
        self.rotary_only = rotary_only
        self._cstruct = None
        self._maps = None

    def mission_slice(self, lo: int, hi: int) -> "Instance":
        """All bases and vehicles with the missions [lo, hi) in load order:
        one mission shard of a single instance."""
        return Instance.from_arrays(
            self.base_id, self.base_kind, self.base_lat, self.base_lon, self.vehicle_id,
            self.vehicle_kind, self.mission_id[lo:hi], self.pickup_lat[lo:hi],
            self.pickup_lon[lo:hi], self.delivery_lat[lo:hi], self.delivery_lon[lo:hi],
            self.rotary_only[lo:hi])

    # -- views in the reference's AoS vocabulary
    @property
    def bases(self) -> list[Base]:
        return [Base(int(i), BaseKind(int(k)), GeoPoint(float(a), float(o)))
                for i, k, a, o in zip(self.base_id, self.base_kind, self.base_lat, self.base_lon)]

    @property
    def fleet(self) -> list[Vehicle]:
        return [Vehicle(int(i), VehicleKind(int(k))) for i, k in zip(self.vehicle_id, self.vehicle_kind)]

    @property
    def missions(self) -> list[Mission]:
        return [Mission(int(i), GeoPoint(float(a), float(b)), GeoPoint(float(c), float(d)), bool(r))
                for i, a, b, c, d, r in zip(self.mission_id, self.pickup_lat, self.pickup_lon,
                                            self.delivery_lat, self.delivery_lon, self.rotary_only)]

    @property
    def n_bases(self) -> int:
        return len(self.base_id)

    @property
    def n_vehicles(self) -> int:
        return len(self.vehicle_id)

    @property
    def n_missions(self) -> int:
        return len(self.mission_id)

    def _index_maps(self):
        if self._maps is None:
            self._maps = ({int(x): k for k, x in enumerate(self.base_id)},
                          {int(x): k for k, x in enumerate(self.vehicle_id)},
                          {int(x): k for k, x in enumerate(self.mission_id)})
        return self._maps

    # model.hpp:46-48 (-1 when unknown); O(1) here, O(n) in the reference.
    def base_index(self, id: int) -> int:
        return self._index_maps()[0].get(int(id), -1)

    def vehicle_index(self, id: int) -> int:
        return self._index_maps()[1].get(int(id), -1)

    def mission_index(self, id: int) -> int:
        return self._index_maps()[2].get(int(id), -1)

    def rotary_count(self) -> int:
        return int(np.count_nonzero(self.vehicle_kind == A.FP_ROTARY))

    def fixed_count(self) -> int:
        return self.n_vehicles - self.rotary_count()

    def aerodrome_count(self) -> int:
        return int(np.count_nonzero(self.base_kind == A.FP_AERODROME))

    def helipad_count(self) -> int:
        return self.n_bases - self.aerodrome_count()

    def c(self) -> A.fp_instance:
        if self._cstruct is None:
            s = A.fp_instance()
            s.n_bases = self.n_bases
            s.base_id, s.base_kind = A.ptr(self.base_id, C.c_int32), A.ptr(self.base_kind, C.c_uint8)
            s.base_lat, s.base_lon = A.ptr(self.base_lat, C.c_double), A.ptr(self.base_lon, C.c_double)
            s.n_vehicles = self.n_vehicles
            s.vehicle_id = A.ptr(self.vehicle_id, C.c_int32)
            s.vehicle_kind = A.ptr(self.vehicle_kind, C.c_uint8)
            s.n_missions = self.n_missions
            s.mission_id = A.ptr(self.mission_id, C.c_int32)
            s.pickup_lat, s.pickup_lon = A.ptr(self.pickup_lat, C.c_double), A.ptr(self.pickup_lon, C.c_double)
            s.delivery_lat = A.ptr(self.delivery_lat, C.c_double)
            s.delivery_lon = A.ptr(self.delivery_lon, C.c_double)
            s.rotary_only = A.ptr(self.rotary_only, C.c_uint8)
            self._cstruct = s
        return self._cstruct


def valid(p) -> bool:
    """proj/src/geo.cpp:12-15: lat in [-90, 90], lon in [-180, 180]."""
    return -90.0 <= p[0] <= 90.0 and -180.0 <= p[1] <= 180.0


_geo_ctx = None


def _geo():
    global _geo_ctx
    if _geo_ctx is None:
        _geo_ctx = _Ctx(0)
    return _geo_ctx


def haversine_km_batch(a_lat, a_lon, b_lat, b_lon, radius_km: float = kEarthRadiusKm,
                       c_lat=None, c_lon=None) -> np.ndarray:
    """Vectorised haversine_km (+ a second leg from the same points when c_*
    is given, i.e. mission_cost_km) on the device, kernel (1)'s arithmetic."""
    arrs = [np.ascontiguousarray(np.atleast_1d(x), np.float64) for x in (a_lat, a_lon, b_lat, b_lon)]
    n = arrs[0].size
    cl = None if c_lat is None else np.ascontiguousarray(np.atleast_1d(c_lat), np.float64)
    co = None if c_lon is None else np.ascontiguousarray(np.atleast_1d(c_lon), np.float64)
    out = np.empty(n, np.float64)
    _check(lib().fp_haversine_batch(_geo().p, n, *(A.ptr(x, C.c_double) for x in arrs),
                                    A.ptr(cl, C.c_double), A.ptr(co, C.c_double), radius_km,
                                    A.ptr(out, C.c_double)))
    return out


def haversine_km(a, b, radius_km: float = kEarthRadiusKm) -> float:
    """proj/include/fleetplace/geo.hpp:22-27 (device arithmetic)."""
    return float(haversine_km_batch(a[0], a[1], b[0], b[1], radius_km)[0])


def mission_cost_km(base, pickup, delivery, radius_km: float = kEarthRadiusKm) -> float:
    """proj/include/fleetplace/geo.hpp:28-30: base->pickup + base->delivery."""
    return float(haversine_km_batch(base[0], base[1], pickup[0], pickup[1], radius_km,
                                    delivery[0], delivery[1])[0])


def validate_instance(inst: Instance) -> None:
    """proj/src/model.cpp:46-74."""
    _check(lib().fp_validate_instance(C.byref(inst.c())))


def compatible_vehicle_base(v: Vehicle, b: Base) -> bool:
    return not (v.kind == VehicleKind.FixedWing and b.kind == BaseKind.Helipad)


def compatible_vehicle_mission(v: Vehicle, m: Mission) -> bool:
    return not (m.rotary_only and v.kind == VehicleKind.FixedWing)


# --------------------------------------------------------------- context ----
class _Ctx:
    def __init__(self, device: int = 0):
        p = C.c_void_p()
        _check(lib().fp_ctx_create(device, C.byref(p)))
        self.p = p
        self.device = device

    def launches(self) -> int:
        return int(lib().fp_ctx_kernel_launches(self.p))

    def last_kernel_ms(self) -> float:
        return float(lib().fp_ctx_last_kernel_ms(self.p))

    def last_copy_ms(self) -> float:
        return float(lib().fp_ctx_last_copy_ms(self.p))

    def __del__(self):
        try:
            if getattr(self, "p", None):
                lib().fp_ctx_destroy(self.p)
                self.p = None
        except Exception:
            pass


class DistanceTable:
    """proj/include/fleetplace/model.hpp:63-66; the table stays resident on the
    device (one context per table). `cost` downloads an (M, B) column-major
    numpy view on first use."""

    def __init__(self, ctx: _Ctx, n_missions: int, n_bases: int, radius_km: float):
        self._ctx = ctx
        self.n_missions, self.n_bases = n_missions, n_bases
        self.earth_radius_km = radius_km
        self._host = None

    @property
    def cost(self) -> np.ndarray:
        if self._host is None:
            flat = np.empty(self.n_missions * self.n_bases, np.float64)
            _check(lib().fp_table_download(self._ctx.p, A.ptr(flat, C.c_double)))
            self._host = flat.reshape(self.n_bases, self.n_missions).T  # (M, B), Fortran order
        return self._host

    @classmethod
    def from_host(cls, cost: np.ndarray, radius_km: float = kEarthRadiusKm, device: int = 0):
        """Makes a caller-built (e.g. the reference's) table resident."""
        cost = np.asarray(cost, np.float64)
        M, B = cost.shape
        flat = np.ascontiguousarray(cost.T).reshape(-1)
        ctx = _Ctx(device)
        _check(lib().fp_table_upload(ctx.p, M, B, A.ptr(flat, C.c_double)))
        t = cls(ctx, M, B, radius_km)
        t._host = flat.reshape(B, M).T
        return t

    def upload(self, cost: np.ndarray) -> None:
        """Replaces the resident table with a host (M, B) table, reusing this
        table's device context (its stream, workspace and buffers)."""
        cost = np.asarray(cost, np.float64)
        M, B = cost.shape
        flat = np.ascontiguousarray(cost.T).reshape(-1)
        _check(lib().fp_table_upload(self._ctx.p, M, B, A.ptr(flat, C.c_double)))
        self.n_missions, self.n_bases = M, B
        self._host = flat.reshape(B, M).T


def build_distance_table(inst: Instance, radius_km: float = kEarthRadiusKm,
                         device: int = 0, row_copy: bool = True) -> DistanceTable:
    """Kernel (1): proj/src/model.cpp:76-90. `row_copy=False`: no eager
    row-major copy for the search (a table that is only ranked; a later
    search on it makes the copy itself)."""
    ctx = _Ctx(device)
    if not row_copy:
        _check(lib().fp_ctx_set_row_copy(ctx.p, 0))
    _check(lib().fp_build_distance_table(ctx.p, C.byref(inst.c()), radius_km,
                                         C.cast(None, C.POINTER(C.c_double))))
    return DistanceTable(ctx, inst.n_missions, inst.n_bases, radius_km)


# ------------------------------------------------------------------ rank ----
@dataclass
class Assignment:
    """proj/include/fleetplace/model.hpp:74-79."""
    placement: dict = field(default_factory=dict)  # vehicle id -> base id
    service: dict = field(default_factory=dict)    # mission id -> vehicle id

    def __eq__(self, other) -> bool:
        return (isinstance(other, Assignment) and self.placement == other.placement
                and self.service == other.service)


@dataclass
class RankedStart:
    """proj/include/fleetplace/rank.hpp:10-14."""
    assignment: Assignment
    unused_bases: list          # base ids, ranking order
    base_totals: np.ndarray     # km, aligned with Instance bases
    # index form kept for the array-level API
    vehicle_base: np.ndarray = None
    mission_vehicle: np.ndarray = None
    unused_index: np.ndarray = None


def device_permutations(seed: int, n: int, passes: int, device: int = 0) -> np.ndarray:
    """The search's permutation stream drawn on the device (fp_permutations):
    shape (2*passes, n), rows perm_a, perm_b of pass 0, 1, ..."""
    out = np.empty(2 * passes * n, np.int32)
    ctx = _Ctx(device)
    _check(lib().fp_permutations(ctx.p, int(seed) & 0xFFFFFFFFFFFFFFFF, n, passes,
                                 A.ptr(out, C.c_int32)))
    return out.reshape(2 * passes, n)


def column_totals(t: DistanceTable) -> np.ndarray:
    """proj/src/rank.cpp:10-23 (bit-identical fixed-order column sums)."""
    out = np.empty(t.n_bases, np.float64)
    _check(lib().fp_column_totals(t._ctx.p, A.ptr(out, C.c_double)))
    return out


@dataclass
class ParallelConfig:
    workers: int = 1


def parallel_rank_totals(t: DistanceTable, pcfg: ParallelConfig) -> np.ndarray:
    """proj/src/parallel.cpp:31-49: bit-identical to column_totals for any
    worker count; here the device does the split."""
    if pcfg.workers < 1:
        raise InvalidArgument("workers must be >= 1")
    return column_totals(t)


def _assignment_from_index(inst: Instance, vb: np.ndarray, mv: np.ndarray) -> Assignment:
    bid, vid, mid = inst.base_id, inst.vehicle_id, inst.mission_id
    placement = {int(vid[v]): int(bid[b]) for v, b in enumerate(vb.tolist()) if b >= 0}
    service = {int(mid[m]): int(vid[v]) for m, v in enumerate(mv.tolist()) if v >= 0}
    return Assignment(dict(sorted(placement.items())), dict(sorted(service.items())))


def rank_bases(inst: Instance, t: DistanceTable) -> RankedStart:
    """Kernel (2): proj/src/rank.cpp:25-124."""
    B, V, M = inst.n_bases, inst.n_vehicles, inst.n_missions
    tot = np.empty(B, np.float64)
    vb = np.empty(V, np.int32)
    mv = np.empty(M, np.int32)
    un = np.empty(B, np.int32)
    rs = A.fp_ranked_start(A.ptr(tot, C.c_double), A.ptr(vb, C.c_int32), A.ptr(mv, C.c_int32),
                           A.ptr(un, C.c_int32), 0)
    _check(lib().fp_rank_bases(t._ctx.p, C.byref(inst.c()), C.byref(rs)))
    un = un[:rs.n_unused].copy()
    return RankedStart(_assignment_from_index(inst, vb, mv), [int(inst.base_id[b]) for b in un],
                       tot, vb, mv, un)


# ---------------------------------------------------------------- search ----
class SearchMode(IntEnum):
    Local = 0
    Tabu = 1


class MoveKind(IntEnum):
    TakeoverByIdleVehicle = 0
    RelocateToEmptyBase = 1
    ReassignToPlacedVehicle = 2


class PoolEntryKind(IntEnum):
    EmptyBase = 0
    IdleVehicle = 1


class PoolEntry(NamedTuple):
    kind: PoolEntryKind
    id: int


@dataclass
class SearchConfig:
    """proj/include/fleetplace/search.hpp:16-26."""
    seed: int = 0
    mode: SearchMode = SearchMode.Local
    tabu_tenure: int = 0
    max_passes: Optional[int] = None
    debug_check_deltas: bool = False


@dataclass
class SearchStats:
    """proj/include/fleetplace/search.hpp:68-76."""
    passes: int = 0
    evaluations: int = 0
    applied_moves: int = 0
    committed_moves: int = 0
    tabu_skips_outer: int = 0
    tabu_skips_inner: int = 0
    final_objective_km: float = 0.0
    # B200 extras (not in the reference): device time and exact fallbacks
    device_ms: float = 0.0
    exact_fallbacks: int = 0
    phase_cycles: tuple = ()
    event_counts: tuple = ()
    init_ms: float = 0.0
    sweep_ms: float = 0.0
    init_part_ms: tuple = ()
    pass_ms: float = 0.0
    pass_launches: int = 0


@dataclass
class MoveProposal:
    kind: MoveKind
    i_entity: int
    j_mission: int
    delta_km: float


def initial_pool(start: RankedStart, inst: Instance) -> list:
    """proj/src/search.cpp:364-377: unused bases in ranking order, then
    placed vehicles serving no mission, in vehicle-id order."""
    pool = [PoolEntry(PoolEntryKind.EmptyBase, b) for b in start.unused_bases]
    served = set(start.assignment.service.values())
    for vid in sorted(start.assignment.placement):
        if vid not in served:
            pool.append(PoolEntry(PoolEntryKind.IdleVehicle, vid))
    return pool


def _state_arrays(a: Assignment, pool: Sequence, inst: Instance):
    """Assignment + pool -> index arrays, raising InfeasibleError where
    SearchState::from (proj/src/search.cpp:14-65) would, in its order."""
    bmap, vmap, mmap = inst._index_maps()
    V, M = inst.n_vehicles, inst.n_missions
    vb = np.full(V, -1, np.int32)
    for vid, bid in sorted(a.placement.items()):
        vi, bi = vmap.get(vid, -1), bmap.get(bid, -1)
        if vi < 0 or bi < 0:
            raise InfeasibleError("assignment references unknown ids")
        vb[vi] = bi
    mv = np.full(M, -1, np.int32)
    for mid, vid in sorted(a.service.items()):
        mi, vi = mmap.get(mid, -1), vmap.get(vid, -1)
        if mi < 0 or vi < 0 or vb[vi] < 0:
            raise InfeasibleError("service references unplaced vehicle")
        mv[mi] = vi
    pk = np.empty(len(pool), np.int32)
    px = np.empty(len(pool), np.int32)
    for k, e in enumerate(pool):
        pk[k] = int(e.kind)
        px[k] = bmap.get(e.id, -1) if e.kind == PoolEntryKind.EmptyBase else vmap.get(e.id, -1)
    return vb, mv, pk, px


@dataclass
class SearchResult:
    """Array-level result of the device search."""
    vehicle_base: np.ndarray
    mission_vehicle: np.ndarray
    stats: SearchStats
    kernel_launches: int


def _fields(arr, ctype, n, nested=None):
    """Column views (numpy, no copies) of the scalar / pointer fields of a
    ctypes struct array; `nested`: the fields of that struct member."""
    base = C.addressof(arr)
    size = C.sizeof(ctype)
    off0 = 0
    if nested is not None:
        off0 = getattr(ctype, nested).offset
        ctype = dict(ctype._fields_)[nested]
    buf = (C.c_char * (size * n)).from_address(base)
    out = {}
    for name, t in ctype._fields_:
        if t in (C.c_double,):
            dt = np.float64
        elif t in (C.c_int32,):
            dt = np.int32
        elif t in (C.c_uint64,):
            dt = np.uint64
        elif issubclass(t, C._Pointer) or t is C.c_void_p:
            dt = np.uint64
        else:
            continue
        out[name] = np.ndarray((n,), dt, buffer=buf, offset=off0 + getattr(ctype, name).offset,
                               strides=(size,))
    return out


def _cfg_c(cfg: SearchConfig) -> A.fp_search_config:
    return A.fp_search_config(int(cfg.seed) & 0xFFFFFFFFFFFFFFFF, int(cfg.mode), int(cfg.tabu_tenure),
                              -1 if cfg.max_passes is None else int(cfg.max_passes),
                              int(bool(cfg.debug_check_deltas)))


def _stats(r: A.fp_search_result) -> SearchStats:
    s = r.stats
    return SearchStats(int(s.passes), int(s.evaluations), int(s.applied_moves), int(s.committed_moves),
                       int(s.tabu_skips_outer), int(s.tabu_skips_inner), float(s.final_objective_km),
                       float(r.device_ms), int(r.exact_fallbacks), tuple(int(x) for x in r.phase_cycles),
                       tuple(int(x) for x in r.event_counts), float(r.init_ms),
                       float(r.sweep_ms), tuple(float(x) for x in r.init_part_ms),
                       float(r.pass_ms), int(r.pass_launches))


def search_arrays(inst: Instance, t: DistanceTable, cfg: SearchConfig, vehicle_base: np.ndarray,
                  mission_vehicle: np.ndarray, pool_kind: np.ndarray,
                  pool_index: np.ndarray) -> SearchResult:
    """Index-form search (the C-ABI call fp_search, host buffers in and out)."""
    vb_in = np.ascontiguousarray(vehicle_base, np.int32)
    mv_in = np.ascontiguousarray(mission_vehicle, np.int32)
    pk = np.ascontiguousarray(pool_kind, np.int32)
    px = np.ascontiguousarray(pool_index, np.int32)
    vb = np.empty(inst.n_vehicles, np.int32)
    mv = np.empty(inst.n_missions, np.int32)
    st = A.fp_search_start(A.ptr(vb_in, C.c_int32), A.ptr(mv_in, C.c_int32), len(pk),
                           A.ptr(pk, C.c_int32), A.ptr(px, C.c_int32))
    res = A.fp_search_result()
    res.vehicle_base, res.mission_vehicle = A.ptr(vb, C.c_int32), A.ptr(mv, C.c_int32)
    c = _cfg_c(cfg)
    _check(lib().fp_search(t._ctx.p, C.byref(inst.c()), C.byref(c), C.byref(st), C.byref(res)))
    return SearchResult(vb, mv, _stats(res), int(res.kernel_launches))


@dataclass
class Sweep:
    """The neighbourhood sweep of a search start (fp_neighbourhood_sweep):
    reloc_* are (V, B) -- entry [v, t] is vehicle v relocating to base t --
    improve_rows (M, ceil(V/32)) bit words, mission_cost (M,)."""
    reloc_sum: np.ndarray
    reloc_err: np.ndarray
    reloc_abs: np.ndarray
    improve_rows: np.ndarray
    mission_cost: np.ndarray
    sweep_ms: float = 0.0
    total_ms: float = 0.0


def neighbourhood_sweep(inst: Instance, t: DistanceTable, vehicle_base, mission_vehicle,
                        pool_kind=None, pool_index=None, device_out=None) -> Sweep:
    """Every relocation's quick delta and every reassignment's improvement
    test of a start on the device (SURVEY.md §8(d)'s sweep; on a mission
    shard: that shard's partial sweep). `device_out`: a torch.device -- the
    results stay there as CUDA tensors (reloc (3, V, B): sum, err, abs)."""
    V, B, M = inst.n_vehicles, inst.n_bases, inst.n_missions
    if device_out is not None:
        return _sweep_to_device(inst, t, vehicle_base, mission_vehicle, device_out)
    vb = np.ascontiguousarray(vehicle_base, np.int32)
    mv = np.ascontiguousarray(mission_vehicle, np.int32)
    pk = np.ascontiguousarray(pool_kind if pool_kind is not None else [], np.int32)
    px = np.ascontiguousarray(pool_index if pool_index is not None else [], np.int32)
    st = A.fp_search_start(A.ptr(vb, C.c_int32), A.ptr(mv, C.c_int32), len(pk),
                           A.ptr(pk, C.c_int32), A.ptr(px, C.c_int32))
    nvw = (V + 31) // 32
    out = Sweep(np.empty((V, B)), np.empty((V, B)), np.empty((V, B)),
                np.empty((M, nvw), np.uint32), np.empty(M))
    r = A.fp_sweep_result(out.reloc_sum.ctypes.data, out.reloc_err.ctypes.data,
                          out.reloc_abs.ctypes.data, out.improve_rows.ctypes.data,
                          out.mission_cost.ctypes.data, 0, 0.0, 0.0)
    _check(lib().fp_neighbourhood_sweep(t._ctx.p, C.byref(inst.c()), C.byref(st), C.byref(r)))
    out.sweep_ms, out.total_ms = float(r.sweep_ms), float(r.total_ms)
    return out


def _sweep_to_device(inst, t, vehicle_base, mission_vehicle, dev) -> Sweep:
    import torch
    V, B, M = inst.n_vehicles, inst.n_bases, inst.n_missions
    vb = np.ascontiguousarray(vehicle_base, np.int32)
    mv = np.ascontiguousarray(mission_vehicle, np.int32)
    pk = np.empty(0, np.int32)
    st = A.fp_search_start(A.ptr(vb, C.c_int32), A.ptr(mv, C.c_int32), 0, A.ptr(pk, C.c_int32),
                           A.ptr(pk, C.c_int32))
    nvw = (V + 31) // 32
    reloc = torch.empty((3, V, B), dtype=torch.float64, device=dev)
    rows = torch.empty((M, nvw), dtype=torch.int32, device=dev)
    mc = torch.empty(M, dtype=torch.float64, device=dev)
    torch.cuda.current_stream(dev).synchronize()
    r = A.fp_sweep_result(reloc[0].data_ptr(), reloc[1].data_ptr(), reloc[2].data_ptr(),
                          rows.data_ptr(), mc.data_ptr(), 1, 0.0, 0.0)
    _check(lib().fp_neighbourhood_sweep(t._ctx.p, C.byref(inst.c()), C.byref(st), C.byref(r)))
    return Sweep(reloc, None, None, rows, mc, float(r.sweep_ms), float(r.total_ms))


def _run_search(start: RankedStart, inst: Instance, t: DistanceTable, cfg: SearchConfig,
                stats: Optional[SearchStats]) -> Assignment:
    if cfg.mode == SearchMode.Tabu:
        if cfg.tabu_tenure < 0:
            raise InvalidArgument("tabu tenure must be positive (0 = auto)")
        if (cfg.tabu_tenure if cfg.tabu_tenure > 0 else 2 * inst.n_missions) <= 0:
            raise InvalidArgument("tabu tenure must be positive")
    vb, mv, pk, px = _state_arrays(start.assignment, initial_pool(start, inst), inst)
    r = search_arrays(inst, t, cfg, vb, mv, pk, px)
    if stats is not None:
        for f in dataclasses.fields(SearchStats):
            setattr(stats, f.name, getattr(r.stats, f.name))
    return _assignment_from_index(inst, r.vehicle_base, r.mission_vehicle)


def local_search(start: RankedStart, inst: Instance, t: DistanceTable, cfg: SearchConfig,
                 stats: Optional[SearchStats] = None) -> Assignment:
    """proj/src/search.cpp:438-444."""
    if cfg.mode != SearchMode.Local:
        raise InvalidArgument("local_search requires SearchMode::Local")
    return _run_search(start, inst, t, cfg, stats)


def tabu_search(start: RankedStart, inst: Instance, t: DistanceTable, cfg: SearchConfig,
                stats: Optional[SearchStats] = None) -> Assignment:
    """proj/src/search.cpp:446-460."""
    if cfg.mode != SearchMode.Tabu:
        raise InvalidArgument("tabu_search requires SearchMode::Tabu")
    return _run_search(start, inst, t, cfg, stats)


def parallel_local_search(start, inst, t, cfg, pcfg: ParallelConfig, stats=None) -> Assignment:
    """proj/src/parallel.cpp:100-128: the reference guarantees the sequential
    trajectory for every worker count; the device path IS that trajectory."""
    if cfg.mode != SearchMode.Local:
        raise InvalidArgument("parallel_local_search requires SearchMode::Local")
    if pcfg.workers < 1:
        raise InvalidArgument("workers must be >= 1")
    return _run_search(start, inst, t, cfg, stats)


def parallel_tabu_search(start, inst, t, cfg, pcfg: ParallelConfig, stats=None) -> Assignment:
    """proj/src/parallel.cpp:250-305 is nondeterministic by design; the device
    path returns the (deterministic) sequential tabu trajectory, which is one
    of the outcomes the reference's contract allows."""
    if cfg.mode != SearchMode.Tabu:
        raise InvalidArgument("parallel_tabu_search requires SearchMode::Tabu")
    if pcfg.workers < 1:
        raise InvalidArgument("workers must be >= 1")
    if cfg.tabu_tenure < 0:
        raise InvalidArgument("tabu tenure must be positive (0 = auto)")
    return _run_search(start, inst, t, cfg, stats)


def enumerate_moves(a: Assignment, pool: Sequence, i: int, j_mission: int, inst: Instance,
                    t: DistanceTable) -> list:
    """proj/src/search.cpp:379-397 with exact fixed-order deltas (device)."""
    vb, mv, pk, px = _state_arrays(a, pool, inst)
    j = inst.mission_index(j_mission)
    st = A.fp_search_start(A.ptr(vb, C.c_int32), A.ptr(mv, C.c_int32), len(pk),
                           A.ptr(pk, C.c_int32), A.ptr(px, C.c_int32))
    kinds = np.empty(3, np.int32)
    deltas = np.empty(3, np.float64)
    n = C.c_int32(0)
    if j < 0:
        raise Error(f"unknown mission id {j_mission}")
    _check(lib().fp_enumerate_moves(t._ctx.p, C.byref(inst.c()), C.byref(st), i, j,
                                    A.ptr(kinds, C.c_int32), A.ptr(deltas, C.c_double), C.byref(n)))
    return [MoveProposal(MoveKind(int(kinds[k])), i, j_mission, float(deltas[k])) for k in range(n.value)]


# ------------------------------------------------------------ feasibility ----
class Rule(IntEnum):
    OneVehiclePerMission = 0
    OneBasePerVehicle = 1
    BaseOccupancy = 2
    ServiceRequiresPlacement = 3
    RotaryOnly = 4
    FixedWingOnHelipad = 5


class Violation(NamedTuple):
    rule: Rule
    subject_id: int
    related_id: int = -1


def check_feasible(a: Assignment, inst: Instance) -> list:
    """proj/src/model.cpp:118-174 (host bookkeeping, O(M) with id maps)."""
    bmap, vmap, mmap = inst._index_maps()
    out, reported = [], set()

    def report(rule, subject, related=-1):
        if (rule, subject) not in reported:
            reported.add((rule, subject))
            out.append(Violation(rule, subject, related))

    load = {}
    for vid, bid in sorted(a.placement.items()):
        vi, bi = vmap.get(vid, -1), bmap.get(bid, -1)
        if vi < 0 or bi < 0:
            report(Rule.OneBasePerVehicle, vid, bid)
            continue
        load[bid] = load.get(bid, 0) + 1
        if inst.vehicle_kind[vi] == A.FP_FIXED and inst.base_kind[bi] == A.FP_HELIPAD:
            report(Rule.FixedWingOnHelipad, vid, bid)
    for bid in sorted(load):
        if load[bid] > 1:
            report(Rule.BaseOccupancy, bid)
    for vid in inst.vehicle_id.tolist():
        if vid not in a.placement:
            report(Rule.OneBasePerVehicle, vid)
    for mid, vid in sorted(a.service.items()):
        mi, vi = mmap.get(mid, -1), vmap.get(vid, -1)
        if mi < 0:
            report(Rule.OneVehiclePerMission, mid, vid)
            continue
        if vi < 0:
            report(Rule.ServiceRequiresPlacement, vid, mid)
            continue
        if vid not in a.placement:
            report(Rule.ServiceRequiresPlacement, vid, mid)
        if inst.rotary_only[mi] and inst.vehicle_kind[vi] == A.FP_FIXED:
            report(Rule.RotaryOnly, mid, vid)
    for mid in inst.mission_id.tolist():
        if mid not in a.service:
            report(Rule.OneVehiclePerMission, mid)
    return out


def objective_km(a: Assignment, inst: Instance, t: DistanceTable) -> float:
    """proj/src/model.cpp:176-192: the fixed mission-order sum, on the device."""
    v = check_feasible(a, inst)
    if v:
        raise InfeasibleError(f"infeasible assignment: {v[0].rule.name}({v[0].subject_id})")
    bmap, vmap, _ = inst._index_maps()
    vb = np.full(inst.n_vehicles, -1, np.int32)
    for vid, bid in a.placement.items():
        vb[vmap[vid]] = bmap[bid]
    mv = np.array([vmap[a.service[int(m)]] for m in inst.mission_id.tolist()], np.int32)
    out = C.c_double(0.0)
    _check(lib().fp_objective_km(t._ctx.p, inst.n_vehicles, A.ptr(vb, C.c_int32),
                                 A.ptr(mv, C.c_int32), C.byref(out)))
    return out.value


# --------------------------------------------------------------- generator ----
def generate_instance(pool_seed: int, aerodromes: int = 274, helipads: int = 104,
                      health_sites: int = 200, missions: int = 80, rotary_only_fraction: float = 0.3,
                      seed: Optional[int] = None, rotary: int = 8, fixed: int = 4,
                      bbox: Optional[tuple] = None) -> Instance:
    """synthesize_pool(pool_seed, bbox, counts) + generate_instance(pool, missions,
    rotary_only_fraction, seed, rotary, fixed) (proj/src/data.cpp:110-180)."""
    seed = pool_seed if seed is None else seed
    B, V, M = aerodromes + helipads, rotary + fixed, missions
    arrs = dict(base_id=np.empty(B, np.int32), base_kind=np.empty(B, np.uint8),
                base_lat=np.empty(B), base_lon=np.empty(B), vehicle_id=np.empty(V, np.int32),
                vehicle_kind=np.empty(V, np.uint8), mission_id=np.empty(M, np.int32),
                pickup_lat=np.empty(M), pickup_lon=np.empty(M), delivery_lat=np.empty(M),
                delivery_lon=np.empty(M), rotary_only=np.empty(M, np.uint8))
    bb = None if bbox is None else np.asarray(bbox, np.float64)
    P = A.ptr
    _check(lib().fp_generate_instance(
        pool_seed, P(bb, C.c_double), aerodromes, helipads, health_sites, missions,
        rotary_only_fraction, seed, rotary, fixed,
        P(arrs["base_id"], C.c_int32), P(arrs["base_kind"], C.c_uint8), P(arrs["base_lat"], C.c_double),
        P(arrs["base_lon"], C.c_double), P(arrs["vehicle_id"], C.c_int32),
        P(arrs["vehicle_kind"], C.c_uint8), P(arrs["mission_id"], C.c_int32),
        P(arrs["pickup_lat"], C.c_double), P(arrs["pickup_lon"], C.c_double),
        P(arrs["delivery_lat"], C.c_double), P(arrs["delivery_lon"], C.c_double),
        P(arrs["rotary_only"], C.c_uint8)))
    return Instance.from_arrays(**arrs)


def survey_instance(n_bases: int, n_missions: int, n_vehicles: int, seed: int = 1) -> Instance:
    """The SURVEY.md §8(d) recipe for the BASELINE.json shapes."""
    a = (274 * n_bases + 189) // 378
    r = (2 * n_vehicles + 1) // 3
    return generate_instance(seed, a, n_bases - a, max(200, n_missions // 50), n_missions, 0.3, seed,
                             r, n_vehicles - r)


def small_generated(seed: int, missions: int = 10, aerodromes: int = 12, helipads: int = 8,
                    rotary: int = 3, fixed: int = 2) -> Instance:
    """helpers::small_generated (proj/tests/test_helpers.hpp:42-50)."""
    return generate_instance(seed, aerodromes, helipads, 30, missions, 0.3, seed, rotary, fixed,
                             bbox=(43.0, 49.0, -82.0, -74.0))


# ------------------------------------------------------------------ batch ----
def search_batch(insts: Sequence[Instance], starts: Sequence[tuple], cfg,
                 tables: Optional[Sequence[Optional[np.ndarray]]] = None,
                 device: int = 0, ctx: Optional["_Ctx"] = None,
                 radius_km: float = kEarthRadiusKm) -> list:
    """Independent searches of one mission count run concurrently, one thread
    block per scenario (C ABI fp_search_batch_configs). `cfg` is one
    SearchConfig for all or a sequence with one per scenario (e.g. the
    multi-attempt protocol: attempt t with seed + t, proj/src/bench.cpp:
    125-128). `starts[s]` is the index-form start (vehicle_base,
    mission_vehicle, pool_kind, pool_index); `tables[s]` a flat column-major
    host table or None to build it on the device (kernel (1), all such
    tables in one launch). `ctx`: a long-lived context (`_Ctx(device)`)
    whose workspace is reused across batches, as a serving process keeps
    one; default a fresh one per call. Returns one SearchResult per
    scenario."""
    n = len(insts)
    ctx = ctx if ctx is not None else _Ctx(device)
    if n == 0:
        return []
    cfgs = [cfg] * n if isinstance(cfg, SearchConfig) else list(cfg)
    if len(cfgs) != n:
        raise InvalidArgument("one SearchConfig per scenario")
    # marshalling is vectorised (a c5 batch has 512 scenarios): the starts
    # and outputs of every scenario live in a few concatenated arrays, the
    # ABI structs are filled column-wise through numpy views of their bytes
    ci = (A.fp_instance * n)(*[x.c() for x in insts])
    keep = []
    tp = None
    if tables is not None:
        tp = (C.POINTER(C.c_double) * n)()
        for k in range(n):
            if tables[k] is not None:
                t = np.ascontiguousarray(tables[k], np.float64).reshape(-1)
                keep.append(t)
                tp[k] = A.ptr(t, C.c_double)
    # the callers' start arrays are used in place (int32, contiguous: no copy)
    cols = [[np.ascontiguousarray(x[f], np.int32) for x in starts] for f in range(4)]
    keep.append(cols)
    st = (A.fp_search_start * n)()
    sv = _fields(st, A.fp_search_start, n)
    for name, f in (("vehicle_base", 0), ("mission_vehicle", 1), ("pool_kind", 2), ("pool_index", 3)):
        sv[name][:] = np.fromiter((a.ctypes.data for a in cols[f]), np.uint64, n)
    sv["pool_size"][:] = np.fromiter((a.size for a in cols[2]), np.int64, n)
    V = np.fromiter((x.n_vehicles for x in insts), np.int64, n)
    M = insts[0].n_missions
    ovb = np.empty(int(V.sum()), np.int32)
    omv = np.empty(n * M, np.int32)
    vo = np.concatenate([[0], np.cumsum(V)[:-1]])
    res = (A.fp_search_result * n)()
    rv = _fields(res, A.fp_search_result, n)
    rv["vehicle_base"][:] = ovb.ctypes.data + 4 * vo
    rv["mission_vehicle"][:] = omv.ctypes.data + 4 * M * np.arange(n)
    cc = (A.fp_search_config * n)(*[_cfg_c(c) for c in cfgs])
    _check(lib().fp_search_batch_configs(ctx.p, n, ci, tp, float(radius_km), cc, st, res))
    ss = _fields(res, A.fp_search_result, n, nested="stats")
    stat_cols = [ss[f].tolist() for f in A.STATS_FIELDS]
    dev_ms, launches = rv["device_ms"].tolist(), rv["kernel_launches"].tolist()
    fallbacks = rv["exact_fallbacks"].tolist()
    out = []
    for k in range(n):
        sk = SearchStats(*(int(c[k]) for c in stat_cols[:6]), float(stat_cols[6][k]),
                         float(dev_ms[k]), int(fallbacks[k]))
        if k == 0:  # the phase clocks describe scenario 0 (fp_search_result)
            sk = _stats(res[0])
        out.append(SearchResult(ovb[vo[k]:vo[k] + V[k]], omv[k * M:(k + 1) * M], sk, int(launches[k])))
    return out
