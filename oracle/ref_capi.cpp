// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin C wrapper around the UNMODIFIED reference implementation
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libfleetplace_ref.so). It converts the index-array form used
// by include/fleetplace_b200.h into the reference's id-keyed types and
// calls the reference's own public API:
//   build_distance_table  proj/src/model.cpp:76-90
//   rank_bases            proj/src/rank.cpp:25-124
//   tabu_search/local_search  proj/src/search.cpp:438-460
//   parallel_*            proj/src/parallel.cpp:31-305
//   enumerate_moves       proj/src/search.cpp:379-397
//   objective_km          proj/src/model.cpp:176-192
//   synthesize_pool/generate_instance  proj/src/data.cpp:110-180
// Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
// legs load this library; the product never does.

#include <chrono>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "fleetplace/bench.hpp"
#include "fleetplace/data.hpp"
#include "fleetplace/errors.hpp"
#include "fleetplace/exact.hpp"
#include "fleetplace/geo.hpp"
#include "fleetplace/model.hpp"
#include "fleetplace/parallel.hpp"
#include "fleetplace/rank.hpp"
#include "fleetplace/search.hpp"
#include "fleetplace_b200.h"

using namespace fleetplace;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return FP_OK;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return FP_ERR_VALIDATION;
  } catch (const InfeasibleError& e) {
    g_err = e.what();
    return FP_ERR_INFEASIBLE;
  } catch (const NoCompatibleVehicleError& e) {
    g_err = e.what();
    return FP_ERR_NO_COMPATIBLE;
  } catch (const PoolTooSmallError& e) {
    g_err = e.what();
    return FP_ERR_POOL_TOO_SMALL;
  } catch (const Error& e) {
    g_err = e.what();
    return FP_ERR_ERROR;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return FP_ERR_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return FP_ERR_LOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FP_ERR_ERROR;
  }
}

Instance to_instance(const fp_instance* in) {
  Instance inst;
  inst.bases.resize(static_cast<std::size_t>(in->n_bases));
  for (int b = 0; b < in->n_bases; ++b)
    inst.bases[b] = {in->base_id[b],
                     in->base_kind[b] ? BaseKind::Helipad : BaseKind::Aerodrome,
                     {in->base_lat[b], in->base_lon[b]}};
  inst.fleet.resize(static_cast<std::size_t>(in->n_vehicles));
  for (int v = 0; v < in->n_vehicles; ++v)
    inst.fleet[v] = {in->vehicle_id[v],
                     in->vehicle_kind[v] ? VehicleKind::FixedWing : VehicleKind::RotaryWing};
  inst.missions.resize(static_cast<std::size_t>(in->n_missions));
  for (int m = 0; m < in->n_missions; ++m)
    inst.missions[m] = {in->mission_id[m],
                        {in->pickup_lat[m], in->pickup_lon[m]},
                        {in->delivery_lat[m], in->delivery_lon[m]},
                        in->rotary_only[m] != 0};
  return inst;
}

DistanceTable to_table(const Instance& inst, const double* cost) {
  DistanceTable t;
  const auto M = static_cast<Eigen::Index>(inst.missions.size());
  const auto B = static_cast<Eigen::Index>(inst.bases.size());
  t.cost.resize(M, B);
  if (M * B > 0) std::memcpy(t.cost.data(), cost, sizeof(double) * M * B);
  return t;
}

Assignment to_assignment(const Instance& inst, const int32_t* vehicle_base,
                         const int32_t* mission_vehicle) {
  Assignment a;
  for (std::size_t v = 0; v < inst.fleet.size(); ++v)
    if (vehicle_base[v] >= 0)
      a.placement[inst.fleet[v].id] = inst.bases[vehicle_base[v]].id;
  for (std::size_t m = 0; m < inst.missions.size(); ++m)
    if (mission_vehicle[m] >= 0)
      a.service[inst.missions[m].id] = inst.fleet[mission_vehicle[m]].id;
  return a;
}

// Index form of an Assignment; ids are looked up through hash-free sorted
// scans of the (small) maps. Unknown ids become -1.
void from_assignment(const Instance& inst, const Assignment& a,
                     int32_t* vehicle_base, int32_t* mission_vehicle) {
  std::map<int, int> bidx, vidx;
  for (std::size_t b = 0; b < inst.bases.size(); ++b) bidx[inst.bases[b].id] = static_cast<int>(b);
  for (std::size_t v = 0; v < inst.fleet.size(); ++v) vidx[inst.fleet[v].id] = static_cast<int>(v);
  for (std::size_t v = 0; v < inst.fleet.size(); ++v) {
    auto it = a.placement.find(inst.fleet[v].id);
    vehicle_base[v] = it == a.placement.end() ? -1 : (bidx.count(it->second) ? bidx[it->second] : -1);
  }
  for (std::size_t m = 0; m < inst.missions.size(); ++m) {
    auto it = a.service.find(inst.missions[m].id);
    mission_vehicle[m] = it == a.service.end() ? -1 : (vidx.count(it->second) ? vidx[it->second] : -1);
  }
}

void copy_stats(const SearchStats& s, fp_search_stats* out) {
  out->passes = s.passes;
  out->evaluations = s.evaluations;
  out->applied_moves = s.applied_moves;
  out->committed_moves = s.committed_moves;
  out->tabu_skips_outer = s.tabu_skips_outer;
  out->tabu_skips_inner = s.tabu_skips_inner;
  out->final_objective_km = s.final_objective_km;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

double ref_haversine_km(double lat_a, double lon_a, double lat_b, double lon_b,
                        double radius_km) {
  return haversine_km({lat_a, lon_a}, {lat_b, lon_b}, radius_km);
}

double ref_mission_cost_km(double base_lat, double base_lon, double p_lat,
                           double p_lon, double d_lat, double d_lon,
                           double radius_km) {
  return mission_cost_km({base_lat, base_lon}, {p_lat, p_lon}, {d_lat, d_lon},
                         radius_km);
}

int ref_generate_instance(uint64_t pool_seed, const double* bbox, int32_t aerodromes,
                          int32_t helipads, int32_t health_sites, int32_t missions,
                          double rotary_only_fraction, uint64_t seed, int32_t rotary,
                          int32_t fixed_wing, int32_t* base_id, uint8_t* base_kind,
                          double* base_lat, double* base_lon, int32_t* vehicle_id,
                          uint8_t* vehicle_kind, int32_t* mission_id, double* pickup_lat,
                          double* pickup_lon, double* delivery_lat, double* delivery_lon,
                          uint8_t* rotary_only) {
  return guarded([&] {
    BoundingBox box;
    if (bbox) box = BoundingBox{bbox[0], bbox[1], bbox[2], bbox[3]};
    const FacilityPool pool = synthesize_pool(
        pool_seed, box, PoolCounts{aerodromes, helipads, health_sites});
    const Instance inst = generate_instance(pool, missions, rotary_only_fraction,
                                            seed, rotary, fixed_wing);
    for (std::size_t b = 0; b < inst.bases.size(); ++b) {
      base_id[b] = inst.bases[b].id;
      base_kind[b] = inst.bases[b].kind == BaseKind::Helipad ? 1 : 0;
      base_lat[b] = inst.bases[b].location.lat_deg;
      base_lon[b] = inst.bases[b].location.lon_deg;
    }
    for (std::size_t v = 0; v < inst.fleet.size(); ++v) {
      vehicle_id[v] = inst.fleet[v].id;
      vehicle_kind[v] = inst.fleet[v].kind == VehicleKind::FixedWing ? 1 : 0;
    }
    for (std::size_t m = 0; m < inst.missions.size(); ++m) {
      mission_id[m] = inst.missions[m].id;
      pickup_lat[m] = inst.missions[m].pickup.lat_deg;
      pickup_lon[m] = inst.missions[m].pickup.lon_deg;
      delivery_lat[m] = inst.missions[m].delivery.lat_deg;
      delivery_lon[m] = inst.missions[m].delivery.lon_deg;
      rotary_only[m] = inst.missions[m].rotary_only ? 1 : 0;
    }
  });
}

int ref_validate_instance(const fp_instance* in) {
  return guarded([&] { validate_instance(to_instance(in)); });
}

int ref_build_distance_table(const fp_instance* in, double radius_km, double* out_cost,
                             double* seconds) {
  return guarded([&] {
    const Instance inst = to_instance(in);
    const auto t0 = std::chrono::steady_clock::now();
    const DistanceTable t = build_distance_table(inst, radius_km);
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (t.cost.rows() * t.cost.cols() > 0)
      std::memcpy(out_cost, t.cost.data(), sizeof(double) * t.cost.rows() * t.cost.cols());
  });
}

int ref_column_totals(int32_t n_missions, int32_t n_bases, const double* cost,
                      int32_t workers, double* out) {
  return guarded([&] {
    DistanceTable t;
    t.cost.resize(n_missions, n_bases);
    if (n_missions * (int64_t)n_bases > 0)
      std::memcpy(t.cost.data(), cost, sizeof(double) * n_missions * (int64_t)n_bases);
    const Eigen::VectorXd v = workers > 0 ? parallel_rank_totals(t, ParallelConfig{workers})
                                          : column_totals(t.cost);
    for (Eigen::Index b = 0; b < v.size(); ++b) out[b] = v(b);
  });
}

int ref_rank_bases(const fp_instance* in, const double* cost, fp_ranked_start* out,
                   double* seconds) {
  return guarded([&] {
    const Instance inst = to_instance(in);
    const DistanceTable t = to_table(inst, cost);
    const auto t0 = std::chrono::steady_clock::now();
    const RankedStart s = rank_bases(inst, t);
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (Eigen::Index b = 0; b < s.base_totals.size(); ++b) out->base_totals[b] = s.base_totals(b);
    from_assignment(inst, s.assignment, out->vehicle_base, out->mission_vehicle);
    std::map<int, int> bidx;
    for (std::size_t b = 0; b < inst.bases.size(); ++b) bidx[inst.bases[b].id] = static_cast<int>(b);
    out->n_unused = static_cast<int32_t>(s.unused_bases.size());
    for (std::size_t k = 0; k < s.unused_bases.size(); ++k)
      out->unused_bases[k] = bidx[s.unused_bases[k]];
  });
}

// Runs the reference search from (assignment, unused bases). The pool's
// EMPTY_BASE entries, in order, are the RankedStart::unused_bases; idle
// vehicles are re-derived by the reference's initial_pool. workers > 0
// selects parallel_local_search / parallel_tabu_search.
int ref_search(const fp_instance* in, const double* cost, const fp_search_config* cfg,
               const fp_search_start* start, int32_t workers, fp_search_result* out,
               double* seconds) {
  return guarded([&] {
    const Instance inst = to_instance(in);
    const DistanceTable t = to_table(inst, cost);
    RankedStart rs;
    rs.assignment = to_assignment(inst, start->vehicle_base, start->mission_vehicle);
    for (int k = 0; k < start->pool_size; ++k)
      if (start->pool_kind[k] == FP_POOL_EMPTY_BASE)
        rs.unused_bases.push_back(start->pool_index[k] >= 0
                                      ? inst.bases[start->pool_index[k]].id
                                      : -2147483647);
    SearchConfig sc;
    sc.seed = cfg->seed;
    sc.mode = cfg->mode == FP_MODE_TABU ? SearchMode::Tabu : SearchMode::Local;
    sc.tabu_tenure = cfg->tabu_tenure;
    if (cfg->max_passes >= 0) sc.max_passes = cfg->max_passes;
    sc.debug_check_deltas = cfg->debug_check_deltas != 0;
    SearchStats st;
    Assignment a;
    const auto t0 = std::chrono::steady_clock::now();
    if (workers > 0) {
      a = sc.mode == SearchMode::Tabu
              ? parallel_tabu_search(rs, inst, t, sc, ParallelConfig{workers}, &st)
              : parallel_local_search(rs, inst, t, sc, ParallelConfig{workers}, &st);
    } else {
      // Deliberately the mode-checked entry points: tabu_search(Local cfg)
      // must throw std::invalid_argument (proj/src/search.cpp:441-452).
      a = cfg->mode == FP_MODE_TABU ? tabu_search(rs, inst, t, sc, &st)
                                    : local_search(rs, inst, t, sc, &st);
    }
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    from_assignment(inst, a, out->vehicle_base, out->mission_vehicle);
    copy_stats(st, &out->stats);
  });
}

// Calls the mode-specific entry point named by `entry` (0 local_search,
// 1 tabu_search) with cfg->mode passed through unchanged, so precondition
// tests can exercise the mismatch errors.
int ref_search_entry(const fp_instance* in, const double* cost, const fp_search_config* cfg,
                     const fp_search_start* start, int32_t entry, fp_search_result* out) {
  return guarded([&] {
    const Instance inst = to_instance(in);
    const DistanceTable t = to_table(inst, cost);
    RankedStart rs;
    rs.assignment = to_assignment(inst, start->vehicle_base, start->mission_vehicle);
    for (int k = 0; k < start->pool_size; ++k)
      if (start->pool_kind[k] == FP_POOL_EMPTY_BASE)
        rs.unused_bases.push_back(inst.bases[start->pool_index[k]].id);
    SearchConfig sc;
    sc.seed = cfg->seed;
    sc.mode = cfg->mode == FP_MODE_TABU ? SearchMode::Tabu : SearchMode::Local;
    sc.tabu_tenure = cfg->tabu_tenure;
    if (cfg->max_passes >= 0) sc.max_passes = cfg->max_passes;
    SearchStats st;
    const Assignment a = entry == 1 ? tabu_search(rs, inst, t, sc, &st)
                                    : local_search(rs, inst, t, sc, &st);
    from_assignment(inst, a, out->vehicle_base, out->mission_vehicle);
    copy_stats(st, &out->stats);
  });
}

int ref_enumerate_moves(const fp_instance* in, const double* cost,
                        const fp_search_start* state, int32_t i, int32_t j_mission_index,
                        int32_t* out_kind, double* out_delta, int32_t* out_count) {
  return guarded([&] {
    const Instance inst = to_instance(in);
    const DistanceTable t = to_table(inst, cost);
    const Assignment a = to_assignment(inst, state->vehicle_base, state->mission_vehicle);
    UnusedPool pool;
    for (int k = 0; k < state->pool_size; ++k) {
      const bool empty = state->pool_kind[k] == FP_POOL_EMPTY_BASE;
      const int idx = state->pool_index[k];
      pool.push_back({empty ? PoolEntryKind::EmptyBase : PoolEntryKind::IdleVehicle,
                      idx < 0 ? -2147483647 : (empty ? inst.bases[idx].id : inst.fleet[idx].id)});
    }
    const auto moves = enumerate_moves(a, pool, i, inst.missions[j_mission_index].id, inst, t);
    *out_count = static_cast<int32_t>(moves.size());
    for (std::size_t k = 0; k < moves.size(); ++k) {
      out_kind[k] = static_cast<int32_t>(moves[k].kind);
      out_delta[k] = moves[k].delta_km;
    }
  });
}

int ref_objective_km(const fp_instance* in, const double* cost, const int32_t* vehicle_base,
                     const int32_t* mission_vehicle, double* out_km) {
  return guarded([&] {
    const Instance inst = to_instance(in);
    const DistanceTable t = to_table(inst, cost);
    *out_km = objective_km(to_assignment(inst, vehicle_base, mission_vehicle), inst, t);
  });
}

int ref_check_feasible_count(const fp_instance* in, const int32_t* vehicle_base,
                             const int32_t* mission_vehicle, int32_t* out_violations) {
  return guarded([&] {
    const Instance inst = to_instance(in);
    *out_violations = static_cast<int32_t>(
        check_feasible(to_assignment(inst, vehicle_base, mission_vehicle), inst).size());
  });
}

int ref_brute_force_optimal_km(const fp_instance* in, double* out_km) {
  return guarded([&] { *out_km = brute_force_optimal(to_instance(in)).objective_km; });
}

}  // extern "C"
