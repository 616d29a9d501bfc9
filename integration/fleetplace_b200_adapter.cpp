// integration/fleetplace_b200_adapter.cpp — the reference-side binding.
//
// Implements the reference's hot-path entry points on top of the C ABI
// (include/fleetplace_b200.h), compiled against the reference's own headers
// (/root/reference/proj/include/fleetplace/*.hpp):
//   build_distance_table  proj/include/fleetplace/model.hpp:68-69
//   column_totals         proj/include/fleetplace/rank.hpp:21
//   rank_bases            proj/include/fleetplace/rank.hpp:30
//   local_search / tabu_search   proj/include/fleetplace/search.hpp:128-138
// A maintainer links this file into the `fleetplace` library and compiles the
// reference's own definitions of those five functions out (oracle/Makefile
// target `acceptance_b200` does it with -D renames), so every caller —
// run_experiment, brute_force_optimal, parallel_local_search(workers=1), the
// CLI, the tests — runs the B200 path. Errors come back as the reference's
// exception types.

#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "fleetplace/errors.hpp"
#include "fleetplace/model.hpp"
#include "fleetplace/rank.hpp"
#include "fleetplace/search.hpp"
#include "fleetplace_b200.h"

namespace fleetplace {
namespace {

[[noreturn]] void raise(fp_status s) {
  const std::string m = fp_last_error();
  switch (s) {
    case FP_ERR_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case FP_ERR_VALIDATION: throw ValidationError("b200", m);
    case FP_ERR_INFEASIBLE: throw InfeasibleError(m);
    case FP_ERR_NO_COMPATIBLE: throw NoCompatibleVehicleError(m);
    case FP_ERR_POOL_TOO_SMALL: throw PoolTooSmallError(m);
    case FP_ERR_LOGIC: throw std::logic_error(m);
    default: throw Error(m);
  }
}

void check(fp_status s) {
  if (s != FP_OK) raise(s);
}

// One context per host thread (fp_ctx is not thread-safe).
struct Ctx {
  fp_ctx* p = nullptr;
  Ctx() { check(fp_ctx_create(0, &p)); }
  ~Ctx() { fp_ctx_destroy(p); }
};
fp_ctx* ctx() {
  thread_local Ctx c;
  return c.p;
}

// Structure-of-arrays view of an Instance for the duration of a call.
struct InstView {
  std::vector<int32_t> bid, vid, mid;
  std::vector<uint8_t> bkind, vkind, ro;
  std::vector<double> blat, blon, plat, plon, dlat, dlon;
  fp_instance c{};
  std::unordered_map<int, int> bidx, vidx, midx;

  explicit InstView(const Instance& inst) {
    for (const Base& b : inst.bases) {
      bidx.emplace(b.id, (int)bid.size());
      bid.push_back(b.id);
      bkind.push_back(b.kind == BaseKind::Helipad ? FP_HELIPAD : FP_AERODROME);
      blat.push_back(b.location.lat_deg);
      blon.push_back(b.location.lon_deg);
    }
    for (const Vehicle& v : inst.fleet) {
      vidx.emplace(v.id, (int)vid.size());
      vid.push_back(v.id);
      vkind.push_back(v.kind == VehicleKind::FixedWing ? FP_FIXED : FP_ROTARY);
    }
    for (const Mission& m : inst.missions) {
      midx.emplace(m.id, (int)mid.size());
      mid.push_back(m.id);
      plat.push_back(m.pickup.lat_deg);
      plon.push_back(m.pickup.lon_deg);
      dlat.push_back(m.delivery.lat_deg);
      dlon.push_back(m.delivery.lon_deg);
      ro.push_back(m.rotary_only ? 1 : 0);
    }
    c = fp_instance{(int32_t)bid.size(), bid.data(), bkind.data(), blat.data(), blon.data(),
                    (int32_t)vid.size(), vid.data(), vkind.data(), (int32_t)mid.size(),
                    mid.data(), plat.data(), plon.data(), dlat.data(), dlon.data(), ro.data()};
  }
  int b(int id) const { auto it = bidx.find(id); return it == bidx.end() ? -1 : it->second; }
  int v(int id) const { auto it = vidx.find(id); return it == vidx.end() ? -1 : it->second; }
  int m(int id) const { auto it = midx.find(id); return it == midx.end() ? -1 : it->second; }
};

void upload(const Eigen::MatrixXd& cost) {
  check(fp_table_upload(ctx(), (int32_t)cost.rows(), (int32_t)cost.cols(), cost.data()));
}

Assignment to_assignment(const InstView& iv, const std::vector<int32_t>& vb,
                         const std::vector<int32_t>& mv) {
  Assignment a;
  for (std::size_t v = 0; v < vb.size(); ++v)
    if (vb[v] >= 0) a.placement[iv.vid[v]] = iv.bid[(std::size_t)vb[v]];
  for (std::size_t m = 0; m < mv.size(); ++m)
    if (mv[m] >= 0) a.service[iv.mid[m]] = iv.vid[(std::size_t)mv[m]];
  return a;
}

Assignment search(const RankedStart& start, const Instance& inst, const DistanceTable& t,
                  const SearchConfig& cfg, SearchStats* stats, int32_t mode) {
  InstView iv(inst);
  // SearchState::from's id checks (proj/src/search.cpp:25-40), with O(1) maps
  std::vector<int32_t> vb(iv.vid.size(), -1), mv(iv.mid.size(), -1);
  for (const auto& [vid, bid] : start.assignment.placement) {
    const int vi = iv.v(vid), bi = iv.b(bid);
    if (vi < 0 || bi < 0) throw InfeasibleError("assignment references unknown ids");
    vb[(std::size_t)vi] = bi;
  }
  for (const auto& [mid, vid] : start.assignment.service) {
    const int mi = iv.m(mid), vi = iv.v(vid);
    if (mi < 0 || vi < 0 || vb[(std::size_t)vi] < 0)
      throw InfeasibleError("service references unplaced vehicle");
    mv[(std::size_t)mi] = vi;
  }
  std::vector<int32_t> pk, px;
  for (const PoolEntry& e : initial_pool(start, inst)) {
    const bool empty = e.kind == PoolEntryKind::EmptyBase;
    pk.push_back(empty ? FP_POOL_EMPTY_BASE : FP_POOL_IDLE_VEHICLE);
    px.push_back(empty ? iv.b(e.id) : iv.v(e.id));
  }
  upload(t.cost);
  fp_search_config c{cfg.seed, mode, cfg.tabu_tenure, cfg.max_passes ? *cfg.max_passes : -1,
                     cfg.debug_check_deltas ? 1 : 0};
  fp_search_start s{vb.data(), mv.data(), (int32_t)pk.size(), pk.data(), px.data()};
  std::vector<int32_t> ovb(vb.size()), omv(mv.size());
  fp_search_result r{};
  r.vehicle_base = ovb.data();
  r.mission_vehicle = omv.data();
  check(fp_search(ctx(), &iv.c, &c, &s, &r));
  if (stats) {
    stats->passes = r.stats.passes;
    stats->evaluations = r.stats.evaluations;
    stats->applied_moves = r.stats.applied_moves;
    stats->committed_moves = r.stats.committed_moves;
    stats->tabu_skips_outer = r.stats.tabu_skips_outer;
    stats->tabu_skips_inner = r.stats.tabu_skips_inner;
    stats->final_objective_km = r.stats.final_objective_km;
  }
  return to_assignment(iv, ovb, omv);
}

}  // namespace

DistanceTable build_distance_table(const Instance& inst, double radius_km) {
  InstView iv(inst);
  DistanceTable t;
  t.earth_radius_km = radius_km;
  t.cost.resize((Eigen::Index)inst.missions.size(), (Eigen::Index)inst.bases.size());
  check(fp_build_distance_table(ctx(), &iv.c, radius_km, t.cost.data()));
  return t;
}

Eigen::VectorXd column_totals(const Eigen::MatrixXd& cost) {
  Eigen::VectorXd out(cost.cols());
  if (cost.cols() == 0) return out;
  upload(cost);
  check(fp_column_totals(ctx(), out.data()));
  return out;
}

RankedStart rank_bases(const Instance& inst, const DistanceTable& t) {
  InstView iv(inst);
  const std::size_t B = iv.bid.size(), V = iv.vid.size(), M = iv.mid.size();
  // validate first, as the reference does (proj/src/rank.cpp:26)
  check(fp_validate_instance(&iv.c));
  upload(t.cost);
  RankedStart start;
  start.base_totals = Eigen::VectorXd((Eigen::Index)B);
  std::vector<int32_t> vb(V), mv(M), unused(B);
  fp_ranked_start r{start.base_totals.data(), vb.data(), mv.data(), unused.data(), 0};
  check(fp_rank_bases(ctx(), &iv.c, &r));
  start.assignment = to_assignment(iv, vb, mv);
  for (int k = 0; k < r.n_unused; ++k) start.unused_bases.push_back(iv.bid[(std::size_t)unused[k]]);
  return start;
}

Assignment local_search(const RankedStart& start, const Instance& inst, const DistanceTable& t,
                        const SearchConfig& cfg, SearchStats* stats) {
  if (cfg.mode != SearchMode::Local)
    throw std::invalid_argument("local_search requires SearchMode::Local");
  return search(start, inst, t, cfg, stats, FP_MODE_LOCAL);
}

Assignment tabu_search(const RankedStart& start, const Instance& inst, const DistanceTable& t,
                       const SearchConfig& cfg, SearchStats* stats) {
  if (cfg.mode != SearchMode::Tabu)
    throw std::invalid_argument("tabu_search requires SearchMode::Tabu");
  return search(start, inst, t, cfg, stats, FP_MODE_TABU);
}

}  // namespace fleetplace
