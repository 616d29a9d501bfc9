// integration/fleetplace_b200_adapter.cpp — the reference-side binding.
//
// Implements the reference's hot-path entry points on top of the C ABI
// (include/fleetplace_b200.h), compiled against the reference's own headers
// (/root/reference/proj/include/fleetplace/*.hpp):
//   build_distance_table  proj/include/fleetplace/model.hpp:68-69
//   column_totals         proj/include/fleetplace/rank.hpp:21
//   rank_bases            proj/include/fleetplace/rank.hpp:30
//   local_search / tabu_search   proj/include/fleetplace/search.hpp:128-138
//   check_feasible / objective_km proj/include/fleetplace/model.hpp:108-119
// A maintainer links this file into the `fleetplace` library and compiles the
// reference's own definitions of those seven functions out (oracle/Makefile
// target `acceptance_b200` does it with -D renames), so every caller —
// run_experiment, brute_force_optimal, parallel_local_search(workers=1), the
// CLI, the tests — runs the B200 path. Errors come back as the reference's
// exception types.
//
// GPU-side configuration (never through SearchConfig): the device is
// FLEETPLACE_DEVICE (default 0) or fleetplace::b200::set_device(). The
// distance table stays resident on the device across calls: a call whose
// matrix has the resident table's data pointer, shape and content hash
// (a 64-bit hash over every entry, multi-threaded) skips the upload.

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
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

int g_device = -1;  // -1: FLEETPLACE_DEVICE or 0

int device_ordinal() {
  if (g_device >= 0) return g_device;
  const char* e = std::getenv("FLEETPLACE_DEVICE");
  return e ? std::max(0, std::atoi(e)) : 0;
}

// The matrix resident in a context: where it came from and its content.
struct Resident {
  const double* ptr = nullptr;
  long long rows = -1, cols = -1;
  unsigned long long hash = 0;
};

// One context per host thread (fp_ctx is not thread-safe).
struct Ctx {
  fp_ctx* p = nullptr;
  int device = -1;
  Resident res;
  ~Ctx() {
    if (p) fp_ctx_destroy(p);
  }
};
Ctx& ctx_state() {
  thread_local Ctx c;
  const int d = device_ordinal();
  if (!c.p || c.device != d) {
    if (c.p) fp_ctx_destroy(c.p);
    c.p = nullptr;
    c.res = Resident{};
    check(fp_ctx_create(d, &c.p));
    c.device = d;
  }
  return c;
}
fp_ctx* ctx() { return ctx_state().p; }

// 64-bit content hash of a table: four independent multiply-xor lanes per
// thread (memory-bound), chunk hashes combined in order.
unsigned long long table_hash(const double* p, std::size_t n) {
  auto chunk = [](const double* q, std::size_t k) {
    unsigned long long a[4] = {0x9E3779B97F4A7C15ull, 0xC2B2AE3D27D4EB4Full, 0x165667B19E3779F9ull,
                               0x27D4EB2F165667C5ull};
    std::size_t i = 0;
    for (; i + 4 <= k; i += 4)
      for (int l = 0; l < 4; ++l) {
        unsigned long long w;
        std::memcpy(&w, q + i + l, 8);
        a[l] = (a[l] ^ w) * 0x100000001B3ull + (a[l] >> 29);
      }
    for (; i < k; ++i) {
      unsigned long long w;
      std::memcpy(&w, q + i, 8);
      a[0] = (a[0] ^ w) * 0x100000001B3ull + (a[0] >> 29);
    }
    return (a[0] * 31 + a[1]) * 31 * 31 + a[2] * 31 + a[3] + k;
  };
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const unsigned T = n < (1u << 22) ? 1u : hw;
  const std::size_t per = (n + T - 1) / T;
  std::vector<unsigned long long> hs(T, 0);
  std::vector<std::thread> ws;
  for (unsigned t = 1; t < T; ++t)
    ws.emplace_back([&, t] {
      const std::size_t lo = std::min(n, t * per), hi = std::min(n, lo + per);
      hs[t] = chunk(p + lo, hi - lo);
    });
  hs[0] = chunk(p, std::min(n, per));
  for (auto& w : ws) w.join();
  unsigned long long h = 0xCBF29CE484222325ull;
  for (unsigned long long x : hs) h = (h ^ x) * 0x100000001B3ull;
  return h;
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

// Makes `cost` the context's resident table unless it already is.
void upload(const Eigen::MatrixXd& cost) {
  Ctx& c = ctx_state();
  const std::size_t n = (std::size_t)cost.rows() * (std::size_t)cost.cols();
  const unsigned long long h = table_hash(cost.data(), n);
  if (c.res.ptr == cost.data() && c.res.rows == cost.rows() && c.res.cols == cost.cols() &&
      c.res.hash == h)
    return;
  c.res = Resident{};
  check(fp_table_upload(c.p, (int32_t)cost.rows(), (int32_t)cost.cols(), cost.data()));
  c.res = Resident{cost.data(), (long long)cost.rows(), (long long)cost.cols(), h};
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

namespace b200 {
// Selects the CUDA device of the calling thread's later calls.
void set_device(int device) { g_device = device < 0 ? -1 : device; }
}  // namespace b200

DistanceTable build_distance_table(const Instance& inst, double radius_km) {
  InstView iv(inst);
  DistanceTable t;
  t.earth_radius_km = radius_km;
  t.cost.resize((Eigen::Index)inst.missions.size(), (Eigen::Index)inst.bases.size());
  Ctx& c = ctx_state();
  c.res = Resident{};
  check(fp_build_distance_table(c.p, &iv.c, radius_km, t.cost.data()));
  // the device copy is this matrix: later calls on it skip the upload (the
  // returned DistanceTable keeps the same heap buffer when moved)
  c.res = Resident{t.cost.data(), (long long)t.cost.rows(), (long long)t.cost.cols(),
                   table_hash(t.cost.data(), (std::size_t)t.cost.rows() * t.cost.cols())};
  return t;
}

// check_feasible (proj/src/model.cpp:118-174): the same rules, report order
// and de-duplication, with id -> index hash maps instead of
// Instance::*_index linear scans (first index wins, like index_of).
std::vector<Violation> check_feasible(const Assignment& a, const Instance& inst) {
  std::unordered_map<int, int> bidx, vidx, midx;
  bidx.reserve(inst.bases.size() * 2);
  vidx.reserve(inst.fleet.size() * 2);
  midx.reserve(inst.missions.size() * 2);
  for (std::size_t i = 0; i < inst.bases.size(); ++i) bidx.emplace(inst.bases[i].id, (int)i);
  for (std::size_t i = 0; i < inst.fleet.size(); ++i) vidx.emplace(inst.fleet[i].id, (int)i);
  for (std::size_t i = 0; i < inst.missions.size(); ++i) midx.emplace(inst.missions[i].id, (int)i);
  auto find = [](const std::unordered_map<int, int>& m, int id) {
    auto it = m.find(id);
    return it == m.end() ? -1 : it->second;
  };
  std::vector<Violation> out;
  std::set<std::pair<Rule, int>> reported;
  auto report = [&](Rule r, int subject, int related = -1) {
    if (reported.insert({r, subject}).second) out.push_back(Violation{r, subject, related});
  };
  std::map<int, int> base_load;
  for (const auto& [vid, bid] : a.placement) {
    const int vi = find(vidx, vid), bi = find(bidx, bid);
    if (vi < 0 || bi < 0) {
      report(Rule::OneBasePerVehicle, vid, bid);
      continue;
    }
    base_load[bid] += 1;
    if (!compatible_vehicle_base(inst.fleet[(std::size_t)vi], inst.bases[(std::size_t)bi]))
      report(Rule::FixedWingOnHelipad, vid, bid);
  }
  for (const auto& [bid, load] : base_load)
    if (load > 1) report(Rule::BaseOccupancy, bid);
  for (const Vehicle& v : inst.fleet)
    if (!a.placement.contains(v.id)) report(Rule::OneBasePerVehicle, v.id);
  for (const auto& [mid, vid] : a.service) {
    const int mi = find(midx, mid), vi = find(vidx, vid);
    if (mi < 0) {
      report(Rule::OneVehiclePerMission, mid, vid);
      continue;
    }
    if (vi < 0) {
      report(Rule::ServiceRequiresPlacement, vid, mid);
      continue;
    }
    if (!a.placement.contains(vid)) report(Rule::ServiceRequiresPlacement, vid, mid);
    if (!compatible_vehicle_mission(inst.fleet[(std::size_t)vi], inst.missions[(std::size_t)mi]))
      report(Rule::RotaryOnly, mid, vid);
  }
  for (const Mission& m : inst.missions)
    if (!a.service.contains(m.id)) report(Rule::OneVehiclePerMission, m.id);
  return out;
}

// objective_km (proj/src/model.cpp:176-192): feasibility as above, then the
// fixed mission-order sum on the device (fp_objective_km, bit-identical).
double objective_km(const Assignment& a, const Instance& inst, const DistanceTable& t) {
  const auto violations = check_feasible(a, inst);
  if (!violations.empty())
    throw InfeasibleError("infeasible assignment: " + to_string(violations.front()));
  InstView iv(inst);
  std::vector<int32_t> vb(iv.vid.size(), -1), mv(iv.mid.size(), -1);
  for (const auto& [vid, bid] : a.placement) vb[(std::size_t)iv.v(vid)] = iv.b(bid);
  for (std::size_t m = 0; m < iv.mid.size(); ++m) mv[m] = iv.v(a.service.at(iv.mid[m]));
  upload(t.cost);
  double km = 0.0;
  check(fp_objective_km(ctx(), (int32_t)vb.size(), vb.data(), mv.data(), &km));
  return km;
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
