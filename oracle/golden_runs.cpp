// oracle/golden_runs.cpp — TEST INFRASTRUCTURE ONLY (never linked by the product).
//
// Long reference runs for the committed goldens (tests/golden/runs.json, made
// by tests/golden/make_run_goldens.py). It drives the UNMODIFIED reference
// (objects from oracle/Makefile) through its own public API, exactly as
// run_experiment does (proj/src/bench.cpp:103-186):
//   synthesize_pool + generate_instance  proj/src/data.cpp:110-180 (SURVEY §8(d) recipe)
//   build_distance_table                 proj/src/model.cpp:76-90
//   rank_bases                           proj/src/rank.cpp:25-124
//   tabu_search / local_search           proj/src/search.cpp:438-460
// and dumps the ranking and the search result in index form.
//
//   golden_runs B M V inst_seed search_seed max_passes(-1 = none) mode(1 tabu, 0 local)
//               table_threads out_prefix
//
// table_threads > 1 fills the table with the reference's own per-entry
// function mission_cost_km (proj/src/geo.cpp:32-36) on several threads, one
// column range each; build_distance_table computes exactly
// cost(m, b) = mission_cost_km(bases[b].location, missions[m], radius) per
// entry (proj/src/model.cpp:82-88), a pure function, so the table bits are
// the same (checked: tests/test_oracle.py::test_golden_runs_parallel_table).
// It exists for c4 only, whose 1e10 entries take ~14 min on one core.

#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "fleetplace/data.hpp"
#include "fleetplace/geo.hpp"
#include "fleetplace/model.hpp"
#include "fleetplace/rank.hpp"
#include "fleetplace/search.hpp"

using namespace fleetplace;

static double secs_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

static void dump(const std::string& path, const void* p, std::size_t n) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) { std::perror(path.c_str()); std::exit(2); }
  if (n && std::fwrite(p, 1, n, f) != n) { std::perror(path.c_str()); std::exit(2); }
  std::fclose(f);
}

int main(int argc, char** argv) {
  if (argc != 10) {
    std::fprintf(stderr, "usage: %s B M V inst_seed search_seed max_passes mode threads out_prefix\n",
                 argv[0]);
    return 2;
  }
  const int B = std::atoi(argv[1]), M = std::atoi(argv[2]), V = std::atoi(argv[3]);
  const std::uint64_t iseed = std::strtoull(argv[4], nullptr, 10);
  const std::uint64_t sseed = std::strtoull(argv[5], nullptr, 10);
  const int max_passes = std::atoi(argv[6]);
  const int mode = std::atoi(argv[7]);
  const int threads = std::atoi(argv[8]);
  const std::string out = argv[9];

  // SURVEY §8(d) recipe (the same as tests/oracle_harness.py ref_survey_instance)
  const int A = (274 * B + 189) / 378, R = (2 * V + 1) / 3;
  const int S = std::max(200, M / 50);
  const FacilityPool pool = synthesize_pool(iseed, BoundingBox{}, PoolCounts{A, B - A, S});
  const Instance inst = generate_instance(pool, M, 0.3, iseed, R, V - R);

  auto t0 = std::chrono::steady_clock::now();
  DistanceTable t;
  if (threads <= 1) {
    t = build_distance_table(inst);
  } else {
    t.earth_radius_km = kEarthRadiusKm;
    t.cost.resize(M, B);
    std::vector<std::thread> ws;
    for (int w = 0; w < threads; ++w)
      ws.emplace_back([&, w] {
        for (int b = w; b < B; b += threads) {
          const GeoPoint& loc = inst.bases[static_cast<std::size_t>(b)].location;
          for (int m = 0; m < M; ++m)
            t.cost(m, b) = mission_cost_km(loc, inst.missions[static_cast<std::size_t>(m)],
                                           kEarthRadiusKm);
        }
      });
    for (auto& w : ws) w.join();
  }
  const double table_s = secs_since(t0);
  if (const char* tp = std::getenv("GOLDEN_DUMP_TABLE"))
    dump(out + ".table.bin", t.cost.data(), sizeof(double) * (std::size_t)M * B), (void)tp;

  t0 = std::chrono::steady_clock::now();
  const RankedStart rs = rank_bases(inst, t);
  const double rank_s = secs_since(t0);

  std::map<int, int> bidx, vidx;
  for (int b = 0; b < B; ++b) bidx[inst.bases[b].id] = b;
  for (int v = 0; v < V; ++v) vidx[inst.fleet[v].id] = v;
  auto index_form = [&](const Assignment& a, std::vector<int32_t>& vb, std::vector<int32_t>& mv) {
    vb.assign(V, -1);
    mv.assign(M, -1);
    for (const auto& [vid, bid] : a.placement) vb[vidx.at(vid)] = bidx.at(bid);
    // Mission ids are dense 0..M-1 in generated instances (proj/src/data.cpp:166-174)
    for (const auto& [mid, vid] : a.service) mv[mid] = vidx.at(vid);
  };
  for (int m = 0; m < M; ++m)
    if (inst.missions[m].id != m) { std::fprintf(stderr, "mission ids not dense\n"); return 3; }

  std::vector<int32_t> rvb, rmv, unused;
  index_form(rs.assignment, rvb, rmv);
  for (int id : rs.unused_bases) unused.push_back(bidx.at(id));
  dump(out + ".totals.bin", rs.base_totals.data(), sizeof(double) * B);
  dump(out + ".rank_vb.bin", rvb.data(), 4 * rvb.size());
  dump(out + ".rank_mv.bin", rmv.data(), 4 * rmv.size());
  dump(out + ".unused.bin", unused.data(), 4 * unused.size());

  SearchConfig sc;
  sc.seed = sseed;
  sc.mode = mode == 1 ? SearchMode::Tabu : SearchMode::Local;
  if (max_passes >= 0) sc.max_passes = max_passes;
  SearchStats st;
  t0 = std::chrono::steady_clock::now();
  const Assignment a = mode == 1 ? tabu_search(rs, inst, t, sc, &st) : local_search(rs, inst, t, sc, &st);
  const double search_s = secs_since(t0);
  std::vector<int32_t> vb, mv;
  index_form(a, vb, mv);
  dump(out + ".vb.bin", vb.data(), 4 * vb.size());
  dump(out + ".mv.bin", mv.data(), 4 * mv.size());

  std::uint64_t bits;
  std::memcpy(&bits, &st.final_objective_km, 8);
  std::printf("{\"bases\": %d, \"missions\": %d, \"vehicles\": %d, \"instance_seed\": %" PRIu64
              ", \"search_seed\": %" PRIu64 ", \"max_passes\": %d, \"mode\": %d, "
              "\"stats\": [%" PRIu64 ", %" PRIu64 ", %" PRIu64 ", %" PRIu64 ", %" PRIu64 ", %" PRIu64
              "], \"final_objective_km\": %.17g, \"final_objective_bits\": \"%016" PRIx64 "\", "
              "\"table_s\": %.3f, \"table_threads\": %d, \"rank_s\": %.3f, \"search_s\": %.3f}\n",
              B, M, V, iseed, sseed, max_passes, mode, st.passes, st.evaluations, st.applied_moves,
              st.committed_moves, st.tabu_skips_outer, st.tabu_skips_inner, st.final_objective_km,
              bits, table_s, threads, rank_s, search_s);
  return 0;
}
