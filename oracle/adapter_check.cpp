// oracle/adapter_check.cpp — TEST INFRASTRUCTURE ONLY.
//
// The drop-in's O(M) check_feasible / objective_km
// (integration/fleetplace_b200_adapter.cpp) against the reference's own
// O(M^2) versions (proj/src/model.cpp:118-192, compiled here under the names
// ref_cpu_* by the acceptance_b200 renames), on the reference test helpers'
// fuzzed assignments (proj/tests/test_helpers.hpp:54-91) plus unknown ids.
//
//   adapter_check [--gpu]
// check_feasible runs on the host; --gpu also compares objective_km (whose
// sum runs on the device). Prints one summary line; exit code = mismatches.

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fleetplace/errors.hpp"
#include "fleetplace/model.hpp"
#include "fleetplace/rank.hpp"
#include "fleetplace/rng.hpp"
#include "test_helpers.hpp"

namespace fleetplace {
std::vector<Violation> ref_cpu_check_feasible(const Assignment& a, const Instance& inst);
double ref_cpu_objective_km(const Assignment& a, const Instance& inst, const DistanceTable& t);
DistanceTable ref_cpu_build_distance_table(const Instance& inst, double radius_km);
RankedStart ref_cpu_rank_bases(const Instance& inst, const DistanceTable& t);
}  // namespace fleetplace

using namespace fleetplace;

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  int cases = 0, bad = 0, feasible = 0, objectives = 0;
  for (std::uint64_t seed = 1; seed <= 40; ++seed) {
    const Instance inst = helpers::small_generated(7000 + seed, 5 + (int)seed % 30);
    const DistanceTable t = ref_cpu_build_distance_table(inst, kEarthRadiusKm);
    Rng rng(seed);
    for (int k = 0; k < 51; ++k) {
      // case 50: the ranked start (feasible by construction)
      Assignment a = k == 50 ? ref_cpu_rank_bases(inst, t).assignment : helpers::fuzz_assignment(inst, rng);
      // ids the instance does not know, on either side
      if (k < 50 && k % 7 == 3) a.placement[9999] = inst.bases[0].id;
      if (k < 50 && k % 11 == 5) a.placement[inst.fleet[0].id] = 8888;
      if (k < 50 && k % 13 == 2) a.service[7777] = inst.fleet[0].id;
      if (k < 50 && k % 17 == 4 && !inst.missions.empty()) a.service[inst.missions[0].id] = 6666;
      ++cases;
      const auto want = ref_cpu_check_feasible(a, inst);
      const auto got = check_feasible(a, inst);
      if (want != got) {
        ++bad;
        std::printf("check_feasible differs: seed %llu case %d (%zu vs %zu violations)\n",
                    (unsigned long long)seed, k, want.size(), got.size());
      }
      feasible += want.empty();
      if (!gpu) continue;
      std::string e1, e2;
      double o1 = -1, o2 = -1;
      try {
        o1 = ref_cpu_objective_km(a, inst, t);
      } catch (const InfeasibleError& e) {
        e1 = e.what();
      }
      try {
        o2 = objective_km(a, inst, t);
      } catch (const InfeasibleError& e) {
        e2 = e.what();
      }
      ++objectives;
      if (e1 != e2 || (e1.empty() && std::memcmp(&o1, &o2, 8) != 0)) {
        ++bad;
        std::printf("objective_km differs: seed %llu case %d: %.17g '%s' vs %.17g '%s'\n",
                    (unsigned long long)seed, k, o1, e1.c_str(), o2, e2.c_str());
      }
    }
  }
  std::printf("adapter_check: %d cases (%d feasible), %d objectives, %d mismatches\n", cases,
              feasible, objectives, bad);
  return bad;
}
