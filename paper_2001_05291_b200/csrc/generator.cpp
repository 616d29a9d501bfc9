// generator.cpp — synthetic instances (host, sequential RNG).
//
// Restates synthesize_pool + generate_instance (proj/src/data.cpp:110-180)
// with the default PoolShape (proj/include/fleetplace/data.hpp:40-45), the
// library's RNG helpers (proj/include/fleetplace/rng.hpp:14-27) and
// standard_normal (proj/src/rng.cpp:9-15). It is the input formatter for the
// benchmark shapes, not part of the accelerated path; the
// sequential mt19937_64 stream has no data parallelism to exploit.
// Identical bits to the reference require the same libm (glibc log/cos/sqrt)
// and no FMA contraction, which holds for this host build (baseline x86-64).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "host_common.hpp"

namespace fpk_host {

namespace {

using Rng = std::mt19937_64;

uint64_t uniform_below(Rng& rng, uint64_t n) {
  const uint64_t threshold = (0 - n) % n;
  uint64_t x = rng();
  while (x < threshold) x = rng();
  return x % n;
}

double uniform_unit(Rng& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

double standard_normal(Rng& rng) {
  double u1 = uniform_unit(rng);
  while (u1 == 0.0) u1 = uniform_unit(rng);
  const double u2 = uniform_unit(rng);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
}

double lerp(double a, double b, double t) { return a + (b - a) * t; }
double clamp_to(double v, double lo, double hi) { return std::min(hi, std::max(lo, v)); }

struct Pt {
  double lat, lon;
};

struct Box {
  double lat_min = 42.0, lat_max = 57.0, lon_min = -96.0, lon_max = -74.0;
};

// PoolShape defaults: 5 clusters, sigma 0.35 deg, urban 0.7, helipads on sites.
constexpr int kClusters = 5;
constexpr double kSigma = 0.35;
constexpr double kUrban = 0.7;
constexpr double kHelipadSiteFraction = 1.0;

Pt sample_point(Rng& rng, const Box& box, const std::vector<Pt>& centers) {
  if (!centers.empty() && uniform_unit(rng) < kUrban) {
    const Pt c = centers[uniform_below(rng, centers.size())];
    const double lat = c.lat + kSigma * standard_normal(rng);
    const double lon = c.lon + kSigma * standard_normal(rng);
    return {clamp_to(lat, box.lat_min, box.lat_max), clamp_to(lon, box.lon_min, box.lon_max)};
  }
  const double lat = lerp(box.lat_min, box.lat_max, uniform_unit(rng));
  const double lon = lerp(box.lon_min, box.lon_max, uniform_unit(rng));
  return {lat, lon};
}

}  // namespace

void generate_instance(uint64_t pool_seed, const double* bbox, int aerodromes, int helipads,
                       int health_sites, int missions, double rotary_only_fraction,
                       uint64_t seed, int rotary, int fixed_wing, int32_t* base_id,
                       uint8_t* base_kind, double* base_lat, double* base_lon,
                       int32_t* vehicle_id, uint8_t* vehicle_kind, int32_t* mission_id,
                       double* pickup_lat, double* pickup_lon, double* delivery_lat,
                       double* delivery_lon, uint8_t* rotary_only) {
  Box box;
  if (bbox) box = Box{bbox[0], bbox[1], bbox[2], bbox[3]};
  // synthesize_pool
  if (aerodromes <= 0 || helipads < 0 || health_sites <= 0)
    throw FpError(FP_ERR_POOL_TOO_SMALL, "pool counts must be positive");
  std::vector<Pt> sites, aeros, helis;
  {
    Rng rng(pool_seed);
    std::vector<Pt> centers;
    for (int c = 0; c < kClusters; ++c) {
      const double lat = lerp(box.lat_min, box.lat_max, uniform_unit(rng));
      const double lon = lerp(box.lon_min, box.lon_max, uniform_unit(rng));
      centers.push_back({lat, lon});
    }
    for (int i = 0; i < health_sites; ++i) sites.push_back(sample_point(rng, box, centers));
    for (int i = 0; i < aerodromes; ++i) aeros.push_back(sample_point(rng, box, centers));
    for (int i = 0; i < helipads; ++i) {
      if (uniform_unit(rng) < kHelipadSiteFraction)
        helis.push_back(sites[uniform_below(rng, sites.size())]);
      else
        helis.push_back(sample_point(rng, box, centers));
    }
  }
  // generate_instance
  if (sites.size() < 2) throw FpError(FP_ERR_POOL_TOO_SMALL, "need at least two health sites");
  if (static_cast<int>(aeros.size()) < fixed_wing)
    throw FpError(FP_ERR_POOL_TOO_SMALL, "need at least one aerodrome per fixed-wing vehicle");
  if (static_cast<int>(aeros.size() + helis.size()) < rotary + fixed_wing)
    throw FpError(FP_ERR_POOL_TOO_SMALL, "fewer bases than vehicles");
  if (rotary + fixed_wing <= 0) throw FpError(FP_ERR_POOL_TOO_SMALL, "fleet must not be empty");
  Rng rng(seed);
  int k = 0;
  for (const Pt& p : aeros) {
    base_id[k] = k;
    base_kind[k] = FP_AERODROME;
    base_lat[k] = p.lat;
    base_lon[k] = p.lon;
    ++k;
  }
  for (const Pt& p : helis) {
    base_id[k] = k;
    base_kind[k] = FP_HELIPAD;
    base_lat[k] = p.lat;
    base_lon[k] = p.lon;
    ++k;
  }
  for (int v = 0; v < rotary + fixed_wing; ++v) {
    vehicle_id[v] = v;
    vehicle_kind[v] = v < rotary ? FP_ROTARY : FP_FIXED;
  }
  const uint64_t n_sites = sites.size();
  for (int m = 0; m < missions; ++m) {
    const uint64_t pick = uniform_below(rng, n_sites);
    uint64_t drop = uniform_below(rng, n_sites - 1);
    if (drop >= pick) ++drop;
    const bool ro = uniform_unit(rng) < rotary_only_fraction;
    mission_id[m] = m;
    pickup_lat[m] = sites[pick].lat;
    pickup_lon[m] = sites[pick].lon;
    delivery_lat[m] = sites[drop].lat;
    delivery_lon[m] = sites[drop].lon;
    rotary_only[m] = ro ? 1 : 0;
  }
}

}  // namespace fpk_host
