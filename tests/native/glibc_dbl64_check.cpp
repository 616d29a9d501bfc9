// Checks csrc/glibc_dbl64.cuh against the libm it restates, bit for bit.
// Built and run by tests/test_glibc_dbl64.py (g++ -O2 -mfma -ffp-contract=off).
// Usage: glibc_dbl64_check <n_random_per_range> <seed>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <random>
#include "glibc_dbl64.cuh"

static int fails = 0;
static long long checked = 0;

static void check(const char* fn, double x, double got, double want) {
  ++checked;
  if (gl64::bits(got) == gl64::bits(want) || (std::isnan(got) && std::isnan(want))) return;
  if (fails++ < 20)
    std::printf("MISMATCH %s(%a) = %a, libm %a\n", fn, x, got, want);
}

// volatile function pointers: the compiler may not fold or inline libm
static double (*volatile lsin)(double) = std::sin;
static double (*volatile lcos)(double) = std::cos;
static double (*volatile lasin)(double) = std::asin;

static void one(double x, int which) {
  if (which & 1) check("sin", x, gl64::sin(x), lsin(x));
  if (which & 2) check("cos", x, gl64::cos(x), lcos(x));
  if (which & 4) check("asin", x, gl64::asin(x), lasin(x));
}

// random arguments uniform in [lo, hi) and around each end (+-64 ulp)
static void range(std::mt19937_64& g, double lo, double hi, long n, int which) {
  std::uniform_real_distribution<double> U(lo, hi);
  for (long i = 0; i < n; ++i) { double x = U(g); one(x, which); one(-x, which); }
  for (double e : {lo, hi}) {
    double a = e, b = e;
    for (int i = 0; i < 64; ++i) {
      one(a, which); one(b, which); one(-a, which); one(-b, which);
      a = std::nextafter(a, 0.0); b = std::nextafter(b, 1e300);
    }
  }
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? std::atol(argv[1]) : 1000000;
  std::mt19937_64 g(argc > 2 ? std::atoll(argv[2]) : 1);
  // sin / cos: every branch of the restated range (|x| < 105414350)
  const double sc[] = {0x1p-40, 0x1p-27, 0x1p-26, 0.126, 0.855469, 1.5707963267948966,
                       2.426265, 3.141592653589793, 6.3, 100.0, 1e5, 1e8};
  for (int i = 0; i + 1 < (int)(sizeof sc / sizeof sc[0]); ++i) range(g, sc[i], sc[i + 1], n, 3);
  // asin: every range of e_asin.c
  const double as[] = {0x1p-40, 0x1p-26, 0.125, 0.25, 0.5, 0.75, 0.921875, 0.953125,
                       0.96875, 0.984375, 0.999, 1.0};
  for (int i = 0; i + 1 < (int)(sizeof as / sizeof as[0]); ++i) range(g, as[i], as[i + 1], n, 4);
  for (double x : {0.0, -0.0, 1.0, -1.0, 1.0000000000000002, (double)INFINITY, -(double)INFINITY, (double)NAN}) one(x, 4);
  for (double x : {0.0, -0.0, (double)INFINITY, (double)NAN}) one(x, 3);
  // the haversine's own arguments: 0.5*|dlat|*deg2rad, 0.5*|dlon|*deg2rad
  // (sin), lat*deg2rad (cos), sqrt(h) (asin) on random coordinates
  const double k = 3.14159265358979323846 / 180.0;
  std::uniform_real_distribution<double> La(-90.0, 90.0), Lo(-180.0, 180.0);
  for (long i = 0; i < 4 * n; ++i) {
    const double a = La(g), b = La(g), c = Lo(g), d = Lo(g);
    one(0.5 * std::fabs(b - a) * k, 1);
    one(0.5 * std::fabs(d - c) * k, 1);
    one(a * k, 2);
    const double sl = std::sin(0.5 * std::fabs(b - a) * k), so = std::sin(0.5 * std::fabs(d - c) * k);
    const double h = sl * sl + std::cos(a * k) * std::cos(b * k) * so * so;
    one(std::fmin(1.0, std::sqrt(h)), 4);
  }
  std::printf("checked %lld arguments, %d mismatches\n", checked, fails);
  return fails != 0;
}
