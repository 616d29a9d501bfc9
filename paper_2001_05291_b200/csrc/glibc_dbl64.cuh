// glibc_dbl64.cuh — sin, cos and asin bit-identical to the glibc libm the
// reference links against (third-party dependency, not in /root/reference:
// Ubuntu GLIBC 2.39-0ubuntu8.5, libm.so.6 build-id
// 0d9969fe206760d250ec30a5a9be18aefbf84ea8, x86-64 FMA variants __sin_fma,
// __cos_fma, __ieee754_asin_fma that the ifunc resolvers pick on any CPU with
// FMA + AVX2).
//
// The reference's haversine (proj/src/geo.cpp:25-29) calls std::sin, std::cos
// and std::asin. CUDA's fp64 versions differ from glibc's in the last bits
// (neither is correctly rounded), so a table built with them was within ~8
// ulp of the reference's, not equal. This file restates glibc's published
// dbl-64 algorithms (sysdeps/ieee754/dbl-64/s_sin.c: do_sin / do_cos /
// TAYLOR_SIN / reduce_sincos; e_asin.c: the Taylor branch, the five
// table-driven polynomial ranges and the Newton square-root branch near 1)
// with every fused multiply-add exactly where GCC contracted one in that
// libm build (read from its disassembly) and every other product and sum a
// separately rounded IEEE operation. The coefficient tables (__sincostab,
// asncs, inroot, powtwo) are glibc's own data: they are not committed here,
// `paper_2001_05291_b200/_glibc_tables.py` extracts them from the image's
// libm.so.6 at build time (checking its build-id) into
// csrc/gen/glibc_dbl64_tables.inc. The scalar polynomial constants below are
// the values of that binary's .rodata (the same script checks them).
//
// Domain: the haversine needs sin on [0, pi], cos on [-pi/2, pi/2] and asin
// on [0, 1]; sin/cos are restated for |x| < 105414350 (glibc's own
// reduce_sincos range; beyond it glibc uses a multi-precision reduction that
// is not restated), asin for every input. Verified against libm itself on
// the host by tests/test_glibc_dbl64.py (every branch, random and edge
// arguments) and, on the device, by tables bit-equal to the reference's.
//
// Compiles as CUDA device code (nvcc) and as host C/C++ (the test harness;
// build it with -ffp-contract=off so the host compiler fuses nothing either).
#pragma once

#include <stdint.h>
#include <string.h>
#include <math.h>

#if defined(__CUDACC__)
#define GL_FN __host__ __device__ __forceinline__
#define GL_TABLE static __device__ const
#else
#define GL_FN static inline
#define GL_TABLE static const
#endif

#if defined(__CUDA_ARCH__)
#define GL_MUL(a, b) __dmul_rn((a), (b))
#define GL_ADD(a, b) __dadd_rn((a), (b))
#define GL_SUB(a, b) __dsub_rn((a), (b))
#define GL_DIV(a, b) __ddiv_rn((a), (b))
#define GL_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define GL_MUL(a, b) ((a) * (b))
#define GL_ADD(a, b) ((a) + (b))
#define GL_SUB(a, b) ((a) - (b))
#define GL_DIV(a, b) ((a) / (b))
#define GL_FMA(a, b, c) fma((a), (b), (c))
#endif

namespace gl64 {

// glibc's tables, extracted from libm.so.6 at build time (_glibc_tables.py)
#include "gen/glibc_dbl64_tables.inc"

GL_FN uint64_t bits(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
#endif
}
GL_FN double from_bits(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double x;
  memcpy(&x, &u, 8);
  return x;
#endif
}
GL_FN uint32_t high_word(double x) { return (uint32_t)(bits(x) >> 32); }
GL_FN double copysign_of(double mag, double sgn) {
  return from_bits((bits(mag) & 0x7fffffffffffffffull) | (bits(sgn) & 0x8000000000000000ull));
}
GL_FN double neg(double x) { return from_bits(bits(x) ^ 0x8000000000000000ull); }

// s_sin.c / usncs.h constants (libm .rodata values)
#define GL_C(name, hex) constexpr double name = hex
GL_C(kSn3, -0x1.5555555555515p-3);
GL_C(kSn5, 0x1.11110e829872fp-7);
GL_C(kCs2, 0x1.0000000000000p-1);
GL_C(kCs4, -0x1.5555555555535p-5);
GL_C(kCs6, 0x1.6c16bedd9e239p-10);
GL_C(kS1, -0x1.5555555555555p-3);
GL_C(kS2, 0x1.1111111110ecep-7);
GL_C(kS3, -0x1.a01a019db08b8p-13);
GL_C(kS4, 0x1.71de27b9a7ed9p-19);
GL_C(kS5, -0x1.addffc2fcdf59p-26);
GL_C(kBig, 0x1.8p45);
GL_C(kHp0, 0x1.921fb54442d18p+0);
GL_C(kHp1, 0x1.1a62633145c07p-54);
GL_C(kMp1, 0x1.921fb58000000p+0);
GL_C(kMp2, -0x1.dde973c000000p-27);
GL_C(kPp3, -0x1.cb3b398000000p-55);
GL_C(kPp4, -0x1.d747f23e32ed7p-83);
GL_C(kHpinv, 0x1.45f306dc9c883p-1);
GL_C(kToint, 0x1.8p52);
// e_asin.c / uasncs.h constants
GL_C(kF1, 0x1.55555555554f9p-3);
GL_C(kF2, 0x1.333333336127dp-4);
GL_C(kF3, 0x1.6db6dae42c0e4p-5);
GL_C(kF4, 0x1.f1c7e04f4ad99p-6);
GL_C(kF5, 0x1.6e442c822d419p-6);
GL_C(kF6, 0x1.292d80f453c72p-6);
GL_C(kRt0, 0x1.fffffffecc1ddp-1);
GL_C(kRt1, 0x1.fffffff757304p-2);
GL_C(kRt2, 0x1.800496769c91ap-2);
GL_C(kRt3, 0x1.4006318d1dab9p-2);
GL_C(kT24, 0x1.0p24);
#undef GL_C

#if defined(__CUDA_ARCH__)
#define GL_LD(t, i) __ldg(&(t)[i])
#else
#define GL_LD(t, i) ((t)[i])
#endif

// TAYLOR_SIN(xx, a, da): t = (POLY(xx)*a - 0.5*da)*xx + da; a + t
GL_FN double taylor_sin(double a, double da) {
  const double xx = GL_MUL(a, a);
  double p = GL_FMA(xx, kS5, kS4);
  p = GL_FMA(xx, p, kS3);
  p = GL_FMA(xx, p, kS2);
  p = GL_FMA(xx, p, kS1);
  const double t1 = GL_FMA(p, a, neg(GL_MUL(da, 0.5)));
  const double t = GL_FMA(xx, t1, da);
  return GL_ADD(a, t);
}

// The table part of do_sin (|x| >= 0.126): sin(Xi + x) from __sincostab at
// Xi = the nearest 1/128 (u = big + |x|).
GL_FN double do_sin_table(double x, double dx) {
  const double ax = fabs(x);
  if (!(x > 0)) dx = neg(dx);
  const double u = GL_ADD(kBig, ax);
  const double xr = GL_SUB(ax, GL_SUB(u, kBig));
  const int k = (int)((uint32_t)bits(u) << 2);
  const double xx = GL_MUL(xr, xr);
  const double s = GL_ADD(xr, GL_FMA(GL_MUL(xr, xx), GL_FMA(xx, kSn5, kSn3), dx));
  const double c = GL_FMA(xr, dx, GL_MUL(xx, GL_FMA(xx, GL_FMA(xx, kCs6, kCs4), kCs2)));
  const double sn = GL_LD(kSinCosTab, k), ssn = GL_LD(kSinCosTab, k + 1);
  const double cs = GL_LD(kSinCosTab, k + 2), ccs = GL_LD(kSinCosTab, k + 3);
  double cor = GL_FMA(s, ccs, ssn);
  cor = GL_FMA(neg(c), sn, cor);
  cor = GL_FMA(s, cs, cor);
  return copysign_of(GL_ADD(sn, cor), x);
}

// do_sin(x, dx): Taylor below 0.126, else the table
GL_FN double do_sin(double x, double dx) {
  if (fabs(x) < 0.126) return taylor_sin(x, dx);
  return do_sin_table(x, dx);
}

// do_cos(x, dx): cos(Xi + x) from __sincostab
GL_FN double do_cos(double x, double dx) {
  if (x < 0) dx = neg(dx);
  const double ax = fabs(x);
  const double u = GL_ADD(kBig, ax);
  const double xr = GL_ADD(GL_SUB(ax, GL_SUB(u, kBig)), dx);
  const int k = (int)((uint32_t)bits(u) << 2);
  const double xx = GL_MUL(xr, xr);
  const double s = GL_FMA(GL_MUL(xr, xx), GL_FMA(xx, kSn5, kSn3), xr);
  const double c = GL_MUL(xx, GL_FMA(xx, GL_FMA(xx, kCs6, kCs4), kCs2));
  const double sn = GL_LD(kSinCosTab, k), ssn = GL_LD(kSinCosTab, k + 1);
  const double cs = GL_LD(kSinCosTab, k + 2), ccs = GL_LD(kSinCosTab, k + 3);
  double cor = GL_FMA(neg(s), ssn, ccs);
  cor = GL_FMA(neg(c), cs, cor);
  cor = GL_FMA(neg(s), sn, cor);
  return GL_ADD(cs, cor);
}

// reduce_sincos: x = n*pi/2 + (a + da), the low bits of t give n mod 4
GL_FN int reduce_sincos(double x, double* a, double* da) {
  const double t = GL_FMA(x, kHpinv, kToint);
  const double xn = GL_SUB(t, kToint);
  const double y = GL_FMA(neg(xn), kMp2, GL_FMA(neg(xn), kMp1, x));
  const int n = (int)(bits(t) & 3);
  const double t2 = GL_FMA(neg(xn), kPp3, y);
  double db = GL_FMA(neg(kPp3), xn, GL_SUB(y, t2));
  const double b = GL_FMA(neg(xn), kPp4, t2);
  db = GL_ADD(db, GL_FMA(neg(xn), kPp4, GL_SUB(t2, b)));
  *a = b;
  *da = db;
  return n;
}

GL_FN double sin(double x) {
  const uint32_t k = high_word(x) & 0x7fffffffu;
  if (k < 0x3e500000u) return x;                        // |x| < 2^-26
  if (k < 0x3feb6000u) return do_sin(x, 0.0);           // |x| < 0.855469
  if (k < 0x400368fdu)                                  // |x| < 2.426265
    return copysign_of(do_cos(GL_SUB(kHp0, fabs(x)), kHp1), x);
  if (k < 0x419921fbu) {                                // |x| < 105414350
    double a, da;
    const int n = reduce_sincos(x, &a, &da);
    const double r = (n & 1) ? do_cos(a, da) : do_sin(a, da);
    return (n & 2) ? neg(r) : r;
  }
  if (k >= 0x7ff00000u) return GL_SUB(x, x);           // inf / nan
  return NAN;                                           // outside the restated range
}

GL_FN double cos(double x) {
  const uint32_t k = high_word(x) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;                      // |x| < 2^-27
  if (k < 0x3feb6000u) return do_cos(x, 0.0);           // |x| < 0.855469
  if (k < 0x400368fdu) {                                // |x| < 2.426265
    const double y = GL_SUB(kHp0, fabs(x));
    const double a = GL_ADD(y, kHp1);
    const double da = GL_ADD(GL_SUB(y, a), kHp1);
    return do_sin(a, da);
  }
  if (k < 0x419921fbu) {
    double a, da;
    const int n = reduce_sincos(x, &a, &da) + 1;
    const double r = (n & 1) ? do_cos(a, da) : do_sin(a, da);
    return (n & 2) ? neg(r) : r;
  }
  if (k >= 0x7ff00000u) return GL_SUB(x, x);
  return NAN;
}

// One table-driven range of e_asin.c: xx = |x| - X[n]; a degree-d polynomial
// T[n+2..n+1+d] (Horner, fused), + T[n+2+d] through xx^2, the linear term
// T[n+1]*xx fused, + T[n+3+d].
GL_FN double asin_poly(double ax, int n, int d) {
  const double xx = GL_SUB(ax, GL_LD(kAsnCs, n));
  double p = GL_LD(kAsnCs, n + 1 + d);
  for (int i = n + d; i >= n + 2; --i) p = GL_FMA(xx, p, GL_LD(kAsnCs, i));
  p = GL_FMA(GL_MUL(xx, xx), p, GL_LD(kAsnCs, n + 2 + d));
  const double t = GL_FMA(xx, GL_LD(kAsnCs, n + 1), p);
  return GL_ADD(t, GL_LD(kAsnCs, n + 3 + d));
}

GL_FN double asin(double x) {
  const uint64_t u = bits(x);
  const uint32_t m = (uint32_t)(u >> 32);
  const uint32_t k = m & 0x7fffffffu;
  const bool pos = (int32_t)m > 0;
  if (k < 0x3e500000u) return x;                        // |x| < 2^-26
  if (k < 0x3fc00000u) {                                // |x| < 0.125: Taylor
    const double x2 = GL_MUL(x, x);
    double p = GL_FMA(x2, kF6, kF5);
    p = GL_FMA(x2, p, kF4);
    p = GL_FMA(x2, p, kF3);
    p = GL_FMA(x2, p, kF2);
    p = GL_FMA(x2, p, kF1);
    return GL_FMA(p, GL_MUL(x2, x), x);
  }
  const double ax = pos ? x : neg(x);
  double res;
  if (k < 0x3fe00000u) {                                // [0.125, 0.5)
    const int n = k < 0x3fd00000u ? 11 * (int)((k & 0x000fffffu) >> 15)
                                  : 11 * (int)((k & 0x000fffffu) >> 14) + 352;
    res = asin_poly(ax, n, 5);
  } else if (k < 0x3fe80000u) {                         // [0.5, 0.75)
    res = asin_poly(ax, 1056 + (int)((k & 0x000fe000u) >> 11) * 3, 6);
  } else if (k < 0x3fed8000u) {                         // [0.75, 0.921875)
    res = asin_poly(ax, 992 + (int)((k & 0x000fe000u) >> 13) * 13, 7);
  } else if (k < 0x3fee8000u) {                         // [0.921875, 0.953125)
    res = asin_poly(ax, 884 + (int)((k & 0x000fe000u) >> 13) * 14, 8);
  } else if (k < 0x3fef0000u) {                         // [0.953125, 0.96875)
    res = asin_poly(ax, 768 + (int)((k & 0x000fe000u) >> 13) * 15, 9);
  } else if (k < 0x3ff00000u) {                         // [0.96875, 1): pi/2 - 2 asin(sqrt(z))
    const double z = GL_MUL(pos ? GL_SUB(1.0, x) : GL_ADD(x, 1.0), 0.5);
    const uint32_t kz = high_word(z);
    double t = GL_MUL(GL_LD(kInRoot, (kz & 0x001fffffu) >> 14), GL_LD(kPowTwo, 511 - (int)(kz >> 21)));
    const double r = GL_FMA(neg(GL_MUL(t, t)), z, 1.0);
    t = GL_MUL(GL_FMA(r, GL_FMA(r, GL_FMA(r, kRt3, kRt2), kRt1), kRt0), t);
    const double c = GL_MUL(z, t);
    const double h = GL_FMA(neg(GL_MUL(t, 0.5)), c, 1.5);  // 1.5 - 0.5*t*c
    const double y = GL_SUB(GL_ADD(c, kT24), kT24);
    const double cc = GL_DIV(GL_FMA(neg(y), y, z), GL_FMA(h, c, y));
    double p = GL_FMA(z, kF6, kF5);
    p = GL_FMA(z, p, kF4);
    p = GL_FMA(z, p, kF3);
    p = GL_FMA(z, p, kF2);
    p = GL_FMA(z, p, kF1);
    p = GL_MUL(p, z);
    const double ycc = GL_ADD(y, cc);
    const double cor = GL_FMA(neg(GL_ADD(ycc, ycc)), p, GL_FMA(-2.0, cc, kHp1));
    const double res1 = GL_FMA(-2.0, y, kHp0);
    res = GL_ADD(cor, res1);
  } else if (k == 0x3ff00000u && (uint32_t)u == 0) {   // |x| == 1
    return pos ? kHp0 : neg(kHp0);
  } else {                                              // |x| > 1, nan
    return GL_DIV(GL_SUB(x, x), GL_SUB(x, x));
  }
  return pos ? res : neg(res);
}

}  // namespace gl64

#undef GL_LD
