// Emission sin/cos for the Fibonacci lattice (emission.cpp:25-26).
//
// The reference evaluates Vec3(rho*cos(phi), rho*sin(phi), z); g++ -O2 turns
// the pair into one glibc sincos() call (objdump of the reference's
// emission.o), which on this image's x86-64 hosts dispatches to the FMA build
// of glibc 2.39's dbl-64 s_sincos.c.  That routine is not correctly rounded
// (it disagrees with the exact value on ~0.3 % of lattice azimuths), so to
// reproduce the reference's rays bit for bit, sincos_glibc() below restates
// its algorithm operation by operation, with every multiply-add fused exactly
// where the FMA build fuses it (read off the disassembly of the installed
// libm's sincos ifunc target):
//   |x| < 2^-27               sin = x, cos = 1
//   |x| < 0.855469            table lookup at u = k/128 (rr_sincostab.h) plus
//                             short polynomials (sin: Taylor to x^11 when
//                             |x| < 0.126)
//   |x| < 2.426265            pi/2 - |x| in 106 bits, then the same kernels
//   |x| < 105414350           Cody-Waite reduction by pi/2 in four pieces
//                             (fused), quadrant swap, the same kernels.
// Above 105414350 (lattices beyond 4.39e7 rays) glibc switches to a
// Payne-Hanek reduction that is not restated here; sincos_glibc then falls
// back to the correctly rounded sincos_cr (<= 1 ulp from glibc).
// tests/native/sincos_check.cpp compares both with the installed libm on
// every lattice azimuth of every config and on random arguments per branch.
// Host (tests) and device share the code; it uses only correctly rounded
// +, -, * and fma.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define RR_HD __host__ __device__ __forceinline__
#else
#define RR_HD inline
#endif

#include "rr_sincostab.h"

namespace rr {

struct DD {
  double hi, lo;
};

RR_HD DD two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return DD{s, (a - (s - bb)) + (b - bb)};
}
RR_HD DD fast_two_sum(double a, double b) {
  const double s = a + b;
  return DD{s, b - (s - a)};
}
RR_HD DD dd_add(DD a, DD b) {
  DD s = two_sum(a.hi, b.hi);
  const DD t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = fast_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return fast_two_sum(s.hi, s.lo);
}
RR_HD DD dd_mul(DD a, DD b) {
  const double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e += a.hi * b.lo + a.lo * b.hi;
  return fast_two_sum(p, e);
}
// a / q for an integer-valued double q (exact residual via fma)
RR_HD DD dd_div_int(DD a, double q) {
  const double h = a.hi / q;
  const double r = fma(-h, q, a.hi);  // a.hi - h*q, exact
  const double l = (r + a.lo) / q;
  return fast_two_sum(h, l);
}

RR_HD void sincos_cr(double x, double* s_out, double* c_out) {
  // pi/2 = P1 + ... + P5 (28 significant bits each)
  const double P1 = 0x1.921fb54p+0, P2 = 0x1.10b4612p-30, P3 = -0x1.676733ap-60, P4 = -0x1.d1fc8f8p-89,
               P5 = -0x1.976b7eep-118;
  const double kd = nearbyint(x * 0.63661977236758138);
  DD r = DD{x - kd * P1, 0.0};  // exact (Sterbenz)
  r = dd_add(r, DD{-(kd * P2), 0.0});
  r = dd_add(r, DD{-(kd * P3), 0.0});
  r = dd_add(r, DD{-(kd * P4), 0.0});
  r = dd_add(r, DD{-(kd * P5), 0.0});
  const DD r2 = dd_mul(r, r);
  DD st = r, ct = DD{1.0, 0.0}, sterm = r, cterm = DD{1.0, 0.0};
  for (int n = 1; n <= 14; ++n) {
    const double a = 2.0 * n;
    sterm = dd_div_int(dd_mul(sterm, r2), a * (a + 1.0));
    cterm = dd_div_int(dd_mul(cterm, r2), (a - 1.0) * a);
    sterm = DD{-sterm.hi, -sterm.lo};
    cterm = DD{-cterm.hi, -cterm.lo};
    st = dd_add(st, sterm);
    ct = dd_add(ct, cterm);
  }
  const double s = st.hi + st.lo, c = ct.hi + ct.lo;
  switch (static_cast<long long>(kd) & 3) {
    case 0: *s_out = s; *c_out = c; break;
    case 1: *s_out = c; *c_out = -s; break;
    case 2: *s_out = -s; *c_out = -c; break;
    default: *s_out = -c; *c_out = s; break;
  }
}

// ---- glibc dbl-64 sincos, FMA build (see the header comment) ----
namespace gsc {
// one copy per side: lanes index it divergently, so global memory (L1), not __constant__
#ifdef __CUDACC__
__device__ static const double kTabDev[RR_SINCOSTAB_SIZE] = {RR_SINCOSTAB_WORDS};
#endif
static const double kTabHost[RR_SINCOSTAB_SIZE] = {RR_SINCOSTAB_WORDS};
RR_HD uint32_t hi_word(double x) {
#ifdef __CUDA_ARCH__
  return static_cast<uint32_t>(__double2hiint(x));
#else
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return static_cast<uint32_t>(b >> 32);
#endif
}
RR_HD uint32_t lo_word(double x) {
#ifdef __CUDA_ARCH__
  return static_cast<uint32_t>(__double2loint(x));
#else
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return static_cast<uint32_t>(b);
#endif
}
RR_HD double tab(int i) {
#ifdef __CUDA_ARCH__
  return kTabDev[i];
#else
  return kTabHost[i];
#endif
}
constexpr double kBig = 0x1.8p+45;  // u = big + |x| puts round(128|x|) in the low word
constexpr double kSn3 = -0x1.5555555555515p-3, kSn5 = 0x1.11110e829872fp-7;
constexpr double kCs2 = 0x1p-1, kCs4 = -0x1.5555555555535p-5, kCs6 = 0x1.6c16bedd9e239p-10;
constexpr double kS1 = -0x1.5555555555555p-3, kS2 = 0x1.1111111110ecep-7, kS3 = -0x1.a01a019db08b8p-13,
                 kS4 = 0x1.71de27b9a7ed9p-19, kS5 = -0x1.addffc2fcdf59p-26;
constexpr double kHp0 = 0x1.921fb54442d18p+0, kHp1 = 0x1.1a62633145c07p-54;  // pi/2 = hp0 + hp1
constexpr double kHpInv = 0x1.45f306dc9c883p-1, kToInt = 0x1.8p+52;
constexpr double kMp1 = 0x1.921fb58000000p+0, kMp2 = -0x1.dde973c000000p-27;
constexpr double kPp3 = -0x1.cb3b398000000p-55, kPp4 = -0x1.d747f23e32ed7p-83;
constexpr double kTaylorMax = 0x1.020c49ba5e354p-3;  // 0.126

struct Tab {
  double xs, sn, ssn, cs, ccs;  // xs = |a| - u: the offset from the table node
};
RR_HD Tab lookup(double aabs) {
  const double u = aabs + kBig;
  const int k = static_cast<int>(lo_word(u) << 2);
  return Tab{aabs - (u - kBig), tab(k), tab(k + 1), tab(k + 2), tab(k + 3)};
}
// sin polynomial of TAYLOR_SIN: ((((s5 xx + s4) xx + s3) xx + s2) xx + s1)
RR_HD double taylor_poly(double xx) {
  double p = fma(xx, kS5, kS4);
  p = fma(xx, p, kS3);
  p = fma(xx, p, kS2);
  return fma(xx, p, kS1);
}
// TAYLOR_SIN(a*a, a, da) = a + ((P a - da/2) a^2 + da)
RR_HD double taylor_sin(double a, double da) {
  const double xx = a * a;
  const double h = da * 0.5;
  return a + fma(xx, fma(taylor_poly(xx), a, -h), da);
}
// do_sin's table branch: |a| >= 0.126; dx already sign-adjusted (a <= 0 -> -da)
RR_HD double sin_tab(const Tab& t, double dx, double a) {
  const double xx = t.xs * t.xs;
  const double s = t.xs + fma(t.xs * xx, fma(xx, kSn5, kSn3), dx);
  const double c = fma(dx, t.xs, xx * fma(fma(xx, kCs6, kCs4), xx, kCs2));
  const double cor = fma(s, t.cs, fma(-c, t.sn, fma(s, t.ccs, t.ssn)));
  return copysign(cor + t.sn, a);
}
// do_cos: dx already sign-adjusted (a < 0 -> -da)
RR_HD double cos_tab(const Tab& t, double dx) {
  const double xc = t.xs + dx;
  const double xx = xc * xc;
  const double s = fma(xc * xx, fma(xx, kSn5, kSn3), xc);
  const double c = xx * fma(fma(xx, kCs6, kCs4), xx, kCs2);
  const double cor = fma(-s, t.sn, fma(-c, t.cs, fma(-t.ssn, s, t.ccs)));
  return cor + t.cs;
}
}  // namespace gsc

// Returns false (outputs untouched) for |x| >= 105414350 or non-finite x.
RR_HD bool sincos_glibc(double x, double* s_out, double* c_out) {
  using namespace gsc;
  const uint32_t k = hi_word(x) & 0x7fffffffu;
  if (k < 0x3e400000u) {  // |x| < 2^-27
    *s_out = x;
    *c_out = 1.0;
    return true;
  }
  if (k < 0x3feb6000u) {  // |x| < 0.855469
    const double ax = fabs(x);
    const Tab t = lookup(ax);
    *s_out = ax < kTaylorMax ? taylor_sin(x, 0.0) : sin_tab(t, x > 0.0 ? 0.0 : -0.0, x);
    *c_out = cos_tab(t, x >= 0.0 ? 0.0 : -0.0);
    return true;
  }
  if (k < 0x400368fdu) {  // |x| < 2.426265: a + da = pi/2 - |x|
    const double y = kHp0 - fabs(x);
    const double a = y + kHp1;
    const double da = (y - a) + kHp1;
    const Tab t = lookup(fabs(a));
    *s_out = copysign(cos_tab(t, a < 0.0 ? -da : da), x);
    *c_out = fabs(a) < kTaylorMax ? taylor_sin(a, da) : sin_tab(t, a <= 0.0 ? -da : da, a);
    return true;
  }
  if (k < 0x419921fbu) {  // |x| < 105414350: reduce_sincos
    const double tt = fma(x, kHpInv, kToInt);
    const double xn = tt - kToInt;
    const int n = static_cast<int>(lo_word(tt) & 3u);
    const double y = fma(-xn, kMp2, fma(-xn, kMp1, x));
    const double t2 = fma(-xn, kPp3, y);
    double db = fma(-xn, kPp3, y - t2);
    double a = fma(-xn, kPp4, t2);
    db = db + fma(-xn, kPp4, t2 - a);
    if (n == 1 || n == 2) {
      a = -a;
      db = -db;
    }
    const Tab t = lookup(fabs(a));
    const double ds = fabs(a) < kTaylorMax ? taylor_sin(a, db) : sin_tab(t, a <= 0.0 ? -db : db, a);
    double dc = cos_tab(t, a < 0.0 ? -db : db);
    if (n & 2) dc = -dc;
    if (n & 1) {
      *s_out = dc;
      *c_out = ds;
    } else {
      *s_out = ds;
      *c_out = dc;
    }
    return true;
  }
  return false;
}

// The emission's sin/cos: glibc's where it is restated, else correctly rounded.
RR_HD void sincos_emit(double x, double* s_out, double* c_out) {
  if (!sincos_glibc(x, s_out, c_out)) sincos_cr(x, s_out, c_out);
}

}  // namespace rr
