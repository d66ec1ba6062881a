// Correctly rounded sin/cos for the Fibonacci lattice (emission.cpp:25-26).
//
// phi = azimuth_step * k reaches ~2e7 rad at k = 8e6; CUDA's double sincos
// (<= 2 ulp) then disagrees with glibc's for a fraction of the rays, which
// would change trajectories.  This evaluates sin/cos in double-double:
// Cody-Waite reduction by pi/2 split into five 28-bit pieces (every k*P_i is
// exact for |k| < 2^25), Taylor series to r^29 in double-double, then one
// rounding.  The value before rounding is accurate to ~2^-100 relative, so
// the result is the correctly rounded sin/cos except for inputs within ~2^-47
// ulp of a rounding boundary; tests/test_emission_sincos.py checks it
// against glibc over every lattice used.  Host (tests) and device share it;
// it uses only +, -, *, / and fma, all correctly rounded on both.
#pragma once

#include <cmath>

#ifdef __CUDACC__
#define RR_HD __host__ __device__ __forceinline__
#else
#define RR_HD inline
#endif

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

}  // namespace rr
