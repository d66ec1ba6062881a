// Test infrastructure.  Compares the device emission's sin/cos
// (paper_1811_05784_b200/csrc/rr_sincos.cuh, compiled for the host) with the
// installed glibc sincos() -- the call the reference's fibonacci_directions
// makes (emission.cpp:25-26, fused by g++ -O2) -- bit for bit:
//   lattice <n> [<n> ...]  every azimuth phi_k = azimuth_step * k, k < n
//   random <count> <seed>  random arguments in each branch of the routine
// Prints "mismatches <bad> of <total> fallback <f> (of which <g> differ)":
// bad counts arguments inside the restated range (|x| < 105414350); fallback
// arguments go through the correctly rounded sincos_cr instead.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>

#include "rr_sincos.cuh"

static long long g_bad = 0, g_total = 0, g_fallback = 0, g_fallback_bad = 0;

static void check(double x) {
  double s, c, gs, gc;
  const bool restated = rr::sincos_glibc(x, &s, &c);
  if (!restated) rr::sincos_cr(x, &s, &c);
  sincos(x, &gs, &gc);
  const bool same = std::memcmp(&s, &gs, 8) == 0 && std::memcmp(&c, &gc, 8) == 0;
  if (!restated) {
    ++g_fallback;
    g_fallback_bad += !same;
    return;
  }
  ++g_total;
  if (!same) {
    if (g_bad < 8) std::printf("x=%a s=%a/%a c=%a/%a\n", x, s, gs, c, gc);
    ++g_bad;
  }
}

static uint64_t splitmix(uint64_t& st) {
  uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  if (std::strcmp(argv[1], "lattice") == 0) {
    // emission.cpp:19-20
    const double golden = (1.0 + std::sqrt(5.0)) / 2.0;
    const double step = 2.0 * M_PI * (1.0 - 1.0 / golden);
    for (int a = 2; a < argc; ++a) {
      const long long n = std::atoll(argv[a]);
      for (long long k = 0; k < n; ++k) check(step * static_cast<double>(k));
    }
  } else {
    const long long count = std::atoll(argv[2]);
    uint64_t st = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 1;
    // branch edges of the routine: 2^-27, 0.126, 0.855469, 2.426265, 105414350
    const double lo[] = {0x1p-30, 0x1p-27, 0.1, 0.126, 0.8, 2.3, 2.4, 100.0, 1e5, 1e7, 1.05e8};
    const double hi[] = {0x1p-27, 0.13, 0.2, 0.86, 2.5, 2.5, 10.0, 1e5, 1e7, 1.0541435e8, 1.0542e8};
    const int nr = sizeof(lo) / sizeof(lo[0]);
    for (long long i = 0; i < count; ++i) {
      const int r = static_cast<int>(i % nr);
      const double u = static_cast<double>(splitmix(st) >> 11) * 0x1p-53;
      double x = lo[r] + (hi[r] - lo[r]) * u;
      if (splitmix(st) & 1) x = -x;
      check(x);
    }
    for (double x : {0.0, -0.0, 0x1p-27, 0.126, 0.855469, 2.426265, 1.5707963267948966, 3.141592653589793})
      check(x);
  }
  std::printf("mismatches %lld of %lld fallback %lld (of which %lld differ)\n", g_bad, g_total, g_fallback,
              g_fallback_bad);
  return g_bad != 0;
}
