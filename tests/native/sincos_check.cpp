// Compares rr::sincos_cr (paper_1811_05784_b200/csrc/rr_sincos.cuh, the
// device emission's sin/cos) with glibc sin/cos on the Fibonacci azimuths
// phi_k = azimuth_step * k (emission.cpp:19-26) for k < n.  Prints the
// number of mismatching k.  Test infrastructure.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "rr_sincos.cuh"

int main(int argc, char** argv) {
  const long long n = argc > 1 ? std::atoll(argv[1]) : 8000000;
  const double golden = (1.0 + std::sqrt(5.0)) / 2.0;
  const double step = 2.0 * M_PI * (1.0 - 1.0 / golden);
  long long bad = 0;
  for (long long k = 0; k < n; ++k) {
    const double phi = step * static_cast<double>(k);
    double s, c;
    rr::sincos_cr(phi, &s, &c);
    if (s != std::sin(phi) || c != std::cos(phi)) {
      if (bad < 5) std::printf("k=%lld phi=%.17g s=%.17g/%.17g c=%.17g/%.17g\n", k, phi, s, std::sin(phi), c, std::cos(phi));
      ++bad;
    }
  }
  std::printf("mismatches %lld of %lld\n", bad, n);
  return bad != 0;
}
