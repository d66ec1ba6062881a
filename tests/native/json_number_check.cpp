// Our JSON number text (include/roomray_b200_artifacts.hpp, Grisu2 restated)
// against nlohmann::json's on random doubles: every bit pattern class
// (uniform bits, decades 1e-320..1e308, integers, subnormals, powers of ten,
// neighbours of round numbers).  Prints the count of mismatches.
#include <json.hpp>

#include <cstdint>
#include <cstring>
#include <iostream>
#include <random>

#include "roomray_b200_artifacts.hpp"

int main(int argc, char** argv) {
  const long n = argc > 1 ? std::atol(argv[1]) : 1000000;
  std::mt19937_64 rng(20240611);
  long bad = 0, tested = 0;
  auto check = [&](double v) {
    if (!std::isfinite(v)) return;
    ++tested;
    const std::string ours = roomray_b200::detail::JOut::number(v).dump();
    const std::string theirs = nlohmann::json(v).dump();
    if (ours != theirs) {
      if (++bad <= 10) std::cout << "mismatch " << theirs << " vs " << ours << "\n";
    }
  };
  std::uniform_real_distribution<double> u(-320.0, 308.0), m(1.0, 10.0);
  for (long i = 0; i < n; ++i) {
    const uint64_t bits = rng();
    double v;
    std::memcpy(&v, &bits, 8);
    check(v);
    check(m(rng) * std::pow(10.0, std::floor(u(rng))));
    check(static_cast<double>(static_cast<int64_t>(rng() >> (rng() % 64))));
    const uint64_t sub = rng() & ((uint64_t{1} << 52) - 1);
    std::memcpy(&v, &sub, 8);
    check(v);
  }
  for (int e = -323; e <= 308; ++e) {
    const double p = std::pow(10.0, e);
    check(p);
    check(std::nextafter(p, 0.0));
    check(std::nextafter(p, HUGE_VAL));
  }
  std::cout << "tested " << tested << " mismatches " << bad << "\n";
  return bad == 0 ? 0 : 1;
}
