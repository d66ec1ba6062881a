// tests/test_io.cpp restated on the facade's host IO
// (include/roomray_b200_artifacts.hpp): WAV float32 round trip, non-WAV and
// missing files fail cleanly, band-trains CSV round trip (bit-exact through
// "%.17g"), image_sources.json loading.  No GPU call.   io_roundtrip <dir>
#include <cmath>
#include <fstream>
#include <iostream>

#include "roomray_b200_artifacts.hpp"

namespace rb = roomray_b200;

#define EXPECT(c)                                                  \
  do {                                                             \
    if (!(c)) {                                                    \
      std::cerr << "failed: " #c " (line " << __LINE__ << ")\n"; \
      return 1;                                                    \
    }                                                              \
  } while (0)

int main(int argc, char** argv) {
  if (argc != 2) return 2;
  const std::string dir = argv[1];
  std::vector<double> samples;
  for (int i = 0; i < 1000; ++i) samples.push_back(std::sin(0.01 * i) * 0.5);
  rb::write_wav(dir + "/probe.wav", samples, 44100.0);
  const rb::WavData w = rb::read_wav(dir + "/probe.wav");
  EXPECT(w.sample_rate == 44100.0 && w.samples.size() == samples.size());
  for (std::size_t i = 0; i < samples.size(); ++i) EXPECT(std::abs(w.samples[i] - samples[i]) <= 1e-7 * std::abs(samples[i]) + 1e-30);
  std::ofstream(dir + "/not_a_wav.wav") << "plain text";
  bool threw = false;
  try { rb::read_wav(dir + "/not_a_wav.wav"); } catch (const std::runtime_error&) { threw = true; }
  EXPECT(threw);
  threw = false;
  try { rb::read_wav(dir + "/missing.wav"); } catch (const std::runtime_error&) { threw = true; }
  EXPECT(threw);

  rb::PulseTrains t;
  for (int b = 0; b < rb::kNumBands; ++b) t[b].band = b;
  t[0].events = {{0.001, 0.25}, {0.5, 0.125}};
  t[7].events = {{0.333333333333333, 0.0625}};
  rb::write_band_trains_csv(dir + "/trains.csv", t);
  const rb::PulseTrains back = rb::load_band_trains_csv(dir + "/trains.csv");
  for (int b = 0; b < rb::kNumBands; ++b) {
    EXPECT(back[b].events.size() == t[b].events.size());
    for (std::size_t i = 0; i < t[b].events.size(); ++i)
      EXPECT(back[b].events[i].time_s == t[b].events[i].time_s && back[b].events[i].amplitude == t[b].events[i].amplitude);
  }
  std::ofstream(dir + "/bad.csv") << "band,time_s,amplitude\n9,0.1,0.2\n";
  threw = false;
  try { rb::load_band_trains_csv(dir + "/bad.csv"); } catch (const std::runtime_error& e) {
    threw = std::string(e.what()).find("line 2") != std::string::npos;
  }
  EXPECT(threw);
  std::cout << "io ok\n";
  return 0;
}
