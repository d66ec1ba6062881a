// Driver for tests/test_gpu_facade.py::test_pipeline_matches_oracle: runs
// roomray_b200::run_trace_pipeline on a run-config file (the reference's
// pipeline.cpp:144-185 shape) and dumps images, the broadband RIR and the
// factors as raw arrays.   pipeline_run <run.json> <out_dir> [oracle.json]
// With an oracle config (pipeline.hpp:47-61) it also runs run_oracle and
// compare(oracle, images, 1e-9, 1.5) — acceptance criterion 4
// (acceptance_main.cpp:239-272) — and prints the report.
#include <algorithm>
#include <cmath>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "roomray_b200_io.hpp"

namespace rb = roomray_b200;

template <typename T>
static void write_all(const std::string& path, const std::vector<T>& v) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

int main(int argc, char** argv) {
  if (argc != 3 && argc != 4) return 2;
  const std::string out = argv[2];
  try {
    const rb::RunConfig cfg = rb::RunConfig::from_json_file(argv[1]);
    const rb::RunArtifacts a = rb::run_trace_pipeline(cfg);
    std::vector<double> img;
    for (const rb::ImageSource& s : a.images) {
      img.insert(img.end(), {s.position.x, s.position.y, s.position.z, s.distance});
      img.insert(img.end(), s.band_energy.begin(), s.band_energy.end());
      img.push_back(s.ray_count);
      img.push_back(s.order);
    }
    write_all(out + "/images.f64", img);
    write_all(out + "/rir.f64", a.rir.samples);
    std::vector<double> fac;
    auto put = [&](const rb::PerceptiveFactors& f) {
      for (const rb::MetricValue* m : {&f.edt_s, &f.t30_s, &f.spl_db, &f.c80_db, &f.d50_pct, &f.ts_ms}) {
        fac.push_back(m->value);
        fac.push_back(m->reliable ? 1.0 : 0.0);
      }
    };
    for (const auto& f : a.metrics.bands) put(f);
    put(a.metrics.mid);
    write_all(out + "/factors.f64", fac);
    std::cout << "pipeline ok: " << a.mesh.faces.size() << " faces, " << a.trace.captures.size() << " captures, "
              << a.images.size() << " images, stages";
    for (const auto& t : a.timings) std::cout << " " << t.name << "=" << t.seconds;
    std::cout << "\n";
    if (argc == 4) {
      const rb::OracleConfig oc = rb::OracleConfig::from_json_file(argv[3]);
      const auto lattice = rb::run_oracle(oc);
      const rb::MatchReport rep = rb::compare(lattice, a.images, 1e-9, 1.5);
      double worst = 0.0;
      for (const rb::MatchedImage& m : rep.matched)
        if (m.order <= 2)
          for (double d : m.energy_delta_db) worst = std::max(worst, std::abs(d));
      std::cout << "acceptance4 oracle=" << lattice.size() << " matched=" << rep.matched.size()
                << " oracle_only=" << rep.unmatched_oracle.size() << " traced_only=" << rep.unmatched_traced.size()
                << " max_pos_err=" << rep.max_position_error << " worst_db=" << worst
                << " within=" << (rep.energy_within(1.5, 2) ? 1 : 0) << "\n";
    }
  } catch (const std::invalid_argument& e) {
    std::cout << "invalid_argument: " << e.what() << "\n";
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "pipeline_run: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
