// Where the C++ facade's run_trace_pipeline time goes: the stages of
// run_trace_pipeline_on (include/roomray_b200_io.hpp) split into device work,
// device->host copies and host-side materialisation of the reference's
// structs.  Same scene.bin as tests/native/pipeline_bench.cpp.
//
//   native_breakdown <scene.bin> <steps> <warmup>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <map>
#include <string>
#include <vector>

#include "roomray_b200_io.hpp"

namespace rb = roomray_b200;
using clk = std::chrono::steady_clock;

template <typename T>
static T get(std::ifstream& f) {
  T v{};
  f.read(reinterpret_cast<char*>(&v), sizeof v);
  return v;
}

int main(int argc, char** argv) {
  if (argc != 4) return 2;
  std::ifstream f(argv[1], std::ios::binary);
  if (!f) return 3;
  const int steps = std::atoi(argv[2]), warmup = std::atoi(argv[3]);
  const int64_t nv = get<int64_t>(f), nf = get<int64_t>(f), nmat = get<int64_t>(f);
  rb::TriangleMesh mesh;
  mesh.vertices.resize(nv);
  for (auto& v : mesh.vertices) v = {get<double>(f), get<double>(f), get<double>(f)};
  mesh.faces.resize(nf);
  for (auto& t : mesh.faces) {
    t.a = get<int32_t>(f);
    t.b = get<int32_t>(f);
    t.c = get<int32_t>(f);
    t.material_id = get<int32_t>(f);
  }
  mesh.materials.resize(nmat);
  for (int64_t m = 0; m < nmat; ++m) {
    mesh.materials[m].name = "m" + std::to_string(m);
    for (int b = 0; b < rb::kNumBands; ++b) mesh.materials[m].absorption[b] = get<double>(f);
  }
  rb::RunConfig cfg;
  cfg.source.position = {get<double>(f), get<double>(f), get<double>(f)};
  cfg.source.ray_count = static_cast<int>(get<int64_t>(f));
  cfg.receiver.center = {get<double>(f), get<double>(f), get<double>(f)};
  cfg.receiver.radius = get<double>(f);
  cfg.max_range = get<double>(f);
  cfg.sample_rate = get<double>(f);
  cfg.max_iterations = static_cast<int>(get<int64_t>(f));
  cfg.merge_coplanar = get<int64_t>(f) != 0;
  if (!f) return 4;

  std::map<std::string, double> acc;
  for (int it = 0; it < warmup + steps; ++it) {
    std::map<std::string, double> st;
    auto last = clk::now();
    auto mark = [&](const char* name) {
      const auto now = clk::now();
      st[name] += std::chrono::duration<double>(now - last).count();
      last = now;
    };
    rb::RunArtifacts a;
    a.mesh = mesh;
    last = clk::now();
    a.tree = rb::build_tree(a.mesh);
    mark("1 tree_build");
    rb::TraceConfig tc;
    tc.max_iterations = cfg.max_iterations;
    tc.speed_of_sound = cfg.speed_of_sound;
    tc.max_range = cfg.max_range;
    rb::detail::TraceHandle th(rb::detail::trace_device(a.tree, cfg.source, cfg.receiver, tc));
    mark("2a trace_device");
    a.trace = rb::detail::trace_result_from(th.h);
    mark("2b trace_to_host");
    rr_air air{cfg.air.enabled ? 1 : 0, cfg.air.temperature_c, cfg.air.relative_humidity, cfg.air.pressure_kpa};
    rr_cluster_options co{rb::ClusterOptions{}.tol_scale, cfg.merge_coplanar ? 1 : 0};
    rr_images* im = nullptr;
    rb::detail::check(rr_build_image_sources(th.h, 0, cfg.source.ray_count, &air, &co, &im));
    mark("3a images_device");
    a.images = rb::detail::images_from(im);
    mark("3b images_to_host");
    a.trains = rb::detail::trains_from(im, cfg.speed_of_sound);
    mark("4a trains_to_host");
    a.rir = rb::detail::rir_from(im, a.trains, cfg.speed_of_sound, cfg.sample_rate);
    mark("4b rir");
    a.metrics = rb::detail::factors_from(im, cfg.speed_of_sound);
    mark("5 metrics");
    rr_images_destroy(im);
    // the same stages through the reference's stage-by-stage API (host
    // vectors between the calls, pipeline.cpp:163-178's sequence)
    last = clk::now();
    const rb::TraceResult tr = rb::trace(a.mesh, a.tree, cfg.source, cfg.receiver, tc);
    mark("s1 trace()");
    const auto imgs = rb::build_image_sources(tr.captures, cfg.source.ray_count, cfg.air, cfg.receiver.center, a.mesh,
                                              a.tree, rb::ClusterOptions{1e-6, cfg.merge_coplanar});
    mark("s2 build_image_sources()");
    const rb::PulseTrains trains = rb::build_pulse_trains(imgs, cfg.speed_of_sound);
    mark("s3 build_pulse_trains()");
    const rb::RoomImpulseResponse rir = rb::synthesize(trains, cfg.sample_rate);
    mark("s4 synthesize()");
    const rb::BandFactors bf = rb::factors(trains);
    mark("s5 factors()");
    if (imgs.size() != a.images.size() || rir.samples != a.rir.samples) {
      std::size_t bad_img = imgs.size(), bad_s = rir.samples.size();
      for (std::size_t i = 0; i < std::min(imgs.size(), a.images.size()); ++i)
        if (imgs[i].distance != a.images[i].distance || imgs[i].face_path != a.images[i].face_path ||
            imgs[i].band_energy != a.images[i].band_energy) {
          bad_img = i;
          break;
        }
      double md = 0.0, peak = 0.0;
      for (std::size_t i = 0; i < std::min(rir.samples.size(), a.rir.samples.size()); ++i) {
        md = std::max(md, std::fabs(rir.samples[i] - a.rir.samples[i]));
        peak = std::max(peak, std::fabs(a.rir.samples[i]));
        if (bad_s == rir.samples.size() && rir.samples[i] != a.rir.samples[i]) bad_s = i;
      }
      std::printf("stage-by-stage vs pipeline: images %zu / %zu, first differing image %zu; samples %zu / %zu, "
                  "first differing %zu, max |diff| %.3g of peak %.3g\n",
                  imgs.size(), a.images.size(), bad_img, rir.samples.size(), a.rir.samples.size(), bad_s, md, peak);
    }
    (void)bf;
    if (it >= warmup)
      for (auto& kv : st) acc[kv.first] += kv.second;
    const auto t0 = clk::now();
    { rb::RunArtifacts gone = std::move(a); }
    if (it >= warmup) acc["9 destroy (untimed in bench)"] += std::chrono::duration<double>(clk::now() - t0).count();
  }
  std::printf("{");
  bool first = true;
  for (const auto& kv : acc) {
    std::printf("%s\"%s\": %.2f", first ? "" : ", ", kv.first.c_str(), 1e3 * kv.second / steps);
    first = false;
  }
  std::printf("}\n");
  return 0;
}
