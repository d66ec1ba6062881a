// Native end-to-end timing of the C++ facade's run_trace_pipeline stages
// (pipeline.cpp:154-183 after loading: tree build, trace, image sources,
// pulse trains + impulse response, perceptive factors), the call a C++
// caller of the reference makes, on a scene given as raw arrays.
//
//   pipeline_bench <scene.bin> <steps> <warmup>
//
// scene.bin (written by bench.py): int64 nv, nf, nmat; f64 vertices[nv*3];
// i32 faces[nf*4]; f64 alpha[nmat*8]; f64 source[3]; int64 ray_count;
// f64 receiver[3], radius, max_range, sample_rate; int64 max_iterations,
// merge_coplanar.  The mesh arrays start in host memory every step (scene
// upload inside the timed region), every output ends in host memory.
// Prints one JSON line: mean seconds per stage and per step, ray*bounces.
#include <chrono>
#include <cstdio>
#include <fstream>
#include <map>
#include <string>
#include <vector>

#include "roomray_b200_io.hpp"

namespace rb = roomray_b200;

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
  std::map<std::string, double> stage;
  double total = 0.0;
  int64_t rb_per_step = 0;
  std::size_t images = 0, captures = 0;
  for (int it = 0; it < warmup + steps; ++it) {
    const auto t0 = std::chrono::steady_clock::now();
    rb::RunArtifacts a;
    a.mesh = mesh;  // host arrays every step (not timed separately: a copy of the loaded mesh)
    const auto t1 = std::chrono::steady_clock::now();
    rb::run_trace_pipeline_on(a, cfg);
    const auto t2 = std::chrono::steady_clock::now();
    if (it >= warmup) {
      total += std::chrono::duration<double>(t2 - t1).count();
      for (const auto& s : a.timings) stage[s.name] += s.seconds;
      rb_per_step = a.trace.ray_bounces;
      images = a.images.size();
      captures = a.trace.captures.size();
    }
    (void)t0;
  }
  std::printf("{\"steps\": %d, \"seconds_per_step\": %.6f, \"ray_bounces_per_step\": %lld, \"images\": %zu, "
              "\"captures\": %zu, \"stage_s\": {",
              steps, total / steps, static_cast<long long>(rb_per_step), images, captures);
  bool first = true;
  for (const auto& kv : stage) {
    std::printf("%s\"%s\": %.6f", first ? "" : ", ", kv.first.c_str(), kv.second / steps);
    first = false;
  }
  std::printf("}}\n");
  return 0;
}
