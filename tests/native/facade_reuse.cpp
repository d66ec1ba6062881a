// Driver for tests/test_gpu_facade.py::test_facade_staging_reuse: the C++
// façade converts every device result through one grow-only page-locked
// staging buffer per host thread (roomray_b200.hpp detail::Staging).  Runs
// run_trace_pipeline_on on a large room, a small room, then the large room
// again, and checks that the repeated run gives identical artifacts (captures,
// image sources, pulse trains, IR, factors) -- i.e. a grown buffer, a call that
// uses only part of it, and the scene upload that shares it leave no stale
// data behind.  Prints "ok <captures> <images>" or the first mismatch.
#include <cstdio>
#include <cstring>
#include <string>

#include "roomray_b200_io.hpp"

namespace rb = roomray_b200;

// a shoebox whose walls are n x n grids of quads (two triangles each)
static rb::TriangleMesh gridded_box(double lx, double ly, double lz, int n) {
  rb::TriangleMesh m;
  rb::Material mat;
  mat.name = "wall";
  for (int b = 0; b < rb::kNumBands; ++b) mat.absorption[b] = 0.05 + 0.02 * b;
  m.materials.push_back(mat);
  const double L[3] = {lx, ly, lz};
  for (int axis = 0; axis < 3; ++axis)
    for (int side = 0; side < 2; ++side) {
      const int u = (axis + 1) % 3, v = (axis + 2) % 3;
      const int base = static_cast<int>(m.vertices.size());
      for (int i = 0; i <= n; ++i)
        for (int j = 0; j <= n; ++j) {
          rb::Vec3 p;
          p[axis] = side ? L[axis] : 0.0;
          p[u] = L[u] * i / n;
          p[v] = L[v] * j / n;
          m.vertices.push_back(p);
        }
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          const int a = base + i * (n + 1) + j, b = a + 1, c = a + (n + 1), d = c + 1;
          m.faces.push_back({a, c, b, 0});
          m.faces.push_back({b, c, d, 0});
        }
    }
  return m;
}

static rb::RunConfig config(double lx, double ly, double lz, int rays) {
  rb::RunConfig c;
  c.source.position = {0.3 * lx, 0.4 * ly, 0.5 * lz};
  c.source.ray_count = rays;
  c.receiver.center = {0.7 * lx, 0.6 * ly, 0.4 * lz};
  c.receiver.radius = 0.5;
  c.max_range = 200.0;
  c.sample_rate = 48000.0;
  c.max_iterations = 30;
  c.merge_coplanar = true;
  return c;
}

static rb::RunArtifacts run(const rb::TriangleMesh& mesh, const rb::RunConfig& cfg) {
  rb::RunArtifacts a;
  a.mesh = mesh;
  rb::run_trace_pipeline_on(a, cfg);
  return a;
}

#define REQUIRE(cond, what)                        \
  do {                                             \
    if (!(cond)) {                                 \
      std::printf("mismatch: %s\n", what);         \
      return 1;                                    \
    }                                              \
  } while (0)

static bool same(const rb::Vec3& a, const rb::Vec3& b) { return std::memcmp(&a, &b, sizeof a) == 0; }
template <typename T>
static bool same_bytes(const T& a, const T& b) {
  return std::memcmp(&a, &b, sizeof a) == 0;
}

int main() {
  const rb::TriangleMesh big = gridded_box(12.0, 9.0, 5.0, 60);  // 43 200 triangles
  const rb::TriangleMesh small = gridded_box(4.0, 3.0, 2.5, 3);  // 108 triangles
  const rb::RunConfig cb = config(12.0, 9.0, 5.0, 60000), cs = config(4.0, 3.0, 2.5, 2000);
  const rb::RunArtifacts a1 = run(big, cb);
  const rb::RunArtifacts s1 = run(small, cs);
  const rb::RunArtifacts a2 = run(big, cb);
  REQUIRE(!a1.trace.captures.empty() && !a1.images.empty() && !s1.images.empty(), "empty artifacts");
  REQUIRE(a1.trace.captures.size() == a2.trace.captures.size(), "capture count");
  for (std::size_t i = 0; i < a1.trace.captures.size(); ++i) {
    const rb::Capture &x = a1.trace.captures[i], &y = a2.trace.captures[i];
    REQUIRE(x.ray_index == y.ray_index && same(x.point, y.point) && same(x.incoming_dir, y.incoming_dir) &&
                same_bytes(x.path_length, y.path_length) && same_bytes(x.band_multiplier, y.band_multiplier) &&
                x.face_history == y.face_history,
            "capture");
  }
  REQUIRE(a1.images.size() == a2.images.size(), "image count");
  for (std::size_t i = 0; i < a1.images.size(); ++i) {
    const rb::ImageSource &x = a1.images[i], &y = a2.images[i];
    REQUIRE(same(x.position, y.position) && same_bytes(x.distance, y.distance) &&
                same_bytes(x.band_energy, y.band_energy) && same_bytes(x.band_multiplier, y.band_multiplier) &&
                x.ray_count == y.ray_count && x.order == y.order && x.face_path == y.face_path &&
                x.projection.has_value() == y.projection.has_value() &&
                (!x.projection || same(*x.projection, *y.projection)),
            "image source");
  }
  for (int b = 0; b < rb::kNumBands; ++b) {
    REQUIRE(a1.trains[b].band == b && a2.trains[b].band == b, "train band");
    REQUIRE(a1.trains[b].events.size() == a1.images.size(), "train length");
    REQUIRE(a1.trains[b].events.size() == a2.trains[b].events.size(), "train size");
    REQUIRE(std::memcmp(a1.trains[b].events.data(), a2.trains[b].events.data(),
                        a1.trains[b].events.size() * sizeof(rb::PulseEvent)) == 0,
            "train events");
    REQUIRE(a1.rir.band_trains[b].events.size() == a1.trains[b].events.size() &&
                std::memcmp(a1.rir.band_trains[b].events.data(), a1.trains[b].events.data(),
                            a1.trains[b].events.size() * sizeof(rb::PulseEvent)) == 0,
            "rir band trains");
    REQUIRE(a1.rir.band_samples[b] == a2.rir.band_samples[b], "band samples");
  }
  REQUIRE(!a1.rir.samples.empty() && a1.rir.samples == a2.rir.samples, "rir samples");
  REQUIRE(same_bytes(a1.metrics.mid.edt_s.value, a2.metrics.mid.edt_s.value) &&
              same_bytes(a1.metrics.mid.t30_s.value, a2.metrics.mid.t30_s.value),
          "factors");
  std::printf("ok %zu %zu %zu\n", a1.trace.captures.size(), a1.images.size(), s1.images.size());
  return 0;
}
