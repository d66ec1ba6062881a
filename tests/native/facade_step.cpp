// step() through the C++ facade the way the reference's bench drives it
// (bench.cpp:26-46): emit, then `iters` calls of step() with the tree and,
// separately, with tree == nullptr (brute force).  Dumps every capture and
// the final rays for tests/test_gpu_facade.py.
//
//   facade_step <in_dir> <out_dir> <ray_count> <iters>
// in_dir: vertices.f64, faces.i32, alpha.f64, params.f64 = {src xyz, recv xyz, radius}
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "roomray_b200.hpp"

namespace rb = roomray_b200;

template <typename T>
std::vector<T> read_all(const std::string& path) {
  std::ifstream f(path, std::ios::binary | std::ios::ate);
  if (!f) throw std::runtime_error("cannot open " + path);
  const auto bytes = static_cast<std::size_t>(f.tellg());
  std::vector<T> v(bytes / sizeof(T));
  f.seekg(0);
  f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(bytes));
  return v;
}

template <typename T>
void write_all(const std::string& path, const std::vector<T>& v) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

static void run(const std::string& out, const std::string& tag, const rb::TriangleMesh& mesh,
                const rb::AccelTree* tree, const rb::SourceConfig& src, const rb::Receiver& recv, int iters) {
  std::vector<rb::Ray> rays = rb::emit(src);
  rb::TraceConfig cfg;  // max_range <= 0: (r/2) sqrt(N), as trace() resolves it
  std::vector<int32_t> c_ray, c_hist;
  std::vector<int64_t> c_off{0};
  std::vector<double> c_f;
  for (int it = 0; it < iters; ++it) {
    for (const rb::Capture& c : rb::step(rays, mesh, tree, recv, cfg)) {
      c_ray.push_back(c.ray_index);
      for (int k = 0; k < 3; ++k) c_f.push_back(c.point[k]);
      for (int k = 0; k < 3; ++k) c_f.push_back(c.incoming_dir[k]);
      c_f.push_back(c.path_length);
      for (double m : c.band_multiplier) c_f.push_back(m);
      c_hist.insert(c_hist.end(), c.face_history.begin(), c.face_history.end());
      c_off.push_back(static_cast<int64_t>(c_hist.size()));
    }
  }
  std::vector<double> r_f;  // origin, dir, path, alive, n_hist, mult
  for (const rb::Ray& r : rays) {
    for (int k = 0; k < 3; ++k) r_f.push_back(r.origin[k]);
    for (int k = 0; k < 3; ++k) r_f.push_back(r.dir[k]);
    r_f.push_back(r.path_length);
    r_f.push_back(r.alive ? 1.0 : 0.0);
    r_f.push_back(static_cast<double>(r.face_history.size()));
    for (double m : r.band_multiplier) r_f.push_back(m);
  }
  write_all(out + "/" + tag + "_cap_ray.i32", c_ray);
  write_all(out + "/" + tag + "_cap_f.f64", c_f);
  write_all(out + "/" + tag + "_cap_off.i64", c_off);
  write_all(out + "/" + tag + "_cap_hist.i32", c_hist);
  write_all(out + "/" + tag + "_rays.f64", r_f);
}

int main(int argc, char** argv) {
  if (argc != 5) {
    std::cerr << "usage: facade_step in_dir out_dir ray_count iters\n";
    return 2;
  }
  const std::string in = argv[1], out = argv[2];
  try {
    const auto v = read_all<double>(in + "/vertices.f64");
    const auto f = read_all<int32_t>(in + "/faces.i32");
    const auto a = read_all<double>(in + "/alpha.f64");
    const auto p = read_all<double>(in + "/params.f64");
    rb::TriangleMesh mesh;
    for (std::size_t i = 0; i + 2 < v.size(); i += 3) mesh.vertices.push_back({v[i], v[i + 1], v[i + 2]});
    for (std::size_t i = 0; i + 3 < f.size(); i += 4) mesh.faces.push_back({f[i], f[i + 1], f[i + 2], f[i + 3]});
    for (std::size_t m = 0; m * 8 < a.size(); ++m) {
      rb::Material mat;
      mat.name = "m" + std::to_string(m);
      for (int b = 0; b < 8; ++b) mat.absorption[b] = a[8 * m + b];
      mesh.materials.push_back(mat);
    }
    rb::SourceConfig src;
    src.position = {p[0], p[1], p[2]};
    src.ray_count = std::atoi(argv[3]);
    rb::Receiver recv;
    recv.center = {p[3], p[4], p[5]};
    recv.radius = p[6];
    const int iters = std::atoi(argv[4]);
    bool threw = false;  // emission.cpp:9-11
    try {
      rb::SourceConfig bad = src;
      bad.ray_count = 0;
      rb::emit(bad);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    if (!threw) {
      std::cerr << "emit(ray_count = 0) did not throw std::invalid_argument\n";
      return 1;
    }
    const rb::AccelTree tree = rb::build_tree(mesh);
    run(out, "tree", mesh, &tree, src, recv, iters);
    run(out, "brute", mesh, nullptr, src, recv, iters);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
