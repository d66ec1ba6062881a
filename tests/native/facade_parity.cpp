// C++ drop-in check: drives the reference-shaped API of include/roomray_b200.hpp
// (build_tree, nearest_hit, trace, build_image_sources, build_pulse_trains,
// synthesize) the way run_trace_pipeline does (pipeline.cpp:154-175) and
// dumps every result as raw arrays for tests/test_gpu_facade.py to compare
// with the oracle.
//
//   facade_parity <in_dir> <out_dir> <ray_count> <max_iterations> <max_range> <merge>
// in_dir: vertices.f64 (nv*3), faces.i32 (nf*4), alpha.f64 (nmat*8),
//         params.f64 = {src xyz, recv xyz, radius, c, fs}
#include <cstdio>
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

int main(int argc, char** argv) {
  if (argc != 7) {
    std::cerr << "usage: facade_parity in_dir out_dir ray_count max_iterations max_range merge\n";
    return 2;
  }
  const std::string in = argv[1], out = argv[2];
  const int n_rays = std::atoi(argv[3]);
  const int max_it = std::atoi(argv[4]);
  const double max_range = std::atof(argv[5]);
  const bool merge = std::atoi(argv[6]) != 0;
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
    // reference error behaviour: empty mesh -> std::invalid_argument (accel_tree.cpp:71-73)
    bool threw = false;
    try {
      rb::build_tree(rb::TriangleMesh{});
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    if (!threw) {
      std::cerr << "empty mesh did not throw std::invalid_argument\n";
      return 1;
    }
    const rb::AccelTree tree = rb::build_tree(mesh);
    write_all(out + "/tree_info.i64",
              std::vector<int64_t>{static_cast<int64_t>(tree.node_count()), tree.root, tree.depth(),
                                   static_cast<int64_t>(tree.leaf_count())});
    // nearest_hit vs nearest_hit_brute from the source along 64 lattice-free directions
    rb::SourceConfig src;
    src.position = {p[0], p[1], p[2]};
    src.ray_count = n_rays;
    rb::Receiver recv;
    recv.center = {p[3], p[4], p[5]};
    recv.radius = p[6];
    std::vector<double> hits;
    for (int k = 0; k < 64; ++k) {
      const double z = 1.0 - (2.0 * k + 1.0) / 64.0, r = std::sqrt(1.0 - z * z), ph = 2.399963229728653 * k;
      const rb::Vec3 d{r * std::cos(ph), r * std::sin(ph), z};
      const auto h = rb::nearest_hit(tree, mesh, src.position, d);
      const auto hb = rb::nearest_hit_brute(tree, src.position, d);
      hits.push_back(h ? h->face_index : -1);
      hits.push_back(h ? h->delta : 0.0);
      hits.push_back(hb ? hb->face_index : -1);
      hits.push_back(hb ? hb->delta : 0.0);
    }
    write_all(out + "/hits.f64", hits);

    rb::TraceConfig cfg;
    cfg.max_iterations = max_it;
    cfg.max_range = max_range;
    cfg.speed_of_sound = p[7];
    const rb::TraceResult tr = rb::trace(mesh, tree, src, recv, cfg);
    std::vector<int32_t> c_ray, c_hist;
    std::vector<int64_t> c_off{0};
    std::vector<double> c_f;  // point, dir, path, mult
    for (const rb::Capture& c : tr.captures) {
      c_ray.push_back(c.ray_index);
      for (int k = 0; k < 3; ++k) c_f.push_back(c.point[k]);
      for (int k = 0; k < 3; ++k) c_f.push_back(c.incoming_dir[k]);
      c_f.push_back(c.path_length);
      for (double m : c.band_multiplier) c_f.push_back(m);
      c_hist.insert(c_hist.end(), c.face_history.begin(), c.face_history.end());
      c_off.push_back(static_cast<int64_t>(c_hist.size()));
    }
    write_all(out + "/cap_ray.i32", c_ray);
    write_all(out + "/cap_f.f64", c_f);
    write_all(out + "/cap_off.i64", c_off);
    write_all(out + "/cap_hist.i32", c_hist);
    write_all(out + "/trace_stats.f64",
              std::vector<double>{static_cast<double>(tr.iterations), tr.truncated ? 1.0 : 0.0,
                                  static_cast<double>(tr.escaped), static_cast<double>(tr.out_of_range), tr.max_range,
                                  static_cast<double>(tr.ray_bounces)});

    rb::AirModel air;
    rb::ClusterOptions opt;
    opt.merge_coplanar = merge;
    const auto images = rb::build_image_sources(tr.captures, n_rays, air, recv.center, mesh, tree, opt);
    std::vector<double> i_f;  // pos, dist, energy, mult, count, order, has_proj, proj
    std::vector<int32_t> i_path;
    std::vector<int64_t> i_off{0};
    for (const rb::ImageSource& s : images) {
      for (int k = 0; k < 3; ++k) i_f.push_back(s.position[k]);
      i_f.push_back(s.distance);
      for (double e : s.band_energy) i_f.push_back(e);
      for (double m : s.band_multiplier) i_f.push_back(m);
      i_f.push_back(s.ray_count);
      i_f.push_back(s.order);
      i_f.push_back(s.projection ? 1.0 : 0.0);
      const rb::Vec3 pr = s.projection.value_or(rb::Vec3{});
      for (int k = 0; k < 3; ++k) i_f.push_back(pr[k]);
      i_path.insert(i_path.end(), s.face_path.begin(), s.face_path.end());
      i_off.push_back(static_cast<int64_t>(i_path.size()));
    }
    write_all(out + "/img_f.f64", i_f);
    write_all(out + "/img_path.i32", i_path);
    write_all(out + "/img_off.i64", i_off);

    const rb::PulseTrains trains = rb::build_pulse_trains(images, cfg.speed_of_sound);
    const rb::RoomImpulseResponse rir = rb::synthesize(trains, p[8]);
    write_all(out + "/rir.f64", rir.samples);
    std::vector<double> bands;
    for (const auto& b : rir.band_samples) bands.insert(bands.end(), b.begin(), b.end());
    write_all(out + "/rir_bands.f64", bands);
    const rb::BandFactors bf = rb::factors(trains);
    std::vector<double> fac;
    auto put = [&](const rb::PerceptiveFactors& f) {
      for (const rb::MetricValue* m : {&f.edt_s, &f.t30_s, &f.spl_db, &f.c80_db, &f.d50_pct, &f.ts_ms}) {
        fac.push_back(m->value);
        fac.push_back(m->reliable ? 1.0 : 0.0);
      }
    };
    for (const auto& f : bf.bands) put(f);
    put(bf.mid);
    write_all(out + "/factors.f64", fac);
    try {
      rb::build_pulse_trains(images, 0.0);
      std::cerr << "c = 0 did not throw\n";
      return 1;
    } catch (const std::invalid_argument&) {
    }
    std::cout << "facade ok: " << tr.captures.size() << " captures, " << images.size() << " images, "
              << rir.samples.size() << " samples\n";
  } catch (const std::exception& e) {
    std::cerr << "facade_parity: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
