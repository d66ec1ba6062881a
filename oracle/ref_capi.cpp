// C entry points over the UNMODIFIED reference sources — TEST INFRASTRUCTURE.
//
// Built by oracle/Makefile together with /root/reference/proj/src/{geometry,
// accel_tree,tracer,emission,air_absorption,image_sources,rir,mesh_gen,
// shoebox}.cpp (compiled in place, against the from-scratch Eigen subset in
// oracle/eigen_shim) into oracle/_ref/libroomray_ref.so.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// load it.  Every function below only marshals plain arrays into the
// reference's own types and calls the reference's public API:
//   build_tree            accel_tree.hpp:38
//   nearest_hit(_brute)   accel_tree.hpp:50-55
//   trace / step          tracer.hpp:43-52   (strided subsets: the trace()
//                         loop of tracer.cpp:108-132 driven over a subset)
//   build_image_sources   image_sources.hpp:58-61
//   build_pulse_trains / synthesize / design_band_filter  rir.hpp:33-45
//   air_beta_bands        air_absorption.hpp:30
//   factors               metrics.hpp:56-60
//   enumerate_images      shoebox.hpp:43
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <memory>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "roomray/accel_tree.hpp"
#include "roomray/air_absorption.hpp"
#include "roomray/emission.hpp"
#include "roomray/image_sources.hpp"
#include "roomray/mesh_gen.hpp"
#include "roomray/metrics.hpp"
#ifdef RREF_HAVE_OBJ
#include "roomray/obj_loader.hpp"
#include "roomray/pipeline.hpp"
#endif
#include "roomray/rir.hpp"
#include "roomray/shoebox.hpp"
#include "roomray/tracer.hpp"

using namespace roomray;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

TriangleMesh make_mesh(const double* verts, int64_t nv, const int32_t* tris,
                       int64_t nf, const double* alpha, int32_t nmat) {
  TriangleMesh mesh;
  mesh.vertices.resize(nv);
  for (int64_t i = 0; i < nv; ++i)
    mesh.vertices[i] = Vec3(verts[3 * i], verts[3 * i + 1], verts[3 * i + 2]);
  mesh.faces.resize(nf);
  for (int64_t f = 0; f < nf; ++f)
    mesh.faces[f] = {tris[4 * f], tris[4 * f + 1], tris[4 * f + 2],
                     tris[4 * f + 3]};
  mesh.materials.resize(nmat);
  for (int32_t m = 0; m < nmat; ++m) {
    mesh.materials[m].name = "m" + std::to_string(m);
    for (int b = 0; b < kNumBands; ++b)
      mesh.materials[m].absorption[b] = alpha[kNumBands * m + b];
  }
  return mesh;
}

struct RefScene {
  TriangleMesh mesh;
  AccelTree tree;
};

struct RefTrace {
  TraceResult result;
  int64_t total_hist = 0;
  int64_t ray_bounces = 0;
};

struct RefImages {
  std::vector<ImageSource> images;
  int64_t total_path = 0;
};

}  // namespace

extern "C" {

const char* rref_last_error() { return g_err.c_str(); }

// Scene = mesh + reference tree (build_tree, accel_tree.cpp:70-87).
void* rref_scene_create(const double* verts, int64_t nv, const int32_t* tris,
                        int64_t nf, const double* alpha, int32_t nmat,
                        int validate) {
  RefScene* s = nullptr;
  int rc = guarded([&] {
    auto scene = std::make_unique<RefScene>();
    scene->mesh = make_mesh(verts, nv, tris, nf, alpha, nmat);
    if (validate) scene->mesh.validate();
    scene->tree = build_tree(scene->mesh);
    s = scene.release();
  });
  return rc == 0 ? s : nullptr;
}

void rref_scene_destroy(void* h) { delete static_cast<RefScene*>(h); }

int64_t rref_tree_size(void* h, int32_t* root, int32_t* depth) {
  auto* s = static_cast<RefScene*>(h);
  *root = s->tree.root;
  *depth = s->tree.depth();
  return static_cast<int64_t>(s->tree.nodes.size());
}

void rref_tree_nodes(void* h, int32_t* left, int32_t* right, int32_t* face,
                     double* lo, double* hi) {
  auto* s = static_cast<RefScene*>(h);
  for (size_t i = 0; i < s->tree.nodes.size(); ++i) {
    const TreeNode& n = s->tree.nodes[i];
    left[i] = n.left;
    right[i] = n.right;
    face[i] = n.face_index;
    for (int k = 0; k < 3; ++k) {
      lo[3 * i + k] = n.box.min[k];
      hi[3 * i + k] = n.box.max[k];
    }
  }
}

int rref_empty_tree_throws() {
  TriangleMesh mesh;
  return guarded([&] { build_tree(mesh); });
}

// nearest_hit (tree) or nearest_hit_brute for n rays.
int rref_nearest_hit(void* h, const double* o, const double* d, int64_t n,
                     int brute, int32_t* face, double* delta, double* point) {
  auto* s = static_cast<RefScene*>(h);
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      const Vec3 org(o[3 * i], o[3 * i + 1], o[3 * i + 2]);
      const Vec3 dir(d[3 * i], d[3 * i + 1], d[3 * i + 2]);
      const auto hit = brute ? nearest_hit_brute(s->mesh, org, dir)
                             : nearest_hit(s->tree, s->mesh, org, dir);
      face[i] = hit ? hit->face_index : -1;
      delta[i] = hit ? hit->delta : 0.0;
      for (int k = 0; k < 3; ++k) point[3 * i + k] = hit ? hit->point[k] : 0.0;
    }
  });
}

int rref_intersect_sphere(const double* o, const double* d, const double* c,
                          double r, double* out) {
  const auto s = intersect_sphere(Vec3(o[0], o[1], o[2]), Vec3(d[0], d[1], d[2]),
                                  Vec3(c[0], c[1], c[2]), r);
  *out = s ? *s : -1.0;
  return s ? 1 : 0;
}

void rref_fibonacci(int n, double* out) {
  const auto dirs = fibonacci_directions(n);
  for (int k = 0; k < n; ++k)
    for (int a = 0; a < 3; ++a) out[3 * k + a] = dirs[k][a];
}

// trace(): tracer.cpp:108-149.  When stride > 1, the same loop is driven over
// the ray subset k = first + i*stride (i < count) of the full-N Fibonacci
// lattice, with max_range resolved against the full N (tracer.cpp:117-118).
// stride <= 0 calls trace() itself; stride >= 1 runs the subset driver, which
// also counts ray-bounces (one per step_ray call on a live ray).
// Capture ray indices are reported as global lattice indices.
void* rref_trace(void* h, const double* src, int32_t ray_count,
                 const double* recv, double radius, int32_t max_iterations,
                 double max_range, int32_t threads, int64_t first,
                 int64_t stride, int64_t count) {
  auto* s = static_cast<RefScene*>(h);
  RefTrace* out = nullptr;
  int rc = guarded([&] {
    auto t = std::make_unique<RefTrace>();
    SourceConfig source;
    source.position = Vec3(src[0], src[1], src[2]);
    source.ray_count = ray_count;
    Receiver receiver{Vec3(recv[0], recv[1], recv[2]), radius};
    TraceConfig config;
    config.max_iterations = max_iterations;
    config.max_range = max_range;
    config.thread_count = threads;
    if (stride <= 0) {
      t->result = trace(s->mesh, s->tree, source, receiver, config);
    } else {
      if (receiver.radius <= 0.0)
        throw std::invalid_argument("receiver radius must be > 0");
      source.validate();
      const auto all = emit(source);
      std::vector<Ray> rays;
      std::vector<int> global;
      if (count <= 0) count = (ray_count - first + stride - 1) / stride;
      for (int64_t i = 0; i < count; ++i) {
        const int64_t k = first + i * stride;
        if (k >= ray_count) break;
        rays.push_back(all[k]);
        global.push_back(static_cast<int>(k));
      }
      TraceConfig resolved = config;
      resolved.max_range = config.resolved_max_range(receiver, ray_count);
      TraceResult& result = t->result;
      result.max_range = resolved.max_range;
      size_t live = rays.size();
      while (live > 0 && result.iterations < config.max_iterations) {
        auto caps = step(rays, s->mesh, &s->tree, receiver, resolved);
        for (auto& c : caps) {
          c.ray_index = global[c.ray_index];
          result.captures.push_back(std::move(c));
        }
        ++result.iterations;
        live = 0;
        for (const Ray& r : rays) live += r.alive ? 1 : 0;
      }
      result.truncated = live > 0;
      for (const Ray& r : rays) {
        if (!r.alive && r.path_length > resolved.max_range)
          ++result.out_of_range;
        else if (!r.alive)
          ++result.escaped;
        t->ray_bounces += static_cast<int64_t>(r.face_history.size());
      }
      t->ray_bounces += static_cast<int64_t>(result.escaped);
      std::sort(result.captures.begin(), result.captures.end(),
                [](const Capture& a, const Capture& b) {
                  if (a.ray_index != b.ray_index)
                    return a.ray_index < b.ray_index;
                  return a.path_length < b.path_length;
                });
    }
    for (const Capture& c : t->result.captures)
      t->total_hist += static_cast<int64_t>(c.face_history.size());
    out = t.release();
  });
  return rc == 0 ? out : nullptr;
}

void rref_trace_info(void* h, int32_t* iterations, int32_t* truncated,
                     int64_t* escaped, int64_t* out_of_range,
                     double* max_range, int64_t* n_captures,
                     int64_t* total_hist, int64_t* ray_bounces) {
  auto* t = static_cast<RefTrace*>(h);
  *iterations = t->result.iterations;
  *truncated = t->result.truncated ? 1 : 0;
  *escaped = static_cast<int64_t>(t->result.escaped);
  *out_of_range = static_cast<int64_t>(t->result.out_of_range);
  *max_range = t->result.max_range;
  *n_captures = static_cast<int64_t>(t->result.captures.size());
  *total_hist = t->total_hist;
  *ray_bounces = t->ray_bounces;
}

void rref_trace_captures(void* h, int32_t* ray, double* point, double* dir,
                         double* path, double* mult, int64_t* hist_off,
                         int32_t* hist) {
  auto* t = static_cast<RefTrace*>(h);
  int64_t off = 0;
  for (size_t i = 0; i < t->result.captures.size(); ++i) {
    const Capture& c = t->result.captures[i];
    ray[i] = c.ray_index;
    for (int k = 0; k < 3; ++k) {
      point[3 * i + k] = c.point[k];
      dir[3 * i + k] = c.incoming_dir[k];
    }
    path[i] = c.path_length;
    for (int b = 0; b < kNumBands; ++b) mult[kNumBands * i + b] = c.band_multiplier[b];
    hist_off[i] = off;
    for (int f : c.face_history) hist[off++] = f;
  }
  hist_off[t->result.captures.size()] = off;
}

void rref_trace_free(void* h) { delete static_cast<RefTrace*>(h); }

// build_image_sources over captures given as arrays (image_sources.cpp:154).
void* rref_image_sources(void* hs, int64_t n, const int32_t* ray,
                         const double* point, const double* dir,
                         const double* path, const double* mult,
                         const int64_t* hist_off, const int32_t* hist,
                         int32_t total_rays, const double* air4,
                         const double* recv, double tol_scale,
                         int merge_coplanar) {
  auto* s = static_cast<RefScene*>(hs);
  RefImages* out = nullptr;
  int rc = guarded([&] {
    std::vector<Capture> caps(n);
    for (int64_t i = 0; i < n; ++i) {
      Capture& c = caps[i];
      c.ray_index = ray[i];
      c.point = Vec3(point[3 * i], point[3 * i + 1], point[3 * i + 2]);
      c.incoming_dir = Vec3(dir[3 * i], dir[3 * i + 1], dir[3 * i + 2]);
      c.path_length = path[i];
      for (int b = 0; b < kNumBands; ++b) c.band_multiplier[b] = mult[kNumBands * i + b];
      c.face_history.assign(hist + hist_off[i], hist + hist_off[i + 1]);
    }
    AirModel air;
    air.enabled = air4[0] != 0.0;
    air.temperature_c = air4[1];
    air.relative_humidity = air4[2];
    air.pressure_kpa = air4[3];
    ClusterOptions opt;
    opt.tol_scale = tol_scale;
    opt.merge_coplanar = merge_coplanar != 0;
    auto r = std::make_unique<RefImages>();
    r->images = build_image_sources(caps, total_rays, air,
                                    Vec3(recv[0], recv[1], recv[2]), s->mesh,
                                    s->tree, opt);
    for (const auto& im : r->images) r->total_path += im.face_path.size();
    out = r.release();
  });
  return rc == 0 ? out : nullptr;
}

void rref_images_info(void* h, int64_t* n, int64_t* total_path) {
  auto* r = static_cast<RefImages*>(h);
  *n = static_cast<int64_t>(r->images.size());
  *total_path = r->total_path;
}

void rref_images_get(void* h, double* pos, double* dist, double* energy,
                     double* mult, int32_t* ray_count, int32_t* order,
                     int32_t* has_proj, double* proj, int64_t* path_off,
                     int32_t* path) {
  auto* r = static_cast<RefImages*>(h);
  int64_t off = 0;
  for (size_t i = 0; i < r->images.size(); ++i) {
    const ImageSource& im = r->images[i];
    for (int k = 0; k < 3; ++k) pos[3 * i + k] = im.position[k];
    dist[i] = im.distance;
    for (int b = 0; b < kNumBands; ++b) {
      energy[kNumBands * i + b] = im.band_energy[b];
      mult[kNumBands * i + b] = im.band_multiplier[b];
    }
    ray_count[i] = im.ray_count;
    order[i] = im.order;
    has_proj[i] = im.projection ? 1 : 0;
    for (int k = 0; k < 3; ++k) proj[3 * i + k] = im.projection ? (*im.projection)[k] : 0.0;
    path_off[i] = off;
    for (int f : im.face_path) path[off++] = f;
  }
  path_off[r->images.size()] = off;
}

void rref_images_free(void* h) { delete static_cast<RefImages*>(h); }

void rref_air_beta_bands(const double* air4, double* beta) {
  AirModel air;
  air.enabled = air4[0] != 0.0;
  air.temperature_c = air4[1];
  air.relative_humidity = air4[2];
  air.pressure_kpa = air4[3];
  const BandArray b = air_beta_bands(air);
  for (int i = 0; i < kNumBands; ++i) beta[i] = b[i];
}

double rref_air_alpha(const double* air4, double f) {
  AirModel air;
  air.enabled = air4[0] != 0.0;
  air.temperature_c = air4[1];
  air.relative_humidity = air4[2];
  air.pressure_kpa = air4[3];
  return air_alpha_db_per_m(air, f);
}

int rref_band_filter(int band, double fs, double* taps) {
  return guarded([&] {
    const auto k = design_band_filter(band, fs);
    std::memcpy(taps, k.data(), sizeof(double) * k.size());
  });
}

// build_pulse_trains + synthesize (rir.cpp:9-96) from image distances and
// band energies; writes the broadband response, returns its length.
// If out == nullptr only the length is computed.  band_mask selects which
// bands' trains are populated (the per-band trick of tests/test_rir.cpp:44).
int64_t rref_synthesize(int64_t n, const double* dist, const double* energy,
                        double c, double fs, int32_t band_mask, double* out,
                        int64_t cap) {
  int64_t len = -1;
  int rc = guarded([&] {
    std::vector<ImageSource> images(n);
    for (int64_t i = 0; i < n; ++i) {
      images[i].distance = dist[i];
      for (int b = 0; b < kNumBands; ++b)
        images[i].band_energy[b] = energy[kNumBands * i + b];
    }
    PulseTrains trains = build_pulse_trains(images, c);
    for (int b = 0; b < kNumBands; ++b)
      if (!(band_mask & (1 << b))) trains[b].events.clear();
    const auto rir = synthesize(trains, fs);
    len = static_cast<int64_t>(rir.samples.size());
    if (out) {
      const int64_t m = std::min(len, cap);
      std::memcpy(out, rir.samples.data(), sizeof(double) * m);
    }
  });
  return rc == 0 ? len : -1;
}

// factors(build_pulse_trains(images, c)) (metrics.cpp:168-180, rir.cpp:9-30):
// out = 9 x 6 x {value, reliable}, bands 0..7 then "mid"; factor order
// edt_s, t30_s, spl_db, c80_db, d50_pct, ts_ms (metrics.hpp:39-46).
int rref_factors(int64_t n, const double* dist, const double* energy, double c, double* out) {
  return guarded([&] {
    std::vector<ImageSource> images(n);
    for (int64_t i = 0; i < n; ++i) {
      images[i].distance = dist[i];
      for (int b = 0; b < kNumBands; ++b) images[i].band_energy[b] = energy[kNumBands * i + b];
    }
    const BandFactors bf = factors(build_pulse_trains(images, c));
    auto put = [&](int slot, const PerceptiveFactors& f) {
      const MetricValue* m[6] = {&f.edt_s, &f.t30_s, &f.spl_db, &f.c80_db, &f.d50_pct, &f.ts_ms};
      for (int k = 0; k < 6; ++k) {
        out[(slot * 6 + k) * 2] = m[k]->value;
        out[(slot * 6 + k) * 2 + 1] = m[k]->reliable ? 1.0 : 0.0;
      }
    };
    for (int b = 0; b < kNumBands; ++b) put(b, bf.bands[b]);
    put(kNumBands, bf.mid);
  });
}

#ifdef RREF_HAVE_OBJ
// parse_material_table + parse_obj (obj_loader.cpp:25-152).  Returns 0 ok,
// 1 ObjParseError (*line set), 2 UnresolvedMaterialError, 3 other error;
// the mesh stays in a handle for rref_obj_get.
struct RefObj {
  TriangleMesh mesh;
  LoadReport report;
};
int rref_parse_obj(const char* obj_text, const char* mat_json, void** out, int32_t* line) {
  *out = nullptr;
  *line = 0;
  try {
    auto r = std::make_unique<RefObj>();
    const auto table = parse_material_table(mat_json);
    r->mesh = parse_obj(obj_text, table, &r->report);
    *out = r.release();
    return 0;
  } catch (const ObjParseError& e) {
    g_err = e.what();
    *line = e.line();
    return 1;
  } catch (const UnresolvedMaterialError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}
void rref_obj_info(void* h, int64_t* nv, int64_t* nf, int64_t* nmat, int64_t* degenerate) {
  auto* r = static_cast<RefObj*>(h);
  *nv = static_cast<int64_t>(r->mesh.vertices.size());
  *nf = static_cast<int64_t>(r->mesh.faces.size());
  *nmat = static_cast<int64_t>(r->mesh.materials.size());
  *degenerate = static_cast<int64_t>(r->report.degenerate_skipped);
}
void rref_obj_get(void* h, double* verts, int32_t* tris, double* alpha) {
  auto* r = static_cast<RefObj*>(h);
  for (std::size_t i = 0; i < r->mesh.vertices.size(); ++i)
    for (int k = 0; k < 3; ++k) verts[3 * i + k] = r->mesh.vertices[i][k];
  for (std::size_t f = 0; f < r->mesh.faces.size(); ++f) {
    const Triangle& t = r->mesh.faces[f];
    tris[4 * f] = t.a;
    tris[4 * f + 1] = t.b;
    tris[4 * f + 2] = t.c;
    tris[4 * f + 3] = t.material_id;
  }
  for (std::size_t m = 0; m < r->mesh.materials.size(); ++m)
    for (int b = 0; b < kNumBands; ++b) alpha[kNumBands * m + b] = r->mesh.materials[m].absorption[b];
}
void rref_obj_free(void* h) { delete static_cast<RefObj*>(h); }
#endif

// Shoebox lattice oracle (shoebox.cpp:43-116): count, then fetch.
void* rref_lattice(const double* dims, const double* walls_alpha /*6x8*/,
                   const double* src, const double* recv, double max_distance,
                   double radius, const double* air4, int64_t* n) {
  std::vector<OracleImageSource>* out = nullptr;
  int rc = guarded([&] {
    ShoeBox box;
    box.dimensions = Vec3(dims[0], dims[1], dims[2]);
    for (int w = 0; w < 6; ++w)
      for (int b = 0; b < kNumBands; ++b)
        box.walls[w].absorption[b] = walls_alpha[kNumBands * w + b];
    AirModel air;
    air.enabled = air4[0] != 0.0;
    air.temperature_c = air4[1];
    air.relative_humidity = air4[2];
    air.pressure_kpa = air4[3];
    out = new std::vector<OracleImageSource>(enumerate_images(
        box, Vec3(src[0], src[1], src[2]), Vec3(recv[0], recv[1], recv[2]),
        max_distance, radius, air));
    *n = static_cast<int64_t>(out->size());
  });
  return rc == 0 ? out : nullptr;
}

void rref_lattice_get(void* h, double* pos, double* dist, int32_t* order,
                      double* energy) {
  auto* v = static_cast<std::vector<OracleImageSource>*>(h);
  for (size_t i = 0; i < v->size(); ++i) {
    const auto& im = (*v)[i];
    for (int k = 0; k < 3; ++k) pos[3 * i + k] = im.position[k];
    dist[i] = im.distance;
    order[i] = im.order;
    for (int b = 0; b < kNumBands; ++b) energy[kNumBands * i + b] = im.band_energy[b];
  }
}

void rref_lattice_hits(void* h, int32_t* hits) {
  auto* v = static_cast<std::vector<OracleImageSource>*>(h);
  for (size_t i = 0; i < v->size(); ++i)
    for (int w = 0; w < 6; ++w) hits[6 * i + w] = (*v)[i].wall_hits[w];
}

// compare (shoebox.cpp:126-182) on plain arrays.
void* rref_compare(int64_t no, const double* opos, const double* oen, const int32_t* oorder, int64_t nt,
                   const double* tpos, const double* ten, double pos_tol, double tol_db, int64_t* counts,
                   double* max_err, double* rms) {
  MatchReport* out = nullptr;
  int rc = guarded([&] {
    std::vector<OracleImageSource> oracle(static_cast<size_t>(no));
    for (int64_t i = 0; i < no; ++i) {
      oracle[i].position = Vec3(opos[3 * i], opos[3 * i + 1], opos[3 * i + 2]);
      oracle[i].order = oorder[i];
      for (int b = 0; b < kNumBands; ++b) oracle[i].band_energy[b] = oen[kNumBands * i + b];
    }
    std::vector<ImageSource> traced(static_cast<size_t>(nt));
    for (int64_t i = 0; i < nt; ++i) {
      traced[i].position = Vec3(tpos[3 * i], tpos[3 * i + 1], tpos[3 * i + 2]);
      for (int b = 0; b < kNumBands; ++b) traced[i].band_energy[b] = ten[kNumBands * i + b];
    }
    out = new MatchReport(compare(oracle, traced, pos_tol, tol_db));
    int64_t members = 0;
    for (const auto& m : out->matched) members += static_cast<int64_t>(m.traced_indices.size());
    counts[0] = static_cast<int64_t>(out->matched.size());
    counts[1] = members;
    counts[2] = static_cast<int64_t>(out->unmatched_oracle.size());
    counts[3] = static_cast<int64_t>(out->unmatched_traced.size());
    *max_err = out->max_position_error;
    for (int b = 0; b < kNumBands; ++b) rms[b] = out->rms_energy_error_db[b];
  });
  return rc == 0 ? out : nullptr;
}

void rref_compare_get(void* h, int32_t* oracle_index, double* pos_err, int32_t* order, double* delta,
                      int64_t* member_off, int32_t* members, int32_t* uo, int32_t* ut) {
  auto* r = static_cast<MatchReport*>(h);
  member_off[0] = 0;
  int64_t k = 0;
  for (size_t g = 0; g < r->matched.size(); ++g) {
    const auto& m = r->matched[g];
    oracle_index[g] = m.oracle_index;
    pos_err[g] = m.position_error;
    order[g] = m.order;
    for (int b = 0; b < kNumBands; ++b) delta[kNumBands * g + b] = m.energy_delta_db[b];
    for (int t : m.traced_indices) members[k++] = t;
    member_off[g + 1] = k;
  }
  for (size_t i = 0; i < r->unmatched_oracle.size(); ++i) uo[i] = r->unmatched_oracle[i];
  for (size_t i = 0; i < r->unmatched_traced.size(); ++i) ut[i] = r->unmatched_traced[i];
}

void rref_compare_free(void* h) { delete static_cast<MatchReport*>(h); }

void rref_lattice_free(void* h) {
  delete static_cast<std::vector<OracleImageSource>*>(h);
}

// Reference mesh generators (mesh_gen.cpp) — used to pin scene fixtures.
// kind 0: box(dims=p[0..2]); 1: icosphere(level); 2: tetra(log2 faces).
void* rref_mesh_gen(int kind, const double* p, int level, int64_t* nv,
                    int64_t* nf) {
  TriangleMesh* out = nullptr;
  int rc = guarded([&] {
    Material m;
    m.name = "g";
    TriangleMesh mesh;
    if (kind == 0) mesh = make_box_mesh(Vec3(p[0], p[1], p[2]), m);
    else if (kind == 1) mesh = make_icosphere(level, m);
    else mesh = make_subdivided_tetrahedron(level, m);
    out = new TriangleMesh(std::move(mesh));
    *nv = static_cast<int64_t>(out->vertices.size());
    *nf = static_cast<int64_t>(out->faces.size());
  });
  return rc == 0 ? out : nullptr;
}

void rref_mesh_get(void* h, double* verts, int32_t* tris) {
  auto* m = static_cast<TriangleMesh*>(h);
  for (size_t i = 0; i < m->vertices.size(); ++i)
    for (int k = 0; k < 3; ++k) verts[3 * i + k] = m->vertices[i][k];
  for (size_t f = 0; f < m->faces.size(); ++f) {
    tris[4 * f] = m->faces[f].a;
    tris[4 * f + 1] = m->faces[f].b;
    tris[4 * f + 2] = m->faces[f].c;
    tris[4 * f + 3] = m->faces[f].material_id;
  }
}

void rref_mesh_free(void* h) { delete static_cast<TriangleMesh*>(h); }

int rref_hardware_threads() {
  return static_cast<int>(std::thread::hardware_concurrency());
}


// The reference's complexity benchmark row (bench.cpp:71-102 with the timing
// loop of bench.cpp:26-46): build the subdivided tetrahedron of 2^k faces
// (mesh_gen.hpp:25), build_tree, then the per-iteration wall time of step()
// over 2^k emitted rays (tree, or brute force when with_tree == 0).
// Returns seconds per iteration (< 0 on error); build seconds and the tree
// depth go to the out-pointers.
double rref_bench_row(int k, int with_tree, int threads, double min_elapsed,
                      int max_repeats, double* build_seconds, int32_t* depth) {
  using Clock = std::chrono::steady_clock;
  double per_iter = -1.0;
  guarded([&] {
    Material reflective;
    reflective.name = "reflective";
    reflective.absorption = BandArray::Zero();
    const TriangleMesh mesh = make_subdivided_tetrahedron(k, reflective);
    const auto b0 = Clock::now();
    const AccelTree tree = build_tree(mesh);
    *build_seconds = std::chrono::duration<double>(Clock::now() - b0).count();
    *depth = tree.depth();
    SourceConfig source;
    source.position = Vec3::Zero();
    source.ray_count = 1 << k;
    auto rays = emit(source);
    Receiver receiver;
    receiver.center = Vec3(1e6, 1e6, 1e6);
    receiver.radius = 1e-3;
    TraceConfig config;
    config.max_range = 1e30;
    config.thread_count = threads;
    const AccelTree* t = with_tree ? &tree : nullptr;
    step(rays, mesh, t, receiver, config);
    double elapsed = 0.0;
    int repeats = 0;
    while (repeats < max_repeats && (repeats < 1 || elapsed < min_elapsed)) {
      const auto s0 = Clock::now();
      step(rays, mesh, t, receiver, config);
      elapsed += std::chrono::duration<double>(Clock::now() - s0).count();
      ++repeats;
    }
    per_iter = elapsed / repeats;
  });
  return per_iter;
}


#ifdef RREF_HAVE_OBJ
// The reference's `roomray trace` file set (pipeline.cpp:144-325): run the
// pipeline on a run config (deterministic: one thread) and write its
// artifacts into out_dir; with an oracle config also run_oracle +
// write_oracle_artifacts and the comparison report of the traced
// image_sources.json (pipeline.cpp:327-514) into out_dir/oracle.
int rref_run_artifacts(const char* run_json, const char* out_dir, const char* oracle_json) {
  return guarded([&] {
    RunConfig config = RunConfig::from_json_file(run_json);
    config.output_dir = out_dir;
    config.deterministic = true;
    config.dump_captures = true;
    config.dump_tree_stats = true;
    const RunArtifacts artifacts = run_trace_pipeline(config);
    write_run_artifacts(config, artifacts);
    if (oracle_json && *oracle_json) {
      OracleConfig oc = OracleConfig::from_json_file(oracle_json);
      oc.output_dir = std::string(out_dir) + "/oracle";
      const auto oracle = run_oracle(oc);
      write_oracle_artifacts(oc, oracle);
      const auto traced = load_image_sources_json(std::string(out_dir) + "/image_sources.json");
      check_comparable(oc, traced);
      write_comparison_report(oc.output_dir + "/comparison.json", compare(oracle, traced.images, 1e-9, 1.5));
    }
  });
}
#endif

}  // extern "C"
