// roomray_b200.hpp — header-only C++ facade over the C ABI (roomray_b200.h).
//
// Re-exposes the reference's C++ API for the ray-propagation path
// (namespace roomray, /root/reference/proj/include/roomray) with the same
// names, argument meaning and exceptions, on Eigen-free value types, so a
// caller such as run_trace_pipeline (pipeline.cpp:154-175) can switch by
// changing the namespace.  All compute runs on the GPU through
// libroomray_b200.so; there is no CPU path.  Link: -lroomray_b200.
//
// Differences from the reference, all outside the hot path:
//  * Vec3 is {x, y, z} with operator[]; BandArray is std::array<double, 8>.
//  * AccelTree holds the device scene (traversed through a device SAH tree);
//    its reference-layout median tree is built and downloaded on first use
//    through nodes() (a method, not a field).
//  * Hit carries delta, point and face_index (lambda / mu are not reported).
//  * RoomImpulseResponse additionally holds the 8 per-band responses.
//  * step() takes std::vector<Ray>& (the reference takes std::span<Ray>);
//    with tree == nullptr it builds a device scene from the mesh for the
//    brute-force scan.  trace() does not call it: the persistent kernel
//    traces each ray to completion.
//  * nearest_hit_brute takes the AccelTree (its device copy of the mesh)
//    where the reference takes the TriangleMesh.
#ifndef ROOMRAY_B200_HPP
#define ROOMRAY_B200_HPP

#include <algorithm>
#include <thread>
#include <array>
#include <cmath>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef __linux__
#include <sys/mman.h>
#endif

#include "roomray_b200.h"

namespace roomray_b200 {

inline constexpr int kNumBands = RR_NUM_BANDS;                       // types.hpp:15
inline constexpr std::array<double, kNumBands> kBandCentersHz = {   // types.hpp:20-21
    62.5, 125.0, 250.0, 500.0, 1000.0, 2000.0, 4000.0, 8000.0};
inline constexpr double kSelfHitEpsilon = 1e-6;                       // types.hpp:31
inline constexpr int kBandFilterTaps = 1023;                          // rir.hpp:40
inline constexpr int kBandFilterDelay = (kBandFilterTaps - 1) / 2;    // rir.hpp:41

struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
  double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  bool operator==(const Vec3& o) const { return x == o.x && y == o.y && z == o.z; }
};
using BandArray = std::array<double, kNumBands>;

inline BandArray band_ones() {
  BandArray a;
  a.fill(1.0);
  return a;
}

// ------------------------------------------------------------------ errors
namespace detail {
inline void check(rr_status s) {
  if (s == RR_OK) return;
  const std::string msg = rr_last_error();
  if (s == RR_INVALID_ARGUMENT) throw std::invalid_argument(msg);  // as the reference
  throw std::runtime_error("roomray_b200: " + msg);
}

// f(t, a, b) for the t-th of up to min(hw, 32) contiguous chunks [a, b) of
// [0, n); one chunk (serial) below `serial_below` items
template <typename F>
inline void parallel_chunks(std::size_t n, F&& f, std::size_t serial_below = std::size_t(1) << 14) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const std::size_t nt = n < serial_below ? 1 : std::min<std::size_t>({hw, 32, n});
  if (nt <= 1) {
    if (n) f(std::size_t(0), std::size_t(0), n);
    return;
  }
  std::vector<std::thread> th;
  const std::size_t chunk = (n + nt - 1) / nt;
  for (std::size_t t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      const std::size_t a = std::min(n, t * chunk), b = std::min(n, a + chunk);
      if (a < b) f(t, a, b);
    });
  for (auto& x : th) x.join();
}

// f(i) for i in [0, n) on the host's hardware threads (the conversions of
// device results into the reference's per-record std::vector types are
// allocation bound); serial below 2^14 records
template <typename F>
inline void parallel_for(std::size_t n, F&& f, std::size_t serial_below = std::size_t(1) << 14) {
  parallel_chunks(
      n, [&](std::size_t, std::size_t a, std::size_t b) {
        for (std::size_t i = a; i < b; ++i) f(i);
      },
      serial_below);
}

// One grow-only page-locked buffer per host thread (rr_host_alloc): device
// results are copied into it at full host-link speed and converted from it,
// so no pageable temporaries are zero-filled and faulted in on every call.
class Staging {
 public:
  Staging() = default;
  Staging(const Staging&) = delete;
  Staging& operator=(const Staging&) = delete;
  ~Staging() {
    if (p_) rr_host_free(p_);  // status ignored: may run after the runtime's teardown
  }
  char* get(std::size_t bytes) {
    if (bytes > cap_) {
      if (p_) check(rr_host_free(p_));
      p_ = nullptr;
      cap_ = 0;
      const std::size_t want = bytes + bytes / 4;
      void* q = nullptr;
      check(rr_host_alloc(static_cast<int64_t>(want), &q));
      p_ = static_cast<char*>(q);
      cap_ = want;
    }
    return p_;
  }

 private:
  char* p_ = nullptr;
  std::size_t cap_ = 0;
};
inline Staging& staging() {
  thread_local Staging s;
  return s;
}

// byte offsets of 256-B aligned arrays carved out of one staging buffer
struct Layout {
  std::size_t bytes = 0;
  template <typename T>
  std::size_t add(std::size_t n) {
    const std::size_t o = (bytes + 255) & ~std::size_t(255);
    bytes = o + n * sizeof(T);
    return o;
  }
};
template <typename T>
inline T* at(char* base, std::size_t off) {
  return reinterpret_cast<T*>(base + off);
}

// v.reserve(n), with transparent huge pages requested for the new storage:
// the reference's record vectors run to hundreds of MB, and faulting them in
// 4-KB pages inside their serial value-initialisation dominated the copies.
template <typename T>
inline void reserve_huge(std::vector<T>& v, std::size_t n) {
  v.reserve(n);
#ifdef __linux__
  constexpr std::uintptr_t kHuge = std::uintptr_t(1) << 21;
  const std::uintptr_t a = (reinterpret_cast<std::uintptr_t>(v.data()) + kHuge - 1) & ~(kHuge - 1);
  const std::uintptr_t e = reinterpret_cast<std::uintptr_t>(v.data() + v.capacity()) & ~(kHuge - 1);
  if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);  // advisory: errors ignored
#endif
}
}  // namespace detail

// ------------------------------------------------------------------ device
/// One GPU and its stream (rr_ctx).  A process-wide instance per device is
/// created on first use; a context is not thread-safe.
class Device {
 public:
  explicit Device(int device = 0) {
    rr_ctx* c = nullptr;
    detail::check(rr_ctx_create(device, &c));
    ctx_.reset(c, [](rr_ctx* p) { rr_ctx_destroy(p); });
  }
  static Device& get(int device = 0) {
    static std::vector<std::unique_ptr<Device>> devs;
    if (device < 0) throw std::invalid_argument("device index must be >= 0");
    if (static_cast<int>(devs.size()) <= device) devs.resize(device + 1);
    if (!devs[device]) devs[device] = std::make_unique<Device>(device);
    return *devs[device];
  }
  rr_ctx* handle() const { return ctx_.get(); }
  int64_t launches() const { return rr_ctx_launches(ctx_.get()); }

 private:
  std::shared_ptr<rr_ctx> ctx_;
};

// ------------------------------------------------------------------ geometry (geometry.hpp)
struct Material {
  std::string name;
  BandArray absorption{};
};

struct Triangle {
  int a = 0, b = 0, c = 0;
  int material_id = 0;
};

struct Aabb {
  Vec3 min, max;
  double diagonal() const {
    const double dx = max.x - min.x, dy = max.y - min.y, dz = max.z - min.z;
    return std::sqrt((dx * dx + dy * dy) + dz * dz);
  }
};

struct Hit {
  double delta = 0.0;
  Vec3 point;
  int face_index = -1;
};

struct TriangleMesh {
  std::vector<Vec3> vertices;
  std::vector<Triangle> faces;
  std::vector<Material> materials;
  std::size_t face_count() const { return faces.size(); }
};

// ------------------------------------------------------------------ tree (accel_tree.hpp)
struct TreeNode {
  Aabb box;
  std::int32_t left = -1;
  std::int32_t right = -1;
  std::int32_t face_index = -1;
  bool is_leaf() const { return face_index >= 0; }
};

/// Device scene + median-split tree, built on the GPU by build_tree.
class AccelTree {
 public:
  std::int32_t root = -1;
  std::size_t node_count() const { return static_cast<std::size_t>(n_nodes_); }
  int depth() const { return depth_; }
  std::size_t leaf_count() const {
    std::size_t n = 0;
    for (const TreeNode& t : nodes()) n += t.is_leaf() ? 1 : 0;
    return n;
  }
  /// Reference-layout nodes (post-order, root last), downloaded once.
  const std::vector<TreeNode>& nodes() const {
    if (nodes_.empty() && n_nodes_ > 0) {
      std::vector<rr_tree_node> raw(static_cast<std::size_t>(n_nodes_));
      detail::check(rr_scene_tree(scene_.get(), raw.data()));
      nodes_.resize(raw.size());
      for (std::size_t i = 0; i < raw.size(); ++i) {
        TreeNode& t = nodes_[i];
        t.box.min = {raw[i].lo[0], raw[i].lo[1], raw[i].lo[2]};
        t.box.max = {raw[i].hi[0], raw[i].hi[1], raw[i].hi[2]};
        t.left = raw[i].left;
        t.right = raw[i].right;
        t.face_index = raw[i].face_index;
      }
    }
    return nodes_;
  }
  rr_scene* handle() const { return scene_.get(); }
  const Aabb& bounds() const { return bounds_; }
  double build_ms() const { return rr_scene_build_ms(scene_.get()); }

 private:
  friend AccelTree build_tree(const TriangleMesh&, int);
  std::shared_ptr<rr_scene> scene_;
  int64_t n_nodes_ = 0;
  int depth_ = 0;
  Aabb bounds_;
  mutable std::vector<TreeNode> nodes_;
};

/// build_tree (accel_tree.hpp:38): uploads the mesh, validates it and builds
/// the reference's median-split tree on the device.  Empty mesh, bad indices
/// or degenerate faces throw std::invalid_argument.
inline AccelTree build_tree(const TriangleMesh& mesh, int device = 0) {
  Device& dev = Device::get(device);
  const std::size_t nv = mesh.vertices.size(), nf = mesh.faces.size(), nm = std::max<std::size_t>(mesh.materials.size(), 1);
  detail::Layout L;
  const std::size_t o_v = L.add<double>(3 * nv), o_f = L.add<int32_t>(4 * nf), o_al = L.add<double>(kNumBands * nm);
  char* base = detail::staging().get(L.bytes);
  double* v = detail::at<double>(base, o_v);
  int32_t* f = detail::at<int32_t>(base, o_f);
  double* alpha = detail::at<double>(base, o_al);
  // repack into the page-locked staging buffer (and the bounds) on the host threads
  std::array<Aabb, 32> part;
  for (auto& p : part) {
    p.min = {HUGE_VAL, HUGE_VAL, HUGE_VAL};
    p.max = {-HUGE_VAL, -HUGE_VAL, -HUGE_VAL};
  }
  detail::parallel_chunks(nv, [&](std::size_t t, std::size_t a, std::size_t b) {
    Aabb& p = part[t];
    for (std::size_t i = a; i < b; ++i)
      for (int k = 0; k < 3; ++k) {
        const double x = mesh.vertices[i][k];
        v[3 * i + k] = x;
        p.min[k] = std::min(p.min[k], x);
        p.max[k] = std::max(p.max[k], x);
      }
  });
  Aabb box = part[0];
  for (const Aabb& p : part)
    for (int k = 0; k < 3; ++k) {
      box.min[k] = std::min(box.min[k], p.min[k]);
      box.max[k] = std::max(box.max[k], p.max[k]);
    }
  detail::parallel_for(nf, [&](std::size_t i) {
    f[4 * i] = mesh.faces[i].a;
    f[4 * i + 1] = mesh.faces[i].b;
    f[4 * i + 2] = mesh.faces[i].c;
    f[4 * i + 3] = mesh.faces[i].material_id;
  });
  std::fill(alpha, alpha + kNumBands * nm, 0.0);
  for (std::size_t m = 0; m < mesh.materials.size(); ++m)
    for (int b = 0; b < kNumBands; ++b) alpha[kNumBands * m + b] = mesh.materials[m].absorption[b];
  rr_scene* s = nullptr;
  detail::check(rr_scene_create(dev.handle(), v, static_cast<int64_t>(nv), f, static_cast<int64_t>(nf), alpha,
                                static_cast<int32_t>(nm), 1, &s));
  AccelTree t;
  t.scene_.reset(s, [](rr_scene* p) { rr_scene_destroy(p); });
  int32_t root = -1, depth = 0;
  detail::check(rr_scene_tree_info(s, &t.n_nodes_, &root, &depth));
  t.root = root;
  t.depth_ = depth;
  t.bounds_ = box;
  return t;
}

/// Batched nearest_hit: one optional Hit per (origin, dir) pair.
inline std::vector<std::optional<Hit>> nearest_hit_batch(const AccelTree& tree, const std::vector<Vec3>& origins,
                                                         const std::vector<Vec3>& dirs, bool brute = false) {
  if (origins.size() != dirs.size()) throw std::invalid_argument("origins and dirs differ in length");
  const std::size_t n = origins.size();
  std::vector<double> o(3 * n), d(3 * n), delta(n), point(3 * n);
  std::vector<int32_t> face(n);
  for (std::size_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      o[3 * i + k] = origins[i][k];
      d[3 * i + k] = dirs[i][k];
    }
  detail::check(rr_nearest_hit_batch(tree.handle(), o.data(), d.data(), static_cast<int64_t>(n), brute ? 1 : 0,
                                     face.data(), delta.data(), point.data()));
  std::vector<std::optional<Hit>> out(n);
  for (std::size_t i = 0; i < n; ++i)
    if (face[i] >= 0) out[i] = Hit{delta[i], {point[3 * i], point[3 * i + 1], point[3 * i + 2]}, face[i]};
  return out;
}

/// nearest_hit (accel_tree.hpp:50-51).  `mesh` must be the mesh the tree
/// was built from (the tree holds its device copy).
inline std::optional<Hit> nearest_hit(const AccelTree& tree, const TriangleMesh& /*mesh*/, const Vec3& origin,
                                      const Vec3& dir) {
  return nearest_hit_batch(tree, {origin}, {dir}, false)[0];
}

/// nearest_hit_brute (accel_tree.hpp:54-55) over the tree's device mesh.
inline std::optional<Hit> nearest_hit_brute(const AccelTree& tree, const Vec3& origin, const Vec3& dir) {
  return nearest_hit_batch(tree, {origin}, {dir}, true)[0];
}

/// nearest_hit_brute with the reference signature: uploads `mesh` first.
inline std::optional<Hit> nearest_hit_brute(const TriangleMesh& mesh, const Vec3& origin, const Vec3& dir) {
  return nearest_hit_brute(build_tree(mesh), origin, dir);
}

// ------------------------------------------------------------------ tracer (tracer.hpp, tracer_types.hpp, emission.hpp)
struct SourceConfig {
  Vec3 position;
  int ray_count = 1;
  BandArray initial_energy = band_ones();  // ignored by emit, as in the reference
};

struct Receiver {
  Vec3 center;
  double radius = 0.1;
};

struct TraceConfig {
  int max_iterations = 1000;
  double speed_of_sound = 343.0;
  double max_range = 0.0;  // <= 0: (r/2)*sqrt(N)
  int thread_count = 1;    // accepted for compatibility; the GPU grid replaces it
  double resolved_max_range(const Receiver& receiver, int ray_count) const {
    if (max_range > 0.0) return max_range;  // tracer.cpp:10-15
    return 0.5 * receiver.radius * std::sqrt(static_cast<double>(ray_count));
  }
};

struct Capture {
  int ray_index = -1;
  Vec3 point;
  Vec3 incoming_dir{0.0, 0.0, 1.0};
  double path_length = 0.0;
  BandArray band_multiplier = band_ones();
  std::vector<int> face_history;
};

struct TraceResult {
  std::vector<Capture> captures;  // sorted by (ray index, path length)
  int iterations = 0;
  bool truncated = false;
  std::size_t escaped = 0;
  std::size_t out_of_range = 0;
  double max_range = 0.0;
  int64_t ray_bounces = 0;  // nearest-hit queries executed (extension)
  double kernel_ms = 0.0;   // device time of the trace kernel (extension)
};

/// Specular mirror bounce u - 2(u.n)n (tracer.hpp:33-37).
inline Vec3 reflect(const Vec3& u, const Vec3& n) {
  const double s = 2.0 * ((u.x * n.x + u.y * n.y) + u.z * n.z);
  return {u.x - s * n.x, u.y - s * n.y, u.z - s * n.z};
}

namespace detail {
struct TraceHandle {
  rr_trace_result* h = nullptr;
  explicit TraceHandle(rr_trace_result* p) : h(p) {}
  ~TraceHandle() {
    if (h) rr_trace_destroy(h);
  }
  TraceHandle(const TraceHandle&) = delete;
  TraceHandle& operator=(const TraceHandle&) = delete;
};
}  // namespace detail

namespace detail {
// host copy of a device trace (TraceResult, tracer.hpp:22-29)
inline TraceResult trace_result_from(rr_trace_result* h) {
  rr_trace_stats st{};
  check(rr_trace_stats_get(h, &st));
  const std::size_t n = static_cast<std::size_t>(st.n_captures);
  Layout L;
  const std::size_t o_ray = L.add<int32_t>(n), o_hist = L.add<int32_t>(std::max<int64_t>(st.total_history, 1)),
                    o_pt = L.add<double>(3 * n), o_dir = L.add<double>(3 * n), o_path = L.add<double>(n),
                    o_mult = L.add<double>(kNumBands * n), o_off = L.add<int64_t>(n + 1);
  char* base = staging().get(L.bytes);
  const int32_t* ray = at<int32_t>(base, o_ray);
  const int32_t* hist = at<int32_t>(base, o_hist);
  const double *point = at<double>(base, o_pt), *dir = at<double>(base, o_dir), *path = at<double>(base, o_path),
               *mult = at<double>(base, o_mult);
  const int64_t* off = at<int64_t>(base, o_off);
  check(rr_trace_captures(h, nullptr, at<int32_t>(base, o_ray), at<double>(base, o_pt), at<double>(base, o_dir),
                          at<double>(base, o_path), at<double>(base, o_mult), at<int64_t>(base, o_off),
                          at<int32_t>(base, o_hist)));
  TraceResult r;
  r.iterations = st.iterations;
  r.truncated = st.truncated != 0;
  r.escaped = static_cast<std::size_t>(st.escaped);
  r.out_of_range = static_cast<std::size_t>(st.out_of_range);
  r.max_range = st.max_range;
  r.ray_bounces = st.ray_bounces;
  r.kernel_ms = rr_trace_kernel_ms(h);
  reserve_huge(r.captures, n);
  r.captures.resize(n);
  parallel_for(n, [&](std::size_t i) {
    Capture& c = r.captures[i];
    c.ray_index = ray[i];
    c.point = {point[3 * i], point[3 * i + 1], point[3 * i + 2]};
    c.incoming_dir = {dir[3 * i], dir[3 * i + 1], dir[3 * i + 2]};
    c.path_length = path[i];
    for (int b = 0; b < kNumBands; ++b) c.band_multiplier[b] = mult[kNumBands * i + b];
    c.face_history.assign(hist + off[i], hist + off[i + 1]);
  });
  return r;
}

// the device trace of the whole lattice for one receiver (caller destroys)
inline rr_trace_result* trace_device(const AccelTree& tree, const SourceConfig& source, const Receiver& receiver,
                                     const TraceConfig& config) {
  rr_source src{{source.position.x, source.position.y, source.position.z}, source.ray_count};
  rr_receiver rc{{receiver.center.x, receiver.center.y, receiver.center.z}, receiver.radius};
  rr_trace_config cfg{};
  cfg.max_iterations = config.max_iterations;
  cfg.speed_of_sound = config.speed_of_sound;
  cfg.max_range = config.max_range;
  rr_trace_result* h = nullptr;
  check(rr_trace(tree.handle(), &src, &rc, 1, &cfg, &h));
  return h;
}
}  // namespace detail

/// trace (tracer.hpp:50-52): the whole Fibonacci lattice on the GPU.
inline TraceResult trace(const TriangleMesh& /*mesh*/, const AccelTree& tree, const SourceConfig& source,
                         const Receiver& receiver, const TraceConfig& config) {
  detail::TraceHandle guard(detail::trace_device(tree, source, receiver, config));
  return detail::trace_result_from(guard.h);
}

/// Ray (tracer_types.hpp:11-18).
struct Ray {
  Vec3 origin{};
  Vec3 dir{0.0, 0.0, 1.0};
  BandArray band_multiplier = band_ones();  // product of (1 - alpha) so far
  double path_length = 0.0;
  std::vector<int> face_history;
  bool alive = true;
};

/// fibonacci_directions (emission.hpp, emission.cpp:17-29), on the host with
/// the C library's sin/cos exactly as the reference evaluates it.
inline std::vector<Vec3> fibonacci_directions(int n) {
  if (n < 1) throw std::invalid_argument("fibonacci_directions needs n >= 1");
  const double golden = (1.0 + std::sqrt(5.0)) / 2.0;
  const double step_phi = 2.0 * M_PI * (1.0 - 1.0 / golden);
  std::vector<Vec3> d(static_cast<std::size_t>(n));
  for (int k = 0; k < n; ++k) {
    const double z = 1.0 - (2.0 * k + 1.0) / n;
    const double rho = std::sqrt(std::max(0.0, 1.0 - z * z));
    const double phi = step_phi * k;
    d[k] = {rho * std::cos(phi), rho * std::sin(phi), z};
  }
  return d;
}

/// emit (emission.hpp:27, emission.cpp:31-43): one live ray per lattice
/// direction at the source, multiplier 1, path 0.
inline std::vector<Ray> emit(const SourceConfig& source) {
  if (source.ray_count < 1) throw std::invalid_argument("source ray_count must be >= 1");
  for (double e : source.initial_energy)
    if (e < 0.0) throw std::invalid_argument("source initial_energy must be >= 0");
  const auto dirs = fibonacci_directions(source.ray_count);
  std::vector<Ray> rays(dirs.size());
  for (std::size_t i = 0; i < dirs.size(); ++i) {
    rays[i].origin = source.position;
    rays[i].dir = dirs[i];
  }
  return rays;
}

/// step (tracer.hpp:43-45, tracer.cpp:19-68): advance every live ray by one
/// wall interaction on the GPU, in place, and return this iteration's
/// receiver captures in ray order.  A null tree selects the brute-force
/// nearest-face search (over a device copy of `mesh`).  max_range <= 0
/// resolves to (r/2)*sqrt(rays.size()) as in the reference's bench.
inline std::vector<Capture> step(std::vector<Ray>& rays, const TriangleMesh& mesh, const AccelTree* tree,
                                 const Receiver& receiver, const TraceConfig& config) {
  std::optional<AccelTree> own;
  if (tree == nullptr) own.emplace(build_tree(mesh));
  const AccelTree& t = tree ? *tree : *own;
  const std::size_t n = rays.size();
  std::size_t cap = 1;
  for (const Ray& r : rays) cap = std::max(cap, r.face_history.size() + 1);
  std::vector<double> o(3 * n), d(3 * n), m(kNumBands * n), path(n);
  std::vector<int32_t> alive(n), hist(n * cap, -1), nh(n);
  for (std::size_t i = 0; i < n; ++i) {
    const Ray& r = rays[i];
    for (int k = 0; k < 3; ++k) o[3 * i + k] = r.origin[k], d[3 * i + k] = r.dir[k];
    for (int b = 0; b < kNumBands; ++b) m[kNumBands * i + b] = r.band_multiplier[b];
    path[i] = r.path_length;
    alive[i] = r.alive ? 1 : 0;
    nh[i] = static_cast<int32_t>(r.face_history.size());
    std::copy(r.face_history.begin(), r.face_history.end(), hist.begin() + i * cap);
  }
  rr_receiver rc{{receiver.center.x, receiver.center.y, receiver.center.z}, receiver.radius};
  rr_trace_config cfg{};
  cfg.max_iterations = config.max_iterations;
  cfg.speed_of_sound = config.speed_of_sound;
  cfg.max_range = config.max_range;
  rr_trace_result* h = nullptr;
  detail::check(rr_step(t.handle(), static_cast<int64_t>(n), o.data(), d.data(), m.data(), path.data(), alive.data(),
                        hist.data(), nh.data(), static_cast<int32_t>(cap), &rc, &cfg, tree ? 0 : 1, &h));
  detail::TraceHandle guard(h);
  for (std::size_t i = 0; i < n; ++i) {
    Ray& r = rays[i];
    r.origin = {o[3 * i], o[3 * i + 1], o[3 * i + 2]};
    r.dir = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
    for (int b = 0; b < kNumBands; ++b) r.band_multiplier[b] = m[kNumBands * i + b];
    r.path_length = path[i];
    r.alive = alive[i] != 0;
    r.face_history.assign(hist.begin() + i * cap, hist.begin() + i * cap + nh[i]);
  }
  rr_trace_stats st{};
  detail::check(rr_trace_stats_get(h, &st));
  const std::size_t nc = static_cast<std::size_t>(st.n_captures);
  std::vector<int32_t> ray(nc), ch(std::max<int64_t>(st.total_history, 1));
  std::vector<double> point(3 * nc), dir(3 * nc), cpath(nc), mult(kNumBands * nc);
  std::vector<int64_t> off(nc + 1);
  detail::check(rr_trace_captures(h, nullptr, ray.data(), point.data(), dir.data(), cpath.data(), mult.data(),
                                  off.data(), ch.data()));
  std::vector<Capture> caps(nc);
  for (std::size_t i = 0; i < nc; ++i) {
    Capture& c = caps[i];
    c.ray_index = ray[i];
    c.point = {point[3 * i], point[3 * i + 1], point[3 * i + 2]};
    c.incoming_dir = {dir[3 * i], dir[3 * i + 1], dir[3 * i + 2]};
    c.path_length = cpath[i];
    for (int b = 0; b < kNumBands; ++b) c.band_multiplier[b] = mult[kNumBands * i + b];
    c.face_history.assign(ch.begin() + off[i], ch.begin() + off[i + 1]);
  }
  return caps;
}

// ------------------------------------------------------------------ air (air_absorption.hpp)
struct AirModel {
  double temperature_c = 20.0;
  double relative_humidity = 50.0;
  double pressure_kpa = 101.325;
  bool enabled = true;
};

/// AirModel::validate (air_absorption.cpp:8-19).
inline void validate(const AirModel& air) {
  rr_air a{air.enabled ? 1 : 0, air.temperature_c, air.relative_humidity, air.pressure_kpa};
  detail::check(rr_air_validate(&a));
}

/// air_alpha_db_per_m (air_absorption.cpp:21-53): ISO 9613-1, dB/m.
inline double air_alpha_db_per_m(const AirModel& air, double frequency_hz) {
  rr_air a{air.enabled ? 1 : 0, air.temperature_c, air.relative_humidity, air.pressure_kpa};
  double out = 0.0;
  detail::check(rr_air_alpha_db_per_m(&a, frequency_hz, &out));
  return out;
}

/// air_beta_bands (air_absorption.hpp:35): energy attenuation per metre.
inline BandArray air_beta_bands(const AirModel& air) {
  rr_air a{air.enabled ? 1 : 0, air.temperature_c, air.relative_humidity, air.pressure_kpa};
  BandArray out{};
  detail::check(rr_air_beta_bands(&a, out.data()));
  return out;
}

// ------------------------------------------------------------------ image sources (image_sources.hpp)
struct ImageSource {
  Vec3 position;
  double distance = 0.0;
  BandArray band_energy{};
  BandArray band_multiplier = band_ones();
  int ray_count = 0;
  int order = 0;
  std::vector<int> face_path;
  std::optional<Vec3> projection;
};

struct ClusterOptions {
  double tol_scale = 1e-6;
  bool merge_coplanar = false;
};

/// retro_propagate (image_sources.hpp:34): point - path * dir.
inline Vec3 retro_propagate(const Capture& c) {
  return {c.point.x - c.path_length * c.incoming_dir.x, c.point.y - c.path_length * c.incoming_dir.y,
          c.point.z - c.path_length * c.incoming_dir.z};
}

/// build_image_sources (image_sources.hpp:58-61): cluster + attach_energy +
/// project on the GPU, sorted by (order, distance, face path).
namespace detail {
// host copy of a device image set (ImageSource list, image_sources.hpp:14-23)
inline std::vector<ImageSource> images_from(rr_images* im) {
  int64_t ni = 0, tp = 0;
  check(rr_images_info(im, &ni, &tp));
  const std::size_t m = static_cast<std::size_t>(ni);
  Layout L;
  const std::size_t o_pos = L.add<double>(3 * m), o_dist = L.add<double>(m), o_en = L.add<double>(kNumBands * m),
                    o_mu = L.add<double>(kNumBands * m), o_proj = L.add<double>(3 * m), o_cnt = L.add<int32_t>(m),
                    o_order = L.add<int32_t>(m), o_hp = L.add<int32_t>(m),
                    o_pth = L.add<int32_t>(std::max<int64_t>(tp, 1)), o_poff = L.add<int64_t>(m + 1);
  char* base = staging().get(L.bytes);
  double *pos = at<double>(base, o_pos), *dist = at<double>(base, o_dist), *en = at<double>(base, o_en),
         *mu = at<double>(base, o_mu), *proj = at<double>(base, o_proj);
  int32_t *cnt = at<int32_t>(base, o_cnt), *order = at<int32_t>(base, o_order), *hp = at<int32_t>(base, o_hp),
          *pth = at<int32_t>(base, o_pth);
  int64_t* poff = at<int64_t>(base, o_poff);
  check(rr_images_get(im, pos, dist, en, mu, cnt, order, hp, proj, poff, pth));
  std::vector<ImageSource> out;
  reserve_huge(out, m);
  out.resize(m);
  parallel_for(m, [&](std::size_t i) {
    ImageSource& s = out[i];
    s.position = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    s.distance = dist[i];
    for (int b = 0; b < kNumBands; ++b) {
      s.band_energy[b] = en[kNumBands * i + b];
      s.band_multiplier[b] = mu[kNumBands * i + b];
    }
    s.ray_count = cnt[i];
    s.order = order[i];
    s.face_path.assign(pth + poff[i], pth + poff[i + 1]);
    if (hp[i]) s.projection = Vec3{proj[3 * i], proj[3 * i + 1], proj[3 * i + 2]};
  });
  return out;
}
}  // namespace detail

inline std::vector<ImageSource> build_image_sources(const std::vector<Capture>& captures, int total_rays,
                                                    const AirModel& air, const Vec3& receiver_center,
                                                    const TriangleMesh& /*mesh*/, const AccelTree& tree,
                                                    const ClusterOptions& options = {}) {
  // the captures as flat arrays in the staging buffer: history offsets by a
  // serial prefix sum, then every record on the host threads
  const std::size_t n = captures.size();
  std::vector<int64_t> off(n + 1, 0);
  for (std::size_t i = 0; i < n; ++i) off[i + 1] = off[i] + static_cast<int64_t>(captures[i].face_history.size());
  detail::Layout L;
  const std::size_t o_ray = L.add<int32_t>(n), o_pt = L.add<double>(3 * n), o_dir = L.add<double>(3 * n),
                    o_path = L.add<double>(n), o_mult = L.add<double>(kNumBands * n),
                    o_hist = L.add<int32_t>(std::max<int64_t>(off[n], 1));
  char* base = detail::staging().get(L.bytes);
  int32_t *ray = detail::at<int32_t>(base, o_ray), *hist = detail::at<int32_t>(base, o_hist);
  double *point = detail::at<double>(base, o_pt), *dir = detail::at<double>(base, o_dir),
         *path = detail::at<double>(base, o_path), *mult = detail::at<double>(base, o_mult);
  hist[0] = 0;
  detail::parallel_for(n, [&](std::size_t i) {
    const Capture& c = captures[i];
    ray[i] = c.ray_index;
    for (int k = 0; k < 3; ++k) {
      point[3 * i + k] = c.point[k];
      dir[3 * i + k] = c.incoming_dir[k];
    }
    path[i] = c.path_length;
    for (int b = 0; b < kNumBands; ++b) mult[kNumBands * i + b] = c.band_multiplier[b];
    std::copy(c.face_history.begin(), c.face_history.end(), hist + off[i]);
  });
  rr_receiver rc{{receiver_center.x, receiver_center.y, receiver_center.z}, 1.0};
  rr_trace_result* h = nullptr;
  detail::check(rr_captures_import(tree.handle(), static_cast<int64_t>(n), nullptr, ray, point, dir, path, mult,
                                   off.data(), hist, &rc, 1, &h));
  detail::TraceHandle guard(h);
  rr_air a{air.enabled ? 1 : 0, air.temperature_c, air.relative_humidity, air.pressure_kpa};
  rr_cluster_options o{options.tol_scale, options.merge_coplanar ? 1 : 0};
  rr_images* im = nullptr;
  detail::check(rr_build_image_sources(h, 0, total_rays, &a, &o, &im));
  std::unique_ptr<rr_images, void (*)(rr_images*)> img(im, [](rr_images* p) { rr_images_destroy(p); });
  return detail::images_from(im);
}

// ------------------------------------------------------------------ RIR (rir.hpp)
struct PulseEvent {
  double time_s = 0.0;
  double amplitude = 0.0;
};

struct BandPulseTrain {
  int band = 0;
  std::vector<PulseEvent> events;
};

using PulseTrains = std::array<BandPulseTrain, kNumBands>;

struct RoomImpulseResponse {
  double sample_rate = 44100.0;
  std::vector<double> samples;                           // broadband
  PulseTrains band_trains;
  std::array<std::vector<double>, kNumBands> band_samples;  // per-band responses (extension)
};

/// build_pulse_trains (rir.cpp:9-30): one event per image per band at
/// t = d / c with amplitude sqrt(E), each train sorted by (time, amplitude).
namespace detail {
// the 8 sorted trains of n events each at [off[b], off[b+1]) of t / a
// (rr_pulse_trains, rr_images_pulse_trains) as PulseTrains, one band per thread
inline PulseTrains trains_unpack(int64_t n, const int64_t* off, const double* t, const double* a) {
  PulseTrains trains;
  parallel_for(
      kNumBands,
      [&](std::size_t b) {
        trains[b].band = static_cast<int>(b);
        auto& ev = trains[b].events;
        reserve_huge(ev, static_cast<std::size_t>(n));
        ev.resize(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) ev[i] = {t[off[b] + i], a[off[b] + i]};
      },
      0);
  return trains;
}

// the trains' events as flat arrays (band b at [off[b], off[b+1])) in the
// staging buffer, one band per thread; `extra_doubles` more doubles are
// reserved after them (returned through *extra)
struct PackedTrains {
  std::array<int64_t, kNumBands + 1> off{};
  double *t = nullptr, *a = nullptr, *extra = nullptr;
};
inline PackedTrains pack_trains(const PulseTrains& trains, std::size_t extra_doubles = 0) {
  PackedTrains p;
  for (int b = 0; b < kNumBands; ++b) p.off[b + 1] = p.off[b] + static_cast<int64_t>(trains[b].events.size());
  const std::size_t total = static_cast<std::size_t>(p.off[kNumBands]);
  Layout L;
  const std::size_t o_t = L.add<double>(std::max<std::size_t>(total, 1)),
                    o_a = L.add<double>(std::max<std::size_t>(total, 1)), o_x = L.add<double>(extra_doubles);
  char* base = staging().get(L.bytes);
  p.t = at<double>(base, o_t);
  p.a = at<double>(base, o_a);
  p.extra = at<double>(base, o_x);
  parallel_for(
      kNumBands,
      [&](std::size_t b) {
        const auto& ev = trains[b].events;
        for (std::size_t i = 0; i < ev.size(); ++i) {
          p.t[p.off[b] + i] = ev[i].time_s;
          p.a[p.off[b] + i] = ev[i].amplitude;
        }
      },
      0);
  return p;
}
}  // namespace detail

/// build_pulse_trains (rir.cpp:9-30): t = d / c and sqrt(E_b) per image and
/// band, sorted by (time, amplitude) on the device (rr_pulse_trains).
inline PulseTrains build_pulse_trains(const std::vector<ImageSource>& images, double speed_of_sound) {
  if (speed_of_sound <= 0.0) throw std::invalid_argument("speed of sound must be > 0");
  const std::size_t n = images.size();
  detail::Layout L;
  const std::size_t o_d = L.add<double>(std::max<std::size_t>(n, 1)),
                    o_e = L.add<double>(kNumBands * std::max<std::size_t>(n, 1)), o_off = L.add<int64_t>(kNumBands + 1),
                    o_t = L.add<double>(kNumBands * std::max<std::size_t>(n, 1)),
                    o_a = L.add<double>(kNumBands * std::max<std::size_t>(n, 1));
  char* base = detail::staging().get(L.bytes);
  double *dist = detail::at<double>(base, o_d), *en = detail::at<double>(base, o_e);
  detail::parallel_for(n, [&](std::size_t i) {
    dist[i] = images[i].distance;
    for (int b = 0; b < kNumBands; ++b) en[kNumBands * i + b] = images[i].band_energy[b];
  });
  int64_t* off = detail::at<int64_t>(base, o_off);
  double *t = detail::at<double>(base, o_t), *a = detail::at<double>(base, o_a);
  detail::check(rr_pulse_trains(Device::get(0).handle(), static_cast<int64_t>(n), dist, en, speed_of_sound, off, t, a));
  return detail::trains_unpack(static_cast<int64_t>(n), off, t, a);
}

/// design_band_filter (rir.cpp:32-58), `taps` taps (reference: 1023).
inline std::vector<double> design_band_filter(int band, double sample_rate, int taps = kBandFilterTaps) {
  std::vector<double> k(static_cast<std::size_t>(std::max(taps, 0)));
  detail::check(rr_band_filter(band, sample_rate, taps, k.data()));
  return k;
}

/// synthesize (rir.cpp:60-96) on the GPU: pulse histograms at
/// lround(t*fs), 8 FIR band filters, broadband sum; length
/// llround(t_last*fs) + delay + 1 as in the reference.
inline RoomImpulseResponse synthesize(const PulseTrains& trains, double sample_rate, int taps = kBandFilterTaps) {
  RoomImpulseResponse rir;
  rir.sample_rate = sample_rate;
  // per band (one thread each): the copy into rir.band_trains, the latest
  // event and the t >= 0 check
  std::array<double, kNumBands> last{};
  std::array<int, kNumBands> negative{};
  detail::parallel_for(
      kNumBands,
      [&](std::size_t b) {
        rir.band_trains[b].band = trains[b].band;
        detail::reserve_huge(rir.band_trains[b].events, trains[b].events.size());
        rir.band_trains[b].events = trains[b].events;
        double m = 0.0;
        for (const PulseEvent& e : trains[b].events) {
          if (e.time_s < 0.0) negative[b] = 1;
          m = std::max(m, e.time_s);
        }
        last[b] = m;
      },
      0);
  for (int b = 0; b < kNumBands; ++b)
    if (negative[b]) throw std::invalid_argument("pulse events cannot precede t = 0");
  std::size_t total = 0;
  for (const auto& tr : trains) total += tr.events.size();
  if (total == 0) return rir;
  const double t_last = *std::max_element(last.begin(), last.end());
  const int64_t length = static_cast<int64_t>(std::llround(t_last * sample_rate)) + (taps - 1) / 2 + 1;
  const detail::PackedTrains p = detail::pack_trains(trains, static_cast<std::size_t>((kNumBands + 1) * length));
  double *band = p.extra, *sum = p.extra + kNumBands * length;
  detail::check(rr_synthesize_trains(Device::get(0).handle(), p.off.data(), p.t, p.a, sample_rate, taps, length, band,
                                     sum));
  rir.samples.assign(sum, sum + length);
  detail::parallel_for(
      kNumBands, [&](std::size_t b) { rir.band_samples[b].assign(band + b * length, band + (b + 1) * length); }, 0);
  return rir;
}

// ------------------------------------------------------------------ metrics (metrics.hpp)
struct MetricValue {
  double value = 0.0;
  bool reliable = false;
};

struct PerceptiveFactors {
  MetricValue edt_s, t30_s, spl_db, c80_db, d50_pct, ts_ms;
};

struct BandFactors {
  std::array<PerceptiveFactors, kNumBands> bands;
  PerceptiveFactors mid;  // 500 Hz / 1 kHz average
};

namespace detail {
inline PerceptiveFactors to_factors(const rr_factors& f) {
  auto m = [](const rr_metric& x) { return MetricValue{x.value, x.reliable != 0}; };
  return PerceptiveFactors{m(f.edt_s), m(f.t30_s), m(f.spl_db), m(f.c80_db), m(f.d50_pct), m(f.ts_ms)};
}
}  // namespace detail

/// factors(const PulseTrains&) (metrics.hpp:56-60) on the GPU.
inline BandFactors factors(const PulseTrains& trains) {
  const detail::PackedTrains p = detail::pack_trains(trains);
  rr_factors out[kNumBands + 1];
  detail::check(rr_band_factors(Device::get(0).handle(), p.off.data(), p.t, p.a, out));
  BandFactors bf;
  for (int b = 0; b < kNumBands; ++b) bf.bands[b] = detail::to_factors(out[b]);
  bf.mid = detail::to_factors(out[kNumBands]);
  return bf;
}

namespace detail {
// build_pulse_trains of a device image set, sorted on the device (no host sort)
inline PulseTrains trains_from(rr_images* im, double speed_of_sound) {
  if (speed_of_sound <= 0.0) throw std::invalid_argument("speed of sound must be > 0");
  int64_t n = 0, tp = 0;
  check(rr_images_info(im, &n, &tp));
  Layout L;
  const std::size_t o_off = L.add<int64_t>(kNumBands + 1), o_t = L.add<double>(kNumBands * std::max<int64_t>(n, 1)),
                    o_a = L.add<double>(kNumBands * std::max<int64_t>(n, 1));
  char* base = staging().get(L.bytes);
  const int64_t* off = at<int64_t>(base, o_off);
  const double *t = at<double>(base, o_t), *a = at<double>(base, o_a);
  check(rr_images_pulse_trains(im, speed_of_sound, at<int64_t>(base, o_off), at<double>(base, o_t),
                               at<double>(base, o_a)));
  return trains_unpack(n, off, t, a);
}

// synthesize(trains) of a device image set (the trains' events are the images')
inline RoomImpulseResponse rir_from(rr_images* im, const PulseTrains& trains, double speed_of_sound,
                                    double sample_rate, int taps = kBandFilterTaps) {
  RoomImpulseResponse rir;
  rir.sample_rate = sample_rate;
  int64_t length = 0;
  check(rr_images_synthesize(im, speed_of_sound, sample_rate, taps, &length, nullptr, nullptr));
  double* band = nullptr;
  if (length > 0) {
    Layout L;
    const std::size_t o_band = L.add<double>(kNumBands * length), o_sum = L.add<double>(length);
    char* base = staging().get(L.bytes);
    band = at<double>(base, o_band);
    double* sum = at<double>(base, o_sum);
    check(rr_images_synthesize(im, speed_of_sound, sample_rate, taps, &length, band, sum));
    rir.samples.assign(sum, sum + length);
  }
  parallel_for(  // one band per thread: the band's copy of the trains and its filtered samples
      kNumBands,
      [&](std::size_t b) {
        rir.band_trains[b].band = trains[b].band;
        reserve_huge(rir.band_trains[b].events, trains[b].events.size());
        rir.band_trains[b].events = trains[b].events;
        if (band) rir.band_samples[b].assign(band + b * length, band + (b + 1) * length);
      },
      0);
  return rir;
}

inline BandFactors factors_from(rr_images* im, double speed_of_sound) {
  rr_factors out[kNumBands + 1];
  check(rr_images_factors(im, speed_of_sound, out));
  BandFactors bf;
  for (int b = 0; b < kNumBands; ++b) bf.bands[b] = to_factors(out[b]);
  bf.mid = to_factors(out[kNumBands]);
  return bf;
}
}  // namespace detail

// ------------------------------------------------------------------ shoebox lattice (shoebox.hpp)
enum BoxWall { kWallX0 = 0, kWallX1, kWallY0, kWallY1, kWallZ0, kWallZ1 };  // shoebox.hpp:13

/// Rectangular room [0,Lx] x [0,Ly] x [0,Lz], one material per wall
/// (shoebox.hpp:16-22).
struct ShoeBox {
  Vec3 dimensions{1.0, 1.0, 1.0};
  std::array<Material, 6> walls{};
  void validate() const {
    for (int a = 0; a < 3; ++a)
      if (dimensions[a] <= 0.0) throw std::invalid_argument("box dimensions must be > 0");
  }
  bool inside(const Vec3& p) const {
    for (int a = 0; a < 3; ++a)
      if (!(p[a] > 0.0) || !(p[a] < dimensions[a])) return false;
    return true;
  }
};

/// OracleImageSource (shoebox.hpp:25-31).
struct OracleImageSource {
  Vec3 position{};
  double distance = 0.0;
  int order = 0;
  std::array<int, 6> wall_hits{};
  BandArray band_energy{};
};

/// enumerate_images (shoebox.hpp:38-43) on the GPU: every mirror-lattice
/// image within max_distance of the receiver, sorted by (distance, cell).
inline std::vector<OracleImageSource> enumerate_images(const ShoeBox& box, const Vec3& source, const Vec3& receiver,
                                                       double max_distance, double receiver_radius,
                                                       const AirModel& air) {
  const double dims[3] = {box.dimensions.x, box.dimensions.y, box.dimensions.z};
  double alpha[6 * kNumBands];
  for (int w = 0; w < 6; ++w)
    for (int b = 0; b < kNumBands; ++b) alpha[kNumBands * w + b] = box.walls[w].absorption[b];
  const double s[3] = {source.x, source.y, source.z}, r[3] = {receiver.x, receiver.y, receiver.z};
  rr_air a{air.enabled ? 1 : 0, air.temperature_c, air.relative_humidity, air.pressure_kpa};
  rr_lattice* h = nullptr;
  detail::check(rr_shoebox_images(Device::get(0).handle(), dims, alpha, s, r, max_distance, receiver_radius, &a, &h));
  std::unique_ptr<rr_lattice, rr_status (*)(rr_lattice*)> guard(h, rr_lattice_destroy);
  int64_t n = 0;
  detail::check(rr_lattice_info(h, &n));
  std::vector<double> pos(3 * n), dist(n), energy(kNumBands * n);
  std::vector<int32_t> order(n), hits(6 * n);
  detail::check(rr_lattice_get(h, pos.data(), dist.data(), order.data(), hits.data(), energy.data()));
  std::vector<OracleImageSource> out(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    OracleImageSource& o = out[i];
    o.position = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    o.distance = dist[i];
    o.order = order[i];
    for (int w = 0; w < 6; ++w) o.wall_hits[w] = hits[6 * i + w];
    for (int b = 0; b < kNumBands; ++b) o.band_energy[b] = energy[kNumBands * i + b];
  }
  return out;
}

/// MatchedImage / MatchReport (shoebox.hpp:47-66).
struct MatchedImage {
  int oracle_index = -1;
  std::vector<int> traced_indices;
  double position_error = 0.0;
  int order = 0;
  BandArray energy_delta_db{};
};

struct MatchReport {
  std::vector<MatchedImage> matched;
  std::vector<int> unmatched_oracle;  // beams the tracer missed
  std::vector<int> unmatched_traced;  // should be empty
  double max_position_error = 0.0;
  BandArray rms_energy_error_db{};
  double pos_tol = 0.0;
  double energy_tol_db = 0.0;
  bool energy_within(double tol_db, int max_order) const {  // shoebox.cpp:118-124
    for (const MatchedImage& m : matched) {
      if (m.order > max_order) continue;
      for (double d : m.energy_delta_db)
        if (std::abs(d) > tol_db) return false;
    }
    return true;
  }
};

/// compare (shoebox.hpp:67-70) on the GPU: cells hashed at 2 * pos_tol
/// instead of the reference's O(T * O) scan; same matches, same tie rule.
inline MatchReport compare(const std::vector<OracleImageSource>& oracle, const std::vector<ImageSource>& traced,
                           double pos_tol, double energy_tol_db) {
  const std::size_t no = oracle.size(), nt = traced.size();
  std::vector<double> opos(3 * no), oen(kNumBands * no), tpos(3 * nt), ten(kNumBands * nt);
  std::vector<int32_t> oord(no);
  for (std::size_t i = 0; i < no; ++i) {
    for (int k = 0; k < 3; ++k) opos[3 * i + k] = oracle[i].position[k];
    for (int b = 0; b < kNumBands; ++b) oen[kNumBands * i + b] = oracle[i].band_energy[b];
    oord[i] = oracle[i].order;
  }
  for (std::size_t i = 0; i < nt; ++i) {
    for (int k = 0; k < 3; ++k) tpos[3 * i + k] = traced[i].position[k];
    for (int b = 0; b < kNumBands; ++b) ten[kNumBands * i + b] = traced[i].band_energy[b];
  }
  rr_match* h = nullptr;
  detail::check(rr_shoebox_compare(Device::get(0).handle(), static_cast<int64_t>(no), opos.data(), oen.data(),
                                   oord.data(), static_cast<int64_t>(nt), tpos.data(), ten.data(), pos_tol,
                                   energy_tol_db, &h));
  std::unique_ptr<rr_match, rr_status (*)(rr_match*)> guard(h, rr_match_destroy);
  int64_t g = 0, nm = 0, nuo = 0, nut = 0;
  MatchReport r;
  r.pos_tol = pos_tol;
  r.energy_tol_db = energy_tol_db;
  detail::check(rr_match_info(h, &g, &nm, &nuo, &nut, &r.max_position_error, r.rms_energy_error_db.data()));
  std::vector<int32_t> oi(g), ord(g), mem(nm);
  std::vector<double> err(g), dd(kNumBands * g);
  std::vector<int64_t> off(g + 1);
  r.unmatched_oracle.resize(nuo);
  r.unmatched_traced.resize(nut);
  detail::check(rr_match_get(h, oi.data(), err.data(), ord.data(), dd.data(), off.data(), mem.data(),
                             r.unmatched_oracle.data(), r.unmatched_traced.data()));
  r.matched.resize(g);
  for (int64_t i = 0; i < g; ++i) {
    MatchedImage& m = r.matched[i];
    m.oracle_index = oi[i];
    m.position_error = err[i];
    m.order = ord[i];
    for (int b = 0; b < kNumBands; ++b) m.energy_delta_db[b] = dd[kNumBands * i + b];
    m.traced_indices.assign(mem.begin() + off[i], mem.begin() + off[i + 1]);
  }
  return r;
}

}  // namespace roomray_b200

#endif  // ROOMRAY_B200_HPP
