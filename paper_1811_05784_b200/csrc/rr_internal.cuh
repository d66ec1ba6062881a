// Internal declarations of the roomray_b200 library (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <atomic>

#include <cstdint>
#include <ctime>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "roomray_b200.h"

namespace rr {

constexpr int kBands = RR_NUM_BANDS;

struct Error : std::runtime_error {
  rr_status code;
  Error(rr_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void invalid(const std::string& m) {
  throw Error(RR_INVALID_ARGUMENT, m);
}

#define RR_CUDA(x)                                                        \
  do {                                                                    \
    cudaError_t rr_e_ = (x);                                              \
    if (rr_e_ != cudaSuccess)                                             \
      throw ::rr::Error(RR_CUDA, std::string(#x) + ": " +                 \
                                     cudaGetErrorString(rr_e_));          \
  } while (0)

#define RR_LAUNCH_CHECK() RR_CUDA(cudaGetLastError())

// Device-side bounds checks of the checked build (libroomray_b200_checked.so,
// -DRR_CHECKED; tests/test_gpu_checked.py): stack depths, node / face /
// history indices.  A failed check prints and traps (the launch fails with
// an error instead of touching memory it must not).  Compiled out otherwise.
#ifdef RR_CHECKED
#define RR_DCHECK(c)                                                               \
  do {                                                                             \
    if (!(c)) {                                                                    \
      printf("RR_DCHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);              \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define RR_DCHECK(c) \
  do {               \
  } while (0)
#endif

// Device buffer, stream-ordered allocation on the owning context's stream.
// RR_ALLOC_TRACE=1 (development): report stream-ordered allocation calls
// that block the host for more than 2 ms
inline bool alloc_trace() {
  static const bool on = std::getenv("RR_ALLOC_TRACE") != nullptr;
  return on;
}
inline double wall_ms() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return 1e3 * static_cast<double>(ts.tv_sec) + 1e-6 * static_cast<double>(ts.tv_nsec);
}
inline void slow_call(const char* what, size_t bytes, double ms) {
  if (ms > 2.0) std::fprintf(stderr, "[rr alloc] %s %zu bytes blocked %.1f ms\n", what, bytes, ms);
}

// Block cache of the context streams (rr_api.cu).  A released block goes
// to its stream's cache instead of cudaFreeAsync and a later allocation on
// the same stream takes it back: everything that touches the block is
// ordered on that one stream, exactly as with cudaFreeAsync ->
// cudaMallocAsync, but with no driver call.  The driver's pool does the same
// in principle, yet on the GPU boxes a steady-state C5 pipeline step saw
// 2-300 ms host stalls inside cudaMallocAsync of sizes the pool had just
// freed (gpurun_out/alloc_trace.log), which the end-to-end time pays.
// Only streams registered by rr_ctx_create are cached; RR_BLOCK_CACHE_MB
// caps the cached bytes (default 16384; 0 turns the cache off).
void* cache_take(size_t bytes, cudaStream_t s, size_t* got);
bool cache_give(void* p, size_t bytes, cudaStream_t s);
void cache_register(cudaStream_t s);
void cache_drop(cudaStream_t s);  // free the stream's blocks (before destroying it)
void cache_trim();                // free every cached block (allocation failure)

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  size_t cap = 0;  // bytes of the block (>= sizeof(T) * n when it came from the cache)
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), cap(o.cap), s(o.s) { o.p = nullptr; o.n = 0; o.cap = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; cap = o.cap; s = o.s;
      o.p = nullptr; o.n = 0; o.cap = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    if (count) {
      const size_t want = sizeof(T) * count;
      p = static_cast<T*>(cache_take(want, stream, &cap));
      if (p) return;
      const double t0 = alloc_trace() ? wall_ms() : 0.0;
      cudaError_t e = cudaMallocAsync(&p, want, stream);
      if (e == cudaErrorMemoryAllocation) {  // cached blocks may hold the memory
        cudaGetLastError();
        cache_trim();
        e = cudaMallocAsync(&p, want, stream);
      }
      if (e != cudaSuccess) {
        p = nullptr;
        n = 0;
        RR_CUDA(e);
      }
      cap = want;
      if (alloc_trace()) slow_call("cudaMallocAsync", want, wall_ms() - t0);
    }
  }
  void release() {
    if (p && !cache_give(p, cap, s)) {
      const double t0 = alloc_trace() ? wall_ms() : 0.0;
      cudaFreeAsync(p, s);
      if (alloc_trace()) slow_call("cudaFreeAsync", cap, wall_ms() - t0);
    }
    p = nullptr;
    n = 0;
    cap = 0;
  }
  size_t bytes() const { return sizeof(T) * n; }
};

// Stage timing for development (RR_TIMING=1 prints CUDA-event intervals).
struct StageTimer {
  cudaStream_t s;
  bool on, stats;  // RR_TIMING set: stage events; RR_TIMING=2: also host-side statistics (slow)
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  std::vector<double> host_ms;  // host wall clock at each mark
  explicit StageTimer(cudaStream_t st)
      : s(st), on(std::getenv("RR_TIMING") != nullptr), stats(on && std::getenv("RR_TIMING")[0] == '2') {
    mark("start");
  }
  static double now_ms() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return 1e3 * static_cast<double>(ts.tv_sec) + 1e-6 * static_cast<double>(ts.tv_nsec);
  }
  void mark(const char* name) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.emplace_back(name, e);
    host_ms.push_back(now_ms());
  }
  ~StageTimer() {
    if (!on) return;
    cudaEventSynchronize(ev.back().second);
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
      std::fprintf(stderr, "[rr timing] %-24s %9.3f ms (host enqueue %8.3f ms)\n", ev[i].first, ms,
                   host_ms[i] - host_ms[i - 1]);
    }
    for (auto& p : ev) cudaEventDestroy(p.second);
  }
};

// Reference-layout node (TreeNode accel_tree.hpp:15-22), same bytes as
// rr_tree_node.
struct RefNode {
  double lo[3], hi[3];
  int32_t left, right, face, pad;
};
static_assert(sizeof(RefNode) == sizeof(rr_tree_node), "layout");

// Traversal node: the two children's conservative fp32 boxes + refs, 64 B
// (one 128-B line holds two nodes).  ref >= 0: internal node index;
// ref < 0: leaf, face = ~ref.
//   a = (L.lo.x, L.hi.x, L.lo.y, L.hi.y)  b = (L.lo.z, L.hi.z, R.lo.x, R.hi.x)
//   c = (R.lo.y, R.hi.y, R.lo.z, R.hi.z)  d = (L.ref, R.ref, -, -)
struct __align__(16) TNode {
  float4 a, b, c;
  int4 d;
};

// 4-wide traversal node collapsed from the reference tree (the even-depth
// internal nodes; children = the grandchildren, or a child leaf): one 128-B
// line, eight independent 16-B loads.  Components are SoA over the 4 slots.
// child >= 0: QNode index; child < 0: leaf, face = ~child; kEmpty: unused.
struct __align__(16) QNode {
  float4 lx, hx, ly, hy, lz, hz;
  int4 child;
  int4 pad;
};
constexpr int32_t kEmpty = static_cast<int32_t>(0x80000000);

// 8-wide compressed traversal node (rr_wide.cu), 80 B = five 16-B loads.
// Child boxes are quantized to 8 bits per plane on a per-node grid
// p + q * 2^e (p fp32, e a power-of-two exponent per axis), rounded outward
// beyond the binary node's conservative fp32 boxes (see rr_wide.cu for the
// error budget), so the filter stays a superset of the fp64 reference's.
//   h  = (px, py, pz, bits: ex | ey << 8 | ez << 16 | imask << 24)
//        e: the biased fp32 exponent of the scale; imask bit k: slot k internal
//   m  = (child_base, tri_base, plane, valid | pair << 8 | cull << 16)
//        internal slot k -> node child_base + popc(imask & ((1 << k) - 1));
//        leaf slot k -> its 1 (or 2, pair bit) faces at tri_base + (faces of
//        the leaf slots before k); cull bit k: slot k's subtree lies in
//        axis-aligned plane `plane` (coplanar-subtree cull)
//   qx = (lo bytes 0-3, lo bytes 4-7, hi bytes 0-3, hi bytes 4-7) of slot k,
//   qy, qz likewise.
struct __align__(16) WNode {
  float4 h;
  int4 m;
  uint4 qx, qy, qz;
};
static_assert(sizeof(WNode) == 80, "WNode");
// leaf ref flag: ~(f | kPairBit) holds faces f and f + 1 (SAH tree, rr_geom.cuh test_leaf)
constexpr int32_t kPairBit = 1 << 30;

struct TravHeader {
  float lo[3], hi[3];  // conservative root box
  int32_t root_ref;    // internal index 0, or ~face for a one-face mesh
  int32_t K;           // nodes [0, K) are the BFS-ordered top levels
  float eps;           // absolute box expansion (metres)
  int32_t depth;
  int32_t root4;       // QNode root (0) or ~face for a one-face mesh
  int32_t K4;          // QNodes [0, K4) are cached in shared memory
};

// Per-face fp64 data for Moller-Trumbore: a, b-a, c-a (geometry.cpp:80-82),
// padded to 80 B for 16-B vector loads.
struct __align__(16) FaceTri {
  double ax, ay, az, e1x, e1y, e1z, e2x, e2y, e2z, pad;
};

}  // namespace rr

// Handles are reference counted: a scene holds its context, a trace result
// or image set holds its scene, so destroying handles in any order (e.g. a
// garbage collector's) never frees memory still reachable from a live one.
struct rr_ctx {
  int refs = 1;
  int device = 0;
  cudaStream_t stream = nullptr;
  std::atomic<int64_t> launches{0};  // the scene build counts from two host threads
  int sm_count = 0;
  int64_t* pinned = nullptr;        // 64 pinned int64 slots for asynchronous read-backs
  cudaEvent_t level_ev[64] = {};    // per-level events of the SAH build
};

struct rr_scene {
  int refs = 1;
  rr_ctx* ctx = nullptr;
  int64_t nv = 0, nf = 0;
  int32_t nmat = 0;
  rr::DevBuf<double> verts;       // nv*3
  rr::DevBuf<int32_t> tris;       // nf*4
  rr::DevBuf<double> oma;         // nmat*8 : 1 - alpha
  rr::DevBuf<rr::FaceTri> tri;    // nf
  rr::DevBuf<float4> tri32;       // nf*3: fp32 a (w = face bits), b-a, c-a (48 B leaf record)
  rr::DevBuf<double> normal;      // nf*3
  rr::DevBuf<int32_t> mat;        // nf
  rr::DevBuf<int32_t> face_plane; // nf: axis-aligned plane id (axis << 29 | index) or -1
  rr::DevBuf<rr::RefNode> ref;    // 2nf-1 (reference layout)
  rr::DevBuf<rr::TNode> tnodes;   // K + nf
  rr::DevBuf<rr::QNode> qnodes;   // 4-wide nodes
  rr::DevBuf<rr::TNode> snodes;   // SAH traversal tree (rr_sah.cu), nf-1 nodes, BFS order
  rr::TravHeader shdr{};          // its header (root box, root ref, eps)
  rr::DevBuf<rr::QNode> s4nodes;  // 4-wide collapse of the SAH tree (pad = slot plane ids)
  rr::DevBuf<rr::WNode> wnodes;   // 8-wide compressed collapse of the SAH tree (rr_wide.cu)
  rr::DevBuf<rr::FaceTri> wtri;   // faces in its leaf order, pad = the face id (int64 bits)
  int32_t wroot = -1;             // WNode root (0) when built
  int32_t wstack = 0;             // bound on the traversal stack occupancy over the 8-wide tree
  bool wide_ok = false;           // every grid step <= 16 (no fp32 overflow in the slab form)
  int32_t wdepth = 0;
  int32_t s4root = -1;
  int32_t sah_depth = 0;
  int64_t n_qnodes = 0;
  rr::DevBuf<rr::TravHeader> dhdr;
  rr::DevBuf<unsigned long long> plane_table;  // 3 hash tables of axis-aligned plane coordinates
  int64_t plane_T = 0;                          // slots per axis table
  bool ref_built = false;         // reference tree (ref, tnodes, qnodes, hdr) built on first use
  rr::TravHeader hdr{};
  int32_t root = -1, depth = 0, K = 0;
  double lo[3]{}, hi[3]{};        // TriangleMesh::bounds (geometry.cpp:41-45)
  float build_ms = 0.f;
  double caps_per_ray = 0.0;      // capture rate of the last trace (buffer sizing)
};

namespace rr {
// rr_build.cu
void build_scene_tree(rr_scene* s);
void ensure_reference_tree(rr_scene* s);
// rr_sah.cu (needs face_plane; runs on its own stream)
void build_sah_tree(rr_scene* s, cudaStream_t st);
void build_sah4(rr_scene* s);  // 4-wide collapse, on demand
// rr_wide.cu
void build_wide(rr_scene* s);  // 8-wide compressed collapse, on demand
// rr_ir.cu
void ir_bin(rr_ctx* ctx, int64_t n, const double* d_dist, const double* d_energy, double c, double fs, int64_t lh,
            double* d_hist);
void ir_filter(rr_ctx* ctx, const double* d_hist, int64_t lh, double fs, int taps, int64_t L, double* d_band_ir,
               double* d_broadband);
void ir_max_amp(rr_ctx* ctx, int64_t n, const double* d_energy, unsigned long long* d_max);
void ir_bin_fixed(rr_ctx* ctx, int64_t n, const double* d_dist, const double* d_energy, double c, double fs,
                  int64_t lh, const unsigned long long* d_max, int64_t n_scale, unsigned long long* d_acc);
void ir_unfix(rr_ctx* ctx, const unsigned long long* d_acc, int64_t total, int64_t n_scale,
              const unsigned long long* d_max, double* d_hist);
// rr_trace.cu
void nearest_hit_batch(rr_scene* s, const double* d_o, const double* d_d,
                       int64_t n, int brute, int32_t* d_face, double* d_delta,
                       double* d_point);
}  // namespace rr
