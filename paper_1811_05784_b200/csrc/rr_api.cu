// C ABI entry points (include/roomray_b200.h): argument checks, uploads,
// error mapping.  All compute runs in the kernels of rr_build.cu,
// rr_trace.cu, rr_images.cu and rr_ir.cu.
#include <functional>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "rr_trace.cuh"

// Block cache of the context streams (rr_internal.cuh DevBuf).
namespace rr {
namespace {
struct CachedBlock {
  void* p;
  size_t bytes;
  cudaStream_t s;
  uint64_t tick;  // release order (oldest evicted first)
};
struct BlockCache {
  std::mutex m;
  std::vector<CachedBlock> blocks;
  std::vector<cudaStream_t> streams;
  size_t held = 0, limit = 0;
  uint64_t tick = 0;
  BlockCache() {
    const char* e = std::getenv("RR_BLOCK_CACHE_MB");
    limit = static_cast<size_t>(e ? std::atoll(e) : 16384) << 20;
  }
  bool known(cudaStream_t s) const {
    for (cudaStream_t t : streams)
      if (t == s) return true;
    return false;
  }
};
BlockCache& cache() {
  static BlockCache* c = new BlockCache;  // never destroyed: DevBufs may outlive static destruction
  return *c;
}
}  // namespace

void* cache_take(size_t bytes, cudaStream_t s, size_t* got) {
  BlockCache& c = cache();
  if (c.limit == 0) return nullptr;
  std::lock_guard<std::mutex> g(c.m);
  // best fit among the stream's blocks of [bytes, bytes * 1.25 + 2 MB]
  const size_t hi = bytes + bytes / 4 + (size_t{2} << 20);
  size_t best = c.blocks.size();
  for (size_t i = 0; i < c.blocks.size(); ++i) {
    const CachedBlock& b = c.blocks[i];
    if (b.s == s && b.bytes >= bytes && b.bytes <= hi && (best == c.blocks.size() || b.bytes < c.blocks[best].bytes))
      best = i;
  }
  if (best == c.blocks.size()) return nullptr;
  void* p = c.blocks[best].p;
  *got = c.blocks[best].bytes;
  c.held -= *got;
  c.blocks[best] = c.blocks.back();
  c.blocks.pop_back();
  return p;
}

bool cache_give(void* p, size_t bytes, cudaStream_t s) {
  BlockCache& c = cache();
  if (c.limit == 0 || bytes > c.limit) return false;
  std::lock_guard<std::mutex> g(c.m);
  if (!c.known(s)) return false;
  while (c.held + bytes > c.limit && !c.blocks.empty()) {  // evict the oldest
    size_t o = 0;
    for (size_t i = 1; i < c.blocks.size(); ++i)
      if (c.blocks[i].tick < c.blocks[o].tick) o = i;
    cudaFreeAsync(c.blocks[o].p, c.blocks[o].s);
    c.held -= c.blocks[o].bytes;
    c.blocks[o] = c.blocks.back();
    c.blocks.pop_back();
  }
  c.blocks.push_back(CachedBlock{p, bytes, s, ++c.tick});
  c.held += bytes;
  return true;
}

void cache_register(cudaStream_t s) {
  BlockCache& c = cache();
  std::lock_guard<std::mutex> g(c.m);
  if (!c.known(s)) c.streams.push_back(s);
}

void cache_drop(cudaStream_t s) {
  BlockCache& c = cache();
  std::lock_guard<std::mutex> g(c.m);
  for (size_t i = 0; i < c.blocks.size();) {
    if (c.blocks[i].s == s) {
      cudaFreeAsync(c.blocks[i].p, s);
      c.held -= c.blocks[i].bytes;
      c.blocks[i] = c.blocks.back();
      c.blocks.pop_back();
    } else {
      ++i;
    }
  }
  for (size_t i = 0; i < c.streams.size(); ++i)
    if (c.streams[i] == s) {
      c.streams[i] = c.streams.back();
      c.streams.pop_back();
      break;
    }
}

void cache_trim() {
  BlockCache& c = cache();
  std::lock_guard<std::mutex> g(c.m);
  for (const CachedBlock& b : c.blocks) cudaFreeAsync(b.p, b.s);
  for (cudaStream_t s : c.streams) cudaStreamSynchronize(s);  // the frees reach the pool
  c.blocks.clear();
  c.held = 0;
}
}  // namespace rr

namespace {

thread_local std::string g_err;

template <typename F>
rr_status guarded(F&& f) {
  try {
    f();
    return RR_OK;
  } catch (const rr::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return RR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RR_RUNTIME;
  }
}

// TriangleMesh::validate (geometry.cpp:47-75): the reference throws at the
// first face (in index order) that fails vertex range, material range or
// area, then checks materials.  key = face*4 + kind.
__global__ void validate_faces_kernel(const double* __restrict__ v, int64_t nv, const int32_t* __restrict__ t,
                                      int64_t nf, int32_t nmat, unsigned long long* __restrict__ first) {
  int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const int32_t a = t[4 * f], b = t[4 * f + 1], c = t[4 * f + 2], m = t[4 * f + 3];
  unsigned long long key = ~0ull;
  if (a < 0 || a >= nv || b < 0 || b >= nv || c < 0 || c >= nv) {
    key = 4ull * f + 0;
  } else if (m < 0 || m >= nmat) {
    key = 4ull * f + 1;
  } else {
    using namespace rr;
    const D3 va = d3(v[3 * a], v[3 * a + 1], v[3 * a + 2]);
    const D3 e1 = d3(v[3 * b], v[3 * b + 1], v[3 * b + 2]) - va;
    const D3 e2 = d3(v[3 * c], v[3 * c + 1], v[3 * c + 2]) - va;
    const D3 n = cross(e1, e2);
    const double area = 0.5 * sqrt(dot(n, n));  // face_area geometry.cpp:22-26
    if (area <= 1e-12) key = 4ull * f + 2;
  }
  if (key != ~0ull) atomicMin(first, key);
}

// Moller-Trumbore operands and face normals (geometry.cpp:9-14, 80-82).
__global__ void face_data_kernel(const double* __restrict__ v, const int32_t* __restrict__ t, int64_t nf,
                                 rr::FaceTri* __restrict__ tri, float4* __restrict__ tri32,
                                 double* __restrict__ normal,
                                 int32_t* __restrict__ mat) {
  using namespace rr;
  int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const int32_t a = t[4 * f], b = t[4 * f + 1], c = t[4 * f + 2];
  const D3 va = d3(v[3 * a], v[3 * a + 1], v[3 * a + 2]);
  const D3 e1 = d3(v[3 * b], v[3 * b + 1], v[3 * b + 2]) - va;
  const D3 e2 = d3(v[3 * c], v[3 * c + 1], v[3 * c + 2]) - va;
  FaceTri ft;
  ft.ax = va.x; ft.ay = va.y; ft.az = va.z;
  ft.e1x = e1.x; ft.e1y = e1.y; ft.e1z = e1.z;
  ft.e2x = e2.x; ft.e2y = e2.y; ft.e2z = e2.z;
  ft.pad = 0.0;
  tri[f] = ft;
  tri32[3 * f] = make_float4(__double2float_rn(va.x), __double2float_rn(va.y), __double2float_rn(va.z),
                             __int_as_float(static_cast<int>(f)));
  tri32[3 * f + 1] = make_float4(__double2float_rn(e1.x), __double2float_rn(e1.y), __double2float_rn(e1.z), 0.f);
  tri32[3 * f + 2] = make_float4(__double2float_rn(e2.x), __double2float_rn(e2.y), __double2float_rn(e2.z), 0.f);
  D3 n = cross(e1, e2);
  const double z = dot(n, n);
  if (z > 0.0) {
    const double s = sqrt(z);
    n = d3(n.x / s, n.y / s, n.z / s);
  }
  normal[3 * f] = n.x;
  normal[3 * f + 1] = n.y;
  normal[3 * f + 2] = n.z;
  mat[f] = t[4 * f + 3];
}

void check_ptr(const void* p, const char* what) {
  if (!p) rr::invalid(std::string(what) + " must not be null");
}

}  // namespace

extern "C" {

const char* rr_last_error(void) { return g_err.c_str(); }
const char* rr_version(void) { return "roomray_b200 0.1 (sm_100a)"; }

rr_status rr_ctx_create(int device, rr_ctx** out) {
  return guarded([&] {
    check_ptr(out, "out");
    int n = 0;
    RR_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) rr::invalid("device index out of range");
    RR_CUDA(cudaSetDevice(device));
    auto c = std::make_unique<rr_ctx>();
    c->device = device;
    RR_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    rr::cache_register(c->stream);
    // keep freed stream-ordered allocations cached in the pool, so the
    // per-call buffers of rr_trace & co. cost no driver round trips
    cudaMemPool_t pool;
    RR_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    RR_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    RR_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
    cudaDeviceProp prop;
    RR_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) rr::invalid("roomray_b200 needs an sm_100a (Blackwell) device");
    RR_CUDA(cudaMallocHost(&c->pinned, sizeof(int64_t) * 64));
    for (cudaEvent_t& e : c->level_ev) RR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    *out = c.release();
  });
}

namespace {
void ctx_release(rr_ctx* ctx) {
  if (--ctx->refs > 0) return;
  cudaSetDevice(ctx->device);
  rr::cache_drop(ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamDestroy(ctx->stream);
  for (cudaEvent_t e : ctx->level_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  delete ctx;
}

void scene_release(rr_scene* scene) {
  if (--scene->refs > 0) return;
  rr_ctx* ctx = scene->ctx;
  cudaSetDevice(ctx->device);
  delete scene;
  cudaStreamSynchronize(ctx->stream);
  ctx_release(ctx);
}
}  // namespace

rr_status rr_ctx_destroy(rr_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    ctx_release(ctx);
  });
}

rr_status rr_host_alloc(int64_t bytes, void** out) {
  return guarded([&] {
    check_ptr(out, "out");
    *out = nullptr;
    if (bytes < 0) throw std::invalid_argument("bytes must be >= 0");
    if (bytes > 0) RR_CUDA(cudaMallocHost(out, static_cast<size_t>(bytes)));
  });
}

rr_status rr_host_free(void* p) {
  return guarded([&] {
    if (p) RR_CUDA(cudaFreeHost(p));
  });
}

void* rr_ctx_stream(rr_ctx* ctx) { return ctx ? reinterpret_cast<void*>(ctx->stream) : nullptr; }
int64_t rr_ctx_launches(rr_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

rr_status rr_scene_create(rr_ctx* ctx, const double* verts, int64_t nv, const int32_t* tris, int64_t nf,
                          const double* alpha, int32_t nmat, int32_t validate, rr_scene** out) {
  return guarded([&] {
    check_ptr(ctx, "ctx");
    check_ptr(out, "out");
    if (nf <= 0) rr::invalid("cannot build a tree over an empty mesh");  // accel_tree.cpp:71-73
    if (nf >= (int64_t(1) << 30)) rr::invalid("face count must be < 2^30");
    check_ptr(verts, "verts");
    check_ptr(tris, "tris");
    if (nmat > 0) check_ptr(alpha, "alpha");
    RR_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    auto s = std::make_unique<rr_scene>();
    s->ctx = ctx;
    s->nv = nv;
    s->nf = nf;
    s->nmat = nmat;
    s->verts.alloc(3 * std::max<int64_t>(nv, 1), st);
    s->tris.alloc(4 * nf, st);
    if (nv > 0) RR_CUDA(cudaMemcpyAsync(s->verts.p, verts, sizeof(double) * 3 * nv, cudaMemcpyHostToDevice, st));
    RR_CUDA(cudaMemcpyAsync(s->tris.p, tris, sizeof(int32_t) * 4 * nf, cudaMemcpyHostToDevice, st));
    const unsigned g = static_cast<unsigned>((nf + 255) / 256);
    if (validate) {
      rr::DevBuf<unsigned long long> first;
      first.alloc(1, st);
      RR_CUDA(cudaMemsetAsync(first.p, 0xff, sizeof(unsigned long long), st));
      validate_faces_kernel<<<g, 256, 0, st>>>(s->verts.p, nv, s->tris.p, nf, nmat, first.p);
      RR_LAUNCH_CHECK();
      ctx->launches++;
      unsigned long long key = 0;
      RR_CUDA(cudaMemcpyAsync(&key, first.p, sizeof key, cudaMemcpyDeviceToHost, st));
      RR_CUDA(cudaStreamSynchronize(st));
      if (key != ~0ull) {
        const long long f = static_cast<long long>(key / 4);
        const int kind = static_cast<int>(key % 4);
        if (kind == 0) rr::invalid("face " + std::to_string(f) + " references a vertex out of range");
        if (kind == 1)
          rr::invalid("face " + std::to_string(f) + " references material " + std::to_string(tris[4 * f + 3]) +
                      " out of range");
        rr::invalid("face " + std::to_string(f) + " is degenerate (area <= 1e-12 m^2)");
      }
      for (int32_t m = 0; m < nmat; ++m)
        for (int b = 0; b < rr::kBands; ++b) {
          const double a = alpha[rr::kBands * m + b];
          if (a < 0.0 || a > 1.0)
            rr::invalid("material 'm" + std::to_string(m) + "' has absorption outside [0,1]");
        }
    }
    // 1 - alpha per band (tracer.cpp:57-58), 8*nmat scalars
    std::vector<double> oma(static_cast<size_t>(rr::kBands) * std::max(nmat, 1), 1.0);
    for (int64_t i = 0; i < static_cast<int64_t>(rr::kBands) * nmat; ++i) oma[i] = 1.0 - alpha[i];
    s->oma.alloc(oma.size(), st);
    RR_CUDA(cudaMemcpyAsync(s->oma.p, oma.data(), sizeof(double) * oma.size(), cudaMemcpyHostToDevice, st));
    s->tri.alloc(nf, st);
    s->tri32.alloc(3 * nf, st);
    s->normal.alloc(3 * nf, st);
    s->mat.alloc(nf, st);
    face_data_kernel<<<g, 256, 0, st>>>(s->verts.p, s->tris.p, nf, s->tri.p, s->tri32.p, s->normal.p, s->mat.p);
    RR_LAUNCH_CHECK();
    ctx->launches++;
    rr::build_scene_tree(s.get());
    RR_CUDA(cudaStreamSynchronize(st));
    ctx->refs++;  // the scene holds its context
    *out = s.release();
  });
}

rr_status rr_scene_destroy(rr_scene* scene) {
  return guarded([&] {
    if (!scene) return;
    scene_release(scene);
  });
}

rr_status rr_scene_tree_info(rr_scene* s, int64_t* n_nodes, int32_t* root, int32_t* depth) {
  return guarded([&] {
    check_ptr(s, "scene");
    if (n_nodes) *n_nodes = 2 * s->nf - 1;
    if (root) *root = s->root;
    if (depth) *depth = s->depth;
  });
}

rr_status rr_scene_tree(rr_scene* s, rr_tree_node* nodes) {
  return guarded([&] {
    check_ptr(s, "scene");
    check_ptr(nodes, "nodes");
    RR_CUDA(cudaSetDevice(s->ctx->device));
    rr::ensure_reference_tree(s);  // built on first use (rr_build.cu)
    RR_CUDA(cudaMemcpyAsync(nodes, s->ref.p, s->ref.bytes(), cudaMemcpyDeviceToHost, s->ctx->stream));
    RR_CUDA(cudaStreamSynchronize(s->ctx->stream));
  });
}

rr_status rr_scene_normals(rr_scene* s, double* normals) {
  return guarded([&] {
    check_ptr(s, "scene");
    check_ptr(normals, "normals");
    RR_CUDA(cudaSetDevice(s->ctx->device));
    RR_CUDA(cudaMemcpyAsync(normals, s->normal.p, s->normal.bytes(), cudaMemcpyDeviceToHost, s->ctx->stream));
    RR_CUDA(cudaStreamSynchronize(s->ctx->stream));
  });
}

double rr_scene_build_ms(rr_scene* s) { return s ? s->build_ms : -1.0; }

rr_status rr_nearest_hit_batch(rr_scene* s, const double* o, const double* d, int64_t n, int32_t brute,
                               int32_t* face, double* delta, double* point) {
  return guarded([&] {
    check_ptr(s, "scene");
    if (n < 0) rr::invalid("n must be >= 0");
    if (n == 0) return;
    check_ptr(o, "origins");
    check_ptr(d, "dirs");
    check_ptr(face, "face");
    check_ptr(delta, "delta");
    check_ptr(point, "point");
    RR_CUDA(cudaSetDevice(s->ctx->device));
    cudaStream_t st = s->ctx->stream;
    rr::DevBuf<double> dob, ddb, ddel, dpt;
    rr::DevBuf<int32_t> dface;
    dob.alloc(3 * n, st);
    ddb.alloc(3 * n, st);
    ddel.alloc(n, st);
    dpt.alloc(3 * n, st);
    dface.alloc(n, st);
    RR_CUDA(cudaMemcpyAsync(dob.p, o, dob.bytes(), cudaMemcpyHostToDevice, st));
    RR_CUDA(cudaMemcpyAsync(ddb.p, d, ddb.bytes(), cudaMemcpyHostToDevice, st));
    rr::nearest_hit_batch(s, dob.p, ddb.p, n, brute, dface.p, ddel.p, dpt.p);
    RR_CUDA(cudaMemcpyAsync(face, dface.p, dface.bytes(), cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaMemcpyAsync(delta, ddel.p, ddel.bytes(), cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaMemcpyAsync(point, dpt.p, dpt.bytes(), cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
  });
}

rr_status rr_trace(rr_scene* s, const rr_source* src, const rr_receiver* recv, int32_t n_recv,
                   const rr_trace_config* cfg, rr_trace_result** out) {
  return guarded([&] {
    check_ptr(s, "scene");
    check_ptr(src, "source");
    check_ptr(recv, "receivers");
    check_ptr(cfg, "config");
    check_ptr(out, "out");
    RR_CUDA(cudaSetDevice(s->ctx->device));
    *out = rr::run_trace(s, src, recv, n_recv, cfg, nullptr);
    (*out)->scene->refs++;
  });
}

rr_status rr_trace_stats_get(rr_trace_result* r, rr_trace_stats* stats) {
  return guarded([&] {
    check_ptr(r, "result");
    check_ptr(stats, "stats");
    *stats = r->stats;
  });
}

rr_status rr_trace_captures(rr_trace_result* r, int32_t* recv, int32_t* ray, double* point, double* dir,
                            double* path, double* mult, int64_t* hist_off, int32_t* hist) {
  return guarded([&] {
    check_ptr(r, "result");
    RR_CUDA(cudaSetDevice(r->scene->ctx->device));
    cudaStream_t st = r->scene->ctx->stream;
    const int64_t n = r->stats.n_captures;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) RR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
    };
    if (n > 0) {
      cp(recv, r->c_recv.p, sizeof(int32_t) * n);
      cp(ray, r->c_ray.p, sizeof(int32_t) * n);
      cp(point, r->c_point.p, sizeof(double) * 3 * n);
      cp(dir, r->c_dir.p, sizeof(double) * 3 * n);
      cp(path, r->c_path.p, sizeof(double) * n);
      cp(mult, r->c_mult.p, sizeof(double) * rr::kBands * n);
      cp(hist, r->c_hist.p, sizeof(int32_t) * r->stats.total_history);
    }
    cp(hist_off, r->c_off.p, sizeof(int64_t) * (n + 1));
    RR_CUDA(cudaStreamSynchronize(st));
  });
}

double rr_trace_kernel_ms(rr_trace_result* r) { return r ? r->kernel_ms : -1.0; }

rr_status rr_step(rr_scene* scene, int64_t n, double* origin, double* dir, double* mult, double* path,
                  int32_t* alive, int32_t* hist, int32_t* n_hist, int32_t hist_cap, const rr_receiver* receiver,
                  const rr_trace_config* config, int32_t brute, rr_trace_result** out) {
  return guarded([&] {
    check_ptr(scene, "scene");
    check_ptr(receiver, "receiver");
    check_ptr(config, "config");
    check_ptr(out, "out");
    if (n > 0) {
      check_ptr(origin, "origin");
      check_ptr(dir, "dir");
      check_ptr(mult, "mult");
      check_ptr(path, "path");
      check_ptr(alive, "alive");
      check_ptr(hist, "hist");
      check_ptr(n_hist, "n_hist");
    }
    RR_CUDA(cudaSetDevice(scene->ctx->device));
    float ms = 0.f;
    *out = rr::step_rays(scene, n, origin, dir, mult, path, alive, hist, n_hist, hist_cap, receiver, config, brute,
                         &ms);
    (*out)->scene->refs++;
  });
}

rr_status rr_captures_import(rr_scene* scene, int64_t n, const int32_t* recv, const int32_t* ray, const double* point,
                             const double* dir, const double* path, const double* mult, const int64_t* hist_off,
                             const int32_t* hist, const rr_receiver* receivers, int32_t n_recv,
                             rr_trace_result** out) {
  return guarded([&] {
    check_ptr(scene, "scene");
    check_ptr(receivers, "receivers");
    check_ptr(out, "out");
    if (n > 0) {
      check_ptr(ray, "ray");
      check_ptr(point, "point");
      check_ptr(dir, "dir");
      check_ptr(path, "path");
      check_ptr(hist_off, "hist_off");
    }
    RR_CUDA(cudaSetDevice(scene->ctx->device));
    *out = rr::import_captures(scene, n, recv, ray, point, dir, path, mult, hist_off, hist, receivers, n_recv);
    (*out)->scene->refs++;
  });
}

rr_status rr_trace_destroy(rr_trace_result* r) {
  return guarded([&] {
    if (!r) return;
    rr_scene* sc = r->scene;
    cudaSetDevice(sc->ctx->device);
    delete r;
    cudaStreamSynchronize(sc->ctx->stream);
    scene_release(sc);
  });
}

}  // extern "C"

// ---------------------------------------------------------------- IR
namespace rr {
void ir_bin(rr_ctx* ctx, int64_t n, const double* d_dist, const double* d_energy, double c, double fs, int64_t lh,
            double* d_hist);
void ir_filter(rr_ctx* ctx, const double* d_hist, int64_t lh, double fs, int taps, int64_t L, double* d_band_ir,
               double* d_broadband);
void band_filter_host(int band, double fs, int taps, double* out, rr_ctx* ctx);
void ir_bin_events(rr_ctx* ctx, const int64_t* d_off, int64_t n, const double* d_time, const double* d_amp, double fs,
                   int64_t lh, double* d_hist);
void air_beta_bands(const rr_air& a, double* beta);
}  // namespace rr

namespace {
__global__ void min_dist_kernel(const double* __restrict__ d, int64_t n, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!(d[i] >= 0.0)) *bad = 1;
}
}  // namespace

extern "C" {

rr_status rr_band_filter(int32_t band, double fs, int32_t taps, double* out) {
  return guarded([&] {
    check_ptr(out, "out");
    static thread_local rr_ctx* ctx = nullptr;
    if (!ctx) {
      if (rr_ctx_create(0, &ctx) != RR_OK) throw rr::Error(RR_CUDA, g_err);
    }
    rr::band_filter_host(band, fs, taps, out, ctx);
  });
}

rr_status rr_ir_bin_device(rr_ctx* ctx, int64_t n, const double* d_dist, const double* d_energy, double c, double fs,
                           int64_t length, double* d_hist) {
  return guarded([&] {
    check_ptr(ctx, "ctx");
    check_ptr(d_hist, "hist");
    if (c <= 0.0) rr::invalid("speed of sound must be > 0");  // rir.cpp:11-13
    if (length <= 0) rr::invalid("length must be > 0");
    RR_CUDA(cudaSetDevice(ctx->device));
    rr::ir_bin(ctx, n, d_dist, d_energy, c, fs, length, d_hist);
  });
}

rr_status rr_ir_filter_device(rr_ctx* ctx, const double* d_hist, double fs, int32_t taps, int64_t length,
                              double* d_band_ir, double* d_broadband) {
  return guarded([&] {
    check_ptr(ctx, "ctx");
    check_ptr(d_hist, "hist");
    RR_CUDA(cudaSetDevice(ctx->device));
    // d_hist holds length + taps samples per band
    rr::ir_filter(ctx, d_hist, length + taps, fs, taps, length, d_band_ir, d_broadband);
  });
}

rr_status rr_synthesize(rr_ctx* ctx, int64_t n, const double* dist, const double* energy, double c, double fs,
                        int32_t taps, int64_t length, double* band_ir, double* broadband) {
  return guarded([&] {
    check_ptr(ctx, "ctx");
    if (c <= 0.0) rr::invalid("speed of sound must be > 0");  // rir.cpp:11-13
    if (n < 0) rr::invalid("n must be >= 0");
    if (n > 0) {
      check_ptr(dist, "dist");
      check_ptr(energy, "energy");
    }
    if (taps < 3) rr::invalid("taps must be >= 3");
    if (fs < 2.0 * 8000.0 * std::sqrt(2.0)) rr::invalid("sample rate too low for the top band edge");
    RR_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    rr::DevBuf<double> dd, de;
    dd.alloc(std::max<int64_t>(n, 1), st);
    de.alloc(rr::kBands * std::max<int64_t>(n, 1), st);
    if (n > 0) {
      RR_CUDA(cudaMemcpyAsync(dd.p, dist, sizeof(double) * n, cudaMemcpyDefault, st));
      RR_CUDA(cudaMemcpyAsync(de.p, energy, sizeof(double) * rr::kBands * n, cudaMemcpyDefault, st));
      rr::DevBuf<int> bad;
      bad.alloc(1, st);
      RR_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
      min_dist_kernel<<<148, 256, 0, st>>>(dd.p, n, bad.p);
      int hb = 0;
      RR_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof hb, cudaMemcpyDeviceToHost, st));
      RR_CUDA(cudaStreamSynchronize(st));
      ctx->launches++;
      if (hb) rr::invalid("pulse events cannot precede t = 0");  // rir.cpp:69-71
    }
    if (length <= 0) rr::invalid("length must be > 0 (see rr_ir_reference_length)");
    const int64_t lh = length + taps;
    rr::DevBuf<double> hist, bands, bb;
    hist.alloc(rr::kBands * lh, st);
    bands.alloc(rr::kBands * length, st);
    bb.alloc(length, st);
    rr::ir_bin(ctx, n, dd.p, de.p, c, fs, lh, hist.p);
    rr::ir_filter(ctx, hist.p, lh, fs, taps, length, bands.p, bb.p);
    if (band_ir)
      RR_CUDA(cudaMemcpyAsync(band_ir, bands.p, bands.bytes(), cudaMemcpyDeviceToHost, st));
    if (broadband) RR_CUDA(cudaMemcpyAsync(broadband, bb.p, bb.bytes(), cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
  });
}

rr_status rr_synthesize_trains(rr_ctx* ctx, const int64_t* band_off, const double* time, const double* amplitude,
                               double fs, int32_t taps, int64_t length, double* band_ir, double* broadband) {
  return guarded([&] {
    check_ptr(ctx, "ctx");
    check_ptr(band_off, "band_off");
    if (band_off[0] != 0) rr::invalid("band_off[0] must be 0");
    for (int b = 0; b < rr::kBands; ++b)
      if (band_off[b + 1] < band_off[b]) rr::invalid("band_off must be non-decreasing");
    const int64_t n = band_off[rr::kBands];
    if (n > 0) {
      check_ptr(time, "time");
      check_ptr(amplitude, "amplitude");
      for (int64_t i = 0; i < n; ++i)
        if (!(time[i] >= 0.0)) rr::invalid("pulse events cannot precede t = 0");  // rir.cpp:69-71
    }
    if (taps < 3) rr::invalid("taps must be >= 3");
    if (fs < 2.0 * 8000.0 * std::sqrt(2.0)) rr::invalid("sample rate too low for the top band edge");
    if (length <= 0) rr::invalid("length must be > 0");
    RR_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const int64_t lh = length + taps;
    rr::DevBuf<int64_t> doff;
    rr::DevBuf<double> dt, da, hist, bands, bb;
    doff.alloc(rr::kBands + 1, st);
    dt.alloc(std::max<int64_t>(n, 1), st);
    da.alloc(std::max<int64_t>(n, 1), st);
    RR_CUDA(cudaMemcpyAsync(doff.p, band_off, sizeof(int64_t) * (rr::kBands + 1), cudaMemcpyHostToDevice, st));
    if (n > 0) {
      RR_CUDA(cudaMemcpyAsync(dt.p, time, sizeof(double) * n, cudaMemcpyHostToDevice, st));
      RR_CUDA(cudaMemcpyAsync(da.p, amplitude, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    }
    hist.alloc(rr::kBands * lh, st);
    bands.alloc(rr::kBands * length, st);
    bb.alloc(length, st);
    rr::ir_bin_events(ctx, doff.p, n, dt.p, da.p, fs, lh, hist.p);
    rr::ir_filter(ctx, hist.p, lh, fs, taps, length, bands.p, bb.p);
    if (band_ir) RR_CUDA(cudaMemcpyAsync(band_ir, bands.p, bands.bytes(), cudaMemcpyDeviceToHost, st));
    if (broadband) RR_CUDA(cudaMemcpyAsync(broadband, bb.p, bb.bytes(), cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
namespace rr {
void band_factors(rr_ctx* ctx, const double* d_t, const double* d_a, int64_t n, rr_factors* d_out);
void image_factors(rr_ctx* ctx, const double* d_dist, const double* d_energy, int64_t n, double c, rr_factors* out);
}  // namespace rr
extern "C" {

rr_status rr_band_schroeder(rr_ctx* ctx, const int64_t* band_off, const double* amplitude, double* level_db) {
  return guarded([&] {
    check_ptr(ctx, "ctx");
    check_ptr(band_off, "band_off");
    if (band_off[0] != 0) rr::invalid("band_off[0] must be 0");
    for (int b = 0; b < rr::kBands; ++b)
      if (band_off[b + 1] < band_off[b]) rr::invalid("band_off must be non-decreasing");
    if (band_off[rr::kBands] > 0) {
      check_ptr(amplitude, "amplitude");
      check_ptr(level_db, "level_db");
    }
    RR_CUDA(cudaSetDevice(ctx->device));
    rr::band_schroeder(ctx, band_off, amplitude, level_db);
  });
}

rr_status rr_band_factors(rr_ctx* ctx, const int64_t* band_off, const double* time, const double* amplitude,
                          rr_factors* out) {
  return guarded([&] {
    check_ptr(ctx, "ctx");
    check_ptr(band_off, "band_off");
    check_ptr(out, "out");
    if (band_off[0] != 0) rr::invalid("band_off[0] must be 0");
    for (int b = 0; b < rr::kBands; ++b)
      if (band_off[b + 1] < band_off[b]) rr::invalid("band_off must be non-decreasing");
    const int64_t n = band_off[rr::kBands];
    if (n > 0) {
      check_ptr(time, "time");
      check_ptr(amplitude, "amplitude");
    }
    RR_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    rr::DevBuf<double> t, a;
    rr::DevBuf<rr_factors> d_out;
    t.alloc(std::max<int64_t>(n, 1), st);
    a.alloc(std::max<int64_t>(n, 1), st);
    d_out.alloc(rr::kBands, st);
    if (n > 0) {
      RR_CUDA(cudaMemcpyAsync(t.p, time, sizeof(double) * n, cudaMemcpyHostToDevice, st));
      RR_CUDA(cudaMemcpyAsync(a.p, amplitude, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    }
    for (int b = 0; b < rr::kBands; ++b)
      rr::band_factors(ctx, t.p + band_off[b], a.p + band_off[b], band_off[b + 1] - band_off[b], d_out.p + b);
    RR_CUDA(cudaMemcpyAsync(out, d_out.p, sizeof(rr_factors) * rr::kBands, cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
    auto avg = [](rr_metric x, rr_metric y) {
      return rr_metric{0.5 * (x.value + y.value), x.reliable && y.reliable};
    };
    out[8] = rr_factors{avg(out[3].edt_s, out[4].edt_s), avg(out[3].t30_s, out[4].t30_s),
                        avg(out[3].spl_db, out[4].spl_db), avg(out[3].c80_db, out[4].c80_db),
                        avg(out[3].d50_pct, out[4].d50_pct), avg(out[3].ts_ms, out[4].ts_ms)};
  });
}

rr_status rr_factors_from_images(rr_ctx* ctx, int64_t n, const double* dist, const double* energy, double c,
                                 rr_factors* out) {
  return guarded([&] {
    check_ptr(ctx, "ctx");
    check_ptr(out, "out");
    if (c <= 0.0) rr::invalid("speed of sound must be > 0");  // rir.cpp:11-13
    if (n < 0) rr::invalid("n must be >= 0");
    if (n > 0) {
      check_ptr(dist, "dist");
      check_ptr(energy, "energy");
    }
    RR_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    rr::DevBuf<double> dd, de;
    dd.alloc(std::max<int64_t>(n, 1), st);
    de.alloc(rr::kBands * std::max<int64_t>(n, 1), st);
    if (n > 0) {
      RR_CUDA(cudaMemcpyAsync(dd.p, dist, sizeof(double) * n, cudaMemcpyDefault, st));
      RR_CUDA(cudaMemcpyAsync(de.p, energy, sizeof(double) * rr::kBands * n, cudaMemcpyDefault, st));
    }
    rr::image_factors(ctx, dd.p, de.p, n, c, out);
  });
}

rr_status rr_images_factors(rr_images* im, double c, rr_factors* out) {
  return guarded([&] {
    check_ptr(im, "images");
    check_ptr(out, "out");
    if (c <= 0.0) rr::invalid("speed of sound must be > 0");
    rr_ctx* ctx = im->scene->ctx;
    RR_CUDA(cudaSetDevice(ctx->device));
    rr::image_factors(ctx, im->dist.p, im->energy.p, im->n, c, out);
  });
}

// Response length of the reference's synthesize (rir.cpp:78-80):
// llround(t_last*fs) + (taps-1)/2 + 1, 0 for no events.
rr_status rr_ir_reference_length(int64_t n, const double* dist, double c, double fs, int32_t taps,
                                 int64_t* length) {
  return guarded([&] {
    check_ptr(length, "length");
    if (c <= 0.0) rr::invalid("speed of sound must be > 0");
    double last = 0.0;
    for (int64_t i = 0; i < n; ++i) last = std::max(last, dist[i] / c);
    *length = n > 0 ? static_cast<int64_t>(std::llround(last * fs)) + (taps - 1) / 2 + 1 : 0;
  });
}

// L2 read-bandwidth probe for the roofline report: every block streams the
// whole (L2-resident) buffer `iters` times with 16-B loads, grid = 4 x SMs.
namespace {
__global__ void l2_read_kernel(const float4* __restrict__ buf, int64_t n4, int iters, float* __restrict__ sink) {
  float acc = 0.f;
  for (int it = 0; it < iters; ++it)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
      const float4 v = __ldcg(buf + i);  // L2 only (bypasses L1)
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 1234.5f) *sink = acc;  // keep the loads
}
}  // namespace

rr_status rr_l2_read_gbs(rr_ctx* ctx, int64_t bytes, int32_t iters, double* gbs) {
  return guarded([&] {
    check_ptr(ctx, "ctx");
    check_ptr(gbs, "gbs");
    if (bytes < (1 << 20) || iters < 1) rr::invalid("bytes >= 1 MiB and iters >= 1 required");
    RR_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const int64_t n4 = bytes / 16;
    rr::DevBuf<float4> buf;
    rr::DevBuf<float> sink;
    buf.alloc(n4, st);
    sink.alloc(1, st);
    RR_CUDA(cudaMemsetAsync(buf.p, 0, buf.bytes(), st));
    const unsigned grid = static_cast<unsigned>(4 * ctx->sm_count);
    l2_read_kernel<<<grid, 512, 0, st>>>(buf.p, n4, 1, sink.p);  // warm: pull into L2
    cudaEvent_t e0, e1;
    RR_CUDA(cudaEventCreate(&e0));
    RR_CUDA(cudaEventCreate(&e1));
    RR_CUDA(cudaEventRecord(e0, st));
    l2_read_kernel<<<grid, 512, 0, st>>>(buf.p, n4, iters, sink.p);
    RR_CUDA(cudaEventRecord(e1, st));
    RR_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    RR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    ctx->launches += 2;
    *gbs = static_cast<double>(n4) * 16.0 * iters / (ms * 1e-3) / 1e9;
  });
}

// ---------------------------------------------------------------- shoebox lattice (rr_shoebox.cu)
rr_status rr_shoebox_images(rr_ctx* ctx, const double* dims, const double* walls_alpha, const double* source,
                            const double* receiver, double max_distance, double receiver_radius, const rr_air* air,
                            rr_lattice** out) {
  return guarded([&] {
    check_ptr(ctx, "ctx");
    check_ptr(dims, "dims");
    check_ptr(walls_alpha, "walls_alpha");
    check_ptr(source, "source");
    check_ptr(receiver, "receiver");
    check_ptr(air, "air");
    check_ptr(out, "out");
    RR_CUDA(cudaSetDevice(ctx->device));
    *out = rr::enumerate_lattice(ctx, dims, walls_alpha, source, receiver, max_distance, receiver_radius, *air);
    ctx->refs++;
  });
}

rr_status rr_lattice_info(rr_lattice* lat, int64_t* n) {
  return guarded([&] {
    check_ptr(lat, "lattice");
    if (n) *n = lat->n;
  });
}

rr_status rr_lattice_get(rr_lattice* lat, double* pos, double* dist, int32_t* order, int32_t* wall_hits,
                         double* energy) {
  return guarded([&] {
    check_ptr(lat, "lattice");
    RR_CUDA(cudaSetDevice(lat->ctx->device));
    cudaStream_t st = lat->ctx->stream;
    const int64_t n = lat->n;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) RR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
    };
    cp(pos, lat->pos.p, sizeof(double) * 3 * n);
    cp(dist, lat->dist.p, sizeof(double) * n);
    cp(order, lat->order.p, sizeof(int32_t) * n);
    cp(wall_hits, lat->hits.p, sizeof(int32_t) * 6 * n);
    cp(energy, lat->energy.p, sizeof(double) * rr::kBands * n);
    RR_CUDA(cudaStreamSynchronize(st));
  });
}

rr_status rr_lattice_destroy(rr_lattice* lat) {
  return guarded([&] {
    if (!lat) return;
    rr_ctx* ctx = lat->ctx;
    cudaSetDevice(ctx->device);
    delete lat;
    cudaStreamSynchronize(ctx->stream);
    ctx_release(ctx);
  });
}

rr_status rr_shoebox_compare(rr_ctx* ctx, int64_t n_oracle, const double* oracle_pos, const double* oracle_energy,
                             const int32_t* oracle_order, int64_t n_traced, const double* traced_pos,
                             const double* traced_energy, double pos_tol, double energy_tol_db, rr_match** out) {
  return guarded([&] {
    check_ptr(ctx, "ctx");
    check_ptr(out, "out");
    if (n_oracle > 0) {
      check_ptr(oracle_pos, "oracle_pos");
      check_ptr(oracle_energy, "oracle_energy");
    }
    if (n_traced > 0) {
      check_ptr(traced_pos, "traced_pos");
      check_ptr(traced_energy, "traced_energy");
    }
    RR_CUDA(cudaSetDevice(ctx->device));
    *out = rr::compare_lattice(ctx, n_oracle, oracle_pos, oracle_energy, oracle_order, n_traced, traced_pos,
                               traced_energy, pos_tol, energy_tol_db);
    ctx->refs++;
  });
}

rr_status rr_lattice_compare_images(rr_lattice* lat, rr_images* traced, double pos_tol, double energy_tol_db,
                                    rr_match** out) {
  return guarded([&] {
    check_ptr(lat, "lattice");
    check_ptr(traced, "images");
    check_ptr(out, "out");
    if (traced->scene->ctx != lat->ctx) rr::invalid("lattice and images belong to different contexts");
    rr_ctx* ctx = lat->ctx;
    RR_CUDA(cudaSetDevice(ctx->device));
    *out = rr::compare_lattice(ctx, lat->n, lat->pos.p, lat->energy.p, lat->order.p, traced->n, traced->pos.p,
                               traced->energy.p, pos_tol, energy_tol_db);
    ctx->refs++;
  });
}

rr_status rr_match_info(rr_match* m, int64_t* n_matched, int64_t* n_members, int64_t* n_unmatched_oracle,
                        int64_t* n_unmatched_traced, double* max_position_error, double* rms_energy_error_db) {
  return guarded([&] {
    check_ptr(m, "match");
    if (n_matched) *n_matched = m->n_matched;
    if (n_members) *n_members = m->n_members;
    if (n_unmatched_oracle) *n_unmatched_oracle = m->n_unmatched_oracle;
    if (n_unmatched_traced) *n_unmatched_traced = m->n_unmatched_traced;
    if (max_position_error) *max_position_error = m->max_position_error;
    if (rms_energy_error_db)
      for (int b = 0; b < rr::kBands; ++b) rms_energy_error_db[b] = m->rms_db[b];
  });
}

rr_status rr_match_get(rr_match* m, int32_t* oracle_index, double* position_error, int32_t* order,
                       double* energy_delta_db, int64_t* member_off, int32_t* members, int32_t* unmatched_oracle,
                       int32_t* unmatched_traced) {
  return guarded([&] {
    check_ptr(m, "match");
    RR_CUDA(cudaSetDevice(m->ctx->device));
    cudaStream_t st = m->ctx->stream;
    const int64_t g = m->n_matched;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) RR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
    };
    cp(oracle_index, m->oracle_index.p, sizeof(int32_t) * g);
    cp(position_error, m->pos_err.p, sizeof(double) * g);
    cp(order, m->order.p, sizeof(int32_t) * g);
    cp(energy_delta_db, m->delta_db.p, sizeof(double) * rr::kBands * g);
    cp(member_off, m->member_off.p, sizeof(int64_t) * (g + 1));
    cp(members, m->members.p, sizeof(int32_t) * m->n_members);
    cp(unmatched_oracle, m->unmatched_oracle.p, sizeof(int32_t) * m->n_unmatched_oracle);
    cp(unmatched_traced, m->unmatched_traced.p, sizeof(int32_t) * m->n_unmatched_traced);
    RR_CUDA(cudaStreamSynchronize(st));
  });
}

rr_status rr_match_destroy(rr_match* m) {
  return guarded([&] {
    if (!m) return;
    rr_ctx* ctx = m->ctx;
    cudaSetDevice(ctx->device);
    delete m;
    cudaStreamSynchronize(ctx->stream);
    ctx_release(ctx);
  });
}

rr_status rr_air_alpha_db_per_m(const rr_air* air, double f, double* alpha) {
  return guarded([&] {
    check_ptr(air, "air");
    check_ptr(alpha, "alpha");
    *alpha = rr::air_alpha(*air, f);
  });
}

rr_status rr_air_validate(const rr_air* air) {
  return guarded([&] {
    check_ptr(air, "air");
    rr::air_validate(*air);
  });
}

rr_status rr_fibonacci_directions(rr_ctx* ctx, int64_t n, int64_t first, int64_t stride, int64_t count,
                                  double* out) {
  return guarded([&] {
    check_ptr(ctx, "ctx");
    if (n < 1) rr::invalid("fibonacci_directions needs n >= 1");  // emission.cpp:18
    if (count < 0 || first < 0 || stride < 1) rr::invalid("bad lattice subset");
    if (count > 0) check_ptr(out, "out");
    RR_CUDA(cudaSetDevice(ctx->device));
    rr::fibonacci_device(ctx, n, first, stride, count, out);
  });
}

rr_status rr_air_beta_bands(const rr_air* air, double* beta) {
  return guarded([&] {
    check_ptr(air, "air");
    check_ptr(beta, "beta");
    rr::air_beta_bands(*air, beta);
  });
}

// ---------------------------------------------------------------- images (K5, rr_images.cu)
rr_status rr_build_image_sources(rr_trace_result* tr, int32_t recv, int64_t total_rays, const rr_air* air,
                                 const rr_cluster_options* opt, rr_images** out) {
  return guarded([&] {
    check_ptr(tr, "trace result");
    check_ptr(air, "air");
    check_ptr(out, "out");
    rr_cluster_options o{1e-6, 0};
    if (opt) o = *opt;
    RR_CUDA(cudaSetDevice(tr->scene->ctx->device));
    *out = rr::build_image_sources(tr, recv, total_rays, *air, o);
    (*out)->scene->refs++;
  });
}

rr_status rr_images_info(rr_images* im, int64_t* n, int64_t* total_path) {
  return guarded([&] {
    check_ptr(im, "images");
    if (n) *n = im->n;
    if (total_path) *total_path = im->total_path;
  });
}

rr_status rr_images_get(rr_images* im, double* pos, double* dist, double* energy, double* mult, int32_t* ray_count,
                        int32_t* order, int32_t* has_proj, double* proj, int64_t* path_off, int32_t* path) {
  return guarded([&] {
    check_ptr(im, "images");
    RR_CUDA(cudaSetDevice(im->scene->ctx->device));
    cudaStream_t st = im->scene->ctx->stream;
    const int64_t n = im->n;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) RR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
    };
    cp(pos, im->pos.p, sizeof(double) * 3 * n);
    cp(dist, im->dist.p, sizeof(double) * n);
    cp(energy, im->energy.p, sizeof(double) * rr::kBands * n);
    cp(mult, im->mult.p, sizeof(double) * rr::kBands * n);
    cp(ray_count, im->ray_count.p, sizeof(int32_t) * n);
    cp(order, im->order.p, sizeof(int32_t) * n);
    cp(has_proj, im->has_proj.p, sizeof(int32_t) * n);
    cp(proj, im->proj.p, sizeof(double) * 3 * n);
    cp(path_off, im->path_off.p, sizeof(int64_t) * (n + 1));
    cp(path, im->path.p, sizeof(int32_t) * im->total_path);
    RR_CUDA(cudaStreamSynchronize(st));
  });
}

rr_status rr_images_get_async(rr_images* im, void* stream, double* pos, double* dist, double* energy, double* mult,
                              int32_t* ray_count, int32_t* order, int32_t* has_proj, double* proj, int64_t* path_off,
                              int32_t* path) {
  return guarded([&] {
    check_ptr(im, "images");
    RR_CUDA(cudaSetDevice(im->scene->ctx->device));
    cudaStream_t ctx = im->scene->ctx->stream;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (st != ctx) {  // the side stream starts after the image build
      cudaEvent_t ev;
      RR_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      RR_CUDA(cudaEventRecord(ev, ctx));
      RR_CUDA(cudaStreamWaitEvent(st, ev, 0));
      RR_CUDA(cudaEventDestroy(ev));
    }
    const int64_t n = im->n;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) RR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
    };
    cp(pos, im->pos.p, sizeof(double) * 3 * n);
    cp(dist, im->dist.p, sizeof(double) * n);
    cp(energy, im->energy.p, sizeof(double) * rr::kBands * n);
    cp(mult, im->mult.p, sizeof(double) * rr::kBands * n);
    cp(ray_count, im->ray_count.p, sizeof(int32_t) * n);
    cp(order, im->order.p, sizeof(int32_t) * n);
    cp(has_proj, im->has_proj.p, sizeof(int32_t) * n);
    cp(proj, im->proj.p, sizeof(double) * 3 * n);
    cp(path_off, im->path_off.p, sizeof(int64_t) * (n + 1));
    cp(path, im->path.p, sizeof(int32_t) * im->total_path);
    if (st != ctx) {  // rr_images_destroy orders its frees after these copies
      if (!im->copies_done) RR_CUDA(cudaEventCreateWithFlags(&im->copies_done, cudaEventDisableTiming));
      RR_CUDA(cudaEventRecord(im->copies_done, st));
    }
  });
}

rr_status rr_images_destroy(rr_images* im) {
  return guarded([&] {
    if (!im) return;
    rr_scene* sc = im->scene;
    cudaSetDevice(sc->ctx->device);
    if (im->copies_done) {  // copies on a caller stream (rr_images_get_async) before the stream-ordered frees
      cudaStreamWaitEvent(sc->ctx->stream, im->copies_done, 0);
      cudaEventDestroy(im->copies_done);
    }
    delete im;
    cudaStreamSynchronize(sc->ctx->stream);
    scene_release(sc);
  });
}

rr_status rr_images_device(rr_images* im, const double** d_dist, const double** d_energy, int64_t* n) {
  return guarded([&] {
    check_ptr(im, "images");
    if (d_dist) *d_dist = im->dist.p;
    if (d_energy) *d_energy = im->energy.p;
    if (n) *n = im->n;
  });
}

}  // extern "C"

// ---------------------------------------------------------------- helpers for rr_shard.cu
namespace rr {
rr_status abi_guard_nccl(const std::function<void()>& f) { return guarded(f); }
void scene_retain(rr_scene* s) { s->refs++; }
void scene_drop(rr_scene* s) { scene_release(s); }
}  // namespace rr

// ---------------------------------------------------------------- pulse trains / IR of a device image set
namespace rr {
void image_trains(rr_ctx* ctx, const double* d_dist, const double* d_energy, int64_t n, double c, double* time,
                  double* amp);
}
namespace {
__global__ void max_dist_kernel(const double* __restrict__ d, int64_t n, unsigned long long* __restrict__ out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, d[i]);
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}
}  // namespace

extern "C" {

rr_status rr_images_pulse_trains(rr_images* im, double c, int64_t* band_off, double* time, double* amplitude) {
  return guarded([&] {
    check_ptr(im, "images");
    if (c <= 0.0) rr::invalid("speed of sound must be > 0");  // rir.cpp:11-13
    rr_ctx* ctx = im->scene->ctx;
    RR_CUDA(cudaSetDevice(ctx->device));
    if (band_off)
      for (int b = 0; b <= rr::kBands; ++b) band_off[b] = b * im->n;
    if (im->n > 0) {
      check_ptr(time, "time");
      check_ptr(amplitude, "amplitude");
      rr::image_trains(ctx, im->dist.p, im->energy.p, im->n, c, time, amplitude);
    }
  });
}

rr_status rr_pulse_trains(rr_ctx* ctx, int64_t n, const double* dist, const double* energy, double c,
                          int64_t* band_off, double* time, double* amplitude) {
  return guarded([&] {
    check_ptr(ctx, "context");
    if (c <= 0.0) rr::invalid("speed of sound must be > 0");  // rir.cpp:11-13
    if (n < 0) rr::invalid("n must be >= 0");
    RR_CUDA(cudaSetDevice(ctx->device));
    if (band_off)
      for (int b = 0; b <= rr::kBands; ++b) band_off[b] = b * n;
    if (n == 0) return;
    check_ptr(dist, "dist");
    check_ptr(energy, "energy");
    check_ptr(time, "time");
    check_ptr(amplitude, "amplitude");
    cudaStream_t st = ctx->stream;
    rr::DevBuf<double> d, e;
    d.alloc(n, st);
    e.alloc(rr::kBands * n, st);
    RR_CUDA(cudaMemcpyAsync(d.p, dist, sizeof(double) * n, cudaMemcpyDefault, st));
    RR_CUDA(cudaMemcpyAsync(e.p, energy, sizeof(double) * rr::kBands * n, cudaMemcpyDefault, st));
    rr::image_trains(ctx, d.p, e.p, n, c, time, amplitude);  // synchronizes the stream
  });
}

rr_status rr_images_synthesize(rr_images* im, double c, double fs, int32_t taps, int64_t* length, double* band_ir,
                               double* broadband) {
  return guarded([&] {
    check_ptr(im, "images");
    check_ptr(length, "length");
    if (c <= 0.0) rr::invalid("speed of sound must be > 0");
    if (taps < 3) rr::invalid("taps must be >= 3");
    rr_ctx* ctx = im->scene->ctx;
    RR_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    if (!band_ir && !broadband) {  // the reference length (rir.cpp:78-80)
      *length = 0;
      if (im->n == 0) return;
      rr::DevBuf<unsigned long long> mx;
      mx.alloc(1, st);
      RR_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(unsigned long long), st));
      max_dist_kernel<<<148, 256, 0, st>>>(im->dist.p, im->n, mx.p);
      RR_LAUNCH_CHECK();
      ctx->launches++;
      unsigned long long bits = 0;
      RR_CUDA(cudaMemcpyAsync(&bits, mx.p, sizeof bits, cudaMemcpyDeviceToHost, st));
      RR_CUDA(cudaStreamSynchronize(st));
      double last;
      std::memcpy(&last, &bits, sizeof last);
      *length = static_cast<int64_t>(std::llround(last / c * fs)) + (taps - 1) / 2 + 1;
      return;
    }
    if (*length <= 0) rr::invalid("length must be > 0");
    const int64_t L = *length, lh = L + taps;
    rr::DevBuf<double> hist, band, bb;
    hist.alloc(rr::kBands * lh, st);
    band.alloc(rr::kBands * L, st);
    bb.alloc(L, st);
    rr::ir_bin(ctx, im->n, im->dist.p, im->energy.p, c, fs, lh, hist.p);
    rr::ir_filter(ctx, hist.p, lh, fs, taps, L, band.p, bb.p);
    if (band_ir) RR_CUDA(cudaMemcpyAsync(band_ir, band.p, sizeof(double) * rr::kBands * L, cudaMemcpyDefault, st));
    if (broadband) RR_CUDA(cudaMemcpyAsync(broadband, bb.p, sizeof(double) * L, cudaMemcpyDefault, st));
    RR_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
