// step (tracer.hpp:43-45, tracer.cpp:19-106): one iteration over a span of
// caller rays, in place.  Used by the reference's complexity bench
// (bench.cpp:26-46, the paper's Table 2: per-iteration time with the tree and
// with brute force) and by callers that drive the loop themselves.
//
// One thread per ray: closest wall (the SAH traversal or, for `brute`, the
// O(M) scan of nearest_hit_brute with the lowest face on ties), receiver
// capture on the segment (warp-aggregated append; the capture copies the
// multipliers and the face history as they were before this wall), escape,
// double-sided normal, reflection, path, band multipliers *= (1 - alpha),
// history append, range kill with max_range = resolved_max_range(receiver, n)
// (tracer.cpp:10-15, 70-71).  Captures come back as a trace result (receiver
// 0), in ray order like the reference's single-threaded step.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <memory>

#include "rr_trace.cuh"

namespace rr {
namespace {

struct StepParams {
  TravHeader hdr;
  const TNode* nodes;
  const FaceTri* tri;
  int64_t nf;
  const double* normal;
  const int32_t* mat;
  const double* oma;
  int64_t n;
  double *origin, *dir, *mult, *path;
  int32_t *alive, *hist, *n_hist;
  int32_t hist_cap;
  double rc[3], rr, max_range;
  int32_t brute;
  // captures: fixed records + multipliers + a history slice of hist_cap
  Capture* caps;
  double* cap_mult;
  int32_t* cap_hist;
  unsigned long long* cap_count;
  int64_t cap_capacity;
  int32_t* bad;
};

__global__ void __launch_bounds__(128, 8) step_kernel(const StepParams p) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if (i >= p.n || !p.alive[i]) return;
  const D3 o = d3(p.origin[3 * i], p.origin[3 * i + 1], p.origin[3 * i + 2]);
  D3 d = d3(p.dir[3 * i], p.dir[3 * i + 1], p.dir[3 * i + 2]);
  HitResult wall{0.0, -1};
  if (p.brute) {  // nearest_hit_brute, accel_tree.cpp:183-191
    for (int64_t f = 0; f < p.nf; ++f) {
      const double t = mt_delta(p.tri, static_cast<int32_t>(f), o, d);
      if (t > 0.0 && (wall.face < 0 || t < wall.delta)) {
        wall.delta = t;
        wall.face = static_cast<int32_t>(f);
      }
    }
  } else {
    wall = closest_hit_pl<16, -2, RegRay>(p.hdr, p.nodes, p.tri, RegRay{o, d}, -2);  // (the tracer's 16-node / register-stack tuning is slower here: one query per thread)
  }
  const int32_t nh = p.n_hist[i];
  const double sd = sphere_delta(o, d, d3(p.rc[0], p.rc[1], p.rc[2]), p.rr);
  bool cap = sd > 0.0 && (wall.face < 0 || sd < wall.delta);
  double L = 0.0;
  if (cap) {
    L = p.path[i] + sd;
    cap = L <= p.max_range;
  }
  const unsigned act = __activemask();
  const unsigned cm = __ballot_sync(act, cap);
  if (cm) {
    const int leader = __ffs(cm) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(p.cap_count, (unsigned long long)__popc(cm));
    base = __shfl_sync(act, base, leader);
    if (cap) {
      const unsigned long long slot = base + __popc(cm & ((1u << lane) - 1u));
      if (slot < static_cast<unsigned long long>(p.cap_capacity)) {
        Capture c;
        const D3 pt = o + sd * d;
        c.p[0] = pt.x; c.p[1] = pt.y; c.p[2] = pt.z;
        c.d[0] = d.x; c.d[1] = d.y; c.d[2] = d.z;
        c.path = L;
        c.ray = static_cast<int32_t>(i);
        c.meta = nh << 8;
        p.caps[slot] = c;
        for (int b = 0; b < kBands; ++b) p.cap_mult[kBands * slot + b] = p.mult[kBands * i + b];
        for (int j = 0; j < nh; ++j) p.cap_hist[slot * p.hist_cap + j] = p.hist[i * p.hist_cap + j];
      }
    }
  }
  if (wall.face < 0) {  // left the mesh
    p.alive[i] = 0;
    return;
  }
  const double* nn = p.normal + 3 * static_cast<int64_t>(wall.face);
  D3 n = d3(__ldg(nn), __ldg(nn + 1), __ldg(nn + 2));
  if (dot(n, d) > 0.0) n = d3(-n.x, -n.y, -n.z);
  const D3 pt = o + wall.delta * d;
  const double s2 = 2.0 * dot(d, n);
  d = d - s2 * n;  // reflect, tracer.hpp:33-37
  p.origin[3 * i] = pt.x; p.origin[3 * i + 1] = pt.y; p.origin[3 * i + 2] = pt.z;
  p.dir[3 * i] = d.x; p.dir[3 * i + 1] = d.y; p.dir[3 * i + 2] = d.z;
  const double path = p.path[i] + wall.delta;
  p.path[i] = path;
  const double* a = p.oma + kBands * p.mat[wall.face];
  for (int b = 0; b < kBands; ++b) p.mult[kBands * i + b] *= a[b];
  if (nh >= p.hist_cap) {
    atomicOr(p.bad, 1);
  } else {
    p.hist[i * p.hist_cap + nh] = wall.face;
    p.n_hist[i] = nh + 1;
  }
  if (path > p.max_range) p.alive[i] = 0;
}

// capture records -> SoA + CSR history for import_captures
__global__ void step_caps_kernel(const Capture* __restrict__ caps, int64_t n, int32_t hist_cap,
                                 const int32_t* __restrict__ cap_hist, const int64_t* __restrict__ off,
                                 int32_t* __restrict__ ray, double* __restrict__ point, double* __restrict__ dir,
                                 double* __restrict__ path, int32_t* __restrict__ hist) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const Capture c = caps[k];
  ray[k] = c.ray;
  for (int q = 0; q < 3; ++q) {
    point[3 * k + q] = c.p[q];
    dir[3 * k + q] = c.d[q];
  }
  path[k] = c.path;
  const int32_t len = static_cast<int32_t>(static_cast<uint32_t>(c.meta) >> 8);
  for (int j = 0; j < len; ++j) hist[off[k] + j] = cap_hist[k * hist_cap + j];
}

__global__ void step_len_kernel(const Capture* __restrict__ caps, int64_t n, int64_t* __restrict__ len) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) len[k] = static_cast<uint32_t>(caps[k].meta) >> 8;
  if (k == n) len[k] = 0;
}

template <typename T>
T* staged(DevBuf<T>& buf, T* src, int64_t count, cudaStream_t st, bool& on_device) {
  cudaPointerAttributes at{};
  RR_CUDA(cudaPointerGetAttributes(&at, src));
  on_device = at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
  if (on_device) return src;
  buf.alloc(std::max<int64_t>(count, 1), st);
  RR_CUDA(cudaMemcpyAsync(buf.p, src, sizeof(T) * count, cudaMemcpyHostToDevice, st));
  return buf.p;
}

template <typename T>
void unstage(const DevBuf<T>& buf, T* dst, int64_t count, bool on_device, cudaStream_t st) {
  if (!on_device) RR_CUDA(cudaMemcpyAsync(dst, buf.p, sizeof(T) * count, cudaMemcpyDeviceToHost, st));
}

}  // namespace

rr_trace_result* step_rays(rr_scene* s, int64_t n, double* origin, double* dir, double* mult, double* path,
                           int32_t* alive, int32_t* hist, int32_t* n_hist, int32_t hist_cap, const rr_receiver* recv,
                           const rr_trace_config* cfg, int32_t brute, float* kernel_ms) {
  if (n < 0) invalid("ray count must be >= 0");
  if (hist_cap < 1) invalid("hist_cap must be >= 1");
  if (!(recv->radius > 0.0)) invalid("receiver radius must be > 0");
  cudaStream_t st = s->ctx->stream;
  const bool sah = s->snodes.p != nullptr;
  if (!sah) ensure_reference_tree(s);
  StepParams p{};
  p.hdr = sah ? s->shdr : s->hdr;
  p.nodes = sah ? s->snodes.p : s->tnodes.p;
  p.tri = s->tri.p;
  p.nf = s->nf;
  p.normal = s->normal.p;
  p.mat = s->mat.p;
  p.oma = s->oma.p;
  p.n = n;
  p.hist_cap = hist_cap;
  for (int k = 0; k < 3; ++k) p.rc[k] = recv->center[k];
  p.rr = recv->radius;
  // resolved_max_range with the span's size as N (tracer.cpp:70-71)
  p.max_range = cfg->max_range > 0.0 ? cfg->max_range : 0.5 * recv->radius * std::sqrt(static_cast<double>(n));
  p.brute = brute;
  DevBuf<double> b_o, b_d, b_m, b_p;
  DevBuf<int32_t> b_a, b_h, b_nh;
  bool dev[7] = {true, true, true, true, true, true, true};
  if (n > 0) {
    p.origin = staged(b_o, origin, 3 * n, st, dev[0]);
    p.dir = staged(b_d, dir, 3 * n, st, dev[1]);
    p.mult = staged(b_m, mult, kBands * n, st, dev[2]);
    p.path = staged(b_p, path, n, st, dev[3]);
    p.alive = staged(b_a, alive, n, st, dev[4]);
    p.hist = staged(b_h, hist, n * static_cast<int64_t>(hist_cap), st, dev[5]);
    p.n_hist = staged(b_nh, n_hist, n, st, dev[6]);
  }
  DevBuf<unsigned long long> cnt;
  DevBuf<int32_t> bad;
  cnt.alloc(1, st);
  bad.alloc(1, st);
  DevBuf<Capture> caps;
  DevBuf<double> cap_mult;
  DevBuf<int32_t> cap_hist;
  int64_t capacity = std::max<int64_t>(1024, n / 8);
  unsigned long long nc = 0;
  cudaEvent_t e0, e1;
  RR_CUDA(cudaEventCreate(&e0));
  RR_CUDA(cudaEventCreate(&e1));
  // the kernel mutates the rays: keep a device copy to re-run after a capture overflow
  DevBuf<double> k_o, k_d, k_m, k_p;
  DevBuf<int32_t> k_a, k_h, k_nh;
  auto keep = [&](auto& dst, auto* src, int64_t count) {
    dst.alloc(std::max<int64_t>(count, 1), st);
    if (count > 0) RR_CUDA(cudaMemcpyAsync(dst.p, src, sizeof(*src) * count, cudaMemcpyDeviceToDevice, st));
  };
  if (n > 0) {
    keep(k_o, p.origin, 3 * n);
    keep(k_d, p.dir, 3 * n);
    keep(k_m, p.mult, kBands * n);
    keep(k_p, p.path, n);
    keep(k_a, p.alive, n);
    keep(k_nh, p.n_hist, n);
  }
  for (int attempt = 0; attempt < 2; ++attempt) {
    caps.alloc(capacity, st);
    cap_mult.alloc(kBands * capacity, st);
    cap_hist.alloc(capacity * static_cast<int64_t>(hist_cap), st);
    p.caps = caps.p;
    p.cap_mult = cap_mult.p;
    p.cap_hist = cap_hist.p;
    p.cap_count = cnt.p;
    p.cap_capacity = capacity;
    p.bad = bad.p;
    RR_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
    RR_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int32_t), st));
    RR_CUDA(cudaEventRecord(e0, st));
    if (n > 0) step_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(p);
    RR_LAUNCH_CHECK();
    RR_CUDA(cudaEventRecord(e1, st));
    s->ctx->launches++;
    RR_CUDA(cudaMemcpyAsync(&nc, cnt.p, sizeof nc, cudaMemcpyDeviceToHost, st));
    int hb = 0;
    RR_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof hb, cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
    if (hb) invalid("a ray's face history exceeds hist_cap");
    if (static_cast<int64_t>(nc) <= capacity) break;
    capacity = static_cast<int64_t>(nc);  // restore the rays and re-run with the exact size
    RR_CUDA(cudaMemcpyAsync(p.origin, k_o.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, st));
    RR_CUDA(cudaMemcpyAsync(p.dir, k_d.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, st));
    RR_CUDA(cudaMemcpyAsync(p.mult, k_m.p, sizeof(double) * kBands * n, cudaMemcpyDeviceToDevice, st));
    RR_CUDA(cudaMemcpyAsync(p.path, k_p.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    RR_CUDA(cudaMemcpyAsync(p.alive, k_a.p, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
    RR_CUDA(cudaMemcpyAsync(p.n_hist, k_nh.p, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
  }
  RR_CUDA(cudaEventElapsedTime(kernel_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (n > 0) {
    unstage(b_o, origin, 3 * n, dev[0], st);
    unstage(b_d, dir, 3 * n, dev[1], st);
    unstage(b_m, mult, kBands * n, dev[2], st);
    unstage(b_p, path, n, dev[3], st);
    unstage(b_a, alive, n, dev[4], st);
    unstage(b_h, hist, n * static_cast<int64_t>(hist_cap), dev[5], st);
    unstage(b_nh, n_hist, n, dev[6], st);
  }
  // captures -> CSR -> trace result (sorted by ray, as step returns them)
  const int64_t m = static_cast<int64_t>(nc);
  DevBuf<int64_t> len, off;
  len.alloc(m + 1, st);
  off.alloc(m + 1, st);
  DevBuf<int32_t> c_ray, c_hist;
  DevBuf<double> c_point, c_dir, c_path;
  c_ray.alloc(std::max<int64_t>(m, 1), st);
  c_point.alloc(3 * std::max<int64_t>(m, 1), st);
  c_dir.alloc(3 * std::max<int64_t>(m, 1), st);
  c_path.alloc(std::max<int64_t>(m, 1), st);
  step_len_kernel<<<static_cast<unsigned>((m + 256) / 256), 256, 0, st>>>(caps.p, m, len.p);
  size_t tb = 0;
  RR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, len.p, off.p, static_cast<int>(m + 1), st));
  DevBuf<uint8_t> tmp;
  tmp.alloc(tb, st);
  RR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, len.p, off.p, static_cast<int>(m + 1), st));
  int64_t th = 0;
  RR_CUDA(cudaMemcpyAsync(&th, off.p + m, sizeof th, cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  c_hist.alloc(std::max<int64_t>(th, 1), st);
  if (m > 0)
    step_caps_kernel<<<static_cast<unsigned>((m + 255) / 256), 256, 0, st>>>(
        caps.p, m, hist_cap, cap_hist.p, off.p, c_ray.p, c_point.p, c_dir.p, c_path.p, c_hist.p);
  RR_LAUNCH_CHECK();
  s->ctx->launches += 4;
  rr_trace_result* out = import_captures(s, m, nullptr, c_ray.p, c_point.p, c_dir.p, c_path.p, cap_mult.p, off.p,
                                         c_hist.p, recv, 1);
  out->stats.max_range = p.max_range;
  out->stats.n_rays = n;
  out->kernel_ms = *kernel_ms;
  return out;
}

}  // namespace rr
