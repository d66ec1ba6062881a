// Capture import: a trace result built from caller-held capture records.
//
// Used by (1) the multi-GPU exchange (shard.py): after the all-to-all of
// capture records each owner rank imports what it received and runs K5 on
// it; (2) the C++ facade's build_image_sources(const std::vector<Capture>&,
// ...) (image_sources.hpp:58-61), whose captures live on the host.
// Pointers may be host or device (UVA, cudaMemcpyDefault).  Records are put
// back into the reference order (receiver, ray index, path length;
// tracer.cpp:143-147) by a radix sort on (receiver, ray, order): captures of
// one ray are made at distinct steps, so order is monotone in path length.
#include <cub/cub.cuh>

#include <algorithm>
#include <memory>

#include "rr_trace.cuh"

namespace rr {
namespace {

__global__ void import_keys_kernel(const int32_t* __restrict__ recv, const int32_t* __restrict__ ray,
                                   const int64_t* __restrict__ off, int64_t n, int32_t n_recv,
                                   unsigned long long* __restrict__ keys, int32_t* __restrict__ idx,
                                   int* __restrict__ bad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t r = recv ? recv[i] : 0;
  const int64_t order = off[i + 1] - off[i];
  if (r < 0 || r >= n_recv || ray[i] < 0 || order < 0 || order >= (1 << 20)) atomicOr(bad, 1);
  keys[i] = (static_cast<unsigned long long>(r & 0xff) << 56) |
            (static_cast<unsigned long long>(static_cast<uint32_t>(ray[i])) << 20) |
            static_cast<unsigned long long>(order & 0xfffff);
  idx[i] = static_cast<int32_t>(i);
}

__global__ void import_len_kernel(const int32_t* __restrict__ perm, const int64_t* __restrict__ off, int64_t n,
                                  int64_t* __restrict__ len) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) len[i] = off[perm[i] + 1] - off[perm[i]];
  if (i == n) len[i] = 0;
}

__global__ void import_gather_kernel(const int32_t* __restrict__ perm, int64_t n, const int32_t* __restrict__ recv,
                                     const int32_t* __restrict__ ray, const double* __restrict__ point,
                                     const double* __restrict__ dir, const double* __restrict__ path,
                                     const double* __restrict__ mult, const int64_t* __restrict__ off,
                                     const int32_t* __restrict__ hist, const int64_t* __restrict__ new_off,
                                     int64_t nf, const int32_t* __restrict__ mat, const double* __restrict__ oma,
                                     int32_t* __restrict__ o_recv,
                                     int32_t* __restrict__ o_ray, double* __restrict__ o_point,
                                     double* __restrict__ o_dir, double* __restrict__ o_path,
                                     double* __restrict__ o_mult, int32_t* __restrict__ o_hist,
                                     int* __restrict__ bad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t s = perm[i];
  o_recv[i] = recv ? recv[s] : 0;
  o_ray[i] = ray[s];
  for (int k = 0; k < 3; ++k) {
    o_point[3 * i + k] = point[3 * s + k];
    o_dir[3 * i + k] = dir[3 * s + k];
  }
  o_path[i] = path[s];
  const int64_t a0 = off[s], len = off[s + 1] - a0, b0 = new_off[i];
  double m[kBands];
  for (int b = 0; b < kBands; ++b) m[b] = 1.0;
  for (int64_t j = 0; j < len; ++j) {
    const int32_t f = hist[a0 + j];
    o_hist[b0 + j] = f;
    if (!mult) {
      if (f < 0 || f >= nf) {
        atomicOr(bad, 2);
        continue;
      }
      // band multiplier = ordered product of (1 - alpha), tracer.cpp:57-58
      const double* a = oma + kBands * mat[f];
      for (int b = 0; b < kBands; ++b) m[b] *= a[b];
    }
  }
  for (int b = 0; b < kBands; ++b) o_mult[kBands * i + b] = mult ? mult[kBands * static_cast<int64_t>(s) + b] : m[b];
}

template <typename T>
const T* stage(DevBuf<T>& buf, const T* src, int64_t count, cudaStream_t st) {
  if (!src) return nullptr;
  buf.alloc(std::max<int64_t>(count, 1), st);
  if (count > 0) RR_CUDA(cudaMemcpyAsync(buf.p, src, sizeof(T) * count, cudaMemcpyDefault, st));
  return buf.p;
}

}  // namespace

rr_trace_result* import_captures(rr_scene* s, int64_t n, const int32_t* recv, const int32_t* ray, const double* point,
                                 const double* dir, const double* path, const double* mult, const int64_t* hist_off,
                                 const int32_t* hist, const rr_receiver* receivers, int32_t n_recv) {
  if (n < 0) invalid("capture count must be >= 0");
  if (n_recv < 1 || n_recv > kMaxRecv) invalid("n_recv must be in [1, 8]");
  for (int r = 0; r < n_recv; ++r)
    if (!(receivers[r].radius > 0.0)) invalid("receiver radius must be > 0");
  if (n >= (int64_t(1) << 31)) invalid("too many captures for one import (< 2^31)");
  cudaStream_t st = s->ctx->stream;
  auto res = std::make_unique<rr_trace_result>();
  res->scene = s;
  for (int r = 0; r < n_recv; ++r) {
    res->recv_center.insert(res->recv_center.end(), receivers[r].center, receivers[r].center + 3);
    res->recv_radius.push_back(receivers[r].radius);
  }
  res->c_off.alloc(n + 1, st);
  res->stats.n_captures = n;
  if (n == 0) {
    RR_CUDA(cudaMemsetAsync(res->c_off.p, 0, sizeof(int64_t), st));
    RR_CUDA(cudaStreamSynchronize(st));
    return res.release();
  }
  DevBuf<int32_t> b_recv, b_ray, b_hist;
  DevBuf<double> b_point, b_dir, b_path, b_mult;
  DevBuf<int64_t> b_off;
  const int64_t* d_off = stage(b_off, hist_off, n + 1, st);
  int64_t h0 = 0, h1 = 0;
  RR_CUDA(cudaMemcpyAsync(&h0, d_off, sizeof h0, cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaMemcpyAsync(&h1, d_off + n, sizeof h1, cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  if (h0 != 0 || h1 < 0) invalid("hist_off must start at 0 and be non-decreasing");
  const int32_t* d_recv = stage(b_recv, recv, n, st);
  const int32_t* d_ray = stage(b_ray, ray, n, st);
  const double* d_point = stage(b_point, point, 3 * n, st);
  const double* d_dir = stage(b_dir, dir, 3 * n, st);
  const double* d_path = stage(b_path, path, n, st);
  const double* d_mult = stage(b_mult, mult, kBands * n, st);
  const int32_t* d_hist = stage(b_hist, hist, h1, st);
  if (h1 > 0 && !d_hist) invalid("hist must not be NULL");

  DevBuf<unsigned long long> keys, keys_o;
  DevBuf<int32_t> idx, idx_o;
  DevBuf<int> bad;
  keys.alloc(n, st);
  keys_o.alloc(n, st);
  idx.alloc(n, st);
  idx_o.alloc(n, st);
  bad.alloc(1, st);
  RR_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  const unsigned g = static_cast<unsigned>((n + 255) / 256);
  import_keys_kernel<<<g, 256, 0, st>>>(d_recv, d_ray, d_off, n, n_recv, keys.p, idx.p, bad.p);
  RR_LAUNCH_CHECK();
  size_t tb = 0;
  RR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, keys_o.p, idx.p, idx_o.p, static_cast<int>(n), 0, 64,
                                          st));
  DevBuf<uint8_t> tmp;
  tmp.alloc(tb, st);
  RR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, keys_o.p, idx.p, idx_o.p, static_cast<int>(n), 0, 64,
                                          st));
  DevBuf<int64_t> len;
  len.alloc(n + 1, st);
  import_len_kernel<<<static_cast<unsigned>((n + 256) / 256), 256, 0, st>>>(idx_o.p, d_off, n, len.p);
  RR_LAUNCH_CHECK();
  tb = 0;
  RR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, len.p, res->c_off.p, static_cast<int>(n + 1), st));
  tmp.alloc(tb, st);
  RR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, len.p, res->c_off.p, static_cast<int>(n + 1), st));
  res->c_recv.alloc(n, st);
  res->c_ray.alloc(n, st);
  res->c_point.alloc(3 * n, st);
  res->c_dir.alloc(3 * n, st);
  res->c_path.alloc(n, st);
  res->c_mult.alloc(kBands * n, st);
  res->c_hist.alloc(std::max<int64_t>(h1, 1), st);
  import_gather_kernel<<<g, 256, 0, st>>>(idx_o.p, n, d_recv, d_ray, d_point, d_dir, d_path, d_mult, d_off, d_hist,
                                          res->c_off.p, s->nf, s->mat.p, s->oma.p, res->c_recv.p,
                                          res->c_ray.p, res->c_point.p, res->c_dir.p, res->c_path.p, res->c_mult.p,
                                          res->c_hist.p, bad.p);
  RR_LAUNCH_CHECK();
  s->ctx->launches += 7;
  int hb = 0;
  RR_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof hb, cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  if (hb & 1) invalid("capture records out of range (receiver, ray or path length)");
  if (hb & 2) invalid("capture face history holds a face index outside the mesh");
  res->stats.total_history = h1;
  return res.release();
}

}  // namespace rr
