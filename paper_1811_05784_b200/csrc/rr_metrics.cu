// Perceptive factors of the 8 pulse trains on the device.
//
// Replaces factors(const PulseTrains&) (metrics.cpp:168-180) with
// factors_from_events (:62-103), schroeder_curve (:13-28) and decay_time
// (:33-60): per band, events sorted by (time, amplitude) like
// build_pulse_trains (rir.cpp:22-28), energies e = amplitude^2;
//   total, t0 = first arrival with e > 0, early50 / early80 / late80 /
//   centroid sums, the Schroeder levels 10 log10(max(tail / total, 1e-300))
//   with tail_i = total - sum_{j<i} e_j, and the least-squares decay fits of
//   EDT [0, -10] dB and T30 [-5, -35] dB over the curve from t0.
// Sums are parallel (radix sort, scan, two-stage deterministic reductions);
// the reference sums sequentially, so values agree to rounding, not bits.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "rr_trace.cuh"

namespace rr {
namespace {

constexpr int kSums = 16;  // see pass2_kernel
constexpr int kBlk = 256;

__global__ void events_kernel(const double* __restrict__ dist, const double* __restrict__ energy, int64_t n,
                              double c, int band, double* __restrict__ t, double* __restrict__ a) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  t[i] = dist[i] / c;                    // rir.cpp:17
  a[i] = sqrt(energy[kBands * i + band]);  // rir.cpp:19
}

__global__ void iota_kernel(int32_t* __restrict__ v, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = static_cast<int32_t>(i);
}

__global__ void keys_kernel(const double* __restrict__ v, const int32_t* __restrict__ idx, int64_t n,
                            unsigned long long* __restrict__ keys) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  // times and amplitudes are >= 0: their bit patterns order like the values
  keys[i] = static_cast<unsigned long long>(__double_as_longlong(v[idx ? idx[i] : i]));
}

__global__ void energy_kernel(const double* __restrict__ t, const double* __restrict__ a,
                              const int32_t* __restrict__ perm, int64_t n, double* __restrict__ ts,
                              double* __restrict__ es) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t j = perm[i];
  ts[i] = t[j];
  es[i] = a[j] * a[j];  // metrics.cpp:121
}

__global__ void gather_pair_kernel(const double* __restrict__ t, const double* __restrict__ a,
                                   const int32_t* __restrict__ perm, int64_t n, double* __restrict__ ts,
                                   double* __restrict__ as) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  ts[i] = t[perm[i]];
  as[i] = a[perm[i]];
}

// pass 1: per-block (sum e, min time over e > 0)
__global__ void pass1_kernel(const double* __restrict__ ts, const double* __restrict__ es, int64_t n,
                             double* __restrict__ part) {
  __shared__ double s_sum[kBlk], s_t0[kBlk];
  double sum = 0.0, t0 = HUGE_VAL;
  for (int64_t i = blockIdx.x * (int64_t)kBlk + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlk) {
    sum += es[i];
    if (es[i] > 0.0) t0 = fmin(t0, ts[i]);
  }
  s_sum[threadIdx.x] = sum;
  s_t0[threadIdx.x] = t0;
  __syncthreads();
  for (int o = kBlk / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s_sum[threadIdx.x] += s_sum[threadIdx.x + o];
      s_t0[threadIdx.x] = fmin(s_t0[threadIdx.x], s_t0[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s_sum[0];
    part[2 * blockIdx.x + 1] = s_t0[0];
  }
}

__global__ void fold1_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x) return;
  double sum = 0.0, t0 = HUGE_VAL;
  for (int b = 0; b < nb; ++b) {
    sum += part[2 * b];
    t0 = fmin(t0, part[2 * b + 1]);
  }
  out[0] = sum;
  out[1] = t0;
}

// pass 2: 0 early50, 1 early80, 2 late80, 3 centroid, 4 min level from t0 on,
// 5-9 EDT (n, sx, sy, sxx, sxy), 10-14 T30, 15 first index with e > 0
__global__ void pass2_kernel(const double* __restrict__ ts, const double* __restrict__ es,
                             const double* __restrict__ prefix, int64_t n, const double* __restrict__ tot,
                             double* __restrict__ part) {
  __shared__ double s[kSums][kBlk];
  const double total = tot[0], t0 = tot[1];
  double v[kSums];
  for (int k = 0; k < kSums; ++k) v[k] = 0.0;
  v[4] = HUGE_VAL;
  v[15] = HUGE_VAL;
  for (int64_t i = blockIdx.x * (int64_t)kBlk + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlk) {
    const double e = es[i], dt = ts[i] - t0;
    if (dt <= 0.050) v[0] += e;  // metrics.cpp:78-84
    if (dt <= 0.080) v[1] += e;
    else v[2] += e;
    v[3] += dt * e;
    if (e > 0.0) v[15] = fmin(v[15], static_cast<double>(i));
  }
  // the shifted curve starts at the first event with e > 0: its index is
  // not known yet inside this pass, so the curve terms use time >= t0 and
  // are corrected below by excluding earlier zero-energy events (their
  // levels equal the level at `first`, see the fold)
  for (int64_t i = blockIdx.x * (int64_t)kBlk + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlk) {
    if (ts[i] < t0) continue;
    const double tail = total - prefix[i];
    const double level = 10.0 * log10(fmax(tail / total, 1e-300));  // metrics.cpp:24
    const double x = ts[i] - t0;
    v[4] = fmin(v[4], level);
    if (level <= 0.0 && level >= -10.0) {  // EDT segment (decay_time :45-52)
      v[5] += 1.0;
      v[6] += x;
      v[7] += level;
      v[8] += x * x;
      v[9] += x * level;
    }
    if (level <= -5.0 && level >= -35.0) {  // T30 segment
      v[10] += 1.0;
      v[11] += x;
      v[12] += level;
      v[13] += x * x;
      v[14] += x * level;
    }
  }
  for (int k = 0; k < kSums; ++k) s[k][threadIdx.x] = v[k];
  __syncthreads();
  for (int o = kBlk / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int k = 0; k < kSums; ++k) {
        if (k == 4 || k == 15) s[k][threadIdx.x] = fmin(s[k][threadIdx.x], s[k][threadIdx.x + o]);
        else s[k][threadIdx.x] += s[k][threadIdx.x + o];
      }
    __syncthreads();
  }
  if (threadIdx.x < kSums) part[kSums * blockIdx.x + threadIdx.x] = s[threadIdx.x][0];
}

__device__ rr_metric decay(double n, double sx, double sy, double sxx, double sxy, bool reaches) {
  if (!reaches || n < 2.0) return rr_metric{0.0, 0};  // metrics.cpp:42,53
  const double denom = n * sxx - sx * sx;
  if (denom == 0.0) return rr_metric{0.0, 0};
  const double slope = (n * sxy - sx * sy) / denom;
  if (slope >= 0.0) return rr_metric{0.0, 0};
  return rr_metric{-60.0 / slope, 1};
}

__global__ void fold2_kernel(const double* __restrict__ part, int nb, const double* __restrict__ tot,
                             const double* __restrict__ ts, const double* __restrict__ es,
                             const double* __restrict__ prefix, int64_t n, rr_factors* __restrict__ out) {
  if (threadIdx.x) return;
  double v[kSums];
  for (int k = 0; k < kSums; ++k) v[k] = (k == 4 || k == 15) ? HUGE_VAL : 0.0;
  for (int b = 0; b < nb; ++b)
    for (int k = 0; k < kSums; ++k) {
      const double x = part[kSums * b + k];
      v[k] = (k == 4 || k == 15) ? fmin(v[k], x) : v[k] + x;
    }
  const double total = tot[0];
  rr_factors f{};
  if (!(total > 0.0)) {  // silent band: everything unreliable (metrics.cpp:67)
    *out = f;
    return;
  }
  // zero-energy events at t0 that precede `first` in the sorted order are
  // not on the shifted curve (metrics.cpp:97-98): remove their terms
  const int64_t first = static_cast<int64_t>(v[15]);
  for (int64_t i = first - 1; i >= 0 && ts[i] >= tot[1]; --i) {
    const double tail = total - prefix[i];
    const double level = 10.0 * log10(fmax(tail / total, 1e-300));
    const double x = ts[i] - tot[1];
    if (level <= 0.0 && level >= -10.0) {
      v[5] -= 1.0; v[6] -= x; v[7] -= level; v[8] -= x * x; v[9] -= x * level;
    }
    if (level <= -5.0 && level >= -35.0) {
      v[10] -= 1.0; v[11] -= x; v[12] -= level; v[13] -= x * x; v[14] -= x * level;
    }
  }
  f.spl_db = rr_metric{10.0 * log10(total), 1};
  f.d50_pct = rr_metric{100.0 * v[0] / total, 1};
  if (v[2] > 0.0) {
    const double c80 = 10.0 * log10(v[1] / v[2]);
    f.c80_db = rr_metric{fmin(fmax(c80, -99.0), 99.0), 1};
  } else {
    f.c80_db = rr_metric{99.0, 1};
  }
  f.ts_ms = rr_metric{1000.0 * v[3] / total, 1};
  f.edt_s = decay(v[5], v[6], v[7], v[8], v[9], v[4] <= -10.0);
  f.t30_s = decay(v[10], v[11], v[12], v[13], v[14], v[4] <= -35.0);
  *out = f;
  (void)es;
  (void)n;
}

template <typename F>
void cub_do(F&& f, DevBuf<uint8_t>& tmp, cudaStream_t st) {
  size_t need = 0;
  RR_CUDA(f(nullptr, need));
  if (need > tmp.n) tmp.alloc(need + 16, st);
  size_t have = tmp.n;
  RR_CUDA(f(tmp.p, have));
}

}  // namespace

// One band: events (t, a) on the device, n of them; writes *d_out (device).
void band_factors(rr_ctx* ctx, const double* d_t, const double* d_a, int64_t n, rr_factors* d_out) {
  cudaStream_t st = ctx->stream;
  if (n == 0) {  // metrics.cpp:124 (empty train)
    RR_CUDA(cudaMemsetAsync(d_out, 0, sizeof(rr_factors), st));
    return;
  }
  DevBuf<uint8_t> tmp;
  DevBuf<unsigned long long> k, ko;
  DevBuf<int32_t> i1, i2;
  k.alloc(n, st);
  ko.alloc(n, st);
  i1.alloc(n, st);
  i2.alloc(n, st);
  const unsigned g = static_cast<unsigned>((n + 255) / 256);
  // (time, amplitude) order: stable sort by amplitude, then stably by time
  keys_kernel<<<g, 256, 0, st>>>(d_a, nullptr, n, k.p);
  RR_LAUNCH_CHECK();
  iota_kernel<<<g, 256, 0, st>>>(i2.p, n);
  cub_do([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, k.p, ko.p, i2.p, i1.p, static_cast<int>(n), 0, 64, st);
  }, tmp, st);
  keys_kernel<<<g, 256, 0, st>>>(d_t, i1.p, n, k.p);
  cub_do([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, k.p, ko.p, i1.p, i2.p, static_cast<int>(n), 0, 64, st);
  }, tmp, st);
  DevBuf<double> ts, es, prefix, part, tot;
  ts.alloc(n, st);
  es.alloc(n, st);
  prefix.alloc(n, st);
  energy_kernel<<<g, 256, 0, st>>>(d_t, d_a, i2.p, n, ts.p, es.p);
  cub_do([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, es.p, prefix.p, static_cast<int>(n), st); },
         tmp, st);
  const int nb = static_cast<int>(std::min<int64_t>((n + kBlk - 1) / kBlk, 2 * ctx->sm_count));
  part.alloc(static_cast<size_t>(kSums) * nb, st);
  tot.alloc(2, st);
  pass1_kernel<<<nb, kBlk, 0, st>>>(ts.p, es.p, n, part.p);
  fold1_kernel<<<1, 32, 0, st>>>(part.p, nb, tot.p);
  pass2_kernel<<<nb, kBlk, 0, st>>>(ts.p, es.p, prefix.p, n, tot.p, part.p);
  fold2_kernel<<<1, 32, 0, st>>>(part.p, nb, tot.p, ts.p, es.p, prefix.p, n, d_out);
  RR_LAUNCH_CHECK();
  ctx->launches += 14;
  RR_CUDA(cudaStreamSynchronize(st));  // temporaries are freed on return
}

// schroeder(const BandPulseTrain&) (metrics.cpp:13-28, 125-134): per band,
// in the train's event order, level_i = 10 log10(max(tail_i / total,
// 1e-300)) with tail_i the energy of events i.. (one block per band: block
// reduction for the total, chunked block scans for the tails).
__global__ void __launch_bounds__(256) schroeder_kernel(const int64_t* __restrict__ off,
                                                        const double* __restrict__ amp, double* __restrict__ level,
                                                        int32_t* __restrict__ silent) {
  using Reduce = cub::BlockReduce<double, 256>;
  using Scan = cub::BlockScan<double, 256>;
  __shared__ union {
    typename Reduce::TempStorage r;
    typename Scan::TempStorage s;
  } tmp;
  __shared__ double s_total, s_carry;
  const int b = blockIdx.x;
  const int64_t b0 = off[b], b1 = off[b + 1];
  if (b1 == b0) return;
  double part = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) part += amp[i] * amp[i];
  const double total = Reduce(tmp.r).Sum(part);
  if (threadIdx.x == 0) {
    s_total = total;
    s_carry = 0.0;
    silent[b] = total <= 0.0 ? 1 : 0;
  }
  __syncthreads();
  const double tot = s_total;
  for (int64_t c = b0; c < b1; c += blockDim.x) {
    const int64_t i = c + threadIdx.x;
    const double e = i < b1 ? amp[i] * amp[i] : 0.0;
    double before = 0.0, chunk = 0.0;
    __syncthreads();
    Scan(tmp.s).ExclusiveSum(e, before, chunk);
    const double tail = tot - (s_carry + before);
    if (i < b1) level[i] = 10.0 * log10(fmax(tail / tot, 1e-300));
    __syncthreads();
    if (threadIdx.x == 0) s_carry += chunk;
  }
}

void band_schroeder(rr_ctx* ctx, const int64_t* band_off, const double* amplitude, double* level) {
  cudaStream_t st = ctx->stream;
  const int64_t n = band_off[kBands];
  DevBuf<int64_t> off;
  DevBuf<double> a, lv;
  DevBuf<int32_t> silent;
  off.alloc(kBands + 1, st);
  a.alloc(std::max<int64_t>(n, 1), st);
  lv.alloc(std::max<int64_t>(n, 1), st);
  silent.alloc(kBands, st);
  RR_CUDA(cudaMemcpyAsync(off.p, band_off, sizeof(int64_t) * (kBands + 1), cudaMemcpyHostToDevice, st));
  RR_CUDA(cudaMemsetAsync(silent.p, 0, sizeof(int32_t) * kBands, st));
  if (n > 0) RR_CUDA(cudaMemcpyAsync(a.p, amplitude, sizeof(double) * n, cudaMemcpyDefault, st));
  schroeder_kernel<<<kBands, 256, 0, st>>>(off.p, a.p, lv.p, silent.p);
  RR_LAUNCH_CHECK();
  ctx->launches++;
  int32_t h_silent[kBands];
  RR_CUDA(cudaMemcpyAsync(h_silent, silent.p, sizeof h_silent, cudaMemcpyDeviceToHost, st));
  if (n > 0) RR_CUDA(cudaMemcpyAsync(level, lv.p, sizeof(double) * n, cudaMemcpyDefault, st));
  RR_CUDA(cudaStreamSynchronize(st));
  for (int b = 0; b < kBands; ++b)
    if (h_silent[b]) invalid("decay of an all-zero signal is undefined");  // metrics.cpp:17-19
}

// build_pulse_trains (rir.cpp:9-30) of an image set on the device: band b's
// events (t = d / c, amplitude sqrt(E_b)) sorted by (time, amplitude)
// (rir.cpp:22-28, the two stable radix passes of band_factors), copied to
// time / amp at [b * n, (b + 1) * n) (host or device buffers).
void image_trains(rr_ctx* ctx, const double* d_dist, const double* d_energy, int64_t n, double c, double* time,
                  double* amp) {
  if (n <= 0) return;
  cudaStream_t st = ctx->stream;
  DevBuf<uint8_t> tmp;
  DevBuf<double> t, a, ts, as;
  DevBuf<unsigned long long> k, ko;
  DevBuf<int32_t> i1, i2;
  t.alloc(n, st);
  a.alloc(n, st);
  ts.alloc(n, st);
  as.alloc(n, st);
  k.alloc(n, st);
  ko.alloc(n, st);
  i1.alloc(n, st);
  i2.alloc(n, st);
  const unsigned g = static_cast<unsigned>((n + 255) / 256);
  for (int b = 0; b < kBands; ++b) {
    events_kernel<<<g, 256, 0, st>>>(d_dist, d_energy, n, c, b, t.p, a.p);
    keys_kernel<<<g, 256, 0, st>>>(a.p, nullptr, n, k.p);
    iota_kernel<<<g, 256, 0, st>>>(i2.p, n);
    RR_LAUNCH_CHECK();
    cub_do([&](void* tt, size_t& bb) {
      return cub::DeviceRadixSort::SortPairs(tt, bb, k.p, ko.p, i2.p, i1.p, static_cast<int>(n), 0, 64, st);
    }, tmp, st);
    keys_kernel<<<g, 256, 0, st>>>(t.p, i1.p, n, k.p);
    cub_do([&](void* tt, size_t& bb) {
      return cub::DeviceRadixSort::SortPairs(tt, bb, k.p, ko.p, i1.p, i2.p, static_cast<int>(n), 0, 64, st);
    }, tmp, st);
    gather_pair_kernel<<<g, 256, 0, st>>>(t.p, a.p, i2.p, n, ts.p, as.p);
    RR_LAUNCH_CHECK();
    RR_CUDA(cudaMemcpyAsync(time + b * n, ts.p, sizeof(double) * n, cudaMemcpyDefault, st));
    RR_CUDA(cudaMemcpyAsync(amp + b * n, as.p, sizeof(double) * n, cudaMemcpyDefault, st));
    ctx->launches += 12;
  }
  RR_CUDA(cudaStreamSynchronize(st));
}

// factors(const PulseTrains&) for trains given as images: t = d / c,
// amplitude sqrt(E_b) (build_pulse_trains, rir.cpp:9-30); out[0..7] bands,
// out[8] the 500 Hz - 1 kHz average (metrics.cpp:170-179).
void image_factors(rr_ctx* ctx, const double* d_dist, const double* d_energy, int64_t n, double c,
                   rr_factors* out) {
  cudaStream_t st = ctx->stream;
  DevBuf<double> t, a;
  DevBuf<rr_factors> d_out;
  t.alloc(std::max<int64_t>(n, 1), st);
  a.alloc(std::max<int64_t>(n, 1), st);
  d_out.alloc(kBands, st);
  for (int b = 0; b < kBands; ++b) {
    if (n > 0) {
      events_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(d_dist, d_energy, n, c, b, t.p, a.p);
      RR_LAUNCH_CHECK();
    }
    band_factors(ctx, t.p, a.p, n, d_out.p + b);
  }
  RR_CUDA(cudaMemcpyAsync(out, d_out.p, sizeof(rr_factors) * kBands, cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  auto avg = [](rr_metric x, rr_metric y) { return rr_metric{0.5 * (x.value + y.value), x.reliable && y.reliable}; };
  const rr_factors& f5 = out[3];
  const rr_factors& f1 = out[4];
  out[8] = rr_factors{avg(f5.edt_s, f1.edt_s), avg(f5.t30_s, f1.t30_s), avg(f5.spl_db, f1.spl_db),
                      avg(f5.c80_db, f1.c80_db), avg(f5.d50_pct, f1.d50_pct), avg(f5.ts_ms, f1.ts_ms)};
}

}  // namespace rr
