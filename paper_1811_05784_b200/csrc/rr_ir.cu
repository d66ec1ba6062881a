// K6 + K7 — impulse-response synthesis.
//
// Replaces build_pulse_trains (rir.cpp:9-30), design_band_filter
// (rir.cpp:32-58) and synthesize (rir.cpp:60-96).  The reference scatters
// every event through all taps (amp * kernel[n] at lround(t*fs) + n - delay).
// That is the convolution of the per-band pulse histogram h_b[c] = sum of
// amplitudes sqrt(E_b) of events with lround(t*fs) == c, with the band
// kernel; here the histogram is built first (K6: 64-bit fixed-point atomics,
// deterministic and order-independent), then convolved (K7: fp64 direct FIR,
// register-blocked sliding window in shared memory).  Linear, so per-GPU
// histograms can be summed (NCCL) before one FIR pass.
#include <cmath>

#include "rr_internal.cuh"

namespace rr {
namespace {

__constant__ double kCentersHz[kBands] = {62.5, 125.0, 250.0, 500.0, 1000.0, 2000.0, 4000.0, 8000.0};

__global__ void max_amp_kernel(const double* __restrict__ energy, int64_t n8, unsigned long long* __restrict__ out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, sqrt(fmax(energy[i], 0.0)));
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// scale = 2^s with n * max_amp * 2^s < 2^62
__device__ __forceinline__ double fixed_scale(unsigned long long max_bits, int64_t n) {
  const double m = __longlong_as_double(static_cast<long long>(max_bits));
  const double worst = fmax(m * static_cast<double>(n), 1e-300);
  int e;
  frexp(worst, &e);  // worst < 2^e
  return ldexp(1.0, 62 - e);
}

// K6: pulse histogram (build_pulse_trains + the lround(t*fs) centring of
// synthesize rir.cpp:86).
// The fixed-point scale depends on (max amplitude, n_scale) only: ranks that
// bin their shares with the global values produce integer histograms whose
// exact sum equals the single-GPU histogram (rr_shard.cu).
__global__ void bin_kernel(const double* __restrict__ dist, const double* __restrict__ energy, int64_t n, double c,
                           double fs, int64_t lh, const unsigned long long* __restrict__ max_bits, int64_t n_scale,
                           unsigned long long* __restrict__ acc) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double scale = fixed_scale(*max_bits, n_scale);
  const double t = dist[i] / c;
  const long long center = llround(t * fs);
  if (center < 0 || center >= lh) return;
  for (int b = 0; b < kBands; ++b) {
    const double a = sqrt(energy[kBands * i + b]);
    const unsigned long long q = static_cast<unsigned long long>(llrint(a * scale));
    if (q) atomicAdd(acc + b * lh + center, q);
  }
}

__global__ void unfix_kernel(const unsigned long long* __restrict__ acc, int64_t total, int64_t n,
                             const unsigned long long* __restrict__ max_bits, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= total) return;
  const double scale = fixed_scale(*max_bits, n);
  out[i] = static_cast<double>(acc[i]) / scale;
}

// Pulse trains given as events (build_pulse_trains output, rir.hpp:12-23):
// band b owns events [off[b], off[b+1]) with times t and amplitudes a.
__global__ void max_abs_kernel(const double* __restrict__ a, int64_t n, unsigned long long* __restrict__ out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(a[i]));
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__global__ void bin_events_kernel(const int64_t* __restrict__ off, const double* __restrict__ time,
                                  const double* __restrict__ amp, int64_t n, double fs, int64_t lh,
                                  const unsigned long long* __restrict__ max_bits,
                                  unsigned long long* __restrict__ pos, unsigned long long* __restrict__ neg) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int b = 0;
  while (b < kBands - 1 && i >= off[b + 1]) ++b;
  const double scale = fixed_scale(*max_bits, n);
  const long long center = llround(time[i] * fs);  // rir.cpp:86
  if (center < 0 || center >= lh) return;
  const double a = amp[i];
  const unsigned long long q = static_cast<unsigned long long>(llrint(fabs(a) * scale));
  if (q) atomicAdd((a < 0.0 ? neg : pos) + b * lh + center, q);
}

__global__ void unfix2_kernel(const unsigned long long* __restrict__ pos, const unsigned long long* __restrict__ neg,
                              int64_t total, int64_t n, const unsigned long long* __restrict__ max_bits,
                              double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= total) return;
  const double scale = fixed_scale(*max_bits, n);
  out[i] = static_cast<double>(pos[i]) / scale - static_cast<double>(neg[i]) / scale;
}

// design_band_filter rir.cpp:32-58 with `taps` taps, delay (taps-1)/2.
__global__ void design_kernel(double fs, int taps, double* __restrict__ k) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kBands * taps) return;
  const int b = i / taps, n = i - b * taps;
  const double fl = kCentersHz[b] / sqrt(2.0), fh = kCentersHz[b] * sqrt(2.0);
  const int delay = (taps - 1) / 2;
  const int m = n - delay;
  double ideal;
  if (m == 0)
    ideal = 2.0 * (fh - fl) / fs;
  else
    ideal = (sin(2.0 * M_PI * fh * m / fs) - sin(2.0 * M_PI * fl * m / fs)) / (M_PI * m);
  const double hann = 0.5 * (1.0 - cos(2.0 * M_PI * n / (taps - 1)));
  k[i] = ideal * hann;
}

constexpr int kFirTile = 512;  // outputs per block
constexpr int kFirR = 4;       // outputs per thread
constexpr int kFirThreads = kFirTile / kFirR;

// K7: out_b[j] = sum_n h_b[j - n + delay] * k_b[n], j in [0, L).
// Thread t owns outputs j0 + t*R + r; the h window slides down one sample per
// tap so each tap costs one shared load of h, one broadcast of k and R FMAs.
__global__ void __launch_bounds__(kFirThreads) fir_kernel(const double* __restrict__ hist, int64_t lh,
                                                          const double* __restrict__ kern, int taps, int64_t L,
                                                          double* __restrict__ band_ir) {
  extern __shared__ double sm[];
  double* ks = sm;             // taps
  double* hs = sm + taps;      // kFirTile + taps
  const int b = blockIdx.y;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * kFirTile;
  const int delay = (taps - 1) / 2;
  const double* h = hist + b * lh;
  for (int i = threadIdx.x; i < taps; i += blockDim.x) ks[i] = kern[b * taps + i];
  // hs[u] = h[j0 + delay - (taps - 1) + u], u in [0, kFirTile + taps - 1)
  const int64_t base = j0 + delay - (taps - 1);
  for (int u = threadIdx.x; u < kFirTile + taps - 1; u += blockDim.x) {
    const int64_t c = base + u;
    hs[u] = (c >= 0 && c < lh) ? h[c] : 0.0;
  }
  __syncthreads();
  const int jl = threadIdx.x * kFirR;  // local output index of r = 0
  // output jl + r at tap n reads hs[jl + r + (taps - 1) - n]
  double acc[kFirR];
  double win[kFirR];
  for (int r = 0; r < kFirR; ++r) {
    acc[r] = 0.0;
    win[r] = hs[jl + r + (taps - 1)];
  }
  for (int n = 0; n < taps; ++n) {
    const double kn = ks[n];
    for (int r = 0; r < kFirR; ++r) acc[r] = fma(win[r], kn, acc[r]);
    // slide: next tap reads one sample earlier
    for (int r = kFirR - 1; r > 0; --r) win[r] = win[r - 1];
    const int u = jl + (taps - 1) - n - 1;
    win[0] = u >= 0 ? hs[u] : 0.0;
  }
  for (int r = 0; r < kFirR; ++r) {
    const int64_t j = j0 + jl + r;
    if (j < L) band_ir[b * L + j] = acc[r];
  }
}

__global__ void sum_bands_kernel(const double* __restrict__ band_ir, int64_t L, double* __restrict__ out) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= L) return;
  double s = 0.0;
  for (int b = 0; b < kBands; ++b) s += band_ir[b * L + j];
  out[j] = s;
}

void check_fs(double fs, int taps) {
  if (taps < 3) invalid("taps must be >= 3");
  if (fs < 2.0 * 8000.0 * std::sqrt(2.0)) invalid("sample rate too low for the top band edge");
}

}  // namespace

// Histogram of pulse trains: d_hist has 8 * lh entries, lh = length + taps.
void ir_bin(rr_ctx* ctx, int64_t n, const double* d_dist, const double* d_energy, double c, double fs, int64_t lh,
            double* d_hist) {
  cudaStream_t st = ctx->stream;
  DevBuf<unsigned long long> acc, mx;
  acc.alloc(kBands * lh, st);
  mx.alloc(1, st);
  RR_CUDA(cudaMemsetAsync(acc.p, 0, acc.bytes(), st));
  RR_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(unsigned long long), st));
  ir_max_amp(ctx, n, d_energy, mx.p);
  ir_bin_fixed(ctx, n, d_dist, d_energy, c, fs, lh, mx.p, std::max<int64_t>(n, 1), acc.p);
  ir_unfix(ctx, acc.p, kBands * lh, std::max<int64_t>(n, 1), mx.p, d_hist);
}

// The three phases of ir_bin, for the multi-GPU pipeline: the max amplitude
// (max-reduced over ranks), the fixed-point binning with the global scale
// (sum-reduced over ranks, exact), the conversion back to fp64.
void ir_max_amp(rr_ctx* ctx, int64_t n, const double* d_energy, unsigned long long* d_max) {
  if (n <= 0) return;
  max_amp_kernel<<<592, 256, 0, ctx->stream>>>(d_energy, kBands * n, d_max);
  RR_LAUNCH_CHECK();
  ctx->launches++;
}

void ir_bin_fixed(rr_ctx* ctx, int64_t n, const double* d_dist, const double* d_energy, double c, double fs,
                  int64_t lh, const unsigned long long* d_max, int64_t n_scale, unsigned long long* d_acc) {
  if (n <= 0) return;
  bin_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(d_dist, d_energy, n, c, fs, lh, d_max,
                                                                              n_scale, d_acc);
  RR_LAUNCH_CHECK();
  ctx->launches++;
}

void ir_unfix(rr_ctx* ctx, const unsigned long long* d_acc, int64_t total, int64_t n_scale,
              const unsigned long long* d_max, double* d_hist) {
  unfix_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, ctx->stream>>>(d_acc, total, n_scale, d_max,
                                                                                     d_hist);
  RR_LAUNCH_CHECK();
  ctx->launches++;
}

// Histogram of explicit pulse trains (times in seconds, signed amplitudes).
void ir_bin_events(rr_ctx* ctx, const int64_t* d_off, int64_t n, const double* d_time, const double* d_amp, double fs,
                   int64_t lh, double* d_hist) {
  cudaStream_t st = ctx->stream;
  DevBuf<unsigned long long> pos, neg, mx;
  pos.alloc(kBands * lh, st);
  neg.alloc(kBands * lh, st);
  mx.alloc(1, st);
  RR_CUDA(cudaMemsetAsync(pos.p, 0, pos.bytes(), st));
  RR_CUDA(cudaMemsetAsync(neg.p, 0, neg.bytes(), st));
  RR_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(unsigned long long), st));
  if (n > 0) {
    max_abs_kernel<<<592, 256, 0, st>>>(d_amp, n, mx.p);
    RR_LAUNCH_CHECK();
    bin_events_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(d_off, d_time, d_amp, n, fs, lh, mx.p,
                                                                              pos.p, neg.p);
    RR_LAUNCH_CHECK();
    ctx->launches += 2;
  }
  unfix2_kernel<<<static_cast<unsigned>((kBands * lh + 255) / 256), 256, 0, st>>>(pos.p, neg.p, kBands * lh,
                                                                                   std::max<int64_t>(n, 1), mx.p,
                                                                                   d_hist);
  RR_LAUNCH_CHECK();
  ctx->launches++;
}

void ir_filter(rr_ctx* ctx, const double* d_hist, int64_t lh, double fs, int taps, int64_t L, double* d_band_ir,
               double* d_broadband) {
  check_fs(fs, taps);
  cudaStream_t st = ctx->stream;
  DevBuf<double> kern;
  kern.alloc(kBands * taps, st);
  design_kernel<<<static_cast<unsigned>((kBands * taps + 255) / 256), 256, 0, st>>>(fs, taps, kern.p);
  RR_LAUNCH_CHECK();
  DevBuf<double> tmp;
  double* bands = d_band_ir;
  if (!bands) {
    tmp.alloc(kBands * L, st);
    bands = tmp.p;
  }
  const size_t smem = sizeof(double) * (taps + kFirTile + taps);
  RR_CUDA(cudaFuncSetAttribute(fir_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  dim3 grid(static_cast<unsigned>((L + kFirTile - 1) / kFirTile), kBands);
  fir_kernel<<<grid, kFirThreads, smem, st>>>(d_hist, lh, kern.p, taps, L, bands);
  RR_LAUNCH_CHECK();
  ctx->launches += 2;
  if (d_broadband) {
    sum_bands_kernel<<<static_cast<unsigned>((L + 255) / 256), 256, 0, st>>>(bands, L, d_broadband);
    RR_LAUNCH_CHECK();
    ctx->launches++;
  }
}

void band_filter_host(int band, double fs, int taps, double* out, rr_ctx* ctx) {
  check_fs(fs, taps);
  if (band < 0 || band >= kBands) invalid("band index out of range");
  cudaStream_t st = ctx->stream;
  DevBuf<double> kern;
  kern.alloc(kBands * taps, st);
  design_kernel<<<static_cast<unsigned>((kBands * taps + 255) / 256), 256, 0, st>>>(fs, taps, kern.p);
  RR_LAUNCH_CHECK();
  ctx->launches++;
  RR_CUDA(cudaMemcpyAsync(out, kern.p + band * taps, sizeof(double) * taps, cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
}

}  // namespace rr
