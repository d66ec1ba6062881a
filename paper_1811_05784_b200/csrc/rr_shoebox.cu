// Rectangular-room mirror-lattice check on the device (shoebox.hpp,
// shoebox.cpp:43-182): enumerate_images and compare.
//
// enumerate_images: one thread per lattice cell (mx, my, mz) in
// [-span, span]^3, span = ceil(max_distance / L) + 1 per axis.  A cell is kept
// when its image lies within max_distance of the receiver; kept cells are
// compacted in linear (= lexicographic (mx, my, mz)) order and then stably
// radix-sorted by distance, which is the reference's sort by (distance, cell)
// (shoebox.cpp:107-112).  Positions, distances, orders and wall hits repeat
// the reference's arithmetic in its operation order (-fmad=false), so they
// are bit-identical; energies use the device exp (within 2 ulp of glibc).
//
// compare: the reference matches every traced image against every oracle
// image (O(T * O), shoebox.cpp:133-149), infeasible at 10^7 lattice images.
// Here the oracle images are hashed into cells of side h = 2 * pos_tol; a
// traced image scans the 27 cells around its own, so every oracle image
// within pos_tol is seen.  The selection rule is the reference's: the
// smallest distance <= pos_tol, the largest oracle index on ties (its loop
// replaces on `dist <= best_dist`).  Members of an oracle image stay in
// traced order (stable sort), energies are summed in that order, and the rms
// is a sequential sum in oracle order, as in shoebox.cpp:152-180.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cmath>
#include <limits>

#include "rr_trace.cuh"

namespace rr {
namespace {

constexpr int kWalls = 6;

struct LatticeParams {
  double L[3], s[3], r[3];
  double max_distance, radius;
  int span[3], n[3];
  double beta[kBands];
  double oma[kWalls][kBands];  // 1 - alpha per wall (shoebox.cpp:59-62)
};

// unfolded_coordinate (shoebox.cpp:20-24); C++ `%` keeps the sign, so odd
// negative cells take the second branch exactly as on the host.
__device__ __forceinline__ double unfolded(int m, double L, double s) {
  if (m % 2 == 0) return m * L + s;
  return (m + 1) * L - s;
}

// axis_wall_hits (shoebox.cpp:29-38).
__device__ __forceinline__ void wall_hits(int m, int& lower, int& upper) {
  const int c = m < 0 ? -m : m;
  if (m > 0) {
    upper = (c + 1) / 2;
    lower = c / 2;
  } else {
    lower = (c + 1) / 2;
    upper = c / 2;
  }
}

__device__ __forceinline__ void cell_of(const LatticeParams& p, int32_t i, int m[3]) {
  const int iz = i % p.n[2];
  const int rest = i / p.n[2];
  m[0] = rest / p.n[1] - p.span[0];
  m[1] = rest % p.n[1] - p.span[1];
  m[2] = iz - p.span[2];
}

__device__ __forceinline__ double image_distance(const LatticeParams& p, const int m[3], D3& pos) {
  pos = d3(unfolded(m[0], p.L[0], p.s[0]), unfolded(m[1], p.L[1], p.s[1]), unfolded(m[2], p.L[2], p.s[2]));
  const D3 v = pos - d3(p.r[0], p.r[1], p.r[2]);
  return sqrt(dot(v, v));  // (position - receiver).norm()
}

struct InRange {
  LatticeParams p;
  __device__ bool operator()(int32_t i) const {
    int m[3];
    cell_of(p, i, m);
    D3 pos;
    return !(image_distance(p, m, pos) > p.max_distance);  // shoebox.cpp:84
  }
};

__global__ void lattice_dist_kernel(LatticeParams p, const int32_t* __restrict__ cells, int64_t n,
                                    unsigned long long* __restrict__ key) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int m[3];
  cell_of(p, cells[k], m);
  D3 pos;
  key[k] = __double_as_longlong(image_distance(p, m, pos));  // d >= 0: bits order like values
}

__global__ void lattice_fill_kernel(LatticeParams p, const int32_t* __restrict__ cells, int64_t n,
                                    double* __restrict__ pos, double* __restrict__ dist, int32_t* __restrict__ order,
                                    int32_t* __restrict__ hits, double* __restrict__ energy) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int m[3];
  cell_of(p, cells[k], m);
  D3 x;
  const double d = image_distance(p, m, x);
  int h[kWalls];
  for (int a = 0; a < 3; ++a) wall_hits(m[a], h[2 * a], h[2 * a + 1]);
  int ord = 0;
  for (int w = 0; w < kWalls; ++w) {
    ord += h[w];
    hits[kWalls * k + w] = h[w];
  }
  pos[3 * k] = x.x;
  pos[3 * k + 1] = x.y;
  pos[3 * k + 2] = x.z;
  dist[k] = d;
  order[k] = ord;
  // E = r^2 / (4 d^2) * exp(-beta d) * prod_w (1 - alpha_w)^hits_w, in the
  // reference's order (shoebox.cpp:91-100)
  const double e0 = p.radius * p.radius / (4.0 * d * d);
  for (int b = 0; b < kBands; ++b) {
    double e = e0 * exp(-p.beta[b] * d);
    for (int w = 0; w < kWalls; ++w)
      for (int t = 0; t < h[w]; ++t) e *= p.oma[w][b];
    energy[kBands * k + b] = e;
  }
}

// ------------------------------------------------------------------ compare
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ long long cell_coord(double x, double inv_h) {
  const double c = floor(x * inv_h);
  const double lim = 4.0e18;  // clamp: far points share a cell (still exact, only slower)
  return static_cast<long long>(fmin(fmax(c, -lim), lim));
}

__device__ __forceinline__ unsigned long long cell_key(long long cx, long long cy, long long cz) {
  return mix64(static_cast<unsigned long long>(cx) + 0x9e3779b97f4a7c15ull *
               mix64(static_cast<unsigned long long>(cy) + 0x632be59bd9b4e019ull *
                     mix64(static_cast<unsigned long long>(cz))));
}

__global__ void oracle_key_kernel(const double* __restrict__ opos, int64_t n, double inv_h,
                                  unsigned long long* __restrict__ key, int32_t* __restrict__ idx) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  key[k] = cell_key(cell_coord(opos[3 * k], inv_h), cell_coord(opos[3 * k + 1], inv_h),
                    cell_coord(opos[3 * k + 2], inv_h));
  idx[k] = static_cast<int32_t>(k);
}

__device__ __forceinline__ double pair_distance(const double* tpos, int64_t t, const double* opos, int32_t o) {
  const D3 v = d3(tpos[3 * t], tpos[3 * t + 1], tpos[3 * t + 2]) - d3(opos[3 * o], opos[3 * o + 1], opos[3 * o + 2]);
  return sqrt(dot(v, v));  // (traced - oracle).norm(), shoebox.cpp:138
}

__global__ void match_kernel(const double* __restrict__ tpos, int64_t nt, const double* __restrict__ opos,
                             const unsigned long long* __restrict__ okey, const int32_t* __restrict__ oidx, int64_t no,
                             double inv_h, double pos_tol, int32_t* __restrict__ best_out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nt) return;
  int32_t best = -1;
  double best_d = pos_tol;
  const long long cx = cell_coord(tpos[3 * t], inv_h), cy = cell_coord(tpos[3 * t + 1], inv_h),
                  cz = cell_coord(tpos[3 * t + 2], inv_h);
  for (int dx = -1; dx <= 1; ++dx)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dz = -1; dz <= 1; ++dz) {
        const unsigned long long key = cell_key(cx + dx, cy + dy, cz + dz);
        int64_t lo = 0, hi = no;  // lower_bound
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (okey[mid] < key) lo = mid + 1;
          else hi = mid;
        }
        for (int64_t j = lo; j < no && okey[j] == key; ++j) {
          const int32_t o = oidx[j];
          const double d = pair_distance(tpos, t, opos, o);
          if (d <= pos_tol && (best < 0 || d < best_d || (d == best_d && o > best))) {
            best = o;
            best_d = d;
          }
        }
      }
  best_out[t] = best;
}

__global__ void member_key_kernel(const int32_t* __restrict__ best, int64_t nt, int32_t* __restrict__ key,
                                  int32_t* __restrict__ idx) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nt) return;
  key[t] = best[t] < 0 ? INT32_MAX : best[t];
  idx[t] = static_cast<int32_t>(t);
}

__global__ void group_kernel(const int32_t* __restrict__ uniq, const int64_t* __restrict__ off, int64_t ng,
                             const int32_t* __restrict__ members, const double* __restrict__ tpos,
                             const double* __restrict__ tenergy, const double* __restrict__ opos,
                             const double* __restrict__ oenergy, const int32_t* __restrict__ oorder,
                             double* __restrict__ pos_err, int32_t* __restrict__ order, double* __restrict__ delta_db,
                             int32_t* __restrict__ matched_flag) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int32_t o = uniq[g];
  double te[kBands];
  for (int b = 0; b < kBands; ++b) te[b] = 0.0;
  double err = 0.0;
  for (int64_t j = off[g]; j < off[g + 1]; ++j) {
    const int32_t t = members[j];
    for (int b = 0; b < kBands; ++b) te[b] += tenergy[kBands * (int64_t)t + b];
    err = fmax(err, pair_distance(tpos, t, opos, o));
  }
  pos_err[g] = err;
  order[g] = oorder ? oorder[o] : 0;
  for (int b = 0; b < kBands; ++b)
    delta_db[kBands * g + b] = 10.0 * log10(fmax(te[b], 1e-300) / fmax(oenergy[kBands * (int64_t)o + b], 1e-300));
  matched_flag[o] = 1;
}

// Sequential (oracle-order) sum of squares per band and the max position
// error: 8 lanes, one band each (shoebox.cpp:175-180).
__global__ void rms_kernel(const double* __restrict__ delta_db, const double* __restrict__ pos_err, int64_t ng,
                           double* __restrict__ out /* 8 rms + max err */) {
  const int b = threadIdx.x;
  if (b < kBands) {
    double sq = 0.0;
    for (int64_t g = 0; g < ng; ++g) {
      const double v = delta_db[kBands * g + b];
      sq += v * v;
    }
    out[b] = ng > 0 ? sqrt(sq / static_cast<double>(ng)) : 0.0;
  } else if (b == kBands) {
    double m = 0.0;
    for (int64_t g = 0; g < ng; ++g) m = fmax(m, pos_err[g]);
    out[kBands] = m;
  }
}

struct Negative {
  const int32_t* v;
  __device__ bool operator()(int32_t i) const { return v[i] < 0; }
};
struct Zero {
  const int32_t* v;
  __device__ bool operator()(int32_t i) const { return v[i] == 0; }
};

inline unsigned blocks(int64_t n, int t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

template <typename F>
void select_indices(int64_t n, F pred, DevBuf<int32_t>& out, int64_t& count, cudaStream_t st) {
  out.alloc(std::max<int64_t>(n, 1), st);
  DevBuf<int32_t> d_count;
  d_count.alloc(1, st);
  size_t tb = 0;
  thrust::counting_iterator<int32_t> it(0);
  RR_CUDA(cub::DeviceSelect::If(nullptr, tb, it, out.p, d_count.p, static_cast<int>(n), pred, st));
  DevBuf<unsigned char> tmp;
  tmp.alloc(tb, st);
  RR_CUDA(cub::DeviceSelect::If(tmp.p, tb, it, out.p, d_count.p, static_cast<int>(n), pred, st));
  int32_t c = 0;
  RR_CUDA(cudaMemcpyAsync(&c, d_count.p, sizeof(c), cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  count = c;
}

template <typename T>
const T* device_view(const T* src, int64_t count, DevBuf<T>& buf, cudaStream_t st) {
  if (!src || count == 0) return src;
  cudaPointerAttributes at{};
  RR_CUDA(cudaPointerGetAttributes(&at, src));
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return src;
  buf.alloc(count, st);
  RR_CUDA(cudaMemcpyAsync(buf.p, src, sizeof(T) * count, cudaMemcpyHostToDevice, st));
  return buf.p;
}

}  // namespace

rr_lattice* enumerate_lattice(rr_ctx* ctx, const double* dims, const double* walls_alpha, const double* source,
                              const double* receiver, double max_distance, double receiver_radius, const rr_air& air) {
  // ShoeBox::validate / inside and the argument checks of shoebox.cpp:48-57
  for (int a = 0; a < 3; ++a)
    if (dims[a] <= 0.0) invalid("box dimensions must be > 0");
  auto inside = [&](const double* p) {
    for (int a = 0; a < 3; ++a)
      if (!(p[a] > 0.0) || !(p[a] < dims[a])) return false;
    return true;
  };
  if (!inside(source) || !inside(receiver)) invalid("source and receiver must be strictly inside the box");
  if (max_distance <= 0.0 || receiver_radius <= 0.0) invalid("max_distance and receiver_radius must be > 0");
  LatticeParams p{};
  int64_t cells = 1;
  for (int a = 0; a < 3; ++a) {
    p.L[a] = dims[a];
    p.s[a] = source[a];
    p.r[a] = receiver[a];
    const double sp = std::ceil(max_distance / dims[a]) + 1.0;
    if (!(sp < 1e6)) invalid("lattice too large: max_distance / box dimension exceeds 10^6");
    p.span[a] = static_cast<int>(sp);
    p.n[a] = 2 * p.span[a] + 1;
    cells *= p.n[a];
  }
  if (cells > INT32_MAX) invalid("lattice too large: more than 2^31 cells");
  p.max_distance = max_distance;
  p.radius = receiver_radius;
  air_beta_bands(air, p.beta);
  for (int w = 0; w < kWalls; ++w)
    for (int b = 0; b < kBands; ++b) p.oma[w][b] = 1.0 - walls_alpha[kBands * w + b];

  cudaStream_t st = ctx->stream;
  auto lat = std::make_unique<rr_lattice>();
  lat->ctx = ctx;
  DevBuf<int32_t> sel;
  int64_t n = 0;
  select_indices(cells, InRange{p}, sel, n, st);
  lat->n = n;
  lat->pos.alloc(3 * std::max<int64_t>(n, 1), st);
  lat->dist.alloc(std::max<int64_t>(n, 1), st);
  lat->order.alloc(std::max<int64_t>(n, 1), st);
  lat->hits.alloc(kWalls * std::max<int64_t>(n, 1), st);
  lat->energy.alloc(kBands * std::max<int64_t>(n, 1), st);
  if (n > 0) {
    DevBuf<unsigned long long> key, key2;
    DevBuf<int32_t> cell2;
    key.alloc(n, st);
    key2.alloc(n, st);
    cell2.alloc(n, st);
    lattice_dist_kernel<<<blocks(n), 256, 0, st>>>(p, sel.p, n, key.p);
    RR_LAUNCH_CHECK();
    size_t tb = 0;
    RR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key2.p, sel.p, cell2.p, static_cast<int>(n), 0, 64,
                                            st));
    DevBuf<unsigned char> tmp;
    tmp.alloc(tb, st);
    RR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, key2.p, sel.p, cell2.p, static_cast<int>(n), 0, 64,
                                            st));
    lattice_fill_kernel<<<blocks(n), 256, 0, st>>>(p, cell2.p, n, lat->pos.p, lat->dist.p, lat->order.p,
                                                   lat->hits.p, lat->energy.p);
    RR_LAUNCH_CHECK();
    ctx->launches += 2;
  }
  ctx->launches += 2;  // select (2 passes)
  RR_CUDA(cudaStreamSynchronize(st));
  return lat.release();
}

rr_match* compare_lattice(rr_ctx* ctx, int64_t no, const double* opos_in, const double* oenergy_in,
                          const int32_t* oorder_in, int64_t nt, const double* tpos_in, const double* tenergy_in,
                          double pos_tol, double energy_tol_db) {
  if (no < 0 || nt < 0) invalid("image counts must be >= 0");
  if (no > INT32_MAX || nt > INT32_MAX) invalid("more than 2^31 images");
  cudaStream_t st = ctx->stream;
  DevBuf<double> b_op, b_oe, b_tp, b_te;
  DevBuf<int32_t> b_oo;
  const double* opos = device_view(opos_in, 3 * no, b_op, st);
  const double* oenergy = device_view(oenergy_in, kBands * no, b_oe, st);
  const int32_t* oorder = device_view(oorder_in, no, b_oo, st);
  const double* tpos = device_view(tpos_in, 3 * nt, b_tp, st);
  const double* tenergy = device_view(tenergy_in, kBands * nt, b_te, st);

  auto m = std::make_unique<rr_match>();
  m->ctx = ctx;
  m->pos_tol = pos_tol;
  m->energy_tol_db = energy_tol_db;
  DevBuf<int32_t> best;
  best.alloc(std::max<int64_t>(nt, 1), st);
  if (nt > 0) {
    if (no == 0 || !(pos_tol >= 0.0)) {
      RR_CUDA(cudaMemsetAsync(best.p, 0xff, sizeof(int32_t) * nt, st));  // nothing can match
    } else {
      const double inv_h = 1.0 / std::max(2.0 * pos_tol, 1e-12);
      DevBuf<unsigned long long> key, key2;
      DevBuf<int32_t> idx, idx2;
      key.alloc(no, st);
      key2.alloc(no, st);
      idx.alloc(no, st);
      idx2.alloc(no, st);
      oracle_key_kernel<<<blocks(no), 256, 0, st>>>(opos, no, inv_h, key.p, idx.p);
      RR_LAUNCH_CHECK();
      size_t tb = 0;
      RR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key2.p, idx.p, idx2.p, static_cast<int>(no), 0, 64,
                                              st));
      DevBuf<unsigned char> tmp;
      tmp.alloc(tb, st);
      RR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, key2.p, idx.p, idx2.p, static_cast<int>(no), 0, 64,
                                              st));
      match_kernel<<<blocks(nt, 128), 128, 0, st>>>(tpos, nt, opos, key2.p, idx2.p, no, inv_h, pos_tol, best.p);
      RR_LAUNCH_CHECK();
      ctx->launches += 2;
    }
  }
  // traced images without an oracle partner, in traced order
  select_indices(nt, Negative{best.p}, m->unmatched_traced, m->n_unmatched_traced, st);
  m->n_members = nt - m->n_unmatched_traced;

  // members grouped by oracle index, traced order inside (stable sort)
  DevBuf<int32_t> mkey, midx, mkey2;
  DevBuf<int32_t> flag;
  flag.alloc(std::max<int64_t>(no, 1), st);
  RR_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int32_t) * std::max<int64_t>(no, 1), st));
  m->members.alloc(std::max<int64_t>(nt, 1), st);
  int64_t ng = 0;
  DevBuf<int32_t> uniq, counts;
  if (m->n_members > 0) {
    mkey.alloc(nt, st);
    midx.alloc(nt, st);
    mkey2.alloc(nt, st);
    member_key_kernel<<<blocks(nt), 256, 0, st>>>(best.p, nt, mkey.p, midx.p);
    RR_LAUNCH_CHECK();
    size_t tb = 0;
    RR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, mkey.p, mkey2.p, midx.p, m->members.p, static_cast<int>(nt),
                                            0, 32, st));
    DevBuf<unsigned char> tmp;
    tmp.alloc(tb, st);
    RR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, mkey.p, mkey2.p, midx.p, m->members.p, static_cast<int>(nt), 0,
                                            32, st));
    uniq.alloc(m->n_members, st);
    counts.alloc(m->n_members, st);
    DevBuf<int32_t> d_ng;
    d_ng.alloc(1, st);
    tb = 0;
    RR_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb, mkey2.p, uniq.p, counts.p, d_ng.p,
                                               static_cast<int>(m->n_members), st));
    DevBuf<unsigned char> tmp2;
    tmp2.alloc(tb, st);
    RR_CUDA(cub::DeviceRunLengthEncode::Encode(tmp2.p, tb, mkey2.p, uniq.p, counts.p, d_ng.p,
                                               static_cast<int>(m->n_members), st));
    int32_t h_ng = 0;
    RR_CUDA(cudaMemcpyAsync(&h_ng, d_ng.p, sizeof(h_ng), cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
    ng = h_ng;
    ctx->launches += 4;
  }
  m->n_matched = ng;
  m->oracle_index.alloc(std::max<int64_t>(ng, 1), st);
  m->member_off.alloc(ng + 1, st);
  m->pos_err.alloc(std::max<int64_t>(ng, 1), st);
  m->order.alloc(std::max<int64_t>(ng, 1), st);
  m->delta_db.alloc(kBands * std::max<int64_t>(ng, 1), st);
  RR_CUDA(cudaMemsetAsync(m->member_off.p, 0, sizeof(int64_t), st));
  DevBuf<double> summary;
  summary.alloc(kBands + 1, st);
  if (ng > 0) {
    RR_CUDA(cudaMemcpyAsync(m->oracle_index.p, uniq.p, sizeof(int32_t) * ng, cudaMemcpyDeviceToDevice, st));
    size_t tb = 0;
    RR_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, counts.p, m->member_off.p + 1, static_cast<int>(ng), st));
    DevBuf<unsigned char> tmp;
    tmp.alloc(tb, st);
    RR_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, counts.p, m->member_off.p + 1, static_cast<int>(ng), st));
    group_kernel<<<blocks(ng), 256, 0, st>>>(m->oracle_index.p, m->member_off.p, ng, m->members.p, tpos, tenergy, opos,
                                             oenergy, oorder, m->pos_err.p, m->order.p, m->delta_db.p, flag.p);
    RR_LAUNCH_CHECK();
    ctx->launches += 2;
  }
  rms_kernel<<<1, 32, 0, st>>>(m->delta_db.p, m->pos_err.p, ng, summary.p);
  RR_LAUNCH_CHECK();
  ctx->launches += 1;
  // oracle images nobody matched, in oracle order
  select_indices(no, Zero{flag.p}, m->unmatched_oracle, m->n_unmatched_oracle, st);
  double h_sum[kBands + 1];
  RR_CUDA(cudaMemcpyAsync(h_sum, summary.p, sizeof(h_sum), cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  for (int b = 0; b < kBands; ++b) m->rms_db[b] = h_sum[b];
  m->max_position_error = h_sum[kBands];
  ctx->launches += 4;  // the two selects
  return m.release();
}

}  // namespace rr
