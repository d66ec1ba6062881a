// K5 — image sources from captures (beam reduction), and the air model.
//
// Replaces build_image_sources (image_sources.cpp:154-170): cluster
// (:82-132, with split_group :28-65 and the coplanar merge :99-128),
// attach_energy (:134-140), project (:142-152) and the final sort.
//
//   1. retro points x = point - path*dir (retro_propagate :9-11);
//   2. captures sorted by exact face path (stable merge sort with a
//      lexicographic path comparator = std::map order, :87-90); one segment
//      per distinct path;
//   3. one thread per segment: sequential mean / spread / sum in capture
//      order (same fp64 order as the reference), rare over-spread segments
//      re-sorted by (x, y, z) in place and chained greedily;
//   4. coplanar merge: exact restatement of the O(I^2) greedy — a claim needs
//      |dx| <= tol, so candidates come from a (2 tol)-grid hash; anchors are
//      resolved in index order by a fixed-point iteration over the (tiny)
//      candidate graph, then each anchor sums its claims in index order;
//   5. energy E = (n/N) exp(-beta d) mult, projection with the tracer's
//      closest-hit, sort by (order, distance, path).
// air_beta_bands (air_absorption.cpp:21-65) is 8 scalars per run and stays
// on the host, as in the reference.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <memory>

#include "rr_trace.cuh"

struct ImgOut {
  double *pos, *dist, *energy, *mult, *proj;
  int32_t *ray_count, *order, *has_proj, *path;
  int64_t* path_off;
  int64_t* path_src;  // per image: start of its path in the capture histories
};

namespace rr {

// AirModel::validate air_absorption.cpp:8-19
void air_validate(const rr_air& a) {
  if (!a.enabled) return;
  if (a.temperature_c < -20.0 || a.temperature_c > 50.0) invalid("air temperature outside [-20, 50] C");
  if (a.relative_humidity < 10.0 || a.relative_humidity > 100.0) invalid("relative humidity outside [10, 100] %");
  if (a.pressure_kpa < 80.0 || a.pressure_kpa > 120.0) invalid("pressure outside [80, 120] kPa");
}

// air_alpha_db_per_m air_absorption.cpp:21-53 (ISO 9613-1)
double air_alpha(const rr_air& a, double f) {
  if (!a.enabled) return 0.0;
  const double tk = a.temperature_c + 273.15;
  const double t_rel = tk / 293.15;
  const double p_rel = a.pressure_kpa / 101.325;
  const double c_sat = -6.8346 * std::pow(273.16 / tk, 1.261) + 4.6151;
  const double h = a.relative_humidity * std::pow(10.0, c_sat) / p_rel;
  const double fro = p_rel * (24.0 + 4.04e4 * h * (0.02 + h) / (0.391 + h));
  const double frn =
      p_rel * std::pow(t_rel, -0.5) * (9.0 + 280.0 * h * std::exp(-4.170 * (std::pow(t_rel, -1.0 / 3.0) - 1.0)));
  const double f2 = f * f;
  const double classical = 1.84e-11 / p_rel * std::sqrt(t_rel);
  const double relax = std::pow(t_rel, -2.5) * (0.01275 * std::exp(-2239.1 / tk) / (fro + f2 / fro) +
                                                0.1068 * std::exp(-3352.0 / tk) / (frn + f2 / frn));
  return 8.686 * f2 * (classical + relax);
}

void air_beta_bands(const rr_air& a, double* beta) {
  static const double centers[kBands] = {62.5, 125.0, 250.0, 500.0, 1000.0, 2000.0, 4000.0, 8000.0};
  air_validate(a);
  for (int b = 0; b < kBands; ++b) beta[b] = air_alpha(a, centers[b]) * std::log(10.0) / 10.0;
}

namespace {

struct PathView {
  const int64_t* off;
  const int32_t* hist;
  __device__ __forceinline__ int cmp(int64_t a, int64_t b) const {
    const int64_t a0 = off[a], a1 = off[a + 1], b0 = off[b], b1 = off[b + 1];
    const int64_t la = a1 - a0, lb = b1 - b0, m = la < lb ? la : lb;
    for (int64_t k = 0; k < m; ++k) {
      const int32_t x = hist[a0 + k], y = hist[b0 + k];
      if (x != y) return x < y ? -1 : 1;
    }
    return la == lb ? 0 : (la < lb ? -1 : 1);
  }
};

// std::lexicographical_compare on face paths (image_sources.cpp:67-69)
struct PathLess {
  PathView pv;
  __device__ bool operator()(int32_t a, int32_t b) const { return pv.cmp(a, b) < 0; }
};

__global__ void retro_kernel(const double* __restrict__ point, const double* __restrict__ dir,
                             const double* __restrict__ path, int64_t c0, int64_t n, double* __restrict__ retro,
                             int32_t* __restrict__ idx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t c = c0 + i;
  for (int k = 0; k < 3; ++k) retro[3 * i + k] = point[3 * c + k] - path[c] * dir[3 * c + k];
  idx[i] = static_cast<int32_t>(c);
}

// Path sort, stage 1: radix key of the first faces (as many as fit in 63 bits
// at ceil(log2(nf + 1)) bits each, at least three;
// face + 1, 0 past the end: a proper prefix sorts first, as in
// std::lexicographical_compare).
__global__ void prefix_key_kernel(const int32_t* __restrict__ idx, int64_t n, PathView pv, int bits, int faces,
                                  unsigned long long* __restrict__ keys) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t c = idx[i], a0 = pv.off[c], len = pv.off[c + 1] - a0;
  unsigned long long k = 0;
  for (int j = 0; j < faces; ++j) {  // face + 1 (0: path ended), lexicographic
    const unsigned long long f = j < len ? static_cast<unsigned long long>(pv.hist[a0 + j]) + 1ull : 0ull;
    k = (k << bits) | f;
  }
  keys[i] = k;
}

// Stage 2: one thread per run of equal prefix keys finishes the order with a
// stable insertion sort on the full comparator (runs are beams of identical
// paths or a handful of paths that share three faces).
// A run needs sorting only if two neighbours in it differ (all-identical
// beams are already in capture order): flag its first element in parallel.
__global__ void prefix_run_flag_kernel(const unsigned long long* __restrict__ keys, int64_t n, PathView pv,
                                       const int32_t* __restrict__ idx, int32_t* __restrict__ dirty) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n) return;
  if (q == 0 || keys[q] != keys[q - 1]) return;  // dirty[] is zeroed beforehand
  if (pv.cmp(idx[q - 1], idx[q]) == 0) return;
  int64_t s = q - 1;
  while (s > 0 && keys[s - 1] == keys[q]) --s;
  atomicOr(dirty + s, 1);
}

__global__ void prefix_run_sort_kernel(const unsigned long long* __restrict__ keys, int64_t n, PathView pv,
                                       const int32_t* dirty, int32_t* __restrict__ idx) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n || (s > 0 && keys[s] == keys[s - 1]) || !dirty[s]) return;
  int64_t e = s + 1;
  while (e < n && keys[e] == keys[s]) ++e;
  if (e - s < 2) return;
  for (int64_t x = s + 1; x < e; ++x) {
    const int32_t v = idx[x];
    int64_t y = x - 1;
    while (y >= s && pv.cmp(idx[y], v) > 0) {
      idx[y + 1] = idx[y];
      --y;
    }
    idx[y + 1] = v;
  }
}

__global__ void head_kernel(const int32_t* __restrict__ idx, int64_t n, PathView pv, int32_t* __restrict__ head) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  head[i] = (i == 0 || pv.cmp(idx[i - 1], idx[i]) != 0) ? 1 : 0;
}

__global__ void group_start_kernel(const int32_t* __restrict__ head, const int32_t* __restrict__ gid, int64_t n,
                                   int64_t* __restrict__ gstart) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && head[i]) gstart[gid[i]] = i;
}

__device__ __forceinline__ D3 ld3(const double* p, int64_t i) { return d3(p[3 * i], p[3 * i + 1], p[3 * i + 2]); }
__device__ __forceinline__ double norm3(D3 a) { return sqrt(dot(a, a)); }

// In-order fp64 sum of the points p[s, e): the loads of 8 iterations are
// issued together, the additions keep the reference's order (same bits as a
// plain loop, without one memory latency per element on long groups).
__device__ __forceinline__ D3 sum_points(const double* __restrict__ p, int64_t s, int64_t e) {
  D3 acc = d3(0, 0, 0);
  int64_t i = s;
  for (; i + 8 <= e; i += 8) {
    D3 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = ld3(p, i + u);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = acc + v[u];
  }
  for (; i < e; ++i) acc = acc + ld3(p, i);
  return acc;
}

__device__ __forceinline__ bool pt_less(const double* retro, int64_t c0, int32_t a, int32_t b) {
  const D3 x = ld3(retro, a - c0), y = ld3(retro, b - c0);
  if (x.x != y.x) return x.x < y.x;
  if (x.y != y.y) return x.y < y.y;
  if (x.z != y.z) return x.z < y.z;
  return a < b;
}

// In-place heapsort of a group's members by retro point (split_group's
// std::sort, image_sources.cpp:46-51; ties only between identical points).
__device__ void heap_sort(int32_t* a, int64_t n, const double* retro, int64_t c0) {
  auto sift = [&](int64_t start, int64_t end) {
    int64_t root = start;
    while (2 * root + 1 < end) {
      int64_t child = 2 * root + 1;
      if (child + 1 < end && pt_less(retro, c0, a[child], a[child + 1])) ++child;
      if (pt_less(retro, c0, a[root], a[child])) {
        const int32_t t = a[root];
        a[root] = a[child];
        a[child] = t;
        root = child;
      } else {
        return;
      }
    }
  };
  for (int64_t s = n / 2 - 1; s >= 0; --s) sift(s, n);
  for (int64_t e = n - 1; e > 0; --e) {
    const int32_t t = a[0];
    a[0] = a[e];
    a[e] = t;
    sift(0, e);
  }
}

// Pass A: spread test; split groups get sorted and their beams counted.
// rs: retro points gathered into path-sorted order (contiguous per group, so
// the sequential fp64 sums below stream instead of chasing indices).
__global__ void gather_retro_kernel(const int32_t* __restrict__ idx, int64_t n, const double* __restrict__ retro,
                                    int64_t c0, double* __restrict__ rs) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t j = idx[i] - c0;
  for (int k = 0; k < 3; ++k) rs[3 * i + k] = retro[3 * j + k];
}

constexpr int64_t kBigGroup = 64;  // groups this large go to group_big_kernel (one block each)

// split groups: sort by retro point and count the beams (split_group)
__device__ void split_count(int32_t* idx, int64_t s, int64_t e, const double* retro, int64_t c0, double tol,
                            int32_t* n_img_g) {
  const int64_t m = e - s;
  heap_sort(idx + s, m, retro, c0);
  int32_t cnt = 1;
  D3 anchor = ld3(retro, idx[s] - c0);
  for (int64_t i = s + 1; i < e; ++i) {
    const D3 p = ld3(retro, idx[i] - c0);
    if (norm3(p - anchor) > tol) {
      ++cnt;
      anchor = p;
    }
  }
  *n_img_g = cnt;
}

// Large groups, one block each (taken from a device list): the block stages
// chunks of retro points in shared memory, thread 0 sums them in capture
// order (the reference's bits), the spread is a block max.
__global__ void __launch_bounds__(256) group_big_kernel(int32_t* __restrict__ idx, const int64_t* __restrict__ gstart,
                                                        int64_t ng, int64_t n, const double* __restrict__ retro,
                                                        const double* __restrict__ rs, int64_t c0, double tol,
                                                        const int32_t* __restrict__ big, const int32_t* __restrict__ n_big,
                                                        int32_t* __restrict__ n_img, int32_t* __restrict__ is_split,
                                                        double* __restrict__ gmean) {
  constexpr int kChunk = 1024;
  __shared__ double sp[3 * kChunk];
  __shared__ double red[256];
  __shared__ double smean[3];
  const int nb = *n_big;
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int64_t g = big[b];
    const int64_t s = gstart[g], e = g + 1 < ng ? gstart[g + 1] : n, m = e - s;
    D3 acc = d3(0, 0, 0);
    for (int64_t c = s; c < e; c += kChunk) {
      const int64_t len = min(static_cast<int64_t>(kChunk), e - c);
      __syncthreads();
      for (int64_t k = threadIdx.x; k < 3 * len; k += blockDim.x) sp[k] = rs[3 * c + k];
      __syncthreads();
      if (threadIdx.x == 0)
        for (int64_t k = 0; k < len; ++k) acc = acc + d3(sp[3 * k], sp[3 * k + 1], sp[3 * k + 2]);
    }
    if (threadIdx.x == 0) {
      smean[0] = acc.x / static_cast<double>(m);
      smean[1] = acc.y / static_cast<double>(m);
      smean[2] = acc.z / static_cast<double>(m);
    }
    __syncthreads();
    const D3 mean = d3(smean[0], smean[1], smean[2]);
    double spread2 = 0.0;
    for (int64_t i = s + threadIdx.x; i < e; i += blockDim.x) {
      const D3 v = ld3(rs, i) - mean;
      const double q = dot(v, v);
      spread2 = (spread2 < q) ? q : spread2;
    }
    red[threadIdx.x] = spread2;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const double spread = sqrt(red[0]);
      if (spread <= tol) {
        n_img[g] = 1;
        is_split[g] = 0;
        gmean[3 * g] = mean.x;
        gmean[3 * g + 1] = mean.y;
        gmean[3 * g + 2] = mean.z;
      } else {
        is_split[g] = 1;
        split_count(idx, s, e, retro, c0, tol, n_img + g);
      }
    }
    __syncthreads();
  }
}

__global__ void group_count_kernel(int32_t* __restrict__ idx, const int64_t* __restrict__ gstart, int64_t ng,
                                   int64_t n, const double* __restrict__ retro, const double* __restrict__ rs,
                                   int64_t c0, double tol, int32_t* __restrict__ n_img,
                                   int32_t* __restrict__ is_split, double* __restrict__ gmean,
                                   int32_t* __restrict__ big, int32_t* __restrict__ n_big) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t s = gstart[g], e = g + 1 < ng ? gstart[g + 1] : n, m = e - s;
  if (m >= kBigGroup) {
    big[atomicAdd(n_big, 1)] = static_cast<int32_t>(g);
    return;
  }
  D3 mean = sum_points(rs, s, e);  // capture order, as the reference
  mean = d3(mean.x / static_cast<double>(m), mean.y / static_cast<double>(m), mean.z / static_cast<double>(m));
  // max of the norms = sqrt of the max squared norm (sqrt is monotone and
  // correctly rounded): one square root per group, the same bits; the max
  // is order-free, so 8 loads go out together
  double spread2 = 0.0;
  int64_t i = s;
  for (; i + 8 <= e; i += 8) {
    D3 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = ld3(rs, i + u);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const D3 w = v[u] - mean;
      const double q = dot(w, w);
      spread2 = (spread2 < q) ? q : spread2;
    }
  }
  for (; i < e; ++i) {
    const D3 v = ld3(rs, i) - mean;
    const double q = dot(v, v);
    spread2 = (spread2 < q) ? q : spread2;
  }
  const double spread = sqrt(spread2);
  if (spread <= tol) {
    n_img[g] = 1;
    is_split[g] = 0;
    gmean[3 * g] = mean.x;  // make_image's position for the unsplit group
    gmean[3 * g + 1] = mean.y;
    gmean[3 * g + 2] = mean.z;
    return;
  }
  is_split[g] = 1;
  split_count(idx, s, e, retro, c0, tol, n_img + g);
}

struct ImgTmp {
  double* pos;      // 3n
  int32_t* count;   // n
  int32_t* order;   // n
  int32_t* rep;     // representative capture (path, mult source)
};

// make_image image_sources.cpp:15-25 over idx[b0, b1)
__device__ void emit_image(const int32_t* idx, int64_t b0, int64_t b1, const double* retro, int64_t c0,
                           const int64_t* off, ImgTmp t, int64_t slot) {
  D3 sum = d3(0, 0, 0);
  int64_t i = b0;
  for (; i + 4 <= b1; i += 4) {
    D3 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = ld3(retro, idx[i + u] - c0);
#pragma unroll
    for (int u = 0; u < 4; ++u) sum = sum + v[u];
  }
  for (; i < b1; ++i) sum = sum + ld3(retro, idx[i] - c0);
  const double m = static_cast<double>(b1 - b0);
  t.pos[3 * slot] = sum.x / m;
  t.pos[3 * slot + 1] = sum.y / m;
  t.pos[3 * slot + 2] = sum.z / m;
  t.count[slot] = static_cast<int32_t>(b1 - b0);
  const int32_t rep = idx[b0];
  t.rep[slot] = rep;
  t.order[slot] = static_cast<int32_t>(off[rep + 1] - off[rep]);
}

__global__ void group_emit_kernel(const int32_t* __restrict__ idx, const int64_t* __restrict__ gstart, int64_t ng,
                                  int64_t n, const double* __restrict__ retro, const double* __restrict__ rs,
                                  int64_t c0, double tol, const int32_t* __restrict__ is_split,
                                  const int32_t* __restrict__ img_off, const int64_t* __restrict__ off,
                                  const double* __restrict__ gmean, ImgTmp t) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t s = gstart[g], e = g + 1 < ng ? gstart[g + 1] : n;
  int64_t slot = img_off[g];
  if (!is_split[g]) {  // make_image over the whole group: the mean computed by the count pass
    t.pos[3 * slot] = gmean[3 * g];
    t.pos[3 * slot + 1] = gmean[3 * g + 1];
    t.pos[3 * slot + 2] = gmean[3 * g + 2];
    t.count[slot] = static_cast<int32_t>(e - s);
    const int32_t rep = idx[s];
    t.rep[slot] = rep;
    t.order[slot] = static_cast<int32_t>(off[rep + 1] - off[rep]);
    return;
  }
  int64_t b0 = s;
  D3 anchor = ld3(retro, idx[s] - c0);
  for (int64_t i = s + 1; i < e; ++i) {
    const D3 p = ld3(retro, idx[i] - c0);
    if (norm3(p - anchor) > tol) {
      emit_image(idx, b0, i, retro, c0, off, t, slot++);
      b0 = i;
      anchor = p;
    }
  }
  emit_image(idx, b0, e, retro, c0, off, t, slot);
}

// ---- coplanar merge
__device__ __forceinline__ void cell_of(const double* pos, int64_t i, double cs, long long* c) {
  for (int k = 0; k < 3; ++k) c[k] = static_cast<long long>(floor(pos[3 * i + k] / cs));
}
__device__ __forceinline__ unsigned long long cell_key(int32_t order, const long long* c) {
  unsigned long long h = 0x9E3779B97F4A7C15ull ^ static_cast<unsigned long long>(order);
  for (int k = 0; k < 3; ++k) {
    h ^= static_cast<unsigned long long>(c[k]) + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 31;
  }
  // 32 bits: runs of equal keys may merge two cells (harmless, see
  // resolve_round_kernel) and the cell sort needs 4 radix passes
  return h & 0xffffffffull;  // never ~0, which marks an empty hash slot
}

// Open-addressing table: sorted cell key -> first index of its run.
__device__ __forceinline__ unsigned long long ht_slot(unsigned long long key, unsigned long long mask) {
  return (key ^ (key >> 29)) & mask;
}

__global__ void ht_insert_kernel(const unsigned long long* __restrict__ skeys, int64_t n,
                                 unsigned long long* tkey, int32_t* __restrict__ tstart, unsigned long long mask) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || (i > 0 && skeys[i] == skeys[i - 1])) return;
  const unsigned long long key = skeys[i];
  for (unsigned long long h = ht_slot(key, mask);; h = (h + 1) & mask) {
    const unsigned long long prev = atomicCAS(tkey + h, ~0ull, key);
    if (prev == ~0ull || prev == key) {
      tstart[h] = static_cast<int32_t>(i);
      return;
    }
  }
}

__device__ __forceinline__ int32_t ht_find(const unsigned long long* __restrict__ tkey,
                                           const int32_t* __restrict__ tstart, unsigned long long mask,
                                           unsigned long long key) {
  for (unsigned long long h = ht_slot(key, mask);; h = (h + 1) & mask) {
    const unsigned long long k = tkey[h];
    if (k == key) return tstart[h];
    if (k == ~0ull) return -1;
  }
}

__global__ void cell_key_kernel(ImgTmp t, int64_t n, double cs, unsigned long long* __restrict__ keys,
                                int32_t* __restrict__ ids) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long c[3];
  cell_of(t.pos, i, cs, c);
  keys[i] = cell_key(t.order[i], c);
  ids[i] = static_cast<int32_t>(i);
}

constexpr int32_t kUndet = -2;
constexpr int32_t kAnchor = -1;

// Candidates in cell-sorted order, contiguous so the threads of one cell
// stream the same records: position, multipliers (of the image's beam) and
// order.
struct Cand {
  const double* pos;   // 3 per entry
  const double* mult;  // 8 per entry
  const int32_t* order;
  const int32_t* id;   // image index
};

__global__ void cand_gather_kernel(ImgTmp t, const double* __restrict__ mult, const int32_t* __restrict__ sids,
                                   int64_t n, double* __restrict__ cpos, double* __restrict__ cmult,
                                   int32_t* __restrict__ corder) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int32_t j = sids[q];
  for (int k = 0; k < 3; ++k) cpos[3 * q + k] = t.pos[3 * j + k];
  const double* m = mult + kBands * static_cast<int64_t>(t.rep[j]);
  for (int b = 0; b < kBands; ++b) cmult[kBands * q + b] = m[b];
  corder[q] = t.order[j];
}

__global__ void owner_init_kernel(int32_t* __restrict__ owner, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) owner[i] = kUndet;
}

// One round of the greedy of image_sources.cpp:103-128 without edge lists.
// Image i is claimed by the smallest-index anchor among its preds
// (j < i with cond(j, i): same order, |pos_i - pos_j| <= tol, multipliers
// within 1e-12); it is an anchor when no pred is.  i is decided once every
// pred below that anchor is decided.  Decisions only move from undecided to
// final, so reading a neighbour's value while it is being written is safe.
// Candidate cells: per axis those met by [p - tol, p + tol] (widened by 1 %
// against rounding of the cell index); cells of 16 tol, so a window mostly
// meets a single cell (one hash probe) while the images of different
// beams stay far apart.
__global__ void resolve_round_kernel(ImgTmp t, const double* __restrict__ mult, int64_t n, double cs, double tol,
                                     const unsigned long long* __restrict__ skeys, Cand cand,
                                     const unsigned long long* __restrict__ tkey, const int32_t* __restrict__ tstart,
                                     unsigned long long mask, int32_t* owner, int32_t* __restrict__ progress) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  volatile int32_t* vo = owner;
  if (vo[i] != kUndet) return;
  const int32_t oi = t.order[i];
  const D3 pi = ld3(t.pos, i);
  const double* mi = mult + kBands * static_cast<int64_t>(t.rep[i]);
  double m8[kBands];
  for (int b = 0; b < kBands; ++b) m8[b] = mi[b];
  long long lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    const double x = t.pos[3 * i + k];
    lo[k] = static_cast<long long>(floor((x - 1.01 * tol) / cs));
    hi[k] = static_cast<long long>(floor((x + 1.01 * tol) / cs));
  }
  int32_t best_anchor = INT32_MAX, min_undet = INT32_MAX;
  for (long long cx = lo[0]; cx <= hi[0]; ++cx)
    for (long long cy = lo[1]; cy <= hi[1]; ++cy)
      for (long long cz = lo[2]; cz <= hi[2]; ++cz) {
        long long cc[3] = {cx, cy, cz};
        const unsigned long long key = cell_key(oi, cc);
        const int32_t start = ht_find(tkey, tstart, mask, key);
        if (start < 0) continue;
        for (int64_t q = start; q < n && skeys[q] == key; ++q) {
          const int32_t j = cand.id[q];
          // ids ascend inside a run: once past i, the best anchor or the
          // smallest undecided pred seen, no later entry can change the outcome
          if (j >= i || j >= best_anchor || j >= min_undet) break;
          if (cand.order[q] != oi) continue;
          // (a hash collision only adds entries of another cell, still in
          // ascending id order; any that meet cond(j, i) are true preds)
          const D3 pj = ld3(cand.pos, q);
          // cond(j, i), j the anchor candidate (image_sources.cpp:111-116)
          if (norm3(pi - pj) > tol) continue;
          const double* mj = cand.mult + kBands * q;
          bool same = true;
          for (int b = 0; b < kBands; ++b) same = same && !(fabs(m8[b] - mj[b]) > 1e-12);
          if (!same) continue;
          const int32_t o = vo[j];
          if (o == kAnchor) best_anchor = j;
          else if (o == kUndet) min_undet = min(min_undet, j);
        }
      }
  if (min_undet < best_anchor) {
    progress[1] = 1;  // still waiting on a smaller undecided pred
    return;
  }
  vo[i] = best_anchor == INT32_MAX ? kAnchor : best_anchor;
  progress[0] = 1;
}

// claims sorted by (owner, index): key owner << cb | index (cb bits hold any
// image index), anchors ~0
__global__ void claim_key_kernel(const int32_t* __restrict__ owner, int64_t n, int cb,
                                 unsigned long long* __restrict__ keys) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t o = owner[i];
  keys[i] = o >= 0 ? (static_cast<unsigned long long>(static_cast<uint32_t>(o)) << cb) | static_cast<uint32_t>(i)
                   : ~0ull;
}

__global__ void claim_start_kernel(const unsigned long long* __restrict__ skeys, int64_t n, int cb,
                                   int32_t* __restrict__ claim_start, int32_t* __restrict__ claim_end) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n || skeys[q] == ~0ull) return;
  const uint32_t a = static_cast<uint32_t>(skeys[q] >> cb);
  if (q == 0 || static_cast<uint32_t>(skeys[q - 1] >> cb) != a) claim_start[a] = static_cast<int32_t>(q);
  if (q + 1 == n || skeys[q + 1] == ~0ull || static_cast<uint32_t>(skeys[q + 1] >> cb) != a)
    claim_end[a] = static_cast<int32_t>(q + 1);
}

constexpr int64_t kBigClaims = 48;  // anchors with this many claims go to merge_big_kernel

__device__ __forceinline__ void merge_write(ImgTmp t, int64_t i, D3 w, int32_t cnt, const int32_t* anchor_rank,
                                            ImgTmp out, int64_t n_out) {
  const int64_t s = anchor_rank[i];
  const double m = static_cast<double>(cnt);
  out.pos[3 * s] = w.x / m;
  out.pos[3 * s + 1] = w.y / m;
  out.pos[3 * s + 2] = w.z / m;
  out.count[s] = cnt;
  out.order[s] = t.order[i];
  // the reference keeps the lexicographically smallest face path
  // (image_sources.cpp:121-123); images are indexed in path order and every
  // claim j > i, so that is always the anchor's own path
  out.rep[s] = t.rep[i];          // path source (lexicographic minimum)
  out.rep[n_out + s] = t.rep[i];  // multiplier source (the anchor's, :113)
}

__device__ __forceinline__ D3 weighted(ImgTmp t, int64_t i) {
  const double c = static_cast<double>(t.count[i]);
  return d3(t.pos[3 * i] * c, t.pos[3 * i + 1] * c, t.pos[3 * i + 2] * c);
}

// merged image per anchor: weighted mean over the anchor and its claims in
// index order (image_sources.cpp:103-128)
__global__ void merge_emit_kernel(ImgTmp t, int64_t n, const int32_t* __restrict__ owner,
                                  const unsigned long long* __restrict__ claims,
                                  const int32_t* __restrict__ claim_start, const int32_t* __restrict__ claim_end,
                                  const int32_t* __restrict__ anchor_rank, ImgTmp out, int64_t n_out,
                                  unsigned long long cmask, int32_t* __restrict__ big, int32_t* __restrict__ n_big) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || owner[i] != kAnchor) return;
  const int64_t q0 = claim_start[i], q1 = q0 >= 0 ? claim_end[i] : q0;
  if (q1 - q0 >= kBigClaims) {
    big[atomicAdd(n_big, 1)] = static_cast<int32_t>(i);
    return;
  }
  int32_t cnt = t.count[i];
  D3 w = weighted(t, i);
  int64_t q = q0;
  for (; q + 4 <= q1; q += 4) {  // gather 4 claims, then add them in index order
    D3 pj[4];
    int32_t cj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int32_t j = static_cast<int32_t>(claims[q + u] & cmask);
      pj[u] = weighted(t, j);
      cj[u] = t.count[j];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      w = w + pj[u];
      cnt += cj[u];
    }
  }
  for (; q < q1; ++q) {
    const int32_t j = static_cast<int32_t>(claims[q] & cmask);
    w = w + weighted(t, j);
    cnt += t.count[j];
  }
  merge_write(t, i, w, cnt, anchor_rank, out, n_out);
}

// anchors with many claims, one block each: the claims' weighted positions
// are staged in shared memory in parallel, thread 0 adds them in order
__global__ void __launch_bounds__(256) merge_big_kernel(ImgTmp t, const unsigned long long* __restrict__ claims,
                                                        const int32_t* __restrict__ claim_start,
                                                        const int32_t* __restrict__ claim_end,
                                                        const int32_t* __restrict__ anchor_rank, ImgTmp out,
                                                        int64_t n_out, unsigned long long cmask,
                                                        const int32_t* __restrict__ big,
                                                        const int32_t* __restrict__ n_big) {
  constexpr int kChunk = 1024;
  __shared__ double sw[3 * kChunk];
  __shared__ int32_t sc[kChunk];
  const int nb = *n_big;
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int64_t i = big[b];
    const int64_t q0 = claim_start[i], q1 = claim_end[i];
    int32_t cnt = t.count[i];
    D3 w = weighted(t, i);
    for (int64_t c = q0; c < q1; c += kChunk) {
      const int64_t len = min(static_cast<int64_t>(kChunk), q1 - c);
      __syncthreads();
      for (int64_t k = threadIdx.x; k < len; k += blockDim.x) {
        const int32_t j = static_cast<int32_t>(claims[c + k] & cmask);
        const D3 v = weighted(t, j);
        sw[3 * k] = v.x;
        sw[3 * k + 1] = v.y;
        sw[3 * k + 2] = v.z;
        sc[k] = t.count[j];
      }
      __syncthreads();
      if (threadIdx.x == 0)
        for (int64_t k = 0; k < len; ++k) {
          w = w + d3(sw[3 * k], sw[3 * k + 1], sw[3 * k + 2]);
          cnt += sc[k];
        }
    }
    if (threadIdx.x == 0) merge_write(t, i, w, cnt, anchor_rank, out, n_out);
    __syncthreads();
  }
}

__global__ void flag_anchor_kernel(const int32_t* __restrict__ owner, int64_t n, int32_t* __restrict__ f) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) f[i] = owner[i] == kAnchor ? 1 : 0;
}

struct EnergyParams {
  TravHeader hdr;
  const TNode* nodes;
  const FaceTri* tri;
  double recv[3];
  double beta[kBands];
  double total_rays;
};

// attach_energy :134-140 + project :142-152
__global__ void energy_kernel(ImgTmp t, const int32_t* __restrict__ mult_src, int64_t n,
                              const double* __restrict__ cmult, EnergyParams ep, double* __restrict__ dist,
                              double* __restrict__ energy, double* __restrict__ mult, int32_t* __restrict__ has_proj,
                              double* __restrict__ proj) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const D3 rc = d3(ep.recv[0], ep.recv[1], ep.recv[2]);
  const D3 tw = ld3(t.pos, i) - rc;
  const double d = norm3(tw);
  dist[i] = d;
  const double frac = static_cast<double>(t.count[i]) / ep.total_rays;
  const double* m = cmult + kBands * static_cast<int64_t>(mult_src[i]);
  for (int b = 0; b < kBands; ++b) {
    mult[kBands * i + b] = m[b];
    energy[kBands * i + b] = (frac * exp((-ep.beta[b]) * d)) * m[b];
  }
  int32_t hp = 0;
  D3 pt = d3(0, 0, 0);
  if (t.order[i] >= 1 && d != 0.0) {
    const D3 dir = d3(tw.x / d, tw.y / d, tw.z / d);
    const HitResult h = closest_hit(ep.hdr, ep.nodes, nullptr, 0, ep.tri, rc, dir);
    if (h.face >= 0) {
      hp = 1;
      pt = rc + h.delta * dir;
    }
  }
  has_proj[i] = hp;
  proj[3 * i] = pt.x;
  proj[3 * i + 1] = pt.y;
  proj[3 * i + 2] = pt.z;
}

// final order (order, distance, face path), image_sources.cpp:163-168: see the final sort

// final sort keys: distance bits (64) or order (32) of image perm[i]
__global__ void final_key_kernel(const int32_t* __restrict__ perm, int64_t n, const double* __restrict__ dist,
                                 const int32_t* __restrict__ order, unsigned long long* __restrict__ kd,
                                 uint32_t* __restrict__ ko) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t s = perm[i];
  if (kd) kd[i] = static_cast<unsigned long long>(__double_as_longlong(dist[s]));
  if (ko) ko[i] = static_cast<uint32_t>(order[s]);
}

// runs of equal (order, distance): insertion sort on the face path
__global__ void final_ties_kernel(int32_t* __restrict__ perm, int64_t n, const double* __restrict__ dist,
                                  const int32_t* __restrict__ order, const int32_t* __restrict__ rep, PathView pv) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  auto same = [&](int64_t a, int64_t b) {
    return order[perm[a]] == order[perm[b]] && dist[perm[a]] == dist[perm[b]];
  };
  if (s > 0 && same(s - 1, s)) return;  // not the first of its run
  if (s + 1 >= n || !same(s, s + 1)) return;  // run of one
  int64_t e = s + 1;
  while (e < n && same(s, e)) ++e;
  for (int64_t x = s + 1; x < e; ++x) {
    const int32_t v = perm[x];
    int64_t y = x - 1;
    while (y >= s && pv.cmp(rep[perm[y]], rep[v]) > 0) {
      perm[y + 1] = perm[y];
      --y;
    }
    perm[y + 1] = v;
  }
}

__global__ void final_len_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ order, int64_t n,
                                 int64_t* __restrict__ len) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) len[i] = order[perm[i]];
  if (i == n) len[i] = 0;
}

__global__ void final_gather_kernel(const int32_t* __restrict__ perm, int64_t n, ImgTmp t,
                                    const double* __restrict__ dist, const double* __restrict__ energy,
                                    const double* __restrict__ mult, const int32_t* __restrict__ has_proj,
                                    const double* __restrict__ proj, PathView pv,
                                    const int64_t* __restrict__ out_off, ImgOut im) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t s = perm[i];
  for (int k = 0; k < 3; ++k) {
    im.pos[3 * i + k] = t.pos[3 * s + k];
    im.proj[3 * i + k] = proj[3 * s + k];
  }
  im.dist[i] = dist[s];
  for (int b = 0; b < kBands; ++b) {
    im.energy[kBands * i + b] = energy[kBands * s + b];
    im.mult[kBands * i + b] = mult[kBands * s + b];
  }
  im.ray_count[i] = t.count[s];
  im.order[i] = t.order[s];
  im.has_proj[i] = has_proj[s];
  const int32_t r = t.rep[s];
  const int64_t a0 = pv.off[r], len = pv.off[r + 1] - a0, o = out_off[i];
  im.path_src[i] = a0;  // path elements are copied by final_path_kernel
  im.path_off[i] = o;
  if (i == n - 1) im.path_off[n] = o + len;
}

// one warp per image copies its face path (coalesced)
__global__ void final_path_kernel(const int64_t* __restrict__ path_off, const int64_t* __restrict__ path_src,
                                  int64_t n, const int32_t* __restrict__ hist, int32_t* __restrict__ path) {
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int64_t o = path_off[i], len = path_off[i + 1] - o, a0 = path_src[i];
  for (int64_t k = lane; k < len; k += 32) path[o + k] = hist[a0 + k];
}

inline unsigned grid(int64_t n, int b = 256) { return static_cast<unsigned>((n + b - 1) / b); }

// [c0, c1) of receiver r in the (receiver, ray, path)-sorted captures
__global__ void recv_range_kernel(const int32_t* __restrict__ recv, int64_t n, int32_t r, int64_t* __restrict__ out) {
  if (threadIdx.x > 1) return;
  const int32_t key = threadIdx.x == 0 ? r : r + 1;  // lower bounds of r and r + 1
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (recv[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  out[threadIdx.x] = lo;
}

__global__ void iota_kernel(int32_t* __restrict__ v, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = static_cast<int32_t>(i);
}

template <typename F>
void cub_call(F&& f, cudaStream_t st) {
  size_t bytes = 0;
  RR_CUDA(f(nullptr, bytes));
  DevBuf<uint8_t> tmp;
  tmp.alloc(bytes + 16, st);
  RR_CUDA(f(tmp.p, bytes));
}

}  // namespace

rr_images* build_image_sources(rr_trace_result* tr, int32_t recv, int64_t total_rays, const rr_air& air,
                               const rr_cluster_options& opt) {
  rr_scene* s = tr->scene;
  rr_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  if (recv < 0 || recv >= static_cast<int32_t>(tr->recv_radius.size())) invalid("receiver index out of range");
  if (total_rays < 1) invalid("total_rays must be >= 1");
  double beta[kBands];
  air_beta_bands(air, beta);
  // receiver range of the (receiver, ray, path)-sorted captures
  const int64_t nc_all = tr->stats.n_captures;
  int64_t range[2] = {0, 0};
  if (nc_all) {
    DevBuf<int64_t> dr;
    dr.alloc(2, st);
    recv_range_kernel<<<1, 32, 0, st>>>(tr->c_recv.p, nc_all, recv, dr.p);
    RR_LAUNCH_CHECK();
    ctx->launches++;
    RR_CUDA(cudaMemcpyAsync(range, dr.p, sizeof range, cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
  }
  const int64_t c0 = range[0], c1 = range[1];
  const int64_t n = c1 - c0;
  auto im = std::make_unique<rr_images>();
  im->scene = s;
  // TriangleMesh::bounds().diagonal() (geometry.hpp:45)
  const double dx = s->hi[0] - s->lo[0], dy = s->hi[1] - s->lo[1], dz = s->hi[2] - s->lo[2];
  const double tol = opt.tol_scale * std::sqrt((dx * dx + dy * dy) + dz * dz);
  if (n == 0) {
    im->path_off.alloc(1, st);
    RR_CUDA(cudaMemsetAsync(im->path_off.p, 0, sizeof(int64_t), st));
    RR_CUDA(cudaStreamSynchronize(st));
    return im.release();
  }
  StageTimer tm(st);
  PathView pv{tr->c_off.p, tr->c_hist.p};
  DevBuf<double> retro;
  DevBuf<int32_t> idx, head, gid;
  retro.alloc(3 * n, st);
  idx.alloc(n, st);
  head.alloc(n, st);
  gid.alloc(n, st);
  retro_kernel<<<grid(n), 256, 0, st>>>(tr->c_point.p, tr->c_dir.p, tr->c_path.p, c0, n, retro.p, idx.p);
  RR_LAUNCH_CHECK();
  if (s->nf < (1 << 21) - 1) {
    // radix sort on the 3-face prefix (stable: ties keep capture order), then
    // per-run stable insertion sorts on the full path
    DevBuf<unsigned long long> pk, pk_s;
    DevBuf<int32_t> idx_s;
    pk.alloc(n, st);
    pk_s.alloc(n, st);
    idx_s.alloc(n, st);
    int bits = 1;
    while ((int64_t(1) << bits) <= s->nf) ++bits;  // face + 1 <= nf
    const int faces = std::max(1, 63 / bits);
    prefix_key_kernel<<<grid(n), 256, 0, st>>>(idx.p, n, pv, bits, faces, pk.p);
    RR_LAUNCH_CHECK();
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, pk.p, pk_s.p, idx.p, idx_s.p, n, 0, bits * faces, st);
    }, st);
    DevBuf<int32_t> dirty;
    dirty.alloc(n, st);
    RR_CUDA(cudaMemsetAsync(dirty.p, 0, dirty.bytes(), st));
    prefix_run_flag_kernel<<<grid(n), 256, 0, st>>>(pk_s.p, n, pv, idx_s.p, dirty.p);
    prefix_run_sort_kernel<<<grid(n), 256, 0, st>>>(pk_s.p, n, pv, dirty.p, idx_s.p);
    RR_LAUNCH_CHECK();
    if (tm.stats) {  // dirty-run statistics (development)
      std::vector<unsigned long long> hk(n);
      std::vector<int32_t> hd(n);
      RR_CUDA(cudaMemcpyAsync(hk.data(), pk_s.p, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost, st));
      RR_CUDA(cudaMemcpyAsync(hd.data(), dirty.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
      RR_CUDA(cudaStreamSynchronize(st));
      int64_t runs = 0, dirty_runs = 0, dirty_elems = 0, max_dirty = 0, max_run = 0;
      for (int64_t a = 0; a < n;) {
        int64_t b = a + 1;
        while (b < n && hk[b] == hk[a]) ++b;
        ++runs;
        max_run = std::max(max_run, b - a);
        if (hd[a]) {
          ++dirty_runs;
          dirty_elems += b - a;
          max_dirty = std::max(max_dirty, b - a);
        }
        a = b;
      }
      std::fprintf(stderr, "[rr timing] prefix runs %lld (max %lld), dirty %lld with %lld captures (max %lld)\n",
                   (long long)runs, (long long)max_run, (long long)dirty_runs, (long long)dirty_elems,
                   (long long)max_dirty);
    }
    idx = std::move(idx_s);
    ctx->launches += 6;
  } else {
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceMergeSort::StableSortKeys(t, b, idx.p, n, PathLess{pv}, st);
    }, st);
  }
  tm.mark("path sort");
  head_kernel<<<grid(n), 256, 0, st>>>(idx.p, n, pv, head.p);
  RR_LAUNCH_CHECK();
  cub_call([&](void* t, size_t& b) { return cub::DeviceScan::InclusiveSum(t, b, head.p, gid.p, n, st); }, st);
  int32_t ng32 = 0;
  RR_CUDA(cudaMemcpyAsync(&ng32, gid.p + n - 1, sizeof ng32, cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  const int64_t ng = ng32;
  // gid is 1-based inclusive; group g starts at the head whose gid == g+1
  DevBuf<int64_t> gstart;
  gstart.alloc(ng + 1, st);
  {
    // shift to 0-based by writing at gid-1
    DevBuf<int32_t> gid0;
    gid0.alloc(n, st);
    cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, head.p, gid0.p, n, st); }, st);
    group_start_kernel<<<grid(n), 256, 0, st>>>(head.p, gid0.p, n, gstart.p);
    RR_LAUNCH_CHECK();
  }
  DevBuf<int32_t> n_img, is_split, img_off;
  n_img.alloc(ng + 1, st);
  is_split.alloc(ng, st);
  img_off.alloc(ng + 1, st);
  DevBuf<double> rs;
  rs.alloc(3 * n, st);
  gather_retro_kernel<<<grid(n), 256, 0, st>>>(idx.p, n, retro.p, c0, rs.p);
  tm.mark("groups: heads");
  DevBuf<double> gmean;
  gmean.alloc(3 * ng, st);
  {
    DevBuf<int32_t> big, n_big;
    big.alloc(std::max<int64_t>(n / kBigGroup + 1, 1), st);
    n_big.alloc(1, st);
    RR_CUDA(cudaMemsetAsync(n_big.p, 0, sizeof(int32_t), st));
    group_count_kernel<<<grid(ng, 128), 128, 0, st>>>(idx.p, gstart.p, ng, n, retro.p, rs.p, c0, tol, n_img.p,
                                                      is_split.p, gmean.p, big.p, n_big.p);
    RR_LAUNCH_CHECK();
    group_big_kernel<<<static_cast<unsigned>(std::min<int64_t>(n / kBigGroup + 1, 2 * ctx->sm_count)), 256, 0, st>>>(
        idx.p, gstart.p, ng, n, retro.p, rs.p, c0, tol, big.p, n_big.p, n_img.p, is_split.p, gmean.p);
    RR_LAUNCH_CHECK();
    ctx->launches += 1;
  }
  tm.mark("groups: count");
  if (tm.stats) {  // group statistics (development)
    std::vector<int64_t> gs(ng + 1);
    std::vector<int32_t> sp(ng);
    RR_CUDA(cudaMemcpyAsync(gs.data(), gstart.p, sizeof(int64_t) * ng, cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaMemcpyAsync(sp.data(), is_split.p, sizeof(int32_t) * ng, cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
    gs[ng] = n;
    int64_t mx = 0, nsplit = 0, mxs = 0;
    for (int64_t g = 0; g < ng; ++g) {
      mx = std::max(mx, gs[g + 1] - gs[g]);
      if (sp[g]) {
        ++nsplit;
        mxs = std::max(mxs, gs[g + 1] - gs[g]);
      }
    }
    std::fprintf(stderr, "[rr timing] groups: %lld, largest %lld, split %lld (largest split %lld)\n", (long long)ng,
                 (long long)mx, (long long)nsplit, (long long)mxs);
  }
  RR_CUDA(cudaMemsetAsync(n_img.p + ng, 0, sizeof(int32_t), st));
  cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, n_img.p, img_off.p, ng + 1, st); },
           st);
  int32_t ni32 = 0;
  RR_CUDA(cudaMemcpyAsync(&ni32, img_off.p + ng, sizeof ni32, cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  int64_t ni = ni32;
  DevBuf<double> tpos;
  DevBuf<int32_t> tcount, torder, trep;
  tpos.alloc(3 * ni, st);
  tcount.alloc(ni, st);
  torder.alloc(ni, st);
  trep.alloc(2 * ni, st);
  ImgTmp T{tpos.p, tcount.p, torder.p, trep.p};
  group_emit_kernel<<<grid(ng, 128), 128, 0, st>>>(idx.p, gstart.p, ng, n, retro.p, rs.p, c0, tol, is_split.p,
                                                   img_off.p, tr->c_off.p, gmean.p, T);
  RR_LAUNCH_CHECK();
  ctx->launches += 8;
  tm.mark("groups");

  // multiplier source per image: the representative capture (beam.front())
  DevBuf<double> mpos;
  DevBuf<int32_t> mcount, morder, mrep;
  ImgTmp M = T;
  const int32_t* mult_src = trep.p;
  if (opt.merge_coplanar && ni > 1) {
    const double cs = 16.0 * tol;
    DevBuf<unsigned long long> keys, skeys;
    DevBuf<int32_t> ids, sids;
    keys.alloc(ni, st);
    skeys.alloc(ni, st);
    ids.alloc(ni, st);
    sids.alloc(ni, st);
    cell_key_kernel<<<grid(ni), 256, 0, st>>>(T, ni, cs, keys.p, ids.p);
    RR_LAUNCH_CHECK();
    tm.mark("merge: cell keys");
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, keys.p, skeys.p, ids.p, sids.p, ni, 0, 32, st);
    }, st);
    tm.mark("merge: cell sort");
    unsigned long long tsize = 1024;
    while (tsize < 2ull * static_cast<unsigned long long>(ni)) tsize <<= 1;
    DevBuf<unsigned long long> tkey;
    DevBuf<int32_t> tstart;
    tkey.alloc(tsize, st);
    tstart.alloc(tsize, st);
    RR_CUDA(cudaMemsetAsync(tkey.p, 0xff, tkey.bytes(), st));
    tm.mark("merge: table alloc");
    ht_insert_kernel<<<grid(ni), 256, 0, st>>>(skeys.p, ni, tkey.p, tstart.p, tsize - 1);
    tm.mark("merge: table insert");
    DevBuf<double> cpos, cmult;
    DevBuf<int32_t> corder, owner, progress;
    cpos.alloc(3 * ni, st);
    cmult.alloc(kBands * ni, st);
    corder.alloc(ni, st);
    owner.alloc(ni, st);
    progress.alloc(2, st);
    cand_gather_kernel<<<grid(ni), 256, 0, st>>>(T, tr->c_mult.p, sids.p, ni, cpos.p, cmult.p, corder.p);
    owner_init_kernel<<<grid(ni), 256, 0, st>>>(owner.p, ni);
    RR_LAUNCH_CHECK();
    ctx->launches += 7;
    tm.mark("merge: cells");
    const Cand cand{cpos.p, cmult.p, corder.p, sids.p};
    for (int round = 0;; ++round) {
      int32_t h[2] = {0, 0};
      RR_CUDA(cudaMemsetAsync(progress.p, 0, 2 * sizeof(int32_t), st));
      resolve_round_kernel<<<grid(ni, 128), 128, 0, st>>>(T, tr->c_mult.p, ni, cs, tol, skeys.p, cand, tkey.p,
                                                          tstart.p, tsize - 1, owner.p, progress.p);
      RR_LAUNCH_CHECK();
      ctx->launches++;
      RR_CUDA(cudaMemcpyAsync(h, progress.p, sizeof h, cudaMemcpyDeviceToHost, st));
      RR_CUDA(cudaStreamSynchronize(st));
      if (!h[1]) {  // nobody left waiting
        if (std::getenv("RR_TIMING")) std::fprintf(stderr, "[rr timing] merge rounds %d\n", round + 1);
        break;
      }
      if (!h[0]) throw Error(RR_RUNTIME, "coplanar merge made no progress");  // impossible: preds are smaller
    }
    tm.mark("merge: resolve");
    DevBuf<unsigned long long> ckeys, cskeys;
    DevBuf<int32_t> claim_start, claim_end;
    ckeys.alloc(ni, st);
    cskeys.alloc(ni, st);
    claim_start.alloc(ni, st);
    claim_end.alloc(ni, st);
    int cb = 1;
    while ((int64_t(1) << cb) < ni) ++cb;  // bits of an image index
    const unsigned long long cmask = (1ull << cb) - 1ull;
    claim_key_kernel<<<grid(ni), 256, 0, st>>>(owner.p, ni, cb, ckeys.p);
    RR_LAUNCH_CHECK();
    cub_call([&](void* t, size_t& b) {  // anchors' ~0 keys stay last: all-ones in the sorted bits
      return cub::DeviceRadixSort::SortKeys(t, b, ckeys.p, cskeys.p, ni, 0, 2 * cb, st);
    }, st);
    RR_CUDA(cudaMemsetAsync(claim_start.p, 0xff, claim_start.bytes(), st));
    claim_start_kernel<<<grid(ni), 256, 0, st>>>(cskeys.p, ni, cb, claim_start.p, claim_end.p);
    RR_LAUNCH_CHECK();
    tm.mark("merge: claims");
    DevBuf<int32_t> aflag, arank;
    aflag.alloc(ni + 1, st);
    arank.alloc(ni + 1, st);
    flag_anchor_kernel<<<grid(ni), 256, 0, st>>>(owner.p, ni, aflag.p);
    RR_LAUNCH_CHECK();
    RR_CUDA(cudaMemsetAsync(aflag.p + ni, 0, sizeof(int32_t), st));
    cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, aflag.p, arank.p, ni + 1, st); },
             st);
    int32_t na = 0;
    RR_CUDA(cudaMemcpyAsync(&na, arank.p + ni, sizeof na, cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
    mpos.alloc(3 * na, st);
    mcount.alloc(na, st);
    morder.alloc(na, st);
    mrep.alloc(2 * static_cast<int64_t>(na), st);
    M = ImgTmp{mpos.p, mcount.p, morder.p, mrep.p};
    // path reps at [0, na), multiplier reps at [na, 2na)
    DevBuf<int32_t> mbig, n_mbig;
    mbig.alloc(ni / kBigClaims + 1, st);
    n_mbig.alloc(1, st);
    RR_CUDA(cudaMemsetAsync(n_mbig.p, 0, sizeof(int32_t), st));
    merge_emit_kernel<<<grid(ni), 256, 0, st>>>(T, ni, owner.p, cskeys.p, claim_start.p, claim_end.p, arank.p, M, na,
                                                cmask, mbig.p, n_mbig.p);
    RR_LAUNCH_CHECK();
    merge_big_kernel<<<static_cast<unsigned>(std::min<int64_t>(ni / kBigClaims + 1, 2 * ctx->sm_count)), 256, 0,
                       st>>>(T, cskeys.p, claim_start.p, claim_end.p, arank.p, M, na, cmask, mbig.p, n_mbig.p);
    RR_LAUNCH_CHECK();
    ctx->launches += 3;
    ni = na;
    mult_src = mrep.p + na;
  }
  tm.mark("coplanar merge");
  EnergyParams ep;
  // projection (image_sources.cpp:142-152) on the SAH tree: closest hits do
  // not depend on the tree (rr_geom.cuh), so this equals the reference's
  if (!s->snodes.p) ensure_reference_tree(s);
  ep.hdr = s->snodes.p ? s->shdr : s->hdr;
  ep.nodes = s->snodes.p ? s->snodes.p : s->tnodes.p;
  ep.tri = s->tri.p;
  for (int k = 0; k < 3; ++k) ep.recv[k] = tr->recv_center[3 * recv + k];
  for (int b = 0; b < kBands; ++b) ep.beta[b] = beta[b];
  ep.total_rays = static_cast<double>(total_rays);
  DevBuf<double> dist, energy, mult, proj;
  DevBuf<int32_t> has_proj;
  dist.alloc(ni, st);
  energy.alloc(kBands * ni, st);
  mult.alloc(kBands * ni, st);
  proj.alloc(3 * ni, st);
  has_proj.alloc(ni, st);
  energy_kernel<<<grid(ni, 128), 128, 0, st>>>(M, mult_src, ni, tr->c_mult.p, ep, dist.p, energy.p, mult.p, has_proj.p,
                                          proj.p);
  RR_LAUNCH_CHECK();
  tm.mark("energy+project");
  DevBuf<int32_t> perm;
  perm.alloc(ni, st);
  {
    iota_kernel<<<grid(ni), 256, 0, st>>>(perm.p, ni);
    RR_LAUNCH_CHECK();
    ctx->launches++;
  }
  {
    // (order, distance) by two stable radix passes (distances are >= 0, so
    // their bits order like the values), then runs of equal (order,
    // distance) — rare exact ties — finish on the face path
    DevBuf<unsigned long long> k64, k64s;
    DevBuf<uint32_t> k32, k32s;
    DevBuf<int32_t> perm2;
    k64.alloc(ni, st);
    k64s.alloc(ni, st);
    k32.alloc(ni, st);
    k32s.alloc(ni, st);
    perm2.alloc(ni, st);
    final_key_kernel<<<grid(ni), 256, 0, st>>>(perm.p, ni, dist.p, M.order, k64.p, nullptr);
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, k64.p, k64s.p, perm.p, perm2.p, ni, 0, 64, st);
    }, st);
    final_key_kernel<<<grid(ni), 256, 0, st>>>(perm2.p, ni, dist.p, M.order, nullptr, k32.p);
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, k32.p, k32s.p, perm2.p, perm.p, ni, 0, 32, st);
    }, st);
    final_ties_kernel<<<grid(ni), 256, 0, st>>>(perm.p, ni, dist.p, M.order, M.rep, pv);
    RR_LAUNCH_CHECK();
    ctx->launches += 11;
  }
  tm.mark("final sort");
  DevBuf<int64_t> len;
  len.alloc(ni + 1, st);
  im->path_off.alloc(ni + 1, st);
  final_len_kernel<<<grid(ni + 1), 256, 0, st>>>(perm.p, M.order, ni, len.p);
  RR_LAUNCH_CHECK();
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, len.p, im->path_off.p, ni + 1, st);
  }, st);
  int64_t tpath = 0;
  RR_CUDA(cudaMemcpyAsync(&tpath, im->path_off.p + ni, sizeof tpath, cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  im->n = ni;
  im->total_path = tpath;
  im->pos.alloc(3 * ni, st);
  im->dist.alloc(ni, st);
  im->energy.alloc(kBands * ni, st);
  im->mult.alloc(kBands * ni, st);
  im->proj.alloc(3 * ni, st);
  im->ray_count.alloc(ni, st);
  im->order.alloc(ni, st);
  im->has_proj.alloc(ni, st);
  im->path.alloc(std::max<int64_t>(tpath, 1), st);
  DevBuf<int64_t> psrc;
  psrc.alloc(std::max<int64_t>(ni, 1), st);
  final_gather_kernel<<<grid(ni), 256, 0, st>>>(perm.p, ni, M, dist.p, energy.p, mult.p, has_proj.p, proj.p, pv,
                                                im->path_off.p,
                                                ImgOut{im->pos.p, im->dist.p, im->energy.p, im->mult.p, im->proj.p,
                                                       im->ray_count.p, im->order.p, im->has_proj.p, im->path.p,
                                                       im->path_off.p, psrc.p});
  RR_LAUNCH_CHECK();
  if (tpath > 0) {
    final_path_kernel<<<grid(32 * ni), 256, 0, st>>>(im->path_off.p, psrc.p, ni, pv.hist, im->path.p);
    RR_LAUNCH_CHECK();
  }
  ctx->launches += 7;
  tm.mark("gather");
  RR_CUDA(cudaStreamSynchronize(st));
  return im.release();
}

}  // namespace rr
