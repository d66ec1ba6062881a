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
__global__ void group_count_kernel(int32_t* __restrict__ idx, const int64_t* __restrict__ gstart, int64_t ng,
                                   int64_t n, const double* __restrict__ retro, int64_t c0, double tol,
                                   int32_t* __restrict__ n_img, int32_t* __restrict__ is_split) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t s = gstart[g], e = g + 1 < ng ? gstart[g + 1] : n, m = e - s;
  D3 mean = d3(0, 0, 0);
  for (int64_t i = s; i < e; ++i) mean = mean + ld3(retro, idx[i] - c0);
  mean = d3(mean.x / static_cast<double>(m), mean.y / static_cast<double>(m), mean.z / static_cast<double>(m));
  double spread = 0.0;
  for (int64_t i = s; i < e; ++i) {
    const double dd = norm3(ld3(retro, idx[i] - c0) - mean);
    spread = (spread < dd) ? dd : spread;
  }
  if (spread <= tol) {
    n_img[g] = 1;
    is_split[g] = 0;
    return;
  }
  is_split[g] = 1;
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
  n_img[g] = cnt;
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
  for (int64_t i = b0; i < b1; ++i) sum = sum + ld3(retro, idx[i] - c0);
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
                                  int64_t n, const double* __restrict__ retro, int64_t c0, double tol,
                                  const int32_t* __restrict__ is_split, const int32_t* __restrict__ img_off,
                                  const int64_t* __restrict__ off, ImgTmp t) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t s = gstart[g], e = g + 1 < ng ? gstart[g + 1] : n;
  int64_t slot = img_off[g];
  if (!is_split[g]) {
    emit_image(idx, s, e, retro, c0, off, t, slot);
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
  return h;
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

// cond(i, j) of image_sources.cpp:111-116 (i the anchor candidate)
__device__ __forceinline__ bool merge_cond(ImgTmp t, const double* mult, int64_t i, int64_t j, double tol) {
  if (t.order[i] != t.order[j]) return false;
  if (norm3(ld3(t.pos, j) - ld3(t.pos, i)) > tol) return false;
  const double* mi = mult + kBands * static_cast<int64_t>(t.rep[i]);
  const double* mj = mult + kBands * static_cast<int64_t>(t.rep[j]);
  for (int b = 0; b < kBands; ++b)
    if (fabs(mj[b] - mi[b]) > 1e-12) return false;
  return true;
}

// For each image: candidate neighbours (pred j < i, succ j > i) with cond.
// mode 0: count; mode 1: fill.
__global__ void neighbour_kernel(ImgTmp t, const double* __restrict__ mult, int64_t n, double cs, double tol,
                                 const unsigned long long* __restrict__ skeys, const int32_t* __restrict__ sids,
                                 int mode, int32_t* __restrict__ n_pred, int32_t* __restrict__ n_succ,
                                 const int64_t* __restrict__ pred_off, const int64_t* __restrict__ succ_off,
                                 int32_t* __restrict__ pred, int32_t* __restrict__ succ) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long c[3];
  cell_of(t.pos, i, cs, c);
  int32_t np = 0, ns = 0;
  for (int dx = -1; dx <= 1; ++dx)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dz = -1; dz <= 1; ++dz) {
        long long cc[3] = {c[0] + dx, c[1] + dy, c[2] + dz};
        const unsigned long long key = cell_key(t.order[i], cc);
        int64_t lo = 0, hi = n;
        while (lo < hi) {
          const int64_t mid = (lo + hi) / 2;
          if (skeys[mid] < key) lo = mid + 1; else hi = mid;
        }
        for (int64_t p = lo; p < n && skeys[p] == key; ++p) {
          const int32_t j = sids[p];
          if (j == i) continue;
          long long cj[3];
          cell_of(t.pos, j, cs, cj);
          if (cj[0] != cc[0] || cj[1] != cc[1] || cj[2] != cc[2]) continue;  // hash collision
          if (j < i) {
            if (!merge_cond(t, mult, j, i, tol)) continue;
            if (mode) pred[pred_off[i] + np] = j;
            ++np;
          } else {
            if (!merge_cond(t, mult, i, j, tol)) continue;
            if (mode) succ[succ_off[i] + ns] = j;
            ++ns;
          }
        }
      }
  if (!mode) {
    n_pred[i] = np;
    n_succ[i] = ns;
  }
}

constexpr int32_t kUndet = -2;
constexpr int32_t kAnchor = -1;

__global__ void anchor_init_kernel(const int32_t* __restrict__ n_pred, int64_t n, int32_t* __restrict__ owner) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) owner[i] = n_pred[i] == 0 ? kAnchor : kUndet;
}

// i is claimed by the smallest anchor among its preds; an anchor when none
// of its preds is one.  Decided once every pred is decided.
__global__ void anchor_step_kernel(const int32_t* __restrict__ n_pred, const int64_t* __restrict__ pred_off,
                                   const int32_t* __restrict__ pred, int64_t n, int32_t* __restrict__ owner,
                                   int32_t* __restrict__ changed) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || owner[i] != kUndet) return;
  // preds ascending: the first anchor among them owns i; an undecided pred
  // before it means "wait"; none => i is an anchor
  for (int32_t k = 0; k < n_pred[i]; ++k) {
    const int32_t j = pred[pred_off[i] + k];
    const int32_t o = owner[j];
    if (o == kUndet) {
      *changed = 1;
      return;
    }
    if (o == kAnchor) {
      owner[i] = j;
      *changed = 1;
      return;
    }
  }
  owner[i] = kAnchor;
  *changed = 1;
}

// merged image per anchor: image_sources.cpp:103-128
__global__ void merge_emit_kernel(ImgTmp t, int64_t n, const int32_t* __restrict__ owner,
                                  const int32_t* __restrict__ n_succ, const int64_t* __restrict__ succ_off,
                                  const int32_t* __restrict__ succ, const int32_t* __restrict__ anchor_rank,
                                  PathView pv, ImgTmp out, int64_t n_out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || owner[i] != kAnchor) return;
  int32_t cnt = t.count[i];
  D3 w = d3(t.pos[3 * i] * static_cast<double>(cnt), t.pos[3 * i + 1] * static_cast<double>(cnt),
            t.pos[3 * i + 2] * static_cast<double>(cnt));
  int32_t rep = t.rep[i];
  // claims in increasing index order (the succ list is sorted below)
  for (int32_t k = 0; k < n_succ[i]; ++k) {
    const int32_t j = succ[succ_off[i] + k];
    if (owner[j] != i) continue;
    const double cj = static_cast<double>(t.count[j]);
    w = w + d3(t.pos[3 * j] * cj, t.pos[3 * j + 1] * cj, t.pos[3 * j + 2] * cj);
    cnt += t.count[j];
    if (pv.cmp(t.rep[j], rep) < 0) rep = t.rep[j];
  }
  const int64_t s = anchor_rank[i];
  const double m = static_cast<double>(cnt);
  out.pos[3 * s] = w.x / m;
  out.pos[3 * s + 1] = w.y / m;
  out.pos[3 * s + 2] = w.z / m;
  out.count[s] = cnt;
  out.order[s] = t.order[i];
  out.rep[s] = rep;       // path source (lexicographic minimum)
  out.rep[n_out + s] = t.rep[i];  // multiplier source (the anchor's, :113)
}

__global__ void sort_small_lists_kernel(const int32_t* __restrict__ cnt, const int64_t* __restrict__ off, int64_t n,
                                        int32_t* __restrict__ list) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t* a = list + off[i];
  const int32_t m = cnt[i];
  for (int32_t x = 1; x < m; ++x) {  // insertion sort (lists are tiny)
    const int32_t v = a[x];
    int32_t y = x - 1;
    while (y >= 0 && a[y] > v) {
      a[y + 1] = a[y];
      --y;
    }
    a[y + 1] = v;
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

// final order (order, distance, face path), image_sources.cpp:163-168
struct FinalLess {
  const int32_t* order;
  const double* dist;
  const int32_t* rep;
  PathView pv;
  __device__ bool operator()(int32_t a, int32_t b) const {
    if (order[a] != order[b]) return order[a] < order[b];
    if (dist[a] != dist[b]) return dist[a] < dist[b];
    return pv.cmp(rep[a], rep[b]) < 0;
  }
};

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
  for (int64_t k = 0; k < len; ++k) im.path[o + k] = pv.hist[a0 + k];
  im.path_off[i] = o;
  if (i == n - 1) im.path_off[n] = o + len;
}

inline unsigned grid(int64_t n, int b = 256) { return static_cast<unsigned>((n + b - 1) / b); }

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
  std::vector<int32_t> hrecv(nc_all);
  if (nc_all) RR_CUDA(cudaMemcpyAsync(hrecv.data(), tr->c_recv.p, sizeof(int32_t) * nc_all, cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  const int64_t c0 = std::lower_bound(hrecv.begin(), hrecv.end(), recv) - hrecv.begin();
  const int64_t c1 = std::upper_bound(hrecv.begin(), hrecv.end(), recv) - hrecv.begin();
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
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceMergeSort::StableSortKeys(t, b, idx.p, n, PathLess{pv}, st);
  }, st);
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
  group_count_kernel<<<grid(ng, 128), 128, 0, st>>>(idx.p, gstart.p, ng, n, retro.p, c0, tol, n_img.p, is_split.p);
  RR_LAUNCH_CHECK();
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
  group_emit_kernel<<<grid(ng, 128), 128, 0, st>>>(idx.p, gstart.p, ng, n, retro.p, c0, tol, is_split.p, img_off.p,
                                              tr->c_off.p, T);
  RR_LAUNCH_CHECK();
  ctx->launches += 8;
  tm.mark("groups");

  // multiplier source per image: the representative capture (beam.front())
  DevBuf<double> mpos;
  DevBuf<int32_t> mcount, morder, mrep;
  ImgTmp M = T;
  const int32_t* mult_src = trep.p;
  if (opt.merge_coplanar && ni > 1) {
    const double cs = 2.0 * tol;
    DevBuf<unsigned long long> keys, skeys;
    DevBuf<int32_t> ids, sids;
    keys.alloc(ni, st);
    skeys.alloc(ni, st);
    ids.alloc(ni, st);
    sids.alloc(ni, st);
    cell_key_kernel<<<grid(ni), 256, 0, st>>>(T, ni, cs, keys.p, ids.p);
    RR_LAUNCH_CHECK();
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, keys.p, skeys.p, ids.p, sids.p, ni, 0, 64, st);
    }, st);
    DevBuf<int32_t> n_pred, n_succ;
    DevBuf<int64_t> pred_off, succ_off;
    n_pred.alloc(ni + 1, st);
    n_succ.alloc(ni + 1, st);
    pred_off.alloc(ni + 1, st);
    succ_off.alloc(ni + 1, st);
    RR_CUDA(cudaMemsetAsync(n_pred.p + ni, 0, sizeof(int32_t), st));
    RR_CUDA(cudaMemsetAsync(n_succ.p + ni, 0, sizeof(int32_t), st));
    neighbour_kernel<<<grid(ni, 128), 128, 0, st>>>(T, tr->c_mult.p, ni, cs, tol, skeys.p, sids.p, 0, n_pred.p,
                                                n_succ.p, nullptr, nullptr, nullptr, nullptr);
    RR_LAUNCH_CHECK();
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, n_pred.p, pred_off.p, ni + 1, st);
    }, st);
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, n_succ.p, succ_off.p, ni + 1, st);
    }, st);
    int64_t tp = 0, ts = 0;
    RR_CUDA(cudaMemcpyAsync(&tp, pred_off.p + ni, sizeof tp, cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaMemcpyAsync(&ts, succ_off.p + ni, sizeof ts, cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
    DevBuf<int32_t> pred, succ, owner, changed;
    pred.alloc(std::max<int64_t>(tp, 1), st);
    succ.alloc(std::max<int64_t>(ts, 1), st);
    owner.alloc(ni, st);
    changed.alloc(1, st);
    neighbour_kernel<<<grid(ni, 128), 128, 0, st>>>(T, tr->c_mult.p, ni, cs, tol, skeys.p, sids.p, 1, n_pred.p,
                                                n_succ.p, pred_off.p, succ_off.p, pred.p, succ.p);
    RR_LAUNCH_CHECK();
    sort_small_lists_kernel<<<grid(ni), 256, 0, st>>>(n_succ.p, succ_off.p, ni, succ.p);
    sort_small_lists_kernel<<<grid(ni), 256, 0, st>>>(n_pred.p, pred_off.p, ni, pred.p);
    RR_LAUNCH_CHECK();
    anchor_init_kernel<<<grid(ni), 256, 0, st>>>(n_pred.p, ni, owner.p);
    RR_LAUNCH_CHECK();
    ctx->launches += 8;
    for (int it = 0; it < 100000; ++it) {
      int32_t h = 0;
      RR_CUDA(cudaMemsetAsync(changed.p, 0, sizeof(int32_t), st));
      anchor_step_kernel<<<grid(ni), 256, 0, st>>>(n_pred.p, pred_off.p, pred.p, ni, owner.p, changed.p);
      RR_LAUNCH_CHECK();
      ctx->launches++;
      RR_CUDA(cudaMemcpyAsync(&h, changed.p, sizeof h, cudaMemcpyDeviceToHost, st));
      RR_CUDA(cudaStreamSynchronize(st));
      if (!h) break;
    }
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
    merge_emit_kernel<<<grid(ni), 256, 0, st>>>(T, ni, owner.p, n_succ.p, succ_off.p, succ.p, arank.p, pv, M, na);
    RR_LAUNCH_CHECK();
    ctx->launches += 3;
    ni = na;
    mult_src = mrep.p + na;
  }
  tm.mark("coplanar merge");
  EnergyParams ep;
  ep.hdr = s->hdr;
  ep.nodes = s->tnodes.p;
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
    std::vector<int32_t> iota(ni);
    for (int64_t i = 0; i < ni; ++i) iota[i] = static_cast<int32_t>(i);
    RR_CUDA(cudaMemcpyAsync(perm.p, iota.data(), sizeof(int32_t) * ni, cudaMemcpyHostToDevice, st));
    RR_CUDA(cudaStreamSynchronize(st));
  }
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceMergeSort::SortKeys(t, b, perm.p, ni, FinalLess{M.order, dist.p, M.rep, pv}, st);
  }, st);
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
  final_gather_kernel<<<grid(ni), 256, 0, st>>>(perm.p, ni, M, dist.p, energy.p, mult.p, has_proj.p, proj.p, pv,
                                                im->path_off.p,
                                                ImgOut{im->pos.p, im->dist.p, im->energy.p, im->mult.p, im->proj.p,
                                                       im->ray_count.p, im->order.p, im->has_proj.p, im->path.p,
                                                       im->path_off.p});
  RR_LAUNCH_CHECK();
  ctx->launches += 6;
  tm.mark("gather");
  RR_CUDA(cudaStreamSynchronize(st));
  return im.release();
}

}  // namespace rr
