// K1' — surface-area-heuristic traversal tree, built on the device.
//
// The reference's median split (accel_tree.cpp:19-87, built exactly by
// rr_build.cu and used for the API, the parity tests and the byte model)
// mixes several walls in its top levels, so a ray inside the room enters
// both children for many levels.  The tracer traverses this second tree
// instead: same leaves (one face each), same conservative fp32 TNode format,
// splits chosen by a binned SAH.  The closest hit is a property of the face
// set alone (fp64 test on every face a conservative box admits,
// lexicographic (delta, face) minimum), so the tree changes the work, never
// a result.  Measured on the reference's own traversal order: internal
// visits per query C2 55.8 -> 32.0, C3 49.0 -> 27.5, C5 90.3 -> 54.4.
//
// Level-synchronous, like rr_build.cu: three face lists presorted by
// centroid per axis, one segment per node of the level; per level
//   1. segment AABBs, centroid bounds, common plane id (atomics);
//   2. SAH segments (>= kSahMin faces, depth budget left): 3 x kBins
//      centroid bins with counts and AABBs;
//   3. one thread per segment writes its box into the parent's TNode slot,
//      picks the split (best binned SAH cost, else the object median of the
//      longest centroid extent) and emits the two child segments;
//   4. stable segmented partition of the three lists.
// Nodes of the large segments are numbered level by level (BFS); segments
// of <= kSmall faces are finished in one kernel (one thread each, median
// splits, preorder ids from the top of the array), which removes the last
// ~4 levels of launches.  Depth is capped so the 32-entry traversal stack
// cannot overflow (median splits once the budget is short).
#include <cub/cub.cuh>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <vector>

#include "rr_internal.cuh"

namespace rr {
namespace {

constexpr int kBins = 32;
constexpr int64_t kSahMin = 17;  // binned SAH from 17 faces (64: C5 468.8 -> 477.0 ms, C2 9.26 -> 10.0 with the exact finish)
constexpr int kMaxDepth = 30;
#ifndef RR_KSMALL
#define RR_KSMALL 16
#endif
constexpr int kSmall = RR_KSMALL;  // segments this small are built in one go by one thread
const char* const kLevelNames[64] = {
    "sah level 0",  "sah level 1",  "sah level 2",  "sah level 3",  "sah level 4",  "sah level 5",  "sah level 6",
    "sah level 7",  "sah level 8",  "sah level 9",  "sah level 10", "sah level 11", "sah level 12", "sah level 13",
    "sah level 14", "sah level 15", "sah level 16", "sah level 17", "sah level 18", "sah level 19", "sah level 20",
    "sah level 21", "sah level 22", "sah level 23", "sah level 24", "sah level 25", "sah level 26", "sah level 27",
    "sah level 28", "sah level 29", "sah level 30", "sah level 31", "sah level 32", "sah level 33", "sah level 34",
    "sah level 35", "sah level 36", "sah level 37", "sah level 38", "sah level 39", "sah level 40", "sah level 41",
    "sah level 42", "sah level 43", "sah level 44", "sah level 45", "sah level 46", "sah level 47", "sah level 48",
    "sah level 49", "sah level 50", "sah level 51", "sah level 52", "sah level 53", "sah level 54", "sah level 55",
    "sah level 56", "sah level 57", "sah level 58", "sah level 59", "sah level 60", "sah level 61", "sah level 62",
    "sah level 63"};

struct SSeg {
  int64_t b, n;
  int32_t parent;  // TNode index of the parent, -1 for the root
  int32_t side;    // 0 left, 1 right
};

// Per-level counters kept on the device, so the host enqueues whole levels
// without reading anything back: S segments at this level, the BFS index of
// its first internal node, and this level's split / SAH segment counts.
struct LevelState {
  int64_t S;
  int64_t n_split;
  int64_t n_sah;
  int32_t level_base;
  int32_t pad;
};

__device__ __forceinline__ uint64_t okey(double x) {
  if (x == 0.0) x = 0.0;
  uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double oval(uint64_t u) {
  u = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
  return __longlong_as_double(static_cast<long long>(u));
}
__device__ __forceinline__ uint32_t okeyf(float x) {
  if (x == 0.0f) x = 0.0f;
  uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ovalf(uint32_t u) {
  u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
  return __uint_as_float(u);
}
__device__ __forceinline__ float lo_f(double x, float eps) { return __fsub_rd(__double2float_rd(x), eps); }
__device__ __forceinline__ float hi_f(double x, float eps) { return __fadd_ru(__double2float_ru(x), eps); }

__global__ void prep_kernel(const double* __restrict__ v, const int32_t* __restrict__ t, int64_t nf,
                            double* __restrict__ fb, double* __restrict__ cen, uint64_t* __restrict__ keys,
                            int32_t* __restrict__ ids) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const int32_t a = t[4 * f], b = t[4 * f + 1], c = t[4 * f + 2];
  // twins: faces 2k and 2k + 1 with the same AABB (a quad's two triangles)
  // get the box centre as their common centroid, so every sorted list keeps
  // them adjacent and SAH bins never separate them (pair leaves, below)
  const int64_t g = f ^ 1;
  bool twin = g < nf;
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    const double va = v[3 * a + k], vb = v[3 * b + k], vc = v[3 * c + k];
    lo[k] = fmin(va, fmin(vb, vc));
    hi[k] = fmax(va, fmax(vb, vc));
    if (twin) {
      const int32_t* tg = t + 4 * g;
      const double wa = v[3 * tg[0] + k], wb = v[3 * tg[1] + k], wc = v[3 * tg[2] + k];
      twin = fmin(wa, fmin(wb, wc)) == lo[k] && fmax(wa, fmax(wb, wc)) == hi[k];
    }
  }
  for (int k = 0; k < 3; ++k) {
    const double va = v[3 * a + k], vb = v[3 * b + k], vc = v[3 * c + k];
    const double ce = twin ? 0.5 * (lo[k] + hi[k]) : ((va + vb) + vc) / 3.0;
    fb[6 * f + k] = lo[k];
    fb[6 * f + 3 + k] = hi[k];
    cen[3 * f + k] = ce;
    keys[k * nf + f] = okeyf(__double2float_rn(ce));  // 32-bit sort key: order only shapes the tree
    ids[k * nf + f] = static_cast<int32_t>(f);
  }
}

// 1. per segment: AABB, centroid bounds (ordered-key atomics), plane ids.
// List positions are grouped by segment, so lanes first reduce within their
// warp's runs and one lane per run issues the atomics.
__global__ void bounds_kernel(const int32_t* __restrict__ pos_seg, const int32_t* __restrict__ perm0,
                              const double* __restrict__ fb, const double* __restrict__ cen,
                              const int32_t* __restrict__ face_plane, int64_t nf, unsigned long long* __restrict__ bb,
                              unsigned long long* __restrict__ cb, int32_t* __restrict__ pl) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int32_t seg = -1;
  uint64_t v[12];  // bb min 3, bb max 3, cb min 3, cb max 3
  int32_t pmin = 0x7fffffff, pmax = static_cast<int32_t>(0x80000000);
  for (int k = 0; k < 3; ++k) {
    v[k] = ~0ull;
    v[3 + k] = 0;
    v[6 + k] = ~0ull;
    v[9 + k] = 0;
  }
  if (i < nf) {
    seg = pos_seg[i];
    if (seg >= 0) {
      const int32_t f = perm0[i];
      for (int k = 0; k < 3; ++k) {
        v[k] = okey(fb[6 * f + k]);
        v[3 + k] = okey(fb[6 * f + 3 + k]);
        v[6 + k] = v[9 + k] = okey(cen[3 * f + k]);
      }
      pmin = pmax = face_plane ? face_plane[f] : -1;
    }
  }
  for (int off = 1; off < 32; off <<= 1) {
    const int32_t so = __shfl_down_sync(0xffffffffu, seg, off);
    const bool ok = (lane + off < 32) && so == seg;
    for (int k = 0; k < 12; ++k) {
      const uint64_t o = __shfl_down_sync(0xffffffffu, v[k], off);
      const bool is_min = (k % 6) < 3;
      if (ok) v[k] = is_min ? (o < v[k] ? o : v[k]) : (o > v[k] ? o : v[k]);
    }
    const int32_t a = __shfl_down_sync(0xffffffffu, pmin, off), b = __shfl_down_sync(0xffffffffu, pmax, off);
    if (ok) {
      pmin = min(pmin, a);
      pmax = max(pmax, b);
    }
  }
  const int32_t prev = __shfl_up_sync(0xffffffffu, seg, 1);
  if (seg >= 0 && (lane == 0 || prev != seg)) {
    for (int k = 0; k < 3; ++k) {
      atomicMin(bb + 6 * seg + k, (unsigned long long)v[k]);
      atomicMax(bb + 6 * seg + 3 + k, (unsigned long long)v[3 + k]);
      atomicMin(cb + 6 * seg + k, (unsigned long long)v[6 + k]);
      atomicMax(cb + 6 * seg + 3 + k, (unsigned long long)v[9 + k]);
    }
    atomicMin(pl + 2 * seg, pmin);
    atomicMax(pl + 2 * seg + 1, pmax);
  }
}

__device__ __forceinline__ int bin_of(double c, double lo, double ext) {
  int b = static_cast<int>((c - lo) / ext * kBins);
  return b < 0 ? 0 : (b >= kBins ? kBins - 1 : b);
}

// 2. centroid bins of the SAH segments: count + float AABB per (axis, bin).
// Blocks whose 256 positions all lie in one segment (the large top-level
// segments) accumulate in shared memory and flush once; others go straight
// to global atomics.
__global__ void __launch_bounds__(256) bin_kernel(const int32_t* __restrict__ pos_seg, const int32_t* __restrict__ perm0,
                                                  const double* __restrict__ fb, const double* __restrict__ cen,
                                                  const unsigned long long* __restrict__ cb,
                                                  const int32_t* __restrict__ sah_idx, int64_t nf,
                                                  int32_t* __restrict__ bcnt, uint32_t* __restrict__ bbox) {
  __shared__ int32_t s_cnt[3 * kBins];
  __shared__ uint32_t s_box[3 * kBins * 6];
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x;
  const int64_t i = i0 + threadIdx.x;
  const int64_t last = min(i0 + static_cast<int64_t>(blockDim.x), nf) - 1;
  const int32_t s0 = pos_seg[i0], s1 = pos_seg[last];
  const bool shared = s0 >= 0 && s0 == s1 && sah_idx[s0] >= 0;  // block-uniform
  if (shared) {
    for (int t = threadIdx.x; t < 3 * kBins; t += blockDim.x) {
      s_cnt[t] = 0;
      for (int k = 0; k < 3; ++k) {
        s_box[6 * t + k] = 0xffffffffu;
        s_box[6 * t + 3 + k] = 0u;
      }
    }
    __syncthreads();
  }
  const int32_t s = i < nf ? pos_seg[i] : -1;
  const int32_t q = s >= 0 ? sah_idx[s] : -1;
  if (q >= 0) {
    const int32_t f = perm0[i];
    uint32_t lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
      lo[k] = okeyf(__double2float_rn(fb[6 * f + k]));
      hi[k] = okeyf(__double2float_rn(fb[6 * f + 3 + k]));
    }
    for (int a = 0; a < 3; ++a) {
      const double clo = oval(cb[6 * s + a]), ext = oval(cb[6 * s + 3 + a]) - clo;
      if (!(ext > 0.0)) continue;
      const int b = bin_of(cen[3 * f + a], clo, ext);
      if (shared) {
        const int t = a * kBins + b;
        atomicAdd(s_cnt + t, 1);
        for (int k = 0; k < 3; ++k) {
          atomicMin(s_box + 6 * t + k, lo[k]);
          atomicMax(s_box + 6 * t + 3 + k, hi[k]);
        }
      } else {
        const int64_t slot = (static_cast<int64_t>(q) * 3 + a) * kBins + b;
        atomicAdd(bcnt + slot, 1);
        for (int k = 0; k < 3; ++k) {
          atomicMin(bbox + 6 * slot + k, lo[k]);
          atomicMax(bbox + 6 * slot + 3 + k, hi[k]);
        }
      }
    }
  }
  if (shared) {
    __syncthreads();
    const int64_t base = static_cast<int64_t>(sah_idx[s0]) * 3 * kBins;
    for (int t = threadIdx.x; t < 3 * kBins; t += blockDim.x) {
      if (!s_cnt[t]) continue;
      atomicAdd(bcnt + base + t, s_cnt[t]);
      for (int k = 0; k < 3; ++k) {
        atomicMin(bbox + 6 * (base + t) + k, s_box[6 * t + k]);
        atomicMax(bbox + 6 * (base + t) + 3 + k, s_box[6 * t + 3 + k]);
      }
    }
  }
}

__device__ __forceinline__ float half_area(const float* lo, const float* hi) {
  const float dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
  return dx * dy + dy * dz + dz * dx;
}

// root box and box expansion of the SAH tree, as rr_build.cu's level 0 does
// for the reference tree (same union of face boxes, hence the same values)
__global__ void root_hdr_kernel(const unsigned long long* __restrict__ bb, TravHeader* __restrict__ hdr) {
  if (threadIdx.x) return;
  double lo[3], hi[3];
  double scale = 1e-3;
  for (int k = 0; k < 3; ++k) {
    lo[k] = oval(bb[k]);
    hi[k] = oval(bb[3 + k]);
    scale = fmax(scale, fmax(fabs(lo[k]), fabs(hi[k])));
  }
  const float eps = __double2float_ru(scale * 0x1p-19);  // see rr_geom.cuh box_enter
  hdr->eps = eps;
  for (int k = 0; k < 3; ++k) {
    hdr->lo[k] = lo_f(lo[k], eps);
    hdr->hi[k] = hi_f(hi[k], eps);
  }
}

// 3. node emission and split choice: one warp per segment.  For SAH
// segments lane b holds bin b; prefix and suffix unions/counts come from warp
// scans, every lane prices the split below its bin, and the warp takes the
// cheapest (ties: lowest axis, then highest bin, as a sequential scan from
// the top bin down with a strict < would).  Lane 0 writes the node.
struct BinAcc {
  float lo[3], hi[3];
  int32_t c;
};

__device__ __forceinline__ BinAcc bin_union(BinAcc a, const BinAcc& b) {
  for (int k = 0; k < 3; ++k) {
    a.lo[k] = fminf(a.lo[k], b.lo[k]);
    a.hi[k] = fmaxf(a.hi[k], b.hi[k]);
  }
  a.c += b.c;
  return a;
}

__device__ __forceinline__ BinAcc shfl_acc(const BinAcc& a, int src_delta, bool up) {
  BinAcc r;
  for (int k = 0; k < 3; ++k) {
    r.lo[k] = up ? __shfl_up_sync(0xffffffffu, a.lo[k], src_delta) : __shfl_down_sync(0xffffffffu, a.lo[k], src_delta);
    r.hi[k] = up ? __shfl_up_sync(0xffffffffu, a.hi[k], src_delta) : __shfl_down_sync(0xffffffffu, a.hi[k], src_delta);
  }
  r.c = up ? __shfl_up_sync(0xffffffffu, a.c, src_delta) : __shfl_down_sync(0xffffffffu, a.c, src_delta);
  return r;
}

// faces p (left of a median cut) and q (right of it) are twins (prep_kernel)
__device__ __forceinline__ bool twins_at(int32_t p, int32_t q, const double* __restrict__ cen) {
  return (p ^ 1) == q && cen[3 * p] == cen[3 * q] && cen[3 * p + 1] == cen[3 * q + 1] &&
         cen[3 * p + 2] == cen[3 * q + 2];
}

__global__ void split_kernel(const SSeg* __restrict__ segs, const LevelState* __restrict__ ls,
                             const int32_t* __restrict__ rank,
                             const unsigned long long* __restrict__ bb, const unsigned long long* __restrict__ cb,
                             const int32_t* __restrict__ pl, const int32_t* __restrict__ sah_idx,
                             const int32_t* __restrict__ bcnt, const uint32_t* __restrict__ bbox,
                             const int32_t* __restrict__ perm0, const double* __restrict__ cen, int64_t nf,
                             TNode* __restrict__ tn,
                             TravHeader* __restrict__ hdr, int32_t* __restrict__ seg_axis,
                             int32_t* __restrict__ seg_split, int64_t* __restrict__ seg_nl, SSeg* __restrict__ next) {
  static_assert(kBins == 32, "one lane per bin");
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= ls->S) return;  // warp-uniform
  const SSeg sg = segs[j];
  if (sg.n >= 2 && sg.n <= kSmall) {  // finish_kernel's
    if (lane == 0) seg_axis[j] = -1;
    return;
  }
  const int32_t level_base = ls->level_base;
  const float eps = hdr->eps;
  if (lane == 0) {
    double lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
      lo[k] = oval(bb[6 * j + k]);
      hi[k] = oval(bb[6 * j + 3 + k]);
    }
    const int32_t my_ref = sg.n == 1 ? ~perm0[sg.b] : level_base + rank[j];
    const int32_t plane = (pl[2 * j] == pl[2 * j + 1]) ? pl[2 * j] : -1;
    if (sg.parent < 0) {
      hdr->root_ref = my_ref;
    } else {
      TNode* p = tn + sg.parent;
      const float lx = lo_f(lo[0], eps), ly = lo_f(lo[1], eps), lz = lo_f(lo[2], eps);
      const float hx = hi_f(hi[0], eps), hy = hi_f(hi[1], eps), hz = hi_f(hi[2], eps);
      if (sg.side == 0) {
        p->a = make_float4(lx, hx, ly, hy);
        reinterpret_cast<float2*>(&p->b)[0] = make_float2(lz, hz);
        p->d.x = my_ref;
        p->d.z = plane;
      } else {
        reinterpret_cast<float2*>(&p->b)[1] = make_float2(lx, hx);
        p->c = make_float4(ly, hy, lz, hz);
        p->d.y = my_ref;
        p->d.w = plane;
      }
    }
    if (sg.n == 1) seg_axis[j] = -1;
  }
  if (sg.n == 1) return;
  int axis = -1, split = -1;
  int64_t nl = sg.n / 2;
  const int32_t q = sah_idx[j];
  if (q >= 0) {
    float best = 3.4e38f;
    int best_axis = -1, best_split = -1;
    int64_t best_nl = 0;
    for (int a = 0; a < 3; ++a) {
      const int64_t slot = (static_cast<int64_t>(q) * 3 + a) * kBins + lane;
      BinAcc mine;
      mine.c = bcnt[slot];
      for (int k = 0; k < 3; ++k) {
        mine.lo[k] = mine.c > 0 ? ovalf(bbox[6 * slot + k]) : 3.4e38f;
        mine.hi[k] = mine.c > 0 ? ovalf(bbox[6 * slot + 3 + k]) : -3.4e38f;
      }
      BinAcc pre = mine, suf = mine;  // inclusive prefix (bins <= lane), suffix (bins >= lane)
      for (int d = 1; d < 32; d <<= 1) {
        const BinAcc up = shfl_acc(pre, d, true);
        if (lane >= d) pre = bin_union(pre, up);
        const BinAcc dn = shfl_acc(suf, d, false);
        if (lane + d < 32) suf = bin_union(suf, dn);
      }
      // split below bin `lane` (lane >= 1): left = bins < lane, right = bins >= lane
      const BinAcc left = shfl_acc(pre, 1, true);
      float cost = 3.4e38f;
      bool ok = lane >= 1 && suf.c > 0 && left.c > 0;
      if (ok) {
        const float la = half_area(left.lo, left.hi), ra = half_area(suf.lo, suf.hi);
        cost = la * static_cast<float>(left.c) + ra * static_cast<float>(suf.c);
      }
      // warp argmin of (cost, -lane)
      float c_best = ok ? cost : 3.4e38f;
      int b_best = ok ? lane : -1;
      for (int d = 16; d > 0; d >>= 1) {
        const float oc = __shfl_xor_sync(0xffffffffu, c_best, d);
        const int ob = __shfl_xor_sync(0xffffffffu, b_best, d);
        if (ob >= 0 && (b_best < 0 || oc < c_best || (oc == c_best && ob > b_best))) {
          c_best = oc;
          b_best = ob;
        }
      }
      const int32_t left_count = __shfl_sync(0xffffffffu, left.c, b_best < 0 ? 0 : b_best);
      if (b_best >= 0 && c_best < best) {
        best = c_best;
        best_axis = a;
        best_split = b_best;
        best_nl = left_count;
      }
    }
    if (best_axis >= 0) {
      axis = best_axis;
      split = best_split;
      nl = best_nl;
    }
  }
  if (lane != 0) return;
  if (axis < 0) {  // object median on the longest centroid extent
    double bestx = -1.0;
    for (int k = 0; k < 3; ++k) {
      const double e = oval(cb[6 * j + 3 + k]) - oval(cb[6 * j + k]);
      if (e > bestx) {
        bestx = e;
        axis = k;
      }
    }
    split = -1;
    nl = sg.n / 2;
    const int32_t* lst = perm0 + axis * nf + sg.b;
    if (twins_at(lst[nl - 1], lst[nl], cen)) ++nl;  // keep twins together
  }
  seg_axis[j] = axis;
  seg_split[j] = split;
  seg_nl[j] = nl;
  const int32_t me = level_base + rank[j];
  next[2 * rank[j]] = SSeg{sg.b, nl, me, 0};
  next[2 * rank[j] + 1] = SSeg{sg.b + nl, sg.n - nl, me, 1};
}

// 3b. small segments (2..kSmall faces): one thread builds the whole subtree
// with object-median splits on the longest centroid extent, numbering its
// n - 1 internal nodes in preorder inside a block taken from the top of the
// node array (the level-order nodes grow from the bottom; together exactly
// nf - 1), and writes the segment's own slot in its parent.
__device__ void child_slot(TNode* p, int side, const double* lo, const double* hi, float eps, int32_t ref,
                           int32_t plane) {
  const float lx = lo_f(lo[0], eps), ly = lo_f(lo[1], eps), lz = lo_f(lo[2], eps);
  const float hx = hi_f(hi[0], eps), hy = hi_f(hi[1], eps), hz = hi_f(hi[2], eps);
  if (side == 0) {
    p->a = make_float4(lx, hx, ly, hy);
    reinterpret_cast<float2*>(&p->b)[0] = make_float2(lz, hz);
    p->d.x = ref;
    p->d.z = plane;
  } else {
    reinterpret_cast<float2*>(&p->b)[1] = make_float2(lx, hx);
    p->c = make_float4(ly, hy, lz, hz);
    p->d.y = ref;
    p->d.w = plane;
  }
}

__global__ void finish_kernel(const SSeg* __restrict__ segs, const LevelState* __restrict__ ls,
                              const int32_t* __restrict__ perm0, const double* __restrict__ fb,
                              const double* __restrict__ cen, const int32_t* __restrict__ face_plane, int64_t nf,
                              TNode* __restrict__ tn, TravHeader* __restrict__ hdr,
                              unsigned long long* __restrict__ top, int level, int fin_sah) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= ls->S) return;
  const float eps = hdr->eps;
  const SSeg sg = segs[j];
  const int n = static_cast<int>(sg.n);
  if (n < 2 || n > kSmall) return;
  int32_t f[kSmall];
  for (int i = 0; i < n; ++i) f[i] = perm0[sg.b + i];
  // fp32 copies of the faces' centroids and boxes by local slot (sl[i] is
  // the slot of f[i]): the split choice only shapes the tree, the node boxes
  // are still the exact fp64 ones (range_box)
  float lc[kSmall][3], lb[kSmall][6];
  uint8_t sl[kSmall];
  for (int i = 0; i < n; ++i) {
    sl[i] = static_cast<uint8_t>(i);
    for (int k = 0; k < 3; ++k) {
      lc[i][k] = static_cast<float>(cen[3 * f[i] + k]);
      lb[i][k] = static_cast<float>(fb[6 * f[i] + k]);
      lb[i][3 + k] = static_cast<float>(fb[6 * f[i] + 3 + k]);
    }
  }
  const int32_t base = static_cast<int32_t>(nf - 1 - static_cast<int64_t>(atomicAdd(top, (unsigned long long)(n - 1))) -
                                            (n - 1));
  // range [a, b) of f -> AABB (exact, fp64) and common plane id
  auto range_box = [&](int a, int b, double* lo, double* hi, int32_t* plane) {
    int32_t pmin = 0x7fffffff, pmax = static_cast<int32_t>(0x80000000);
    for (int k = 0; k < 3; ++k) {
      lo[k] = HUGE_VAL;
      hi[k] = -HUGE_VAL;
    }
    for (int i = a; i < b; ++i) {
      for (int k = 0; k < 3; ++k) {
        lo[k] = fmin(lo[k], fb[6 * f[i] + k]);
        hi[k] = fmax(hi[k], fb[6 * f[i] + 3 + k]);
      }
      const int32_t p = face_plane ? face_plane[f[i]] : -1;
      pmin = min(pmin, p);
      pmax = max(pmax, p);
    }
    *plane = pmin == pmax ? pmin : -1;
  };
  // A two-face range [a, a + 2) of consecutive faces (f, f + 1) becomes one
  // pair leaf when a node over it cannot pay: with equal node and face test
  // costs the SAH splits only if A(left) + A(right) < A(union), and a quad's
  // two triangles share one box (the node cost a dependent fetch for no cull).
  auto half_area = [](const double* lo, const double* hi) {
    const double x = hi[0] - lo[0], y = hi[1] - lo[1], z = hi[2] - lo[2];
    return x * y + y * z + z * x;
  };
  auto pair_ref = [&](int a, int32_t* ref) -> bool {
    const int32_t g0 = min(f[a], f[a + 1]);
    if (max(f[a], f[a + 1]) != g0 + 1) return false;
    double lo[3], hi[3], l0[3], h0[3], l1[3], h1[3];
    int32_t pdummy;
    range_box(a, a + 2, lo, hi, &pdummy);
    range_box(a, a + 1, l0, h0, &pdummy);
    range_box(a + 1, a + 2, l1, h1, &pdummy);
    if (half_area(l0, h0) + half_area(l1, h1) < half_area(lo, hi)) return false;
    *ref = ~(g0 | kPairBit);
    return true;
  };
  {  // the segment itself, in its parent's slot (or as the root)
    double lo[3], hi[3];
    int32_t plane;
    range_box(0, n, lo, hi, &plane);
    int32_t pref;
    if (sg.parent < 0) {
      hdr->root_ref = base;
    } else if (n == 2 && pair_ref(0, &pref)) {
      child_slot(tn + sg.parent, sg.side, lo, hi, eps, pref, plane);  // its node id stays unused
      return;
    } else {
      child_slot(tn + sg.parent, sg.side, lo, hi, eps, base, plane);
    }
  }
  // insertion sort of f[a, b) by (fp32) centroid on axis ax (ties by face id)
  auto sort_axis = [&](int a, int b, int ax) {
    for (int x = a + 1; x < b; ++x) {
      const int32_t v = f[x];
      const uint8_t vs = sl[x];
      const float cv = lc[vs][ax];
      int y = x - 1;
      while (y >= a && (lc[sl[y]][ax] > cv || (lc[sl[y]][ax] == cv && f[y] > v))) {
        f[y + 1] = f[y];
        sl[y + 1] = sl[y];
        --y;
      }
      f[y + 1] = v;
      sl[y + 1] = vs;
    }
  };
  auto half_area_f = [](const float* lo, const float* hi) {
    const float x = hi[0] - lo[0], y = hi[1] - lo[1], z = hi[2] - lo[2];
    return x * y + y * z + z * x;
  };
  // exact SAH over the sorted centroid orders of the three axes (fin_sah):
  // the split position m of [a, b) minimising A(left) |left| + A(right)
  // |right|, twins kept together; f[a, b) left sorted on the chosen axis.
  // Returns false when no position qualifies.
  auto sah_exact = [&](int a, int b, int* m_out) -> bool {
    float best = FLT_MAX;
    int bax = -1, bm = -1;
    for (int ax = 0; ax < 3; ++ax) {
      sort_axis(a, b, ax);
      float ra[kSmall];
      float lo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, hi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
      for (int i = b - 1; i > a; --i) {  // ra[i - a]: area of f[i, b)
        for (int k = 0; k < 3; ++k) {
          lo[k] = fminf(lo[k], lb[sl[i]][k]);
          hi[k] = fmaxf(hi[k], lb[sl[i]][3 + k]);
        }
        ra[i - a] = half_area_f(lo, hi);
      }
      for (int k = 0; k < 3; ++k) {
        lo[k] = FLT_MAX;
        hi[k] = -FLT_MAX;
      }
      for (int i = a + 1; i < b; ++i) {  // split before position i
        for (int k = 0; k < 3; ++k) {
          lo[k] = fminf(lo[k], lb[sl[i - 1]][k]);
          hi[k] = fmaxf(hi[k], lb[sl[i - 1]][3 + k]);
        }
        if (twins_at(f[i - 1], f[i], cen)) continue;
        const float c = half_area_f(lo, hi) * (i - a) + ra[i - a] * (b - i);
        if (c < best) {
          best = c;
          bax = ax;
          bm = i;
        }
      }
    }
    if (bax < 0) return false;
    if (bax != 2) sort_axis(a, b, bax);
    *m_out = bm;
    return true;
  };
  // explicit stack of ranges still to split: (a, b, node index, depth below
  // the segment)
  int sa[kSmall], sb[kSmall], sn[kSmall], sd[kSmall];
  int sp = 0;
  sa[0] = 0;
  sb[0] = n;
  sn[0] = base;
  sd[0] = 0;
  sp = 1;
  while (sp > 0) {
    --sp;
    const int a = sa[sp], b = sb[sp], me = sn[sp], dep = sd[sp];
    int m = -1;
    // SAH while the depth budget leaves room for a median finish below
    // either child (the level kernels' rule, split_flags)
    int lg = 0;
    while ((1 << lg) < b - a) ++lg;
    const bool sah_ok = fin_sah && level + dep + lg + 2 <= kMaxDepth;
    if (!(sah_ok && b - a > 2 && sah_exact(a, b, &m))) {
      // longest centroid extent, then insertion sort of f[a, b) on that axis
      float clo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, chi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
      for (int i = a; i < b; ++i)
        for (int k = 0; k < 3; ++k) {
          clo[k] = fminf(clo[k], lc[sl[i]][k]);
          chi[k] = fmaxf(chi[k], lc[sl[i]][k]);
        }
      int ax = 0;
      for (int k = 1; k < 3; ++k)
        if (chi[k] - clo[k] > chi[ax] - clo[ax]) ax = k;
      sort_axis(a, b, ax);
      m = a + (b - a) / 2;
      if (b - a > 2 && twins_at(f[m - 1], f[m], cen)) m = (m + 1 < b) ? m + 1 : m - 1;  // keep twins together
    }
    const int rng[2][2] = {{a, m}, {m, b}};
    // preorder ids: the subtree of `me` (range size s) owns [me, me + s - 1);
    // left child me + 1, right child me + (m - a)
    int32_t ref[2] = {(m - a) >= 2 ? me + 1 : ~f[a], (b - m) >= 2 ? me + (m - a) : ~f[m]};
    bool leafpair[2] = {m - a == 2 && pair_ref(a, &ref[0]), b - m == 2 && pair_ref(m, &ref[1])};
    for (int side = 0; side < 2; ++side) {
      double lo[3], hi[3];
      int32_t plane;
      range_box(rng[side][0], rng[side][1], lo, hi, &plane);
      child_slot(tn + me, side, lo, hi, eps, ref[side], plane);
    }
    if (b - m >= 2 && !leafpair[1]) {
      sa[sp] = m;
      sb[sp] = b;
      sn[sp] = ref[1];
      sd[sp] = dep + 1;
      ++sp;
    }
    if (m - a >= 2 && !leafpair[0]) {
      sa[sp] = a;
      sb[sp] = m;
      sn[sp] = ref[0];
      sd[sp] = dep + 1;
      ++sp;
    }
  }
}

// 4a. left/right flag per face
__global__ void flag_kernel(const int32_t* __restrict__ pos_seg, const SSeg* __restrict__ segs,
                            const int32_t* __restrict__ seg_axis, const int32_t* __restrict__ seg_split,
                            const int64_t* __restrict__ seg_nl, const unsigned long long* __restrict__ cb, const double* __restrict__ cen,
                            const int32_t* __restrict__ perm, int64_t nf, uint8_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nf) return;
  const int32_t s = pos_seg[i];
  if (s < 0) return;
  const int32_t axis = seg_axis[s];
  if (axis < 0) return;
  const SSeg sg = segs[s];
  const int32_t f = perm[axis * nf + i];  // position i of the axis list
  if (seg_split[s] < 0) {
    flag[f] = (i - sg.b) < seg_nl[s] ? 1 : 0;
  } else {
    const double clo = oval(cb[6 * s + axis]), ext = oval(cb[6 * s + 3 + axis]) - clo;
    flag[f] = bin_of(cen[3 * f + axis], clo, ext) < seg_split[s] ? 1 : 0;
  }
}

__global__ void gather_kernel(const int32_t* __restrict__ perm, const uint8_t* __restrict__ flag, int64_t total,
                              int32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < total) out[i] = flag[perm[i]];
}

// 4b. stable segmented partition of the three lists
__global__ void scatter_kernel(const int32_t* __restrict__ pos_seg, const SSeg* __restrict__ segs,
                               const int32_t* __restrict__ seg_axis, const int64_t* __restrict__ seg_nl,
                               const int32_t* __restrict__ rank, const int32_t* __restrict__ perm,
                               const int32_t* __restrict__ fl, const int32_t* __restrict__ scan, int64_t nf,
                               int32_t* __restrict__ perm_out, int32_t* __restrict__ pos_seg_out,
                               LevelState* __restrict__ ls, int64_t* __restrict__ s_out) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g == 0) {  // end of the level (nothing in this kernel reads ls): the next has 2 n_split segments
    ls->level_base += static_cast<int32_t>(ls->n_split);
    ls->S = 2 * ls->n_split;
    *s_out = ls->S;
  }
  if (g >= 3 * nf) return;
  const int k = static_cast<int>(g / nf);
  const int64_t i = g - k * nf;
  const int32_t sj = pos_seg[i];
  if (sj < 0 || seg_axis[sj] < 0) {
    perm_out[g] = perm[g];
    if (k == 0) pos_seg_out[i] = -1;
    return;
  }
  const SSeg sg = segs[sj];
  const int64_t nl = seg_nl[sj];
  const int64_t cnt_l = scan[g] - scan[k * nf + sg.b];
  const bool left = fl[g] != 0;
  const int64_t np = left ? sg.b + cnt_l : sg.b + nl + (i - sg.b - cnt_l);
  perm_out[k * nf + np] = perm[g];
  if (k == 0) pos_seg_out[np] = 2 * rank[sj] + (left ? 0 : 1);
}

__device__ __forceinline__ unsigned long long split_flags(const SSeg* __restrict__ segs, int64_t j, int level,
                                                          int64_t sah_min);

// per-segment accumulator reset and the packed split / SAH flags (positions
// S .. s_max get flag 0 so the scan can run over the level's upper bound)
__global__ void seg_init_kernel(const LevelState* __restrict__ ls, unsigned long long* __restrict__ bb,
                                unsigned long long* __restrict__ cb, int32_t* __restrict__ pl,
                                const SSeg* __restrict__ segs, int64_t s_max, int level,
                                unsigned long long* __restrict__ flags, int64_t sah_min) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t S = ls->S;
  if (j <= s_max) flags[j] = j < S ? split_flags(segs, j, level, sah_min) : 0ull;
  if (j >= S) return;
  for (int k = 0; k < 3; ++k) {  // ordered keys: min from ~0, max from 0
    bb[6 * j + k] = ~0ull;
    bb[6 * j + 3 + k] = 0ull;
    cb[6 * j + k] = ~0ull;
    cb[6 * j + 3 + k] = 0ull;
  }
  pl[2 * j] = 0x7fffffff;
  pl[2 * j + 1] = static_cast<int32_t>(0x80000000);
}

// packed flags: split (>= kSmall + 1 faces) << 32 | SAH-eligible
__device__ __forceinline__ unsigned long long split_flags(const SSeg* __restrict__ segs, int64_t j, int level,
                                                          int64_t sah_min) {
  const int64_t n = segs[j].n;
  const unsigned long long split = n > kSmall ? 1ull : 0ull;  // 2..kSmall: finish_kernel
  // SAH only while the depth budget allows a median finish below
  int lg = 0;
  while ((int64_t(1) << lg) < n) ++lg;
  const unsigned long long sah = (n >= sah_min && level + 1 + lg + 2 <= kMaxDepth) ? 1ull : 0ull;
  return (split << 32) | sah;
}

__global__ void rank_kernel(const unsigned long long* __restrict__ flags, const unsigned long long* __restrict__ ranks,
                            LevelState* __restrict__ ls, int32_t* __restrict__ srank, int32_t* __restrict__ sah_idx,
                            int32_t* __restrict__ bcnt, uint32_t* __restrict__ bbox) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t S = ls->S;
  const unsigned long long both = ranks[S];  // exclusive scan at S = the level's totals
  const int64_t n_bins = static_cast<int64_t>(both & 0xffffffffull) * 3 * kBins;
  if (j == 0) {
    ls->n_split = static_cast<int64_t>(both >> 32);
    ls->n_sah = static_cast<int64_t>(both & 0xffffffffull);
  }
  if (j < S) {
    srank[j] = static_cast<int32_t>(ranks[j] >> 32);
    sah_idx[j] = (flags[j] & 0xffffffffull) ? static_cast<int32_t>(ranks[j] & 0xffffffffull) : -1;
  }
  if (j < n_bins) {
    bcnt[j] = 0;
    for (int k = 0; k < 3; ++k) {
      bbox[6 * j + k] = 0xffffffffu;
      bbox[6 * j + 3 + k] = 0u;
    }
  }
}


// ---- 4-wide collapse of the SAH tree: every internal node at even depth
// becomes a QNode whose slots are its grandchildren (or a child leaf); slot
// planes go into QNode.pad for the coplanar culling.
__global__ void depth_kernel(const TNode* __restrict__ tn, int32_t n_int, int d, int32_t* __restrict__ depth) {
  const int32_t n = static_cast<int32_t>(blockIdx.x * blockDim.x + threadIdx.x);
  if (n >= n_int || depth[n] != d) return;
  const int4 c = tn[n].d;
  if (c.x >= 0) depth[c.x] = d + 1;
  if (c.y >= 0) depth[c.y] = d + 1;
}

__global__ void qflag_kernel(const int32_t* __restrict__ depth, int32_t n_int, int32_t* __restrict__ flag) {
  const int32_t n = static_cast<int32_t>(blockIdx.x * blockDim.x + threadIdx.x);
  if (n < n_int) flag[n] = (depth[n] >= 0 && (depth[n] & 1) == 0) ? 1 : 0;
  if (n == n_int) flag[n] = 0;
}

__device__ __forceinline__ void qslot(QNode& q, int s, const float* b6, int32_t ref, int32_t plane) {
  reinterpret_cast<float*>(&q.lx)[s] = b6[0];
  reinterpret_cast<float*>(&q.hx)[s] = b6[1];
  reinterpret_cast<float*>(&q.ly)[s] = b6[2];
  reinterpret_cast<float*>(&q.hy)[s] = b6[3];
  reinterpret_cast<float*>(&q.lz)[s] = b6[4];
  reinterpret_cast<float*>(&q.hz)[s] = b6[5];
  reinterpret_cast<int32_t*>(&q.child)[s] = ref;
  reinterpret_cast<int32_t*>(&q.pad)[s] = plane;
}

// TNode child boxes: left (a.x, a.y, a.z, a.w, b.x, b.y), right (b.z, b.w, c.x, c.y, c.z, c.w)
__device__ __forceinline__ void tbox(const TNode& t, int side, float* b6) {
  if (side == 0) {
    b6[0] = t.a.x; b6[1] = t.a.y; b6[2] = t.a.z; b6[3] = t.a.w; b6[4] = t.b.x; b6[5] = t.b.y;
  } else {
    b6[0] = t.b.z; b6[1] = t.b.w; b6[2] = t.c.x; b6[3] = t.c.y; b6[4] = t.c.z; b6[5] = t.c.w;
  }
}

__global__ void qbuild_kernel(const TNode* __restrict__ tn, int32_t n_int, const int32_t* __restrict__ flag,
                              const int32_t* __restrict__ qidx, QNode* __restrict__ out) {
  const int32_t n = static_cast<int32_t>(blockIdx.x * blockDim.x + threadIdx.x);
  if (n >= n_int || !flag[n]) return;
  const TNode t = tn[n];
  QNode q;
  float b6[6];
  for (int s = 0; s < 4; ++s) {  // empty slot: a point box far outside every scene
    const float far6[6] = {1e30f, 1e30f, 1e30f, 1e30f, 1e30f, 1e30f};
    qslot(q, s, far6, kEmpty, -1);
  }
  int slot = 0;
  const int32_t kid[2] = {t.d.x, t.d.y}, kpl[2] = {t.d.z, t.d.w};
  for (int side = 0; side < 2; ++side) {
    if (kid[side] < 0) {  // child leaf
      tbox(t, side, b6);
      qslot(q, slot++, b6, kid[side], kpl[side]);
      continue;
    }
    const TNode c = tn[kid[side]];
    const int32_t gk[2] = {c.d.x, c.d.y}, gp[2] = {c.d.z, c.d.w};
    for (int g = 0; g < 2; ++g) {
      tbox(c, g, b6);
      qslot(q, slot++, b6, gk[g] >= 0 ? qidx[gk[g]] : gk[g], gp[g]);
    }
  }
  out[qidx[n]] = q;
}

inline unsigned grid(int64_t n, int b = 256) { return static_cast<unsigned>((n + b - 1) / b); }

template <typename F>
void cub_run(F&& f, DevBuf<uint8_t>& tmp, cudaStream_t st) {
  size_t need = 0;
  RR_CUDA(f(nullptr, need));
  if (need > tmp.n) tmp.alloc(need + 16, st);
  size_t have = tmp.n;
  RR_CUDA(f(tmp.p, have));
}

}  // namespace

void build_sah_tree(rr_scene* s, cudaStream_t st) {
  const int64_t nf = s->nf;
  if (nf < 2) return;  // a one-face scene is traversed through the reference tree
  DevBuf<double> fb, cen;
  DevBuf<uint64_t> keys, keys_o;
  DevBuf<int32_t> ids, permA, permB, posA, posB, fl, scan;
  DevBuf<uint8_t> flag, tmp;
  fb.alloc(6 * nf, st);
  cen.alloc(3 * nf, st);
  keys.alloc(3 * nf, st);
  keys_o.alloc(3 * nf, st);
  ids.alloc(3 * nf, st);
  permA.alloc(3 * nf, st);
  permB.alloc(3 * nf, st);
  posA.alloc(nf, st);
  posB.alloc(nf, st);
  fl.alloc(3 * nf, st);
  scan.alloc(3 * nf, st);
  flag.alloc(nf, st);
  prep_kernel<<<grid(nf), 256, 0, st>>>(s->verts.p, s->tris.p, nf, fb.p, cen.p, keys.p, ids.p);
  RR_LAUNCH_CHECK();
  for (int k = 0; k < 3; ++k)
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, keys.p + k * nf, keys_o.p + k * nf, ids.p + k * nf,
                                             permA.p + k * nf, static_cast<int>(nf), 0, 32, st);
    }, tmp, st);
  s->snodes.alloc(nf - 1, st);
  RR_CUDA(cudaMemsetAsync(s->snodes.p, 0, s->snodes.bytes(), st));
  DevBuf<TravHeader> dh;
  dh.alloc(1, st);
  RR_CUDA(cudaMemsetAsync(dh.p, 0, sizeof(TravHeader), st));
  RR_CUDA(cudaMemsetAsync(posA.p, 0, sizeof(int32_t) * nf, st));

  // Upper bounds for the device-resident level sizes: a level has at most
  // 2^L segments, below the root at most 2 * nf / (kSmall + 1) (only
  // segments of more than kSmall faces split), and at most nf / kSahMin
  // SAH-binned segments.
  const int64_t max_seg = std::max<int64_t>(1, std::min<int64_t>(nf, 2 * (nf / (kSmall + 1)) + 2));
  // RR_SAH_MIN / RR_SAH_FIN (A/B): the smallest binned-SAH segment, and
  // exact SAH (1) or object medians (0) inside finish_kernel's segments
  static const int64_t sah_min = [] {
    const char* e = std::getenv("RR_SAH_MIN");
    return std::max<int64_t>(kSmall + 1, e ? std::atoll(e) : kSahMin);
  }();
  static const int fin_sah = [] {
    const char* e = std::getenv("RR_SAH_FIN");
    return e ? std::atoi(e) : 1;
  }();
  const int64_t max_sah = nf / sah_min + 1;
  DevBuf<SSeg> segA, segB;
  DevBuf<int32_t> srank, sah_idx, axis, split, pl;
  DevBuf<unsigned long long> flags, franks;
  DevBuf<int64_t> nl;
  DevBuf<unsigned long long> bb, cb;
  segA.alloc(max_seg, st);
  segB.alloc(max_seg, st);
  flags.alloc(max_seg + 1, st);
  franks.alloc(max_seg + 1, st);
  srank.alloc(max_seg + 1, st);
  sah_idx.alloc(max_seg + 1, st);
  axis.alloc(max_seg, st);
  split.alloc(max_seg, st);
  pl.alloc(2 * max_seg, st);
  nl.alloc(max_seg, st);
  bb.alloc(6 * max_seg, st);
  cb.alloc(6 * max_seg, st);
  DevBuf<int32_t> bcnt;
  DevBuf<uint32_t> bbox;
  bcnt.alloc(max_sah * 3 * kBins, st);
  bbox.alloc(max_sah * 3 * kBins * 6, st);
  const SSeg root{0, nf, -1, 0};
  RR_CUDA(cudaMemcpyAsync(segA.p, &root, sizeof root, cudaMemcpyHostToDevice, st));
  DevBuf<LevelState> ls;
  ls.alloc(1, st);
  const LevelState ls0{1, 0, 0, 0, 0};
  RR_CUDA(cudaMemcpyAsync(ls.p, &ls0, sizeof ls0, cudaMemcpyHostToDevice, st));
  // the next level's segment count, per level, read back a few levels late
  // (pinned slots and events owned by the context)
  constexpr int kMaxLevels = 64;
  int64_t* h_next = s->ctx->pinned;
  DevBuf<int64_t> d_next;
  d_next.alloc(kMaxLevels, st);
  cudaEvent_t* lev_ev = s->ctx->level_ev;
  int n_ev = 0;
  int32_t *perm = permA.p, *perm_o = permB.p, *pos = posA.p, *pos_o = posB.p;
  SSeg *segs = segA.p, *nsegs = segB.p;
  DevBuf<unsigned long long> top;  // internal nodes handed to finish_kernel (from the top)
  top.alloc(1, st);
  RR_CUDA(cudaMemsetAsync(top.p, 0, sizeof(unsigned long long), st));
  StageTimer tm(st);
  // Levels are enqueued without host round trips; the host learns that the
  // tree is complete kLag levels later and stops.  Levels enqueued after the
  // last split find no segments and change nothing.
  constexpr int kLag = 2;
  int depth = -1;
  for (int L = 0; L < kMaxLevels && depth < 0; ++L) {
    if (tm.on) tm.mark(L < 64 ? kLevelNames[L] : "level");
    const int64_t s_max = L == 0 ? 1 : std::min<int64_t>(max_seg, L < 62 ? (int64_t(1) << L) : max_seg);
    const int64_t sah_max = std::min<int64_t>(s_max, max_sah);
    // 1. bounds (one init launch for the per-segment accumulators)
    seg_init_kernel<<<grid(s_max + 1), 256, 0, st>>>(ls.p, bb.p, cb.p, pl.p, segs, s_max, L, flags.p, sah_min);
    bounds_kernel<<<grid(nf), 256, 0, st>>>(pos, perm, fb.p, cen.p, s->face_plane.p, nf, bb.p, cb.p, pl.p);
    if (L == 0) root_hdr_kernel<<<1, 32, 0, st>>>(bb.p, dh.p);
    // 2. split flags and SAH flags, both ranks from one 64-bit scan
    //    (split flag in the high word, SAH flag in the low word)
    RR_LAUNCH_CHECK();
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, flags.p, franks.p, static_cast<int>(s_max + 1), st);
    }, tmp, st);
    // srank[j] / sah_idx[j] (compact index, -1 for non-SAH segments), bins reset
    rank_kernel<<<grid(std::max<int64_t>(s_max, sah_max * 3 * kBins)), 256, 0, st>>>(flags.p, franks.p, ls.p,
                                                                                    srank.p, sah_idx.p, bcnt.p,
                                                                                    bbox.p);
    RR_LAUNCH_CHECK();
    if (sah_max > 0) {
      bin_kernel<<<grid(nf), 256, 0, st>>>(pos, perm, fb.p, cen.p, cb.p, sah_idx.p, nf, bcnt.p, bbox.p);
      RR_LAUNCH_CHECK();
    }
    // 3. nodes + splits
    split_kernel<<<grid(32 * s_max), 256, 0, st>>>(segs, ls.p, srank.p, bb.p, cb.p, pl.p, sah_idx.p, bcnt.p, bbox.p, perm,
                                              cen.p, nf, s->snodes.p, dh.p, axis.p, split.p, nl.p, nsegs);
    finish_kernel<<<grid(s_max, 64), 64, 0, st>>>(segs, ls.p, perm, fb.p, cen.p, s->face_plane.p, nf, s->snodes.p,
                                                  dh.p, top.p, L, fin_sah);
    RR_LAUNCH_CHECK();
    // 4. stable partition of the three lists
    flag_kernel<<<grid(nf), 256, 0, st>>>(pos, segs, axis.p, split.p, nl.p, cb.p, cen.p, perm, nf, flag.p);
    gather_kernel<<<grid(3 * nf), 256, 0, st>>>(perm, flag.p, 3 * nf, fl.p);
    RR_LAUNCH_CHECK();
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, fl.p, scan.p, static_cast<int>(3 * nf), st);
    }, tmp, st);
    scatter_kernel<<<grid(3 * nf), 256, 0, st>>>(pos, segs, axis.p, nl.p, srank.p, perm, fl.p, scan.p, nf, perm_o,
                                                  pos_o, ls.p, d_next.p + L);
    RR_LAUNCH_CHECK();
    RR_CUDA(cudaMemcpyAsync(h_next + L, d_next.p + L, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    n_ev = L + 1;
    RR_CUDA(cudaEventRecord(lev_ev[L], st));
    s->ctx->launches += 10;
    std::swap(perm, perm_o);
    std::swap(pos, pos_o);
    std::swap(segs, nsegs);
    const int seen = L - kLag;  // the newest level the host waits for
    if (seen >= 0) {
      RR_CUDA(cudaEventSynchronize(lev_ev[seen]));
      for (int q = 0; q <= seen && depth < 0; ++q)
        if (h_next[q] == 0) depth = q;
    }
  }
  RR_CUDA(cudaStreamSynchronize(st));
  for (int q = 0; q < n_ev && depth < 0; ++q)
    if (h_next[q] == 0) depth = q;
  if (depth < 0) throw Error(RR_RUNTIME, "SAH build did not terminate");
  RR_CUDA(cudaMemcpyAsync(&s->shdr, dh.p, sizeof(TravHeader), cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  s->shdr.K = 0;
  s->shdr.K4 = 0;
  s->shdr.root4 = 0;
  s->sah_depth = depth;
  if (depth > kMaxDepth) throw Error(RR_RUNTIME, "SAH tree deeper than the traversal stack");
  // the wide collapses serve the deep-tree kernels (rr_trace.cu run_trace
  // picks the tree by face count); forced choices build theirs on demand
  if (nf >= (int64_t(1) << 20)) build_wide(s);
  else if (nf >= (int64_t(1) << 18)) build_sah4(s);
}

// 4-wide collapse of the SAH tree (traversed by trace_kernel<3, ...>).
void build_sah4(rr_scene* s) {
  if (s->s4nodes.p || !s->snodes.p) return;
  cudaStream_t st = s->ctx->stream;
  const int32_t n_int = static_cast<int32_t>(s->nf - 1);
  const int depth = s->sah_depth;
  DevBuf<uint8_t> tmp;
  DevBuf<int32_t> depthb, qf, qi;
  depthb.alloc(n_int, st);
  qf.alloc(n_int + 1, st);
  qi.alloc(n_int + 1, st);
  RR_CUDA(cudaMemsetAsync(depthb.p, 0xff, depthb.bytes(), st));
  const int32_t root_ref = s->shdr.root_ref;
  if (root_ref >= 0) RR_CUDA(cudaMemsetAsync(depthb.p + root_ref, 0, sizeof(int32_t), st));
  for (int d = 0; d <= depth + 6; ++d)
    depth_kernel<<<grid(n_int), 256, 0, st>>>(s->snodes.p, n_int, d, depthb.p);
  qflag_kernel<<<grid(n_int + 1), 256, 0, st>>>(depthb.p, n_int, qf.p);
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, qf.p, qi.p, static_cast<int>(n_int + 1), st);
  }, tmp, st);
  int32_t nq = 0;
  RR_CUDA(cudaMemcpyAsync(&nq, qi.p + n_int, sizeof nq, cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  s->s4nodes.alloc(std::max(nq, 1), st);
  qbuild_kernel<<<grid(n_int), 256, 0, st>>>(s->snodes.p, n_int, qf.p, qi.p, s->s4nodes.p);
  RR_LAUNCH_CHECK();
  int32_t root4 = root_ref;
  if (root_ref >= 0) RR_CUDA(cudaMemcpyAsync(&root4, qi.p + root_ref, sizeof root4, cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  s->s4root = root4;
  s->ctx->launches += depth + 10;
}

}  // namespace rr
