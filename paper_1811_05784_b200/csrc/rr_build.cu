// K1 — device build of the reference median-split tree.
//
// Replaces build_tree / Builder::build_range (accel_tree.cpp:19-87).  The
// reference splits each face range at mid = begin + n/2 after nth_element on
// the total order (centroid[axis], face index), axis = first argmax of the
// range box extent (accel_tree.cpp:30-41).  Because that order is total, the
// set of faces sent left is unique, so the tree is a function of the input
// alone and is rebuilt here level-synchronously:
//   * three face lists presorted by (centroid[k], face) (CUB radix sort,
//     stable => ties by face index, accel_tree.cpp:38-39);
//   * per level: segmented box reduction (warp-segmented + u64 atomics on
//     order-preserving keys, exact min/max), axis choice, split flags from the
//     chosen axis' list (rank < n/2), and a stable segmented partition of all
//     three lists (one scan) so each stays sorted inside its child segments.
// Node numbering follows the reference post-order (left subtree, right
// subtree, node; root last, accel_tree.cpp:43-46): a range [b, b+n) whose
// subtree starts at s has its node at s + 2n - 2 and children starting at s
// and s + 2*(n/2) - 1.  Segment sizes depend on nf only, so the host knows
// every level's segment count without a device round trip.
//
// The same pass emits the traversal layout used by the tracer: TNode pairs of
// conservative fp32 child boxes (outward-rounded and expanded by eps), with
// the top D levels in BFS order at [0, K) (cached in shared memory by the
// tracer) and deeper subtrees in preorder at K + begin + (left edges below
// level D).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <exception>
#include <map>
#include <thread>

#include "rr_internal.cuh"

namespace rr {
namespace {

constexpr int kMaxCachedNodes = 511;   // 32 KB of TNodes in shared memory
constexpr int kMaxCachedQNodes = 384;  // 48 KB of QNodes in shared memory

__device__ __forceinline__ uint64_t ord_key(double x) {
  if (x == 0.0) x = 0.0;  // -0 == +0 in the reference comparisons
  uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(uint64_t u) {
  u = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
  return __longlong_as_double(static_cast<long long>(u));
}

struct Seg {
  int64_t b, n, s;   // range [b, b+n), post-order base of the subtree
  int32_t parent;    // traversal index of the parent node, -1 for the root
  int32_t side;      // 0 left child, 1 right child
  int32_t lam;       // left edges on the path below level D
  int32_t pad;
};

// Centroid (geometry.cpp:16-19), face bounds (geometry.cpp:28-35), sort keys.
__global__ void face_prep_kernel(const double* __restrict__ v,
                                 const int32_t* __restrict__ t, int64_t nf,
                                 double* __restrict__ fb,  // nf*6 lo,hi
                                 uint64_t* __restrict__ keys,  // 3*nf
                                 int32_t* __restrict__ ids) {  // 3*nf
  int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const int32_t a = t[4 * f], b = t[4 * f + 1], c = t[4 * f + 2];
  for (int k = 0; k < 3; ++k) {
    const double va = v[3 * a + k], vb = v[3 * b + k], vc = v[3 * c + k];
    const double cen = ((va + vb) + vc) / 3.0;
    double lo = va, hi = va;  // Aabb::extend: std::min/std::max
    lo = (vb < lo) ? vb : lo;
    hi = (hi < vb) ? vb : hi;
    lo = (vc < lo) ? vc : lo;
    hi = (hi < vc) ? vc : hi;
    fb[6 * f + k] = lo;
    fb[6 * f + 3 + k] = hi;
    keys[k * nf + f] = ord_key(cen);
    ids[k * nf + f] = static_cast<int32_t>(f);
  }
}

// Segmented min/max of face bounds over each active segment.
__global__ void seg_box_kernel(const int32_t* __restrict__ pos_seg,
                               const int32_t* __restrict__ perm0,
                               const double* __restrict__ fb, int64_t nf,
                               unsigned long long* __restrict__ bmin,
                               unsigned long long* __restrict__ bmax) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int32_t seg = -1;
  uint64_t mn[3] = {~0ull, ~0ull, ~0ull}, mx[3] = {0, 0, 0};
  if (i < nf) {
    seg = pos_seg[i];
    if (seg >= 0) {
      const int32_t f = perm0[i];
      for (int k = 0; k < 3; ++k) {
        mn[k] = ord_key(fb[6 * f + k]);
        mx[k] = ord_key(fb[6 * f + 3 + k]);
      }
    }
  }
  for (int off = 1; off < 32; off <<= 1) {
    const int32_t so = __shfl_down_sync(0xffffffffu, seg, off);
    const bool ok = (lane + off < 32) && so == seg;
    for (int k = 0; k < 3; ++k) {
      const uint64_t a = __shfl_down_sync(0xffffffffu, mn[k], off);
      const uint64_t b = __shfl_down_sync(0xffffffffu, mx[k], off);
      if (ok) {
        mn[k] = a < mn[k] ? a : mn[k];
        mx[k] = b > mx[k] ? b : mx[k];
      }
    }
  }
  const int32_t sp = __shfl_up_sync(0xffffffffu, seg, 1);
  const bool head = seg >= 0 && (lane == 0 || sp != seg);
  if (head) {
    for (int k = 0; k < 3; ++k) {
      atomicMin(bmin + 3 * seg + k, (unsigned long long)mn[k]);
      atomicMax(bmax + 3 * seg + k, (unsigned long long)mx[k]);
    }
  }
}

__global__ void split_flag_kernel(const Seg* __restrict__ segs, int64_t S,
                                  int32_t* __restrict__ flag) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < S) flag[j] = segs[j].n >= 2 ? 1 : 0;
}

__device__ __forceinline__ float lo_f(double x, float eps) {
  return __fsub_rd(__double2float_rd(x), eps);
}
__device__ __forceinline__ float hi_f(double x, float eps) {
  return __fadd_ru(__double2float_ru(x), eps);
}

// Node emission, axis choice, child segments.
__global__ void seg_node_kernel(const Seg* __restrict__ segs, int64_t S,
                                const int32_t* __restrict__ rank,
                                const unsigned long long* __restrict__ bmin,
                                const unsigned long long* __restrict__ bmax,
                                const int32_t* __restrict__ perm0, int level,
                                int D, int32_t level_base, int32_t K,
                                RefNode* __restrict__ ref, TNode* __restrict__ tn,
                                TravHeader* __restrict__ hdr,
                                int32_t* __restrict__ seg_axis,
                                Seg* __restrict__ next,
                                int32_t* __restrict__ node_level,
                                int32_t* __restrict__ node_tidx) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= S) return;
  const Seg sg = segs[j];
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    lo[k] = ord_val(bmin[3 * j + k]);
    hi[k] = ord_val(bmax[3 * j + k]);
  }
  float eps;
  if (level == 0) {
    double scale = 1e-3;
    for (int k = 0; k < 3; ++k) scale = fmax(scale, fmax(fabs(lo[k]), fabs(hi[k])));
    eps = __double2float_ru(scale * 0x1p-19);  // see rr_geom.cuh box_enter
    hdr->eps = eps;
    for (int k = 0; k < 3; ++k) {
      hdr->lo[k] = lo_f(lo[k], eps);
      hdr->hi[k] = hi_f(hi[k], eps);
    }
  } else {
    eps = hdr->eps;
  }
  const int64_t node = sg.s + 2 * sg.n - 2;
  RefNode r;
  for (int k = 0; k < 3; ++k) {
    r.lo[k] = lo[k];
    r.hi[k] = hi[k];
  }
  r.pad = 0;
  int32_t my_ref;
  if (sg.n == 1) {
    r.face = perm0[sg.b];
    r.left = r.right = -1;
    my_ref = ~r.face;
    seg_axis[j] = -1;
  } else {
    const int64_t nl = sg.n / 2, nr = sg.n - nl;
    r.face = -1;
    r.left = static_cast<int32_t>(sg.s + 2 * nl - 2);
    r.right = static_cast<int32_t>((sg.s + 2 * nl - 1) + 2 * nr - 2);
    // axis = first argmax of the box extent (accel_tree.cpp:30-32)
    const double ex = hi[0] - lo[0], ey = hi[1] - lo[1], ez = hi[2] - lo[2];
    int axis = 0;
    double best = ex;
    if (ey > best) { axis = 1; best = ey; }
    if (ez > best) { axis = 2; }
    seg_axis[j] = axis;
    my_ref = level < D ? level_base + rank[j]
                       : K + static_cast<int32_t>(sg.b) + sg.lam;
    const int32_t lam_l = (level + 1 < D) ? 0 : (level + 1 == D ? 0 : sg.lam + 1);
    const int32_t lam_r = (level + 1 < D) ? 0 : (level + 1 == D ? 0 : sg.lam);
    Seg L{sg.b, nl, sg.s, my_ref, 0, lam_l, 0};
    Seg R{sg.b + nl, nr, sg.s + 2 * nl - 1, my_ref, 1, lam_r, 0};
    next[2 * rank[j]] = L;
    next[2 * rank[j] + 1] = R;
  }
  ref[node] = r;
  node_level[node] = level;
  node_tidx[node] = my_ref;
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
    } else {
      reinterpret_cast<float2*>(&p->b)[1] = make_float2(lx, hx);
      p->c = make_float4(ly, hy, lz, hz);
      p->d.y = my_ref;
    }
  }
}

// flag[face] = goes left, from the chosen axis' sorted list.
__global__ void face_flag_kernel(const int32_t* __restrict__ pos_seg,
                                 const Seg* __restrict__ segs,
                                 const int32_t* __restrict__ seg_axis,
                                 const int32_t* __restrict__ perm, int64_t nf,
                                 uint8_t* __restrict__ flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nf) return;
  const int32_t sj = pos_seg[i];
  if (sj < 0) return;
  const int32_t axis = seg_axis[sj];
  if (axis < 0) return;
  const Seg sg = segs[sj];
  flag[perm[axis * nf + i]] = (i - sg.b) < sg.n / 2 ? 1 : 0;
}

__global__ void gather_flag_kernel(const int32_t* __restrict__ perm,
                                   const uint8_t* __restrict__ flag,
                                   int64_t total, int32_t* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < total) out[i] = flag[perm[i]];
}

// Stable segmented partition of the three lists.
__global__ void scatter_kernel(const int32_t* __restrict__ pos_seg,
                               const Seg* __restrict__ segs,
                               const int32_t* __restrict__ seg_axis,
                               const int32_t* __restrict__ rank,
                               const int32_t* __restrict__ perm,
                               const int32_t* __restrict__ fl,
                               const int32_t* __restrict__ scan, int64_t nf,
                               int32_t* __restrict__ perm_out,
                               int32_t* __restrict__ pos_seg_out) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= 3 * nf) return;
  const int k = static_cast<int>(g / nf);
  const int64_t i = g - k * nf;
  const int32_t sj = pos_seg[i];
  if (sj < 0 || seg_axis[sj] < 0) {
    perm_out[g] = perm[g];
    if (k == 0) pos_seg_out[i] = -1;
    return;
  }
  const Seg sg = segs[sj];
  const int64_t nl = sg.n / 2;
  const int64_t cnt_l = scan[g] - scan[k * nf + sg.b];
  const bool left = fl[g] != 0;
  const int64_t np = left ? sg.b + cnt_l : sg.b + nl + (i - sg.b - cnt_l);
  perm_out[k * nf + np] = perm[g];
  if (k == 0) pos_seg_out[np] = 2 * rank[sj] + (left ? 0 : 1);
}

// ---- 4-wide collapse: the even-depth internal nodes of the reference tree
// become QNodes, indexed in the order of their BVH2 traversal index (BFS top
// levels first, then preorder) so the cached prefix is the top of the tree.
__global__ void q_flag_kernel(const RefNode* __restrict__ ref, const int32_t* __restrict__ level,
                              const int32_t* __restrict__ tidx, int64_t n_nodes, int32_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_nodes) return;
  if (ref[i].face < 0 && (level[i] & 1) == 0) flag[tidx[i]] = 1;
}

__device__ __forceinline__ void q_child(const RefNode* __restrict__ ref, const int32_t* __restrict__ tidx,
                                        const int32_t* __restrict__ qidx, int32_t c, float eps, QNode& q,
                                        int slot) {
  const RefNode& n = ref[c];
  reinterpret_cast<float*>(&q.lx)[slot] = lo_f(n.lo[0], eps);
  reinterpret_cast<float*>(&q.hx)[slot] = hi_f(n.hi[0], eps);
  reinterpret_cast<float*>(&q.ly)[slot] = lo_f(n.lo[1], eps);
  reinterpret_cast<float*>(&q.hy)[slot] = hi_f(n.hi[1], eps);
  reinterpret_cast<float*>(&q.lz)[slot] = lo_f(n.lo[2], eps);
  reinterpret_cast<float*>(&q.hz)[slot] = hi_f(n.hi[2], eps);
  reinterpret_cast<int32_t*>(&q.child)[slot] = n.face >= 0 ? ~n.face : qidx[tidx[c]];
}

__global__ void q_build_kernel(const RefNode* __restrict__ ref, const int32_t* __restrict__ level,
                               const int32_t* __restrict__ tidx, const int32_t* __restrict__ qidx,
                               int64_t n_nodes, const TravHeader* __restrict__ hdr, QNode* __restrict__ q) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_nodes) return;
  const RefNode n = ref[i];
  if (n.face >= 0 || (level[i] & 1)) return;
  const float eps = hdr->eps;
  QNode out;
  for (int s = 0; s < 4; ++s) {
    // empty slot: a point box far outside every scene, never a usable hit
    reinterpret_cast<float*>(&out.lx)[s] = 1e30f;
    reinterpret_cast<float*>(&out.hx)[s] = 1e30f;
    reinterpret_cast<float*>(&out.ly)[s] = 1e30f;
    reinterpret_cast<float*>(&out.hy)[s] = 1e30f;
    reinterpret_cast<float*>(&out.lz)[s] = 1e30f;
    reinterpret_cast<float*>(&out.hz)[s] = 1e30f;
    reinterpret_cast<int32_t*>(&out.child)[s] = kEmpty;
  }
  out.pad = make_int4(0, 0, 0, 0);
  int slot = 0;
  const int32_t kids[2] = {n.left, n.right};
  for (int k = 0; k < 2; ++k) {
    const RefNode& c = ref[kids[k]];
    if (c.face >= 0) {
      q_child(ref, tidx, qidx, kids[k], eps, out, slot++);
    } else {
      q_child(ref, tidx, qidx, c.left, eps, out, slot++);
      q_child(ref, tidx, qidx, c.right, eps, out, slot++);
    }
  }
  out.pad.x = slot;
  q[qidx[tidx[i]]] = out;
}

// ---- axis-aligned plane ids (coplanar-subtree culling, rr_geom.cuh).
// A face is flat on axis k when its three vertices share coordinate k
// exactly (a valid face has at most one such axis); a node is flat when its
// box has zero extent on k, i.e. all its faces lie on one plane x_k = c.
__device__ __forceinline__ int flat_axis(const double* lo, const double* hi) {
  for (int k = 0; k < 3; ++k)
    if (lo[k] == hi[k]) return k;
  return -1;
}

// Axis-aligned plane ids: the flat faces' plane coordinates go into one
// open-addressing hash table per axis (size T, a power of two, ~0 = empty);
// a plane's id is (axis << 29) | its slot.  Ids are only compared for
// equality (coplanar culling), so no order is needed.
__device__ __forceinline__ uint64_t plane_slot0(uint64_t key, uint64_t mask) {
  key ^= key >> 33;
  key *= 0xff51afd7ed558ccdull;
  key ^= key >> 33;
  return key & mask;
}

__global__ void plane_insert_kernel(const double* __restrict__ fb, int64_t nf, unsigned long long* __restrict__ table,
                                    int64_t T) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const int k = flat_axis(fb + 6 * f, fb + 6 * f + 3);
  if (k < 0) return;
  const unsigned long long key = ord_key(fb[6 * f + k]);
  unsigned long long* t = table + k * T;
  for (uint64_t h = plane_slot0(key, T - 1);; h = (h + 1) & (T - 1)) {
    const unsigned long long prev = atomicCAS(t + h, ~0ull, key);
    if (prev == ~0ull || prev == key) return;
  }
}

__device__ __forceinline__ int32_t plane_lookup(const unsigned long long* __restrict__ table, int64_t T, int k,
                                                double c) {
  const unsigned long long key = ord_key(c);
  const unsigned long long* t = table + k * T;
  for (uint64_t h = plane_slot0(key, T - 1);; h = (h + 1) & (T - 1)) {
    const unsigned long long v = t[h];
    if (v == key) return static_cast<int32_t>((k << 29) | static_cast<int32_t>(h));
    if (v == ~0ull) return -1;
  }
}

__global__ void face_plane_kernel(const double* __restrict__ fb, int64_t nf,
                                  const unsigned long long* __restrict__ table, int64_t T,
                                  int32_t* __restrict__ face_plane) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const int k = flat_axis(fb + 6 * f, fb + 6 * f + 3);
  face_plane[f] = k < 0 ? -1 : plane_lookup(table, T, k, fb[6 * f + k]);
}

__global__ void node_plane_kernel(const RefNode* __restrict__ ref, const int32_t* __restrict__ tidx,
                                  int64_t n_nodes, const unsigned long long* __restrict__ table,
                                  int64_t T, TNode* __restrict__ tn) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_nodes || ref[i].face >= 0) return;
  int32_t pl[2];
  const int32_t kids[2] = {ref[i].left, ref[i].right};
  for (int s = 0; s < 2; ++s) {
    const RefNode& c = ref[kids[s]];
    const int k = flat_axis(c.lo, c.hi);
    pl[s] = k < 0 ? -1 : plane_lookup(table, T, k, c.lo[k]);
  }
  tn[tidx[i]].d.z = pl[0];
  tn[tidx[i]].d.w = pl[1];
}

__global__ void vert_bounds_kernel(const double* __restrict__ v, int64_t nv,
                                   unsigned long long* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  uint64_t mn[3] = {~0ull, ~0ull, ~0ull}, mx[3] = {0, 0, 0};
  for (; i < nv; i += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < 3; ++k) {
      const uint64_t u = ord_key(v[3 * i + k]);
      mn[k] = u < mn[k] ? u : mn[k];
      mx[k] = u > mx[k] ? u : mx[k];
    }
  for (int off = 16; off > 0; off >>= 1)
    for (int k = 0; k < 3; ++k) {
      const uint64_t a = __shfl_xor_sync(0xffffffffu, mn[k], off);
      const uint64_t b = __shfl_xor_sync(0xffffffffu, mx[k], off);
      mn[k] = a < mn[k] ? a : mn[k];
      mx[k] = b > mx[k] ? b : mx[k];
    }
  if ((threadIdx.x & 31) == 0)
    for (int k = 0; k < 3; ++k) {
      atomicMin(out + k, (unsigned long long)mn[k]);
      atomicMax(out + 3 + k, (unsigned long long)mx[k]);
    }
}

__global__ void unmap_bounds_kernel(const unsigned long long* in, double* out) {
  if (threadIdx.x < 6) out[threadIdx.x] = ord_val(in[threadIdx.x]);
}

inline unsigned grid_for(int64_t n, int block = 256) {
  return static_cast<unsigned>((n + block - 1) / block);
}

}  // namespace

namespace {
// Host plan of the reference median tree: per-level segment size multisets
// (they depend on nf only), the cached top-K node count and level bases.
struct LevelPlan {
  int n_levels = 0, D = 0;
  int64_t K = 0, max_seg = 1;
  std::vector<int64_t> seg_count, split_count;
  std::vector<int32_t> level_base;
};

LevelPlan plan_levels(int64_t nf) {
  std::vector<std::map<int64_t, int64_t>> levels;
  levels.push_back({{nf, 1}});
  for (;;) {
    std::map<int64_t, int64_t> nx;
    for (auto [sz, cnt] : levels.back())
      if (sz >= 2) {
        nx[sz / 2] += cnt;
        nx[sz - sz / 2] += cnt;
      }
    if (nx.empty()) break;
    levels.push_back(nx);
  }
  const int n_levels = static_cast<int>(levels.size());
  std::vector<int64_t> seg_count(n_levels), split_count(n_levels);
  for (int L = 0; L < n_levels; ++L) {
    int64_t c = 0, sp = 0;
    for (auto [sz, cnt] : levels[L]) {
      c += cnt;
      if (sz >= 2) sp += cnt;
    }
    seg_count[L] = c;
    split_count[L] = sp;
  }
  int D = 0;
  int64_t K = 0;
  while (D < n_levels && K + split_count[D] <= kMaxCachedNodes) {
    K += split_count[D];
    ++D;
  }
  std::vector<int32_t> level_base(n_levels, 0);
  for (int L = 1; L < n_levels; ++L)
    level_base[L] = level_base[L - 1] + static_cast<int32_t>(split_count[L - 1]);
  int64_t max_seg = 1;
  for (auto c : seg_count) max_seg = std::max(max_seg, c);

  LevelPlan lp;
  lp.n_levels = n_levels;
  lp.D = D;
  lp.K = K;
  lp.max_seg = max_seg;
  lp.seg_count = seg_count;
  lp.split_count = split_count;
  lp.level_base = level_base;
  return lp;
}
}  // namespace

// Scene build: face plane ids, the SAH traversal tree (rr_sah.cu) and the
// mesh bounds.  The reference-layout median tree (accel_tree.cpp:19-87) is
// built on first use only (ensure_reference_tree): traversal, projection
// and nearest_hit run on the SAH tree, so run_trace_pipeline never needs it.
void build_scene_tree(rr_scene* s) {
  cudaStream_t st = s->ctx->stream;
  const int64_t nf = s->nf;
  cudaEvent_t e0, e1;
  RR_CUDA(cudaEventCreate(&e0));
  RR_CUDA(cudaEventCreate(&e1));
  RR_CUDA(cudaEventRecord(e0, st));
  StageTimer tm(st);
  const LevelPlan lp = plan_levels(nf);
  s->depth = lp.n_levels - 1;
  s->K = static_cast<int32_t>(lp.K);
  s->root = static_cast<int32_t>(2 * nf - 2);

  DevBuf<double> fb;
  fb.alloc(6 * nf, st);
  {
    DevBuf<uint64_t> keys;
    DevBuf<int32_t> ids;
    keys.alloc(3 * nf, st);
    ids.alloc(3 * nf, st);
    face_prep_kernel<<<grid_for(nf), 256, 0, st>>>(s->verts.p, s->tris.p, nf, fb.p, keys.p, ids.p);
    RR_LAUNCH_CHECK();
    s->ctx->launches++;
  }
  // ---- axis-aligned plane ids: one hash table of plane coordinates per
  // axis; ids for faces (here) and for tree children (reference tree)
  DevBuf<unsigned long long>& table = s->plane_table;
  {
    int64_t T = 1024;
    while (T < 2 * nf) T <<= 1;  // load factor <= 1/2 per axis
    if (T > (int64_t(1) << 29)) invalid("too many faces for 29-bit plane slots");
    s->plane_T = T;
    table.alloc(3 * T, st);
    RR_CUDA(cudaMemsetAsync(table.p, 0xff, table.bytes(), st));
    plane_insert_kernel<<<grid_for(nf), 256, 0, st>>>(fb.p, nf, table.p, T);
    RR_LAUNCH_CHECK();
    s->face_plane.alloc(nf, st);
    face_plane_kernel<<<grid_for(nf), 256, 0, st>>>(fb.p, nf, table.p, T, s->face_plane.p);
    RR_LAUNCH_CHECK();
    s->ctx->launches += 2;
  }
  tm.mark("build: plane tables");
  build_sah_tree(s, st);
  tm.mark("build: SAH tree");
  // ---- TriangleMesh::bounds over all vertices (image-source tolerance)
  DevBuf<unsigned long long> vb;
  vb.alloc(6, st);
  RR_CUDA(cudaMemsetAsync(vb.p, 0xff, sizeof(unsigned long long) * 3, st));
  RR_CUDA(cudaMemsetAsync(vb.p + 3, 0x00, sizeof(unsigned long long) * 3, st));
  const int64_t nv = std::max<int64_t>(s->nv, 1);
  vert_bounds_kernel<<<std::min<unsigned>(grid_for(nv), 1184u), 256, 0, st>>>(s->verts.p, s->nv, vb.p);
  RR_LAUNCH_CHECK();
  DevBuf<double> vbd;
  vbd.alloc(6, st);
  unmap_bounds_kernel<<<1, 32, 0, st>>>(vb.p, vbd.p);
  RR_LAUNCH_CHECK();
  s->ctx->launches += 2;
  double hb[6];
  RR_CUDA(cudaMemcpyAsync(hb, vbd.p, sizeof hb, cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaEventRecord(e1, st));
  RR_CUDA(cudaStreamSynchronize(st));
  for (int k = 0; k < 3; ++k) {
    s->lo[k] = hb[k];
    s->hi[k] = hb[3 + k];
  }
  RR_CUDA(cudaEventElapsedTime(&s->build_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

// The reference median tree in its own layout (RefNode, for
// AccelTree::nodes) and as TNodes / 4-wide QNodes for the diagnostic
// traversals (RR_SAH=0, nearest_hit_batch brute = 3): level-synchronous
// exact-median split of three presorted face lists (accel_tree.cpp:19-47).
void ensure_reference_tree(rr_scene* s) {
  if (s->ref_built) return;
  cudaStream_t st = s->ctx->stream;
  const int64_t nf = s->nf;
  StageTimer tm(st);
  const LevelPlan lp = plan_levels(nf);
  const int n_levels = lp.n_levels, D = lp.D;
  const int64_t K = lp.K, max_seg = lp.max_seg;
  const std::vector<int64_t>& seg_count = lp.seg_count;
  const std::vector<int64_t>& split_count = lp.split_count;
  const std::vector<int32_t>& level_base = lp.level_base;
  // ---- buffers
  DevBuf<double> fb;
  fb.alloc(6 * nf, st);
  DevBuf<uint64_t> keys, keys_out;
  keys.alloc(3 * nf, st);
  keys_out.alloc(3 * nf, st);
  DevBuf<int32_t> ids, permA, permB, fl, scan, pos_a, pos_b;
  ids.alloc(3 * nf, st);
  permA.alloc(3 * nf, st);
  permB.alloc(3 * nf, st);
  fl.alloc(3 * nf, st);
  scan.alloc(3 * nf, st);
  pos_a.alloc(nf, st);
  pos_b.alloc(nf, st);
  DevBuf<uint8_t> flag;
  flag.alloc(nf, st);
  DevBuf<Seg> segA, segB;
  segA.alloc(max_seg, st);
  segB.alloc(max_seg, st);
  DevBuf<int32_t> sflag, srank, saxis;
  sflag.alloc(max_seg, st);
  srank.alloc(max_seg, st);
  saxis.alloc(max_seg, st);
  DevBuf<int32_t> nlevel, ntidx;
  nlevel.alloc(2 * nf - 1, st);
  ntidx.alloc(2 * nf - 1, st);
  DevBuf<unsigned long long> bmin, bmax;
  bmin.alloc(3 * max_seg, st);
  bmax.alloc(3 * max_seg, st);

  s->ref.alloc(2 * nf - 1, st);
  s->tnodes.alloc(K + nf, st);
  RR_CUDA(cudaMemsetAsync(s->tnodes.p, 0, s->tnodes.bytes(), st));
  s->dhdr.alloc(1, st);
  RR_CUDA(cudaMemsetAsync(s->dhdr.p, 0, sizeof(TravHeader), st));

  face_prep_kernel<<<grid_for(nf), 256, 0, st>>>(s->verts.p, s->tris.p, nf, fb.p, keys.p, ids.p);
  RR_LAUNCH_CHECK();
  s->ctx->launches++;

  // ---- CUB scratch
  size_t tmp_sort = 0, tmp_scan = 0, tmp_scan2 = 0;
  RR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, keys.p, keys_out.p, ids.p, permA.p,
                                          static_cast<int>(nf), 0, 64, st));
  RR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, fl.p, scan.p, static_cast<int>(3 * nf), st));
  RR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan2, sflag.p, srank.p, static_cast<int>(max_seg), st));
  DevBuf<uint8_t> tmp;
  tmp.alloc(std::max(tmp_sort, std::max(tmp_scan, tmp_scan2)) + 16, st);
  for (int k = 0; k < 3; ++k) {
    size_t t = tmp.n;
    RR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, t, keys.p + k * nf, keys_out.p + k * nf, ids.p + k * nf,
                                            permA.p + k * nf, static_cast<int>(nf), 0, 64, st));
    s->ctx->launches += 4;
  }

  // ---- level loop
  RR_CUDA(cudaMemsetAsync(pos_a.p, 0, sizeof(int32_t) * nf, st));
  const Seg root{0, nf, 0, -1, 0, 0, 0};
  RR_CUDA(cudaMemcpyAsync(segA.p, &root, sizeof(Seg), cudaMemcpyHostToDevice, st));
  int32_t* perm = permA.p;
  int32_t* perm_o = permB.p;
  int32_t* pos = pos_a.p;
  int32_t* pos_o = pos_b.p;
  Seg* segs = segA.p;
  Seg* nsegs = segB.p;
  for (int L = 0; L < n_levels; ++L) {
    const int64_t S = seg_count[L];
    RR_CUDA(cudaMemsetAsync(bmin.p, 0xff, sizeof(unsigned long long) * 3 * S, st));
    RR_CUDA(cudaMemsetAsync(bmax.p, 0x00, sizeof(unsigned long long) * 3 * S, st));
    seg_box_kernel<<<grid_for(nf), 256, 0, st>>>(pos, perm, fb.p, nf, bmin.p, bmax.p);
    RR_LAUNCH_CHECK();
    split_flag_kernel<<<grid_for(S), 256, 0, st>>>(segs, S, sflag.p);
    RR_LAUNCH_CHECK();
    size_t t = tmp.n;
    RR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, t, sflag.p, srank.p, static_cast<int>(S), st));
    seg_node_kernel<<<grid_for(S), 256, 0, st>>>(segs, S, srank.p, bmin.p, bmax.p, perm, L, D,
                                                 level_base[L], static_cast<int32_t>(K), s->ref.p,
                                                 s->tnodes.p, s->dhdr.p, saxis.p, nsegs, nlevel.p, ntidx.p);
    RR_LAUNCH_CHECK();
    s->ctx->launches += 4;
    if (split_count[L] == 0) break;
    face_flag_kernel<<<grid_for(nf), 256, 0, st>>>(pos, segs, saxis.p, perm, nf, flag.p);
    RR_LAUNCH_CHECK();
    gather_flag_kernel<<<grid_for(3 * nf), 256, 0, st>>>(perm, flag.p, 3 * nf, fl.p);
    RR_LAUNCH_CHECK();
    t = tmp.n;
    RR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, t, fl.p, scan.p, static_cast<int>(3 * nf), st));
    scatter_kernel<<<grid_for(3 * nf), 256, 0, st>>>(pos, segs, saxis.p, srank.p, perm, fl.p, scan.p, nf,
                                                     perm_o, pos_o);
    RR_LAUNCH_CHECK();
    s->ctx->launches += 4;
    std::swap(perm, perm_o);
    std::swap(pos, pos_o);
    std::swap(segs, nsegs);
  }

  tm.mark("reference tree: levels");
  node_plane_kernel<<<grid_for(2 * nf - 1), 256, 0, st>>>(s->ref.p, ntidx.p, 2 * nf - 1, s->plane_table.p, s->plane_T,
                                                         s->tnodes.p);
  RR_LAUNCH_CHECK();
  s->ctx->launches++;
  // ---- 4-wide collapse
  int32_t k4 = 0;
  {
    const int64_t n_nodes = 2 * nf - 1, span = K + nf;
    DevBuf<int32_t> qflag, qidx;
    qflag.alloc(span + 1, st);
    qidx.alloc(span + 1, st);
    RR_CUDA(cudaMemsetAsync(qflag.p, 0, sizeof(int32_t) * (span + 1), st));
    q_flag_kernel<<<grid_for(n_nodes), 256, 0, st>>>(s->ref.p, nlevel.p, ntidx.p, n_nodes, qflag.p);
    RR_LAUNCH_CHECK();
    size_t t = tmp.n;
    size_t need = 0;
    RR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, qflag.p, qidx.p, static_cast<int>(span + 1), st));
    if (need > t) tmp.alloc(need, st);
    t = tmp.n;
    RR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, t, qflag.p, qidx.p, static_cast<int>(span + 1), st));
    int32_t counts[2] = {0, 0};
    RR_CUDA(cudaMemcpyAsync(&counts[0], qidx.p + span, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaMemcpyAsync(&counts[1], qidx.p + K, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
    s->n_qnodes = counts[0];
    s->qnodes.alloc(std::max<int64_t>(counts[0], 1), st);
    q_build_kernel<<<grid_for(n_nodes), 256, 0, st>>>(s->ref.p, nlevel.p, ntidx.p, qidx.p, n_nodes, s->dhdr.p,
                                                      s->qnodes.p);
    RR_LAUNCH_CHECK();
    s->ctx->launches += 3;
    k4 = std::min<int32_t>(counts[1], kMaxCachedQNodes);
  }

  tm.mark("reference tree: 4-wide collapse");
  RR_CUDA(cudaMemcpyAsync(&s->hdr, s->dhdr.p, sizeof(TravHeader), cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  s->hdr.K = static_cast<int32_t>(K);
  s->hdr.K4 = k4;
  s->hdr.root4 = nf == 1 ? s->hdr.root_ref : 0;
  s->hdr.depth = s->depth;
  RR_CUDA(cudaMemcpyAsync(s->dhdr.p, &s->hdr, sizeof(TravHeader), cudaMemcpyHostToDevice, st));
  RR_CUDA(cudaStreamSynchronize(st));
  s->ref_built = true;
}

}  // namespace rr
