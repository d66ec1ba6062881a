// K1'' — 8-wide compressed collapse of the SAH traversal tree (rr_sah.cu).
//
// Deep scenes (C3, C5: 4.4e5 - 2e6 faces) make the binary traversal a chain
// of ~50 dependent node fetches per ray-bounce against a 128 MB node array
// that does not fit in the 126 MB L2 (the round-1 C5 tracer: 1.2 KB of DRAM
// traffic per ray-bounce at 20 % of HBM bandwidth).  Collapsing the binary
// tree into 8-wide nodes with 8-bit quantized child boxes (the compressed
// wide BVH layout of Ylitie, Karras and Laine, HPG 2017, restated for this
// tracer's exactness contract) cuts the chain to ~1/3 and the node array to
// ~80 B per 7 binary nodes, which keeps it L2-resident; the faces are copied
// into leaf order so a node's leaf faces are contiguous.
//
// Build: a bottom-up SAH-optimal distribution pass over the binary tree
// (dp_up_kernel), then level-synchronous from the root (one thread per wide
// node):
//   expand: the slots of the node's optimal distribution (dp_unfold; the
//           A/B alternative opens the internal child of largest surface area
//           until 8 slots are used); leaf slots are the SAH tree's own 1- or
//           2-face leaves, or two sibling single-face leaves as one pair
//           slot over their parent's box;
//   scan:   exclusive sum of (internal children, leaf faces) per node, so a
//           node's internal children are contiguous one level down and its
//           leaf faces contiguous in `wtri`;
//   write:  the WNode (quantized boxes, masks, plane cull bits), the next
//           frontier, the leaf faces (FaceTri with the face id in `pad`).
//
// Exactness.  The traversal only filters; the closest hit is still the
// lexicographic (delta, face) minimum of the fp64 tests of every admitted
// face (accel_tree.cpp:148-153), so any superset of the reference's boxes
// gives identical results.  Each slot's box is the binary node's
// conservative fp32 child box (exact box + eps, rounded outward; eps =
// scale * 2^-19 bounds the fp32 slab error, rr_geom.cuh box_enter) widened
// by another eps/4 and rounded outward onto the grid (quant_axis),
// evaluated in fp64 on the exact grid values.  The node traversal evaluates
// a plane as fma(q - 1, A, B) (rr_geom.cuh visit_w8; q - 1 is exact, one
// packed FADD from the byte-permuted 2^23 + q): three roundings, A = grid *
// inv, B = fma(p, inv, -o * inv) and the final fma, each below 6 * scale *
// 2^-24 = 0.19 eps in space units (|(q - 1) * grid|, |p - o| <= 6 scale),
// where box_enter has one.  The binary box's eps covers box_enter's error
// (o, inv, o * inv and the fma: below eps / 2, rr_geom.cuh), so the two
// extra roundings (0.38 eps) stay inside the rest of eps plus the eps/4.
#include <cub/cub.cuh>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>

#include "rr_geom.cuh"

namespace rr {
namespace {

constexpr int kW = 8;

struct Slot {
  float b[6];  // lo x, hi x, lo y, hi y, lo z, hi z (the TNode child box)
  int32_t ref;  // binary ref: >= 0 internal, < 0 leaf (~f or ~(f | kPairBit))
  int32_t plane;
  int32_t ref2;  // >= 0: a pair slot of faces leaf_face(ref) and ref2 (two sibling leaves, RR_W8_PAIRS)
};

__device__ __forceinline__ void tnode_slot(const TNode& t, int side, Slot& s) {
  if (side == 0) {
    s.b[0] = t.a.x; s.b[1] = t.a.y; s.b[2] = t.a.z; s.b[3] = t.a.w; s.b[4] = t.b.x; s.b[5] = t.b.y;
    s.ref = t.d.x;
    s.plane = t.d.z;
    s.ref2 = -1;
  } else {
    s.b[0] = t.b.z; s.b[1] = t.b.w; s.b[2] = t.c.x; s.b[3] = t.c.y; s.b[4] = t.c.z; s.b[5] = t.c.w;
    s.ref = t.d.y;
    s.plane = t.d.w;
    s.ref2 = -1;
  }
}

__device__ __forceinline__ float half_area(const Slot& s) {
  const float dx = s.b[1] - s.b[0], dy = s.b[3] - s.b[2], dz = s.b[5] - s.b[4];
  return dx * dy + dy * dz + dz * dx;
}

constexpr int32_t kEmptySlot = INT32_MIN;  // an unused slot of the 8 (ref)

// ---- SAH-optimal collapse (RR_W8_DP; Ylitie, Karras and Laine 2017, sec.
// 4.1, restated for fixed 1-2-face leaves).  For every binary node n and
// i = 1..8, G(n, i) is the least SAH cost of covering n's subtree with at
// most i slots of one wide node, n itself never a slot:
//   F(c, k) = cost of child c as <= k slots = min(S(c), G(c, k)), with
//             S(c) = A(c) c_node + G(c, 8) (c its own wide node) or
//             A(c) c_face nfaces(c) (a leaf slot), G(c, 1) = inf;
//   D(n, j) = min over k of F(left, k) + F(right, j - k);
//   G(n, i) = min over 2 <= j <= i of D(n, j).
// Bottom-up (the second child to finish processes its parent), then each
// wide node unfolds G(n, 8) through the recorded choices (expand_kernel).
constexpr float kInfCost = 3.0e38f;

struct alignas(16) DpRec {
  float g[8];       // G(n, 1..8)
  uint32_t bestj;   // nibble i-1: the j <= i achieving G(n, i)
  uint32_t argk;    // nibble j-1: the k of D(n, j)
  uint32_t pad[2];
};

__global__ void dp_init_kernel(const TNode* __restrict__ tn, int32_t n_int, int32_t* __restrict__ parent,
                               int32_t* __restrict__ need, int32_t* __restrict__ arrived) {
  const int32_t n = static_cast<int32_t>(blockIdx.x * blockDim.x + threadIdx.x);
  if (n >= n_int) return;
  const TNode t = tn[n];
  int c = 0;
  if (t.d.x >= 0) { parent[t.d.x] = n; ++c; }
  if (t.d.y >= 0) { parent[t.d.y] = n; ++c; }
  need[n] = c;
  arrived[n] = 0;
}

// internal node c whose two children are single-face leaves: the faces
// (they can share one pair slot, RR_W8_PAIRS)
__device__ __forceinline__ bool pair_faces(const TNode* __restrict__ tn, int32_t c, int32_t* f1, int32_t* f2) {
  const int4 d = tn[c].d;
  if (d.x >= 0 || d.y >= 0 || leaf_faces(d.x) != 1 || leaf_faces(d.y) != 1) return false;
  *f1 = leaf_face(d.x);
  *f2 = leaf_face(d.y);
  return true;
}

// F(c, k), k = 1..8, of slot s (its box from the parent's TNode); an
// internal child whose two children are single faces may also become one
// pair slot, cost A(c) c_face 2 (pairs != 0)
__device__ __forceinline__ void dp_child(const TNode* __restrict__ tn, const Slot& s, const DpRec* __restrict__ rec,
                                         float c_node, float c_face, int pairs, float* F) {
  const float A = half_area(s);
  if (s.ref < 0) {
    const float v = A * c_face * static_cast<float>(leaf_faces(s.ref));
#pragma unroll
    for (int k = 0; k < 8; ++k) F[k] = v;
    return;
  }
  float g[8];
  const float4* r = reinterpret_cast<const float4*>(rec + s.ref);
  const float4 g0 = __ldcg(r), g1 = __ldcg(r + 1);  // written by another thread of this launch
  g[0] = g0.x; g[1] = g0.y; g[2] = g0.z; g[3] = g0.w; g[4] = g1.x; g[5] = g1.y; g[6] = g1.z; g[7] = g1.w;
  int32_t f1, f2;
  const float Sp = (pairs && pair_faces(tn, s.ref, &f1, &f2)) ? A * c_face * 2.0f : kInfCost;
  const float S = fminf(A * c_node + g[7], Sp);
#pragma unroll
  for (int k = 0; k < 8; ++k) F[k] = fminf(S, g[k]);
}

// the choice dp_child's min made for child s given k slots: 0 split it
// further, 1 one slot as it is, 2 one pair slot
__device__ __forceinline__ int dp_single(const TNode* __restrict__ tn, const Slot& s, const DpRec* __restrict__ rec,
                                         float c_node, float c_face, int pairs, int k) {
  if (s.ref < 0) return 1;
  int32_t f1, f2;
  const float A = half_area(s);
  const float Sp = (pairs && pair_faces(tn, s.ref, &f1, &f2)) ? A * c_face * 2.0f : kInfCost;
  const float Sw = A * c_node + rec[s.ref].g[7];
  if (k > 1 && fminf(Sw, Sp) > rec[s.ref].g[k - 1]) return 0;
  return Sp < Sw ? 2 : 1;
}

__global__ void dp_up_kernel(const TNode* __restrict__ tn, int32_t n_int, const int32_t* __restrict__ parent,
                             const int32_t* __restrict__ need, int32_t* __restrict__ arrived, DpRec* __restrict__ rec,
                             float c_node, float c_face, int pairs) {
  int32_t n = static_cast<int32_t>(blockIdx.x * blockDim.x + threadIdx.x);
  if (n >= n_int || need[n] != 0) return;
  for (;;) {
    const TNode t = tn[n];
    Slot sl, sr;
    tnode_slot(t, 0, sl);
    tnode_slot(t, 1, sr);
    float FL[8], FR[8];
    dp_child(tn, sl, rec, c_node, c_face, pairs, FL);
    dp_child(tn, sr, rec, c_node, c_face, pairs, FR);
    DpRec o;
    o.g[0] = kInfCost;
    o.bestj = 0;
    o.argk = 0;
    float gi = kInfCost;
    uint32_t bj = 1;
    for (int j = 2; j <= 8; ++j) {
      float d = kInfCost;
      int bk = 1;
      for (int k = 1; k < j; ++k) {
        const float v = FL[k - 1] + FR[j - k - 1];
        if (v < d) {
          d = v;
          bk = k;
        }
      }
      o.argk |= static_cast<uint32_t>(bk) << (4 * (j - 1));
      if (d < gi) {
        gi = d;
        bj = static_cast<uint32_t>(j);
      }
      o.g[j - 1] = gi;
      o.bestj |= bj << (4 * (j - 1));
    }
    rec[n] = o;
    __threadfence();
    const int32_t p = parent[n];
    if (p < 0) return;
    if (atomicAdd(arrived + p, 1) + 1 < need[p]) return;
    __threadfence();
    n = p;
  }
}

// the slots of binary node n as one wide node: G(n, 8) unfolded
__device__ __forceinline__ int dp_unfold(const TNode* __restrict__ tn, const DpRec* __restrict__ rec, int32_t root,
                                         float c_node, float c_face, int pairs, Slot* s) {
  int32_t st_n[8];
  int st_i[8];
  int sp = 0, cnt = 0;
  st_n[sp] = root;
  st_i[sp++] = 8;
  while (sp > 0) {
    --sp;
    const int32_t n = st_n[sp];
    const int i = st_i[sp];
    const DpRec& r = rec[n];
    const int j = static_cast<int>((r.bestj >> (4 * (i - 1))) & 0xfu);
    const int k = static_cast<int>((r.argk >> (4 * (j - 1))) & 0xfu);
    const TNode t = tn[n];
    for (int side = 0; side < 2; ++side) {
      Slot c;
      tnode_slot(t, side, c);
      const int kk = side == 0 ? k : j - k;
      const int how = dp_single(tn, c, rec, c_node, c_face, pairs, kk);
      if (how == 2) {  // the two leaves of c as one pair slot over c's box
        int32_t f1 = 0, f2 = 0;
        pair_faces(tn, c.ref, &f1, &f2);
        c.ref = ~(f1 | kPairBit);
        c.ref2 = f2;
        s[cnt++] = c;
      } else if (how == 1) {
        s[cnt++] = c;
      } else {
        st_n[sp] = c.ref;
        st_i[sp++] = kk;
      }
    }
  }
  return cnt;
}

// expand frontier node i into <= 8 slots; packed (internal << 32 | faces).
// order: place the children in the 8 slots by direction (Ylitie, Karras and
// Laine 2017): slot s stands for the ray octant s (bit a set: negative
// direction along axis a) and takes the child nearest to that octant's
// rays' entry side, i.e. the one minimising dot(centroid - centre, sign(s)),
// chosen greedily by cost; a ray of octant o then meets the children roughly
// front to back in the slot order s = j ^ o, j = 0..7 (trace_kernel_w8's
// group traversal).  Any slot order gives the same closest hits.
__global__ void expand_kernel(const TNode* __restrict__ tn, const int32_t* __restrict__ frontier, int32_t n,
                              Slot* __restrict__ slots, int32_t* __restrict__ nslot,
                              unsigned long long* __restrict__ packed, int order, const DpRec* __restrict__ rec,
                              float c_node, float c_face, int pairs) {
  const int32_t i = static_cast<int32_t>(blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= n) return;
  Slot s[kW];
  int cnt = 2;
  if (rec) {
    cnt = dp_unfold(tn, rec, frontier[i], c_node, c_face, pairs, s);
  } else {
    const TNode t = tn[frontier[i]];
    tnode_slot(t, 0, s[0]);
    tnode_slot(t, 1, s[1]);
  }
  while (!rec && cnt < kW) {
    int best = -1;
    float ba = -1.f;
    for (int k = 0; k < cnt; ++k)
      if (s[k].ref >= 0) {
        const float a = half_area(s[k]);
        if (a > ba) {
          ba = a;
          best = k;
        }
      }
    if (best < 0) break;
    const TNode c = tn[s[best].ref];
    tnode_slot(c, 0, s[best]);
    tnode_slot(c, 1, s[cnt]);
    ++cnt;
  }
  unsigned long long ni = 0, nfc = 0;
  for (int k = 0; k < cnt; ++k) {
    if (s[k].ref >= 0) ++ni;
    else nfc += leaf_faces(s[k].ref);
  }
  int at[kW];  // slot of child k
  for (int k = 0; k < cnt; ++k) at[k] = k;
  if (order) {
    float lo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, hi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    for (int k = 0; k < cnt; ++k)
      for (int a = 0; a < 3; ++a) {
        lo[a] = fminf(lo[a], s[k].b[2 * a]);
        hi[a] = fmaxf(hi[a], s[k].b[2 * a + 1]);
      }
    float c[kW][3];
    for (int k = 0; k < cnt; ++k)
      for (int a = 0; a < 3; ++a) c[k][a] = 0.5f * (s[k].b[2 * a] + s[k].b[2 * a + 1]) - 0.5f * (lo[a] + hi[a]);
    uint32_t free_child = (1u << cnt) - 1u, free_slot = 0xffu;
    for (int it = 0; it < cnt; ++it) {
      float best = FLT_MAX;
      int bk = -1, bs = -1;
      for (int k = 0; k < cnt; ++k) {
        if (!((free_child >> k) & 1u)) continue;
        for (int sl = 0; sl < kW; ++sl) {
          if (!((free_slot >> sl) & 1u)) continue;
          const float cost = ((sl & 1) ? -c[k][0] : c[k][0]) + ((sl & 2) ? -c[k][1] : c[k][1]) +
                             ((sl & 4) ? -c[k][2] : c[k][2]);
          if (cost < best || bk < 0) {
            best = cost;
            bk = k;
            bs = sl;
          }
        }
      }
      at[bk] = bs;
      free_child &= ~(1u << bk);
      free_slot &= ~(1u << bs);
    }
  }
  Slot* out = slots + static_cast<int64_t>(i) * kW;
  for (int k = 0; k < kW; ++k) out[k].ref = kEmptySlot;
  for (int k = 0; k < cnt; ++k) out[at[k]] = s[k];
  nslot[i] = cnt;
  packed[i] = (ni << 32) | nfc;
}

// Grid of one axis: plane(q) = p + (q - 1) * 2^(e-127), q in [0, 255]
// (p fp32, exact in fp64).  Each slot gets the floor / ceiling of its
// margin-widened box on the grid: the traversal evaluates t = fma(q - 1, A,
// B) with A = 2^(e-127) * inv (exact), whose error the margin covers.
// RR_QEXACT 0 (A/B, round 2 before): t = fma(2^23 + q, A, C) with
// C = fl(B - (2^23 + 1) A), whose rounding is up to half a grid step, so
// each slot got one more grid step below and above (C5: 18.9 instead of
// 18.0 node visits and 4.7 instead of 4.4 face tests per ray-bounce,
// 458 instead of 436 ms).  Returns the biased exponent.
__device__ __forceinline__ uint32_t quant_axis(const Slot* s, int ax, double m, float* p_out, uint32_t* lo8,
                                               uint32_t* hi8) {
  double lo = 1e300, hi = -1e300;
  for (int k = 0; k < kW; ++k) {
    if (s[k].ref == kEmptySlot) continue;
    lo = fmin(lo, static_cast<double>(s[k].b[2 * ax]) - m);
    hi = fmax(hi, static_cast<double>(s[k].b[2 * ax + 1]) + m);
  }
  const float p = __double2float_rd(lo);
  const double pd = static_cast<double>(p);
  // smallest power of two with (hi - p) <= 254 * scale (q = plane step + 1;
  // RR_QEXACT 0: 253, one step of slack below and above)
  const double span = RR_QEXACT ? 254.0 : 253.0;
  int e = static_cast<int>(ceil(log2((hi - pd) / span)));
  while (ldexp(span, e) < hi - pd) ++e;
  while (e > -126 && ldexp(span, e - 1) >= hi - pd) --e;
  e = max(e, -126);
  // RR_QMANT mantissa bits: the smallest 2^(e-1) (1 + j / 2^M) that still
  // spans the box (a finer grid than the power of two, same decode cost)
  uint32_t field = static_cast<uint32_t>(e + 127) << RR_QMANT;
  double sc = ldexp(1.0, e);
  if (RR_QMANT > 0 && e - 1 >= -126) {
    for (int j = 1; j < (1 << RR_QMANT); ++j) {
      const double c = ldexp(1.0 + static_cast<double>(j) / (1 << RR_QMANT), e - 1);
      if (c * span >= hi - pd) {
        sc = c;
        field = (static_cast<uint32_t>(e - 1 + 127) << RR_QMANT) | static_cast<uint32_t>(j);
        break;
      }
    }
  }
  lo8[0] = lo8[1] = hi8[0] = hi8[1] = 0;
  for (int k = 0; k < kW; ++k) {
    if (s[k].ref == kEmptySlot) continue;
    // q - 1 = floor(..) - 1 and ceil(..) + 1 (RR_QEXACT: floor(..) and ceil(..))
    double ql = floor((static_cast<double>(s[k].b[2 * ax]) - m - pd) / sc) + (RR_QEXACT ? 1.0 : 0.0);
    double qh = ceil((static_cast<double>(s[k].b[2 * ax + 1]) + m - pd) / sc) + (RR_QEXACT ? 1.0 : 2.0);
    ql = fmin(fmax(ql, 0.0), 255.0);
    qh = fmin(fmax(qh, 0.0), 255.0);
    lo8[k >> 2] |= static_cast<uint32_t>(ql) << (8 * (k & 3));
    hi8[k >> 2] |= static_cast<uint32_t>(qh) << (8 * (k & 3));
  }
  *p_out = p;
  return field;
}

__global__ void write_kernel(const Slot* __restrict__ slots, const int32_t* __restrict__ nslot,
                             const unsigned long long* __restrict__ offs, int32_t n, int32_t level_base,
                             int32_t next_base, int32_t tri_base, const int32_t* __restrict__ acc,
                             const FaceTri* __restrict__ tri,
                             double margin, WNode* __restrict__ out, FaceTri* __restrict__ wtri,
                             int32_t* __restrict__ next_frontier, int32_t* __restrict__ next_acc,
                             int32_t* __restrict__ bound, int32_t* __restrict__ emax, int64_t n_faces) {
  const int32_t i = static_cast<int32_t>(blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= n) return;
  Slot s[kW];
  const int cnt = nslot[i];
  for (int k = 0; k < kW; ++k) s[k] = slots[static_cast<int64_t>(i) * kW + k];
  const unsigned long long o = offs[i];
  const int32_t ci = static_cast<int32_t>(o >> 32);  // rank of my first internal child in the next level
  const int32_t ti = tri_base + static_cast<int32_t>(o & 0xffffffffu);
  WNode w;
  float p[3];
  uint32_t e[3], lo8[3][2], hi8[3][2];
  for (int ax = 0; ax < 3; ++ax) e[ax] = quant_axis(s, ax, margin, &p[ax], lo8[ax], hi8[ax]);
  uint32_t imask = 0, valid = 0, pair = 0, cull = 0;
  // plane for the cull: the first slot plane (a subtree inside an axis-aligned
  // wall usually has all its slots in that wall)
  int32_t plane = -1;
  for (int k = 0; k < kW; ++k)
    if (s[k].ref != kEmptySlot && s[k].plane >= 0) {
      plane = s[k].plane;
      break;
    }
  // stack occupancy bound below this node: every slot but the one taken
  // pushed (trace_kernel_w8 pushes leaf slots too)
  const int32_t a = acc[i] + cnt - 1;
  int ni = 0, nfc = 0;
  for (int k = 0; k < kW; ++k) {
    if (s[k].ref == kEmptySlot) continue;
    valid |= 1u << k;
    if (plane >= 0 && s[k].plane == plane) cull |= 1u << k;
    if (s[k].ref >= 0) {
      imask |= 1u << k;
      next_frontier[ci + ni] = s[k].ref;
      next_acc[ci + ni] = a;
      ++ni;
    } else {
      const int32_t f0 = leaf_face(s[k].ref);
      const int nl = leaf_faces(s[k].ref);
      if (nl == 2) pair |= 1u << k;
      for (int j = 0; j < nl; ++j) {
        const int32_t fj = (j == 1 && s[k].ref2 >= 0) ? s[k].ref2 : f0 + j;
        RR_DCHECK(ti + nfc + j < n_faces && fj < n_faces);
        FaceTri ft = tri[fj];
        ft.pad = __longlong_as_double(static_cast<long long>(fj));
        wtri[ti + nfc + j] = ft;
      }
      nfc += nl;
    }
  }
  atomicMax(bound, a);
  atomicMax(emax, static_cast<int32_t>(max(e[0], max(e[1], e[2])) >> RR_QMANT));
  // h.w: the three (8 + RR_QMANT)-bit scale fields (RR_QMANT 0: the
  // internal mask in the top byte too)
  constexpr int kF = 8 + RR_QMANT;
  w.h = make_float4(p[0], p[1], p[2],
                    __int_as_float(static_cast<int>(e[0] | (e[1] << kF) | (e[2] << (2 * kF)) |
                                                    (RR_QMANT == 0 ? imask << 24 : 0u))));
  // bits: valid | pair << 8 | cull << 16 | internal << 24 (the internal mask
  // also in h.w, next to the exponents)
  w.m = make_int4(next_base + ci, ti, plane, static_cast<int>(valid | (pair << 8) | (cull << 16) | (imask << 24)));
  w.qx = make_uint4(lo8[0][0], lo8[0][1], hi8[0][0], hi8[0][1]);
  w.qy = make_uint4(lo8[1][0], lo8[1][1], hi8[1][0], hi8[1][1]);
  w.qz = make_uint4(lo8[2][0], lo8[2][1], hi8[2][0], hi8[2][1]);
  out[level_base + i] = w;
}

inline unsigned grid(int64_t n, int b = 256) { return static_cast<unsigned>(std::max<int64_t>(1, (n + b - 1) / b)); }

}  // namespace

void build_wide(rr_scene* s) {
  if (s->wnodes.p || !s->snodes.p || s->shdr.root_ref < 0 || s->nf < 3) return;
  cudaStream_t st = s->ctx->stream;
  const int64_t nf = s->nf;
  const int32_t n_int = static_cast<int32_t>(nf - 1);
  // every wide node consumes >= 1 binary internal node
  DevBuf<WNode> nodes;
  nodes.alloc(n_int, st);
  s->wtri.alloc(nf, st);
  DevBuf<int32_t> fr[2], ac[2], nslot, bound;  // bound: [stack bound, largest grid exponent]
  DevBuf<Slot> slots;
  DevBuf<unsigned long long> packed, offs;
  DevBuf<uint8_t> tmp;
  bound.alloc(2, st);
  RR_CUDA(cudaMemsetAsync(bound.p, 0, 2 * sizeof(int32_t), st));
  fr[0].alloc(1, st);
  ac[0].alloc(1, st);
  const int32_t root = s->shdr.root_ref, zero = 0;
  RR_CUDA(cudaMemcpyAsync(fr[0].p, &root, sizeof root, cudaMemcpyHostToDevice, st));
  RR_CUDA(cudaMemcpyAsync(ac[0].p, &zero, sizeof zero, cudaMemcpyHostToDevice, st));
  const double margin = 0.25 * static_cast<double>(s->shdr.eps);
  // RR_W8_ORDER=0: children in expansion order (A/B)
  static const int slot_order = [] {
    const char* e = std::getenv("RR_W8_ORDER");
    return e ? std::atoi(e) : 1;
  }();
  // RR_W8_DP (A/B): SAH-optimal collapse (1; C5 visits per ray-bounce
  // 19.73 -> 18.89, trace 468.2 -> 458.0 ms) or the greedy largest-area
  // expansion (0).
  static const int use_dp = [] {
    const char* e = std::getenv("RR_W8_DP");
    return e ? std::atoi(e) : 1;
  }();
  // RR_W8_PAIRS: two sibling single-face leaves may share one slot (a pair
  // leaf of arbitrary faces, copied next to each other in wtri); RR_W8_CFACE:
  // the face-test cost in node visits.  The warp-cooperative leaf tests make
  // a face test cheap, so pairs pay almost always (C5, node visits / face
  // tests per ray-bounce, ms): no pairs 17.93 / 4.38 404.4; c_face 2: 17.93
  // / 4.38 404.5, 1: 17.80 / 4.51 400.8, 0.5: 17.62 / 4.81 396.1, 0.25:
  // 17.56 / 4.98 394.8, 0.1 394.8, 0.05: 17.55 / 5.05 394.6, 0.01 394.6.
  static const int pairs = [] {
    const char* e = std::getenv("RR_W8_PAIRS");
    return e ? std::atoi(e) : 1;
  }();
  static const float c_face = [] {
    const char* e = std::getenv("RR_W8_CFACE");
    return e ? static_cast<float>(std::atof(e)) : 0.05f;
  }();
  const float c_node = 1.0f;
  DevBuf<DpRec> rec;
  if (use_dp) {
    DevBuf<int32_t> parent, need, arrived;
    parent.alloc(n_int, st);
    need.alloc(n_int, st);
    arrived.alloc(n_int, st);
    rec.alloc(n_int, st);
    RR_CUDA(cudaMemsetAsync(parent.p, 0xff, sizeof(int32_t) * n_int, st));
    dp_init_kernel<<<grid(n_int), 256, 0, st>>>(s->snodes.p, n_int, parent.p, need.p, arrived.p);
    RR_LAUNCH_CHECK();
    dp_up_kernel<<<grid(n_int), 256, 0, st>>>(s->snodes.p, n_int, parent.p, need.p, arrived.p, rec.p, c_node,
                                              c_face, pairs);
    RR_LAUNCH_CHECK();
    s->ctx->launches += 3;
  }
  int32_t n = 1, base = 0, depth = 0;
  int64_t tri_done = 0;
  while (n > 0) {
    slots.alloc(static_cast<int64_t>(n) * kW, st);
    nslot.alloc(n, st);
    packed.alloc(n + 1, st);
    offs.alloc(n + 1, st);
    expand_kernel<<<grid(n), 256, 0, st>>>(s->snodes.p, fr[0].p, n, slots.p, nslot.p, packed.p, slot_order,
                                           use_dp ? rec.p : nullptr, c_node, c_face, pairs);
    RR_LAUNCH_CHECK();
    RR_CUDA(cudaMemsetAsync(packed.p + n, 0, sizeof(unsigned long long), st));
    size_t need = 0;
    RR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, packed.p, offs.p, n + 1, st));
    if (need > tmp.n) tmp.alloc(need, st);
    RR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, need, packed.p, offs.p, n + 1, st));
    unsigned long long tot = 0;
    RR_CUDA(cudaMemcpyAsync(&tot, offs.p + n, sizeof tot, cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
    const int32_t n_next = static_cast<int32_t>(tot >> 32);
    const int64_t n_tri = static_cast<int64_t>(tot & 0xffffffffu);
    if (base + n + n_next > n_int) throw Error(RR_RUNTIME, "8-wide collapse: node count bound exceeded");
    fr[1].alloc(std::max(n_next, 1), st);
    ac[1].alloc(std::max(n_next, 1), st);
    write_kernel<<<grid(n), 256, 0, st>>>(slots.p, nslot.p, offs.p, n, base, base + n,
                                          static_cast<int32_t>(tri_done), ac[0].p, s->tri.p, margin, nodes.p,
                                          s->wtri.p, fr[1].p, ac[1].p, bound.p, bound.p + 1, nf);
    RR_LAUNCH_CHECK();
    s->ctx->launches += 5;
    tri_done += n_tri;
    base += n;
    n = n_next;
    ++depth;
    std::swap(fr[0], fr[1]);
    std::swap(ac[0], ac[1]);
  }
  if (tri_done != nf) throw Error(RR_RUNTIME, "8-wide collapse: leaf faces do not cover the mesh");
  int32_t h_bound[2] = {0, 0};
  RR_CUDA(cudaMemcpyAsync(h_bound, bound.p, sizeof h_bound, cudaMemcpyDeviceToHost, st));
  // compact copy of the node array
  s->wnodes.alloc(base, st);
  RR_CUDA(cudaMemcpyAsync(s->wnodes.p, nodes.p, sizeof(WNode) * base, cudaMemcpyDeviceToDevice, st));
  RR_CUDA(cudaStreamSynchronize(st));
  s->wroot = 0;
  s->wstack = h_bound[0] + 1;
  // fma(2^23 + q, A, C) with |A| = 2^e |inv| <= 2^e * 1e30 stays finite for
  // grid steps 2^e <= 16 (scenes up to ~2 km); larger scenes use the binary tree
  s->wide_ok = h_bound[1] <= 127 + 4;
  s->wdepth = depth;
  s->ctx->launches += 1;
}

}  // namespace rr
