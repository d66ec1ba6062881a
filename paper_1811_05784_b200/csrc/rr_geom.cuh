// Device geometry shared by the tracer kernels.
//
// fp64 parts restate the reference operation order exactly; the library is
// compiled with -fmad=false so no FMA is contracted into them (the oracle is
// compiled for baseline x86-64 with -ffp-contract=off).  The fp32 box test is
// a conservative filter only: node boxes are rounded outward and expanded by
// eps = scale * 2^-19, which dominates the fp32 origin/slab rounding error,
// so every box the fp64 reference could enter is entered here too, and the
// closest hit is decided by the fp64 triangle test alone.
#pragma once

#include <cfloat>
#include <cstdint>

#include "rr_internal.cuh"

namespace rr {

struct D3 {
  double x, y, z;
};

__device__ __forceinline__ D3 d3(double x, double y, double z) { return D3{x, y, z}; }
__device__ __forceinline__ D3 operator+(D3 a, D3 b) { return d3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ D3 operator-(D3 a, D3 b) { return d3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ D3 operator*(double s, D3 a) { return d3(s * a.x, s * a.y, s * a.z); }
// Eigen-shim dot order: (x*x' + y*y') + z*z'
__device__ __forceinline__ double dot(D3 a, D3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__device__ __forceinline__ D3 cross(D3 a, D3 b) {
  return d3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

constexpr int32_t kPop = 0x7fffffff;
constexpr int32_t kDone = 0x7ffffffe;
// an internal node to visit (not a leaf, not kDone / kPop): one unsigned compare
__device__ __forceinline__ bool is_inner(int32_t n) { return static_cast<uint32_t>(n) < static_cast<uint32_t>(kDone); }
constexpr int kStack = 32;   // BVH2: one push per level, depth <= 30
constexpr int kStack4 = 48;  // 4-wide: <= 3 pushes per level, depth <= 15

// Moller-Trumbore, geometry.cpp:77-106 (double-sided, det == 0 rejected,
// delta > kSelfHitEpsilon = 1e-6).  Returns delta or -1.
__device__ __forceinline__ double mt_delta(const FaceTri* __restrict__ tri, int32_t f, D3 o, D3 d) {
  const double2* p = reinterpret_cast<const double2*>(tri + f);
  const double2 q0 = __ldg(p), q1 = __ldg(p + 1), q2 = __ldg(p + 2), q3 = __ldg(p + 3), q4 = __ldg(p + 4);
  const D3 va = d3(q0.x, q0.y, q1.x);
  const D3 e1 = d3(q1.y, q2.x, q2.y);
  const D3 e2 = d3(q3.x, q3.y, q4.x);
  const D3 pv = cross(d, e2);
  const double det = dot(e1, pv);
  if (det == 0.0) return -1.0;
  const double inv = 1.0 / det;
  const D3 tv = o - va;
  const double lambda = dot(tv, pv) * inv;
  if (lambda < 0.0 || lambda > 1.0) return -1.0;
  const D3 qv = cross(tv, e1);
  const double mu = dot(d, qv) * inv;
  if (mu < 0.0 || lambda + mu > 1.0) return -1.0;
  const double delta = dot(e2, qv) * inv;
  if (delta <= 1e-6) return -1.0;
  return delta;
}

// intersect_sphere, geometry.cpp:115-128.  Returns delta or -1.
__device__ __forceinline__ double sphere_delta(D3 o, D3 d, D3 c, double r) {
  const D3 oc = o - c;
  const double b = dot(d, oc);
  const double cc = dot(oc, oc) - r * r;
  const double disc = b * b - cc;
  if (disc < 0.0) return -1.0;
  const double sq = sqrt(disc);
  const double nr = -b - sq;
  if (nr > 0.0) return nr;
  const double fr = -b + sq;
  if (fr > 0.0) return fr;
  return -1.0;
}

// Per-segment fp32 ray for the box filter.
struct RayF {
  float ox, oy, oz, ix, iy, iz;
  float nx, ny, nz;  // -(o * inv) for the fused slab test
  double shift;  // the fp32 origin sits at o + shift*d (shift > 0 only for far origins)
};

__device__ __forceinline__ float inv_dir(double dk) {
  float f = __double2float_rn(dk);
  float a = fabsf(f);
  if (a < 1e-30f) f = copysignf(1e-30f, dk);
  return __frcp_rn(f);  // correctly rounded, as 1.0f / f
}

// Origins farther than 4*scale from 0 are moved (in fp64) to the root box
// entry so that fp32 rounding of the origin stays below eps.
__device__ __forceinline__ bool make_rayf(const TravHeader& h, D3 o, D3 d, RayF& r) {
  const double scale = static_cast<double>(h.eps) * 0x1p19;
  double shift = 0.0;
  if (fabs(o.x) > 4.0 * scale || fabs(o.y) > 4.0 * scale || fabs(o.z) > 4.0 * scale) {
    double tn = 0.0, tf = 1e300;
    const double oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
    for (int k = 0; k < 3; ++k) {
      const double lo = static_cast<double>(h.lo[k]) - 2.0 * h.eps;
      const double hi = static_cast<double>(h.hi[k]) + 2.0 * h.eps;
      if (dd[k] == 0.0) {
        if (oo[k] < lo || oo[k] > hi) return false;
        continue;
      }
      double a = (lo - oo[k]) / dd[k], b = (hi - oo[k]) / dd[k];
      if (a > b) { const double t = a; a = b; b = t; }
      tn = fmax(tn, a);
      tf = fmin(tf, b);
    }
    if (tn > tf * (1.0 + 1e-9) + 1e-9) return false;
    shift = fmax(0.0, tn * (1.0 - 1e-9) - 4.0 * h.eps);
    o = o + shift * d;
  }
  r.ox = __double2float_rn(o.x);
  r.oy = __double2float_rn(o.y);
  r.oz = __double2float_rn(o.z);
  r.ix = inv_dir(d.x);
  r.iy = inv_dir(d.y);
  r.iz = inv_dir(d.z);
  r.nx = -(r.ox * r.ix);
  r.ny = -(r.oy * r.iy);
  r.nz = -(r.oz * r.iz);
  r.shift = shift;
  return true;
}

// Upper bound on (delta - shift) in fp32 for pruning.
__device__ __forceinline__ float prune_bound(double delta, double shift) {
  return __double2float_ru(delta - shift) * (1.0f + 0x1p-20f) + 1e-30f;
}

// Slab test of one fp32 box; returns entry t (>= 0) or +inf when missed /
// beyond tmax.
__device__ __forceinline__ float box_enter(const RayF& r, float lx, float hx, float ly, float hy, float lz, float hz,
                                           float tmax) {
  // fused slab distances l*inv - o*inv: besides the rounding of o and inv
  // (each below scale * 2^-22 in space units), the rounded product o*inv
  // adds at most |o| * 2^-24 <= scale * 2^-22 (|o| <= 4 scale, make_rayf);
  // together below the eps = scale * 2^-19 expansion of every box.
  const float x0 = __fmaf_rn(lx, r.ix, r.nx), x1 = __fmaf_rn(hx, r.ix, r.nx);
  const float y0 = __fmaf_rn(ly, r.iy, r.ny), y1 = __fmaf_rn(hy, r.iy, r.ny);
  const float z0 = __fmaf_rn(lz, r.iz, r.nz), z1 = __fmaf_rn(hz, r.iz, r.nz);
  const float tn = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fmaxf(fminf(z0, z1), 0.0f));
  const float tf = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fminf(fmaxf(z0, z1), tmax));
  return tn <= tf ? tn : __int_as_float(0x7f800000);
}

// 8-wide tracer options (rr_trace_w8.cuh)
#ifndef RR_PF8
#define RR_PF8 0  // prefetch a stashed leaf's faces: 1 into L2, 2 into L1 (with the evict-first face loads: 0 406.5 ms, 1 409.0)
#endif
#ifndef RR_GST
#define RR_GST 1  // group entries hold the node's child / face bases: no refetch at the pop (0: A/B)
#endif
#ifndef RR_HCS
#define RR_HCS 0  // A/B: face-history stores with the streaming (evict-first) hint (neutral)
#endif
#ifndef RR_OCT
#define RR_OCT 1  // octant flags re-derived from the octant word at each visit: 7 -> 3 spill reloads per visit (C5 486.5 -> 482.8 ms; 0: A/B)
#endif
#ifndef RR_HIT2
#define RR_HIT2 1  // 8-wide slot test with the clamps folded into the 3-input min / max (C5 506 -> 493 ms; 0: A/B)
#endif
#ifndef RR_FCG
#define RR_FCG 2  // face loads L1 evict-first, so the nodes and spill slots keep L1 (C5 414.3 -> 409.0 ms; 0: default
                  // caching, 1: L2 only 429.0, 3: L1 no-allocate 414.9)
#endif
#ifndef RR_HBUF
#define RR_HBUF 0  // 8-wide tracer: face history buffered per 32-B sector (rr_trace_w8.cuh; A/B)
#endif
#ifndef RR_QEXACT
#define RR_QEXACT 1  // 8-wide planes as fma(q - 1, A, B), no extra grid step (C5 458 -> 436 ms; 0: A/B)
#endif
#ifndef RR_COOP
#define RR_COOP 1  // 8-wide tracer: batched leaf tests spread over the whole warp (C5 434.7 -> 428.8 ms; 0: A/B)
#endif
#ifndef RR_PIPE
// 8-wide visit: ALU-pipe work moved to the FMA pipe (bit mask; see wbyte,
// visit_w8).  ncu (C5): ALU pipe 63 % busy, FMA pipe 22 %, issue 70 %: the
// ALU pipe (one warp instruction per 2 cycles per SMSP, like the FMA pipe)
// took the byte permutes, min / max, selects and compares.  1: near / far
// planes by IMADs (427.3 -> 423.3 ms), 2: top bytes as mad.hi (ptxas emits
// one LEA.HI with the 2^23 bits folded in: 425.6; 1|2 421.8), 8: hit mask
// from FADD2 sign bits (LEA.HI) gathered by IMADs (1|2|8 417.0); forcing
// IMAD.HI instead of LEA.HI costs 19 %.  Tried and slower:
// byte 2 by two IMADs (427.0), the nearest-slot keys by IMADs (421.6), the
// octant permutation of the group mask as an L1 table (427.1).
#define RR_PIPE 11
#endif
#ifndef RR_RSM
#define RR_RSM 1  // 8-wide tracer: the fp32 ray terms in shared memory (C5 417.9 -> 415.3 ms at the 196 KB carveout; 0: A/B)
#endif
#ifndef RR_NEL
#define RR_NEL 0  // A/B: 8-wide node loads with the L1 evict-last hint
#endif
#ifndef RR_QMANT
#define RR_QMANT 2  // 8-wide grid scales with 2 mantissa bits (0: powers of two; A/B)
#endif
#ifndef RR_FFMA2
#define RR_FFMA2 1
#endif
// (f0, f1) * a + c in one packed fp32x2 FMA (Blackwell FFMA2), each lane
// rounded like __fmaf_rn
__device__ __forceinline__ float2 fma2(float f0, float f1, float a, float c) {
  float2 r;
  asm("{\n\t.reg .b64 F, A, C, D;\n\tmov.b64 F, {%2, %3};\n\tmov.b64 A, {%4, %4};\n\tmov.b64 C, {%5, %5};\n\t"
      "fma.rn.f32x2 D, F, A, C;\n\tmov.b64 {%0, %1}, D;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(f0), "f"(f1), "f"(a), "f"(c));
  return r;
}

// (f0 - (2^23 + 1), f1 - (2^23 + 1)) * a + c, two slots per packed FADD +
// FFMA: f = 2^23 + q from the byte permute, so f - (2^23 + 1) = q - 1 exactly
__device__ __forceinline__ float2 fma2q(float f0, float f1, float a, float c) {
  float2 r;
  asm("{\n\t.reg .b64 F, K, A, C, D;\n\tmov.b64 F, {%2, %3};\n\tmov.b64 K, {%6, %6};\n\tmov.b64 A, {%4, %4};\n\t"
      "mov.b64 C, {%5, %5};\n\tadd.rn.f32x2 F, F, K;\n\tfma.rn.f32x2 D, F, A, C;\n\tmov.b64 {%0, %1}, D;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(f0), "f"(f1), "f"(a), "f"(c), "f"(-8388609.0f));
  return r;
}

__device__ __forceinline__ TNode load_node(const TNode* __restrict__ g, const TNode* s, int32_t n, int32_t K) {
  if (n < K) return s[n];
  const float4* p = reinterpret_cast<const float4*>(g + n);
  TNode t;
  t.a = __ldg(p);
  t.b = __ldg(p + 1);
  t.c = __ldg(p + 2);
  const int4* q = reinterpret_cast<const int4*>(p + 3);
  t.d = __ldg(q);
  return t;
}

// Closest hit: lexicographic min of (delta, face) over all faces the fp64
// triangle test accepts (accel_tree.cpp:148-153); visits a superset of the
// leaves the reference's pruned traversal visits.
struct HitResult {
  double delta;
  int32_t face;
};

// rplane: plane id of the face the ray leaves (or -2).  Children whose whole
// subtree lies on that axis-aligned plane are skipped: a ray leaving the
// plane with |d_axis| > 1e-6 meets it only at delta ~ 1e-14 / |d_axis|, which
// the reference's fp64 test rejects (delta <= kSelfHitEpsilon), so the
// closest hit is unchanged.
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Leaf refs: ~f holds face f; in the SAH tree ~(f | kPairBit) holds faces f
// and f + 1 together (a quad's two triangles share one box, so the node
// over them only cost a dependent fetch; rr_sah.cu finish_kernel).
__device__ __forceinline__ int32_t leaf_face(int32_t leaf) { return ~leaf & (kPairBit - 1); }
__device__ __forceinline__ int leaf_faces(int32_t leaf) { return (~leaf & kPairBit) ? 2 : 1; }

// fp64 test of a leaf's faces into best (lexicographic (delta, face)
// minimum, accel_tree.cpp:148-153); true if best changed
__device__ __forceinline__ bool test_leaf(const FaceTri* __restrict__ tri, int32_t leaf, D3 o, D3 d,
                                          HitResult& best) {
  const int32_t f0 = leaf_face(leaf);
  const int nfc = leaf_faces(leaf);
  if (nfc == 2) prefetch_l1(tri + f0 + 1);
  bool better = false;
#pragma unroll 1
  for (int k = 0; k < nfc; ++k) {
    const int32_t f = f0 + k;
    const double t = mt_delta(tri, f, o, d);
    if (t > 0.0 && (best.face < 0 || t < best.delta || (t == best.delta && f < best.face))) {
      best.delta = t;
      best.face = f;
      better = true;
    }
  }
  return better;
}

template <bool PF = false>
__device__ __forceinline__ HitResult closest_hit(const TravHeader& h, const TNode* __restrict__ nodes,
                                                 const TNode* smem, int32_t K, const FaceTri* __restrict__ tri,
                                                 D3 o, D3 d, int32_t* n_visit = nullptr, int32_t rplane = -2) {
  HitResult best{0.0, -1};
  RayF r;
  if (!make_rayf(h, o, d, r)) return best;
  float tbest = FLT_MAX;
  int32_t node;
  if (h.root_ref < 0) {
    node = h.root_ref;
  } else {
    const float t = box_enter(r, h.lo[0], h.hi[0], h.lo[1], h.hi[1], h.lo[2], h.hi[2], tbest);
    node = (t == __int_as_float(0x7f800000)) ? kDone : h.root_ref;
  }
  int32_t st_n[kStack];
  float st_t[kStack];
  int sp = 0;
  int32_t visits = 0;
  while (node != kDone) {
    if (node >= 0 && node != kPop) {
      ++visits;
      const TNode nd = load_node(nodes, smem, node, K);
      if (PF) {  // start fetching both children while the boxes are tested
        prefetch_l1(nd.d.x >= 0 ? static_cast<const void*>(nodes + nd.d.x)
                                : static_cast<const void*>(tri + leaf_face(nd.d.x)));
        prefetch_l1(nd.d.y >= 0 ? static_cast<const void*>(nodes + nd.d.y)
                                : static_cast<const void*>(tri + leaf_face(nd.d.y)));
      }
      float tl = box_enter(r, nd.a.x, nd.a.y, nd.a.z, nd.a.w, nd.b.x, nd.b.y, tbest);
      float tr = box_enter(r, nd.b.z, nd.b.w, nd.c.x, nd.c.y, nd.c.z, nd.c.w, tbest);
      if (nd.d.z == rplane) tl = __int_as_float(0x7f800000);
      if (nd.d.w == rplane) tr = __int_as_float(0x7f800000);
      const bool hl = tl != __int_as_float(0x7f800000), hr = tr != __int_as_float(0x7f800000);
      if (hl && hr) {
        const bool lf = tl <= tr;
        st_n[sp] = lf ? nd.d.y : nd.d.x;
        st_t[sp] = lf ? tr : tl;
        ++sp;
        node = lf ? nd.d.x : nd.d.y;
      } else if (hl) {
        node = nd.d.x;
      } else if (hr) {
        node = nd.d.y;
      } else {
        node = kPop;
      }
    } else if (node < 0) {
      if (test_leaf(tri, node, o, d, best)) tbest = prune_bound(best.delta, r.shift);
      node = kPop;
    }
    if (node == kPop) {
      node = kDone;
      while (sp > 0) {
        --sp;
        if (st_t[sp] <= tbest) {
          node = st_n[sp];
          break;
        }
      }
    }
  }
  if (n_visit) *n_visit = visits;
  return best;
}

// Same contract as closest_hit, for warp-synchronous callers: a reached leaf
// is stashed (its triangle prefetched into L1) and traversal goes on; the
// stashed fp64 tests run together when at least LEAFT of the lanes still in
// the loop hold one or some lane cannot continue without its test, so the
// Moller-Trumbore code runs with most lanes active instead of ~2.  Pruning
// uses the bound of the leaves tested so far (looser while a leaf waits), so
// the candidate set still holds the closest face; stack entries are packed
// (node, t) pairs, one 8-B local access per push / pop.
struct RegRay {  // ray held in registers
  D3 o, d;
  __device__ __forceinline__ D3 org() const { return o; }
  __device__ __forceinline__ D3 dir() const { return d; }
};

// CNT: count internal-node visits and leaf tests into *cnt (instrumented build)
// UNR: internal nodes a lane may process per vote round (amortises the votes)
__device__ __forceinline__ int mt32(const float4* __restrict__ tri32, int32_t f, const RayF& r, float dx, float dy,
                                    float dz, float S, float* tlo, float* tup);

// SMS: the bottom SMS stack entries live in shared memory (sst: this
// thread's column, stride 128), the rest in local memory.  F32L: a batched
// leaf first goes through the conservative fp32 classification (mt32) and
// only leaves it cannot reject run the fp64 test.
template <int LEAFT, int STUCKT = 1, typename RAY = RegRay, bool CNT = false, int UNR = 1, int SMS = 0,
          bool F32L = false, int TOS = 0, bool PFL = true>  // STUCKT < 0: >= 1/|STUCKT| of lanes; TOS: newest entries in registers (0-2); PFL: prefetch stashed leaves
__device__ __forceinline__ HitResult closest_hit_pl(const TravHeader& h, const TNode* __restrict__ nodes,
                                                    const FaceTri* __restrict__ tri, const RAY& ray,
                                                    int32_t rplane, unsigned long long* cnt = nullptr,
                                                    int2* sst = nullptr, const float4* __restrict__ tri32 = nullptr) {
  HitResult best{0.0, -1};
  RayF r;
  if (!make_rayf(h, ray.org(), ray.dir(), r)) return best;
  const float kInf = __int_as_float(0x7f800000);
  float tbest = FLT_MAX;
  int32_t node;
  if (h.root_ref < 0) {
    node = h.root_ref;
  } else {
    const float t = box_enter(r, h.lo[0], h.hi[0], h.lo[1], h.hi[1], h.lo[2], h.hi[2], tbest);
    node = (t == kInf) ? kDone : h.root_ref;
  }
  int2 st[kStack - SMS];
  int sp = 0;
  int2 top[TOS > 0 ? TOS : 1] = {};  // TOS: the newest entries (top[0] newest), kept out of local memory
  int n_top = 0;
  int32_t leaf = 0;  // stashed leaf (< 0) or 0
  if (node < 0 && node != kDone) {  // one-face scene: the root is a leaf
    leaf = node;
    node = kDone;
  }
  auto pop = [&]() {
    node = kDone;
    while (TOS > 0 && n_top > 0) {
      const int2 e = top[0];
#pragma unroll
      for (int k = 0; k + 1 < TOS; ++k) top[k] = top[k + 1];
      --n_top;
      if (__int_as_float(e.y) <= tbest) {
        node = e.x;
        return;
      }
    }
    while (sp > 0) {
      --sp;
      const int2 e = (SMS > 0 && sp < SMS) ? sst[sp * 128] : st[sp - SMS];
      if (__int_as_float(e.y) <= tbest) {
        node = e.x;
        break;
      }
    }
  };
  while (node != kDone || leaf != 0) {
#pragma unroll 1
    for (int u = 0; u < UNR && is_inner(node) && (u == 0 || leaf == 0); ++u) {
      if (CNT) ++cnt[0];
      const float4* q = reinterpret_cast<const float4*>(nodes + node);
      const float4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
      const int4 dd = __ldg(reinterpret_cast<const int4*>(q + 3));
      float tl = box_enter(r, a.x, a.y, a.z, a.w, b.x, b.y, tbest);
      float tr = box_enter(r, b.z, b.w, c.x, c.y, c.z, c.w, tbest);
      if (dd.z == rplane) tl = kInf;
      if (dd.w == rplane) tr = kInf;
      const bool hl = tl != kInf, hr = tr != kInf;
      if (hl && hr) {
        const bool lf = tl <= tr;
        const int2 e = make_int2(lf ? dd.y : dd.x, __float_as_int(lf ? tr : tl));
        if (TOS > 0) {
          RR_DCHECK(n_top < TOS || sp < kStack - SMS);
          if (n_top == TOS) st[sp++] = top[TOS - 1];  // the oldest register entry spills
#pragma unroll
          for (int k = TOS - 1; k > 0; --k) top[k] = top[k - 1];
          top[0] = e;
          n_top = min(n_top + 1, TOS);
        } else {
          if (SMS > 0 && sp < SMS) sst[sp * 128] = e;
          else st[sp - SMS] = e;
          ++sp;
        }
        node = lf ? dd.x : dd.y;
      } else if (hl) {
        node = dd.x;
      } else if (hr) {
        node = dd.y;
      } else {
        pop();
      }
      if (node < 0 && leaf == 0) {  // stash a reached leaf and keep traversing
        leaf = node;
        if (PFL) prefetch_l1(tri + leaf_face(leaf));
        pop();
      }
    }
    // test when enough lanes hold a leaf, enough are stuck behind theirs, or
    // no lane can advance without a test (nothing to decide if none holds one)
    const unsigned act = __activemask();
    const unsigned hv = __ballot_sync(act, leaf != 0);
    if (hv == 0) continue;
    const bool can = is_inner(node);
    const bool must = leaf != 0 && !can;
    const unsigned mv = __ballot_sync(act, must);
    const unsigned cv = __ballot_sync(act, can);
    const int na = __popc(act);
    const bool enough_stuck = STUCKT > 0 ? __popc(mv) >= STUCKT : __popc(mv) * (-STUCKT) >= na;
    if (enough_stuck || cv == 0 || __popc(hv) * LEAFT >= 32 * na) {
      if (leaf != 0) {
        if (CNT) cnt[1] += leaf_faces(leaf);
        bool test = true;
        if (F32L && leaf_faces(leaf) == 1) {
          const D3 dd = ray.dir();
          float lo, up;
          test = mt32(tri32, leaf_face(leaf), r, __double2float_rn(dd.x), __double2float_rn(dd.y),
                      __double2float_rn(dd.z), h.eps * 0x1p19f, &lo, &up) != 0;
        }
        if (test && test_leaf(tri, leaf, ray.org(), ray.dir(), best)) tbest = prune_bound(best.delta, r.shift);
        leaf = 0;
        if (node < 0) {  // the leaf that waited for the slot
          leaf = node;
          if (PFL) prefetch_l1(tri + leaf_face(leaf));
          pop();
        }
      }
    }
  }
  return best;
}

// closest_hit_pl over the 4-wide collapse of the SAH tree: one QNode visit
// replaces two binary levels (half the dependent node fetches); hit slots
// are ordered by entry distance, the nearest taken next and the others
// pushed (leaves included, so a popped entry may be a leaf); coplanar slots
// culled via QNode.pad; same postponed, warp-batched leaf tests.
template <int LEAFT, int STUCKT, typename RAY, int UNR = 1, int TOS = 0, bool CNT = false>
__device__ __forceinline__ HitResult closest_hit4_pl(const TravHeader& h, const QNode* __restrict__ q4,
                                                     int32_t root4, const FaceTri* __restrict__ tri,
                                                     const RAY& ray, int32_t rplane,
                                                     unsigned long long* cnt = nullptr) {
  HitResult best{0.0, -1};
  RayF r;
  if (!make_rayf(h, ray.org(), ray.dir(), r)) return best;
  const float kInf = __int_as_float(0x7f800000);
  float tbest = FLT_MAX;
  int32_t node;
  if (root4 < 0) {
    node = root4;
  } else {
    const float t = box_enter(r, h.lo[0], h.hi[0], h.lo[1], h.hi[1], h.lo[2], h.hi[2], tbest);
    node = (t == kInf) ? kDone : root4;
  }
  int2 st[kStack4];
  int sp = 0;
  int2 top[TOS > 0 ? TOS : 1] = {};  // TOS: the newest entries in registers (top[0] newest)
  int n_top = 0;
  int32_t leaf = 0;
  auto push = [&](int2 e) {
    RR_DCHECK(sp < kStack4);
    if (TOS > 0) {
      if (n_top == TOS) st[sp++] = top[TOS - 1];
#pragma unroll
      for (int k = TOS - 1; k > 0; --k) top[k] = top[k - 1];
      top[0] = e;
      n_top = min(n_top + 1, TOS);
    } else {
      st[sp++] = e;
    }
  };
  auto pop = [&]() {
    node = kDone;
    while (TOS > 0 && n_top > 0) {
      const int2 e = top[0];
#pragma unroll
      for (int k = 0; k + 1 < TOS; ++k) top[k] = top[k + 1];
      --n_top;
      if (__int_as_float(e.y) <= tbest) {
        node = e.x;
        return;
      }
    }
    while (sp > 0) {
      --sp;
      const int2 e = st[sp];
      if (__int_as_float(e.y) <= tbest) {
        node = e.x;
        break;
      }
    }
  };
  while (node != kDone || leaf != 0) {
#pragma unroll 1
    for (int u = 0; u < UNR && node >= 0 && node != kDone && (u == 0 || leaf == 0); ++u) {
      if (CNT) ++cnt[0];
      const float4* p = reinterpret_cast<const float4*>(q4 + node);
      const float4 lx = __ldg(p), hx = __ldg(p + 1), ly = __ldg(p + 2), hy = __ldg(p + 3);
      const float4 lz = __ldg(p + 4), hz = __ldg(p + 5);
      const int4 ch = __ldg(reinterpret_cast<const int4*>(p + 6));
      const int4 pl = __ldg(reinterpret_cast<const int4*>(p + 7));
      float t0 = box_enter(r, lx.x, hx.x, ly.x, hy.x, lz.x, hz.x, tbest);
      float t1 = box_enter(r, lx.y, hx.y, ly.y, hy.y, lz.y, hz.y, tbest);
      float t2 = box_enter(r, lx.z, hx.z, ly.z, hy.z, lz.z, hz.z, tbest);
      float t3 = box_enter(r, lx.w, hx.w, ly.w, hy.w, lz.w, hz.w, tbest);
      if (pl.x == rplane || ch.x == kEmpty) t0 = kInf;
      if (pl.y == rplane || ch.y == kEmpty) t1 = kInf;
      if (pl.z == rplane || ch.z == kEmpty) t2 = kInf;
      if (pl.w == rplane || ch.w == kEmpty) t3 = kInf;
      // sort the four (t, ref) pairs ascending (5 compare-exchanges)
      int32_t c0 = ch.x, c1 = ch.y, c2 = ch.z, c3 = ch.w;
      auto cx = [](float& ta, int32_t& ca, float& tb, int32_t& cb) {
        const bool sw = tb < ta;
        const float tt = sw ? tb : ta;
        tb = sw ? ta : tb;
        ta = tt;
        const int32_t cc = sw ? cb : ca;
        cb = sw ? ca : cb;
        ca = cc;
      };
      cx(t0, c0, t1, c1);
      cx(t2, c2, t3, c3);
      cx(t0, c0, t2, c2);
      cx(t1, c1, t3, c3);
      cx(t1, c1, t2, c2);
      // push the far hits (descending), continue with the nearest
      if (t3 != kInf) push(make_int2(c3, __float_as_int(t3)));
      if (t2 != kInf) push(make_int2(c2, __float_as_int(t2)));
      if (t1 != kInf) push(make_int2(c1, __float_as_int(t1)));
      if (t0 != kInf) {
        node = c0;
      } else {
        pop();
      }
      if (node < 0 && leaf == 0) {  // stash a reached leaf and keep traversing
        leaf = node;
        prefetch_l1(tri + leaf_face(leaf));
        pop();
      }
    }
    if (node < 0 && leaf == 0) {  // a popped leaf (or a leaf root) with no node visit
      leaf = node;
      prefetch_l1(tri + leaf_face(leaf));
      pop();
    }
    const unsigned act = __activemask();
    const unsigned hv = __ballot_sync(act, leaf != 0);
    if (hv == 0) continue;  // no lane holds a leaf: nothing to decide
    const bool can = node >= 0 && node != kDone;
    const bool must = leaf != 0 && !can;
    const unsigned mv = __ballot_sync(act, must);
    const unsigned cv = __ballot_sync(act, can);
    const int na = __popc(act);
    const bool enough_stuck = STUCKT > 0 ? __popc(mv) >= STUCKT : __popc(mv) * (-STUCKT) >= na;
    if (enough_stuck || cv == 0 || __popc(hv) * LEAFT >= 32 * na) {
      if (leaf != 0) {
        if (CNT) cnt[1] += leaf_faces(leaf);
        if (test_leaf(tri, leaf, ray.org(), ray.dir(), best)) tbest = prune_bound(best.delta, r.shift);
        leaf = 0;
        if (node < 0) {  // the leaf that waited for the slot
          leaf = node;
          prefetch_l1(tri + leaf_face(leaf));
          pop();
        }
      }
    }
  }
  return best;
}

// ---------------------------------------------------------------------------
// fp32 triangle classification.  The fp64 Moller-Trumbore decides every hit;
// this filter only sorts leaves into
//   0: the fp64 test certainly rejects it,
//   1: uncertain (kept as a candidate for the fp64 test),
//   2: the fp64 test certainly accepts it, with delta in [tlo, tup]
//      (shifted frame), so tup may tighten the pruning bound.
// u = (O-A).(D x E2), v = D.((O-A) x E1), t = E2.((O-A) x E1), det =
// E1.(D x E2) are computed in fp32 from fp32-rounded inputs; each carries an
// absolute error below K * (product of the L1 norms of its three factors),
// K = 2^-19 (>= 32 units of fp32 roundoff), with |O-A| widened by the scene
// scale S to cover the rounding of O and A.  Outside the margins the signs
// of the exact quantities, hence the fp64 decisions, are known.
__device__ __forceinline__ int mt32(const float4* __restrict__ tri32, int32_t f, const RayF& r, float dx, float dy,
                                    float dz, float S, float* tlo, float* tup) {
  const float4 A = __ldg(tri32 + 3 * f), E1 = __ldg(tri32 + 3 * f + 1), E2 = __ldg(tri32 + 3 * f + 2);
  const float px = dy * E2.z - dz * E2.y, py = dz * E2.x - dx * E2.z, pz = dx * E2.y - dy * E2.x;
  float det = E1.x * px + E1.y * py + E1.z * pz;
  const float tx = r.ox - A.x, ty = r.oy - A.y, tz = r.oz - A.z;
  float u = tx * px + ty * py + tz * pz;
  const float qx = ty * E1.z - tz * E1.y, qy = tz * E1.x - tx * E1.z, qz = tx * E1.y - ty * E1.x;
  float v = dx * qx + dy * qy + dz * qz;
  float t = E2.x * qx + E2.y * qy + E2.z * qz;
  const float K = 0x1p-19f;
  const float nd = fabsf(dx) + fabsf(dy) + fabsf(dz);
  const float n1 = fabsf(E1.x) + fabsf(E1.y) + fabsf(E1.z);
  const float n2 = fabsf(E2.x) + fabsf(E2.y) + fabsf(E2.z);
  const float nt = fabsf(tx) + fabsf(ty) + fabsf(tz) + S;
  const float m_det = K * n1 * nd * n2, m_u = K * nt * nd * n2, m_v = K * nd * nt * n1, m_t = K * n2 * nt * n1;
  if (det < 0.0f) {
    det = -det;
    u = -u;
    v = -v;
    t = -t;
  }
  if (u < -m_u || v < -m_v || u + v > det + (m_u + m_v + m_det)) return 0;
  if (det <= m_det) {  // near-parallel: undecidable here
    *tlo = 0.0f;
    *tup = __int_as_float(0x7f800000);
    return 1;
  }
  const float lo = (t - m_t) / (det + m_det) * (1.0f - 0x1p-20f);
  const float hi = (t + m_t) / (det - m_det) * (1.0f + 0x1p-20f);
  const float sh = static_cast<float>(r.shift);
  if (hi + sh < 0.5e-6f) return 0;  // delta <= kSelfHitEpsilon for sure
  *tlo = lo;
  *tup = hi;
  const bool robust = u >= m_u && v >= m_v && u + v <= det - (m_u + m_v + m_det) && lo + sh > 2e-6f;
  return robust ? 2 : 1;
}

constexpr int kCand = 16;

// fp64-leaf traversal kept out of line: the rare fallback of closest_hit_f.
static __device__ __noinline__ HitResult closest_hit_slow(const TravHeader& h, const TNode* __restrict__ nodes,
                                                   const FaceTri* __restrict__ tri, D3 o, D3 d) {
  return closest_hit(h, nodes, nullptr, 0, tri, o, d);
}

// Closest hit with an fp32 traversal (boxes + mt32) and fp64 resolution:
// leaves of class 1/2 become candidates, robust hits tighten the pruning
// bound, and the fp64 Moller-Trumbore picks the lexicographic (delta, face)
// minimum among the candidates that can still win.  Same result as
// closest_hit: a leaf holding the fp64-closest face is never pruned (its
// entry <= that delta <= the bound) and never classed 0.
__device__ __forceinline__ HitResult closest_hit_f(const TravHeader& h, const TNode* __restrict__ nodes,
                                                   const float4* __restrict__ tri32, const FaceTri* __restrict__ tri,
                                                   D3 o, D3 d) {
  HitResult best{0.0, -1};
  RayF r;
  if (!make_rayf(h, o, d, r)) return best;
  const float dx = __double2float_rn(d.x), dy = __double2float_rn(d.y), dz = __double2float_rn(d.z);
  const float S = h.eps * 0x1p19f;
  float tbest = FLT_MAX;
  int32_t cand[kCand];
  float cand_lo[kCand];
  int nc = 0;
  int32_t node;
  if (h.root_ref < 0) {
    node = h.root_ref;
  } else {
    const float t = box_enter(r, h.lo[0], h.hi[0], h.lo[1], h.hi[1], h.lo[2], h.hi[2], tbest);
    node = (t == __int_as_float(0x7f800000)) ? kDone : h.root_ref;
  }
  int32_t st_n[kStack];
  float st_t[kStack];
  int sp = 0;
  bool overflow = false;
  auto flush = [&](int32_t f) {  // fp64 decision for one candidate
    const double t = mt_delta(tri, f, o, d);
    if (t > 0.0 && (best.face < 0 || t < best.delta || (t == best.delta && f < best.face))) {
      best.delta = t;
      best.face = f;
      tbest = fminf(tbest, prune_bound(t, r.shift));
    }
  };
  while (node != kDone) {
    if (node >= 0 && node != kPop) {
      const float4* p = reinterpret_cast<const float4*>(nodes + node);
      const float4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
      const int4 dd = __ldg(reinterpret_cast<const int4*>(p + 3));
      const float tl = box_enter(r, a.x, a.y, a.z, a.w, b.x, b.y, tbest);
      const float tr = box_enter(r, b.z, b.w, c.x, c.y, c.z, c.w, tbest);
      const bool hl = tl != __int_as_float(0x7f800000), hr = tr != __int_as_float(0x7f800000);
      if (hl && hr) {
        const bool lf = tl <= tr;
        st_n[sp] = lf ? dd.y : dd.x;
        st_t[sp] = lf ? tr : tl;
        ++sp;
        node = lf ? dd.x : dd.y;
      } else if (hl) {
        node = dd.x;
      } else if (hr) {
        node = dd.y;
      } else {
        node = kPop;
      }
    } else if (node < 0) {
      const int32_t f = ~node;
      float lo, hi;
      const int cls = mt32(tri32, f, r, dx, dy, dz, S, &lo, &hi);
      if (cls == 2) tbest = fminf(tbest, hi);
      if (cls != 0 && lo <= tbest) {
        if (nc == kCand) {  // pathological: redo this ray with fp64 leaf tests
          overflow = true;
          break;
        }
        cand[nc] = f;
        cand_lo[nc] = lo;
        ++nc;
      }
      node = kPop;
    }
    if (node == kPop) {
      node = kDone;
      while (sp > 0) {
        --sp;
        if (st_t[sp] <= tbest) {
          node = st_n[sp];
          break;
        }
      }
    }
  }
  if (overflow) return closest_hit_slow(h, nodes, tri, o, d);
  for (int k = 0; k < nc; ++k)
    if (cand_lo[k] <= tbest) flush(cand[k]);
  return best;
}

__device__ __forceinline__ QNode load_qnode(const QNode* __restrict__ g, const QNode* s, int32_t n, int32_t K4) {
  if (n < K4) return s[n];
  const float4* p = reinterpret_cast<const float4*>(g + n);
  QNode q;
  q.lx = __ldg(p);
  q.hx = __ldg(p + 1);
  q.ly = __ldg(p + 2);
  q.hy = __ldg(p + 3);
  q.lz = __ldg(p + 4);
  q.hz = __ldg(p + 5);
  q.child = __ldg(reinterpret_cast<const int4*>(p + 6));
  return q;
}

// Closest hit over the 4-wide collapse of the reference tree.  Same result
// contract as closest_hit: lexicographic min of (delta, face) over the faces
// the fp64 test accepts, visiting a superset of the reference's leaves.
// Leaf children are tested as soon as their box is entered (shrinking the
// pruning bound early); internal children are visited nearest first.
__device__ __forceinline__ HitResult closest_hit4(const TravHeader& h, const QNode* __restrict__ nodes,
                                                  const QNode* smem, int32_t K4, const FaceTri* __restrict__ tri,
                                                  D3 o, D3 d) {
  HitResult best{0.0, -1};
  RayF r;
  if (!make_rayf(h, o, d, r)) return best;
  float tbest = FLT_MAX;
  const float kInf = __int_as_float(0x7f800000);
  int32_t node;
  if (h.root4 < 0) {
    node = h.root4;
  } else {
    const float t = box_enter(r, h.lo[0], h.hi[0], h.lo[1], h.hi[1], h.lo[2], h.hi[2], tbest);
    node = (t == kInf) ? kDone : h.root4;
  }
  int32_t st_n[kStack4];
  float st_t[kStack4];
  int sp = 0;
  while (node != kDone) {
    if (node >= 0 && node != kPop) {
      const QNode q = load_qnode(nodes, smem, node, K4);
      const float lx[4] = {q.lx.x, q.lx.y, q.lx.z, q.lx.w}, hx[4] = {q.hx.x, q.hx.y, q.hx.z, q.hx.w};
      const float ly[4] = {q.ly.x, q.ly.y, q.ly.z, q.ly.w}, hy[4] = {q.hy.x, q.hy.y, q.hy.z, q.hy.w};
      const float lz[4] = {q.lz.x, q.lz.y, q.lz.z, q.lz.w}, hz[4] = {q.hz.x, q.hz.y, q.hz.z, q.hz.w};
      const int32_t ch[4] = {q.child.x, q.child.y, q.child.z, q.child.w};
      float t[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) t[s] = box_enter(r, lx[s], hx[s], ly[s], hy[s], lz[s], hz[s], tbest);
      // leaves first (their hits tighten tbest)
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        if (t[s] != kInf && ch[s] < 0 && ch[s] != kEmpty) {
          const int32_t f = ~ch[s];
          const double dt = mt_delta(tri, f, o, d);
          if (dt > 0.0 && (best.face < 0 || dt < best.delta || (dt == best.delta && f < best.face))) {
            best.delta = dt;
            best.face = f;
            tbest = prune_bound(dt, r.shift);
          }
        }
      }
      // internal children, nearest first
      int32_t cn[4];
      float ct[4];
      int m = 0;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        if (t[s] <= tbest && ch[s] >= 0) {
          // insertion into the sorted (ascending t) list
          int k = m++;
          while (k > 0 && ct[k - 1] > t[s]) {
            ct[k] = ct[k - 1];
            cn[k] = cn[k - 1];
            --k;
          }
          ct[k] = t[s];
          cn[k] = ch[s];
        }
      }
      if (m == 0) {
        node = kPop;
      } else {
        for (int k = m - 1; k >= 1; --k) {
          st_n[sp] = cn[k];
          st_t[sp] = ct[k];
          ++sp;
        }
        node = cn[0];
      }
    } else if (node < 0) {  // one-face mesh
      const int32_t f = ~node;
      const double dt = mt_delta(tri, f, o, d);
      if (dt > 0.0) {
        best.delta = dt;
        best.face = f;
      }
      node = kPop;
    }
    if (node == kPop) {
      node = kDone;
      while (sp > 0) {
        --sp;
        if (st_t[sp] <= tbest) {
          node = st_n[sp];
          break;
        }
      }
    }
  }
  return best;
}


// ---------------------------------------------------------------------------
// 8-wide compressed traversal (WNode, rr_wide.cu).  Leaf refs index the
// leaf-ordered face copy: ~(t | kPairBit) holds wtri[t] and wtri[t + 1];
// the face id travels in FaceTri.pad.

// Moller-Trumbore on a leaf-ordered face (mt_delta's operations), face id out
__device__ __forceinline__ double mt_delta_w(const FaceTri* __restrict__ wtri, int32_t t, D3 o, D3 d, int32_t* face) {
  const double2* p = reinterpret_cast<const double2*>(wtri + t);
#if RR_FCG == 2  // A/B: face loads marked L1 evict-first
  double2 q0, q1, q2, q3, q4;
  asm("ld.global.nc.L1::evict_first.v2.f64 {%0, %1}, [%2];" : "=d"(q0.x), "=d"(q0.y) : "l"(p));
  asm("ld.global.nc.L1::evict_first.v2.f64 {%0, %1}, [%2];" : "=d"(q1.x), "=d"(q1.y) : "l"(p + 1));
  asm("ld.global.nc.L1::evict_first.v2.f64 {%0, %1}, [%2];" : "=d"(q2.x), "=d"(q2.y) : "l"(p + 2));
  asm("ld.global.nc.L1::evict_first.v2.f64 {%0, %1}, [%2];" : "=d"(q3.x), "=d"(q3.y) : "l"(p + 3));
  asm("ld.global.nc.L1::evict_first.v2.f64 {%0, %1}, [%2];" : "=d"(q4.x), "=d"(q4.y) : "l"(p + 4));
#elif RR_FCG == 3  // A/B: face loads not allocated in L1
  double2 q0, q1, q2, q3, q4;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(q0.x), "=d"(q0.y) : "l"(p));
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(q1.x), "=d"(q1.y) : "l"(p + 1));
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(q2.x), "=d"(q2.y) : "l"(p + 2));
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(q3.x), "=d"(q3.y) : "l"(p + 3));
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(q4.x), "=d"(q4.y) : "l"(p + 4));
#elif RR_FCG  // A/B: face loads cached in L2 only (L1 left to the nodes)
  const double2 q0 = __ldcg(p), q1 = __ldcg(p + 1), q2 = __ldcg(p + 2), q3 = __ldcg(p + 3), q4 = __ldcg(p + 4);
#else
  const double2 q0 = __ldg(p), q1 = __ldg(p + 1), q2 = __ldg(p + 2), q3 = __ldg(p + 3), q4 = __ldg(p + 4);
#endif
  *face = static_cast<int32_t>(__double_as_longlong(q4.y));
  const D3 va = d3(q0.x, q0.y, q1.x);
  const D3 e1 = d3(q1.y, q2.x, q2.y);
  const D3 e2 = d3(q3.x, q3.y, q4.x);
  const D3 pv = cross(d, e2);
  const double det = dot(e1, pv);
  if (det == 0.0) return -1.0;
  const double inv = 1.0 / det;
  const D3 tv = o - va;
  const double lambda = dot(tv, pv) * inv;
  if (lambda < 0.0 || lambda > 1.0) return -1.0;
  const D3 qv = cross(tv, e1);
  const double mu = dot(d, qv) * inv;
  if (mu < 0.0 || lambda + mu > 1.0) return -1.0;
  const double delta = dot(e2, qv) * inv;
  if (delta <= 1e-6) return -1.0;
  return delta;
}

__device__ __forceinline__ bool test_leaf_w(const FaceTri* __restrict__ wtri, int32_t leaf, D3 o, D3 d,
                                            HitResult& best) {
  const int32_t t0 = leaf_face(leaf);
  const int nfc = leaf_faces(leaf);
  bool better = false;
#pragma unroll 1
  for (int k = 0; k < nfc; ++k) {
    int32_t f;
    const double t = mt_delta_w(wtri, t0 + k, o, d, &f);
    if (t > 0.0 && (best.face < 0 || t < best.delta || (t == best.delta && f < best.face))) {
      best.delta = t;
      best.face = f;
      better = true;
    }
  }
  return better;
}

// One 8-wide node visit (WNode, rr_wide.cu) for one lane's ray: entry
// distances of the 8 slots, the mask of slots hit within tmax and not
// culled, and the slot refs.  A plane of slot k is p + (q - 1) * 2^e; with
// F = 2^23 + q (one byte permute builds its fp32 bits), q - 1 = F - (2^23 +
// 1) exactly (one packed FADD per two slots) and the slab distance is
// fma(q - 1, A, B), A = scale * inv, B = fma(p, inv, -o * inv); the
// builder's margin covers the three roundings.  The per-axis grid scale is
// 2^e (1 + j / 4) (RR_QMANT 2 mantissa bits in a 10-bit field whose shift
// is the fp32 bits; powers of two: C5 17.9 -> 18.0 visits, 434 -> 437 ms).
// (RR_QEXACT 0: fma(F, A, C), C = fl(B - (2^23 + 1) * A), one FADD less per
// two slots but C's rounding of up to half a grid step needs an extra grid
// step on each side of every slot box: 5 % slower on C5.)
struct WVisit {
  float t[8];
  uint32_t hit;      // slots hit
  uint32_t imask;    // internal slots
  int32_t child;     // first internal child
  int32_t tri;       // first leaf face
  uint32_t leafm, pairm;
};

// integer multiply-adds on the FMA pipe (the node visit is heavy on the ALU
// pipe: byte permutes, min / max, selects, compares)
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t imad_hi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// (a0 - b0, a1 - b1), one packed FADD
__device__ __forceinline__ float2 fsub2(float a0, float a1, float b0, float b1) {
  float2 r;
  asm("{\n\t.reg .b64 A, B, D;\n\tmov.b64 A, {%2, %3};\n\tmov.b64 B, {%4, %5};\n\t"
      "sub.rn.f32x2 D, A, B;\n\tmov.b64 {%0, %1}, D;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
  return r;
}
__device__ __forceinline__ float wbyte(uint32_t w, int k) {
  // byte k & 3 of w as the fp32 2^23 + byte.  RR_PIPE & 2: the top byte as
  // hi32(w * 2^8) + 0x4b000000 (one LEA.HI; byte 2 by two IMADs too: slower)
  if ((RR_PIPE & 2) && (k & 3) == 3) return __uint_as_float(imad_hi(w, 256u, 0x4b000000u));
  return __uint_as_float(__byte_perm(w, 0x4b000000u, 0x7440u | static_cast<uint32_t>(k & 3)));
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

__device__ __forceinline__ void visit_w8(const WNode* __restrict__ wn, int32_t node, const RayF& r, bool px, bool py,
                                         bool pz, float tmax, int32_t rplane, WVisit& v) {
  const float4* q = reinterpret_cast<const float4*>(wn + node);
#if RR_NEL  // A/B: node loads marked L1 evict-last (the faces stream through)
  float4 hh;
  int4 mm;
  uint4 qx, qy, qz;
  asm("ld.global.nc.L1::evict_last.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(hh.x), "=f"(hh.y), "=f"(hh.z), "=f"(hh.w) : "l"(q));
  asm("ld.global.nc.L1::evict_last.v4.s32 {%0, %1, %2, %3}, [%4];"
      : "=r"(mm.x), "=r"(mm.y), "=r"(mm.z), "=r"(mm.w) : "l"(q + 1));
  asm("ld.global.nc.L1::evict_last.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(qx.x), "=r"(qx.y), "=r"(qx.z), "=r"(qx.w) : "l"(q + 2));
  asm("ld.global.nc.L1::evict_last.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(qy.x), "=r"(qy.y), "=r"(qy.z), "=r"(qy.w) : "l"(q + 3));
  asm("ld.global.nc.L1::evict_last.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(qz.x), "=r"(qz.y), "=r"(qz.z), "=r"(qz.w) : "l"(q + 4));
#else
  const float4 hh = __ldg(q);
  const int4 mm = __ldg(reinterpret_cast<const int4*>(q + 1));
  const uint4 qx = __ldg(reinterpret_cast<const uint4*>(q + 2));
  const uint4 qy = __ldg(reinterpret_cast<const uint4*>(q + 3));
  const uint4 qz = __ldg(reinterpret_cast<const uint4*>(q + 4));
#endif
  const uint32_t hw = __float_as_uint(hh.w);
  // grid scales: (8 + RR_QMANT)-bit fields = the fp32 bits of 2^(e-127) (1 + j / 2^M)
  constexpr int kF = 8 + RR_QMANT;
  constexpr uint32_t kFM = (1u << kF) - 1u;
  const float ax = __uint_as_float((hw & kFM) << (23 - RR_QMANT)) * r.ix;
  const float ay = __uint_as_float(((hw >> kF) & kFM) << (23 - RR_QMANT)) * r.iy;
  const float az = __uint_as_float(((hw >> (2 * kF)) & kFM) << (23 - RR_QMANT)) * r.iz;
#if RR_QEXACT
  const float cx = __fmaf_rn(hh.x, r.ix, r.nx);
  const float cy = __fmaf_rn(hh.y, r.iy, r.ny);
  const float cz = __fmaf_rn(hh.z, r.iz, r.nz);
#define RR_WFMA2 fma2q
#else
  const float cx = __fmaf_rn(-8388609.0f, ax, __fmaf_rn(hh.x, r.ix, r.nx));
  const float cy = __fmaf_rn(-8388609.0f, ay, __fmaf_rn(hh.y, r.iy, r.ny));
  const float cz = __fmaf_rn(-8388609.0f, az, __fmaf_rn(hh.z, r.iz, r.nz));
#define RR_WFMA2 fma2
#endif
  // near / far plane words per axis from the ray's octant
#if RR_PIPE & 1
  // RR_PIPE & 1: near = lo + b (hi - lo), far = hi - b (hi - lo), b = 1 for
  // a negative direction, as IMADs (FMA pipe) instead of 12 SELs (ALU pipe)
  const uint32_t bx = px ? 0u : 1u, by = py ? 0u : 1u, bz = pz ? 0u : 1u;
  const uint32_t dx0 = imad(qx.x, 0xffffffffu, qx.z), dx1 = imad(qx.y, 0xffffffffu, qx.w);
  const uint32_t dy0 = imad(qy.x, 0xffffffffu, qy.z), dy1 = imad(qy.y, 0xffffffffu, qy.w);
  const uint32_t dz0 = imad(qz.x, 0xffffffffu, qz.z), dz1 = imad(qz.y, 0xffffffffu, qz.w);
  const uint32_t nx0 = imad(bx, dx0, qx.x), nx1 = imad(bx, dx1, qx.y), fx0 = imad(0u - bx, dx0, qx.z),
                 fx1 = imad(0u - bx, dx1, qx.w);
  const uint32_t ny0 = imad(by, dy0, qy.x), ny1 = imad(by, dy1, qy.y), fy0 = imad(0u - by, dy0, qy.z),
                 fy1 = imad(0u - by, dy1, qy.w);
  const uint32_t nz0 = imad(bz, dz0, qz.x), nz1 = imad(bz, dz1, qz.y), fz0 = imad(0u - bz, dz0, qz.z),
                 fz1 = imad(0u - bz, dz1, qz.w);
#else
  const uint32_t nx0 = px ? qx.x : qx.z, nx1 = px ? qx.y : qx.w, fx0 = px ? qx.z : qx.x, fx1 = px ? qx.w : qx.y;
  const uint32_t ny0 = py ? qy.x : qy.z, ny1 = py ? qy.y : qy.w, fy0 = py ? qy.z : qy.x, fy1 = py ? qy.w : qy.y;
  const uint32_t nz0 = pz ? qz.x : qz.z, nz1 = pz ? qz.y : qz.w, fz0 = pz ? qz.z : qz.x, fz1 = pz ? qz.w : qz.y;
#endif
  const uint32_t bits = static_cast<uint32_t>(mm.w);
  const uint32_t cull = mm.z == rplane ? (bits >> 16) & 0xffu : 0u;
  uint32_t hit = 0;
#if RR_FFMA2
  // two slots per packed FFMA2 (fma.rn.f32x2: each lane rounds like FFMA)
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    const uint32_t wnx = k < 4 ? nx0 : nx1, wfx = k < 4 ? fx0 : fx1;
    const uint32_t wny = k < 4 ? ny0 : ny1, wfy = k < 4 ? fy0 : fy1;
    const uint32_t wnz = k < 4 ? nz0 : nz1, wfz = k < 4 ? fz0 : fz1;
    const float2 nx = RR_WFMA2(wbyte(wnx, k), wbyte(wnx, k + 1), ax, cx);
    const float2 ny = RR_WFMA2(wbyte(wny, k), wbyte(wny, k + 1), ay, cy);
    const float2 nz = RR_WFMA2(wbyte(wnz, k), wbyte(wnz, k + 1), az, cz);
    const float2 fx = RR_WFMA2(wbyte(wfx, k), wbyte(wfx, k + 1), ax, cx);
    const float2 fy = RR_WFMA2(wbyte(wfy, k), wbyte(wfy, k + 1), ay, cy);
    const float2 fz = RR_WFMA2(wbyte(wfz, k), wbyte(wfz, k + 1), az, cz);
#if RR_HIT2
    // entry clamped at 0 and exit at tmax (>= 0) inside the 3-input min / max:
    // max(tn, 0) <= min(tf, tmax) is the test below, one compare per slot
    const float tn0 = fmax3(nx.x, ny.x, fmaxf(nz.x, 0.0f)), tf0 = fmin3(fx.x, fy.x, fminf(fz.x, tmax));
    const float tn1 = fmax3(nx.y, ny.y, fmaxf(nz.y, 0.0f)), tf1 = fmin3(fx.y, fy.y, fminf(fz.y, tmax));
    v.t[k] = tn0;
    v.t[k + 1] = tn1;
#if RR_PIPE & 8
    // RR_PIPE & 8: the misses from the sign bits of tf - tn (one packed FADD,
    // sign bit = hi32(bits * 2)) gathered by IMADs, all on the FMA pipe:
    // fl(tf - tn) < 0 exactly when tn > tf (a NaN counts as a hit)
    const float2 dd = fsub2(tf0, tf1, tn0, tn1);
    hit = imad(imad_hi(__float_as_uint(dd.x), 2u, 0u), 1u << k, hit);
    hit = imad(imad_hi(__float_as_uint(dd.y), 2u, 0u), 2u << k, hit);
#else
    hit |= (tn0 <= tf0 ? 1u : 0u) << k;
    hit |= (tn1 <= tf1 ? 2u : 0u) << k;
#endif
#else
    const float tn0 = fmax3(nx.x, ny.x, nz.x), tf0 = fmin3(fx.x, fy.x, fz.x);
    const float tn1 = fmax3(nx.y, ny.y, nz.y), tf1 = fmin3(fx.y, fy.y, fz.y);
    v.t[k] = tn0;
    v.t[k + 1] = tn1;
    if (tn0 <= fminf(tf0, tmax) && tf0 >= 0.0f) hit |= 1u << k;
    if (tn1 <= fminf(tf1, tmax) && tf1 >= 0.0f) hit |= 2u << k;
#endif
  }
#else
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t wnx = k < 4 ? nx0 : nx1, wfx = k < 4 ? fx0 : fx1;
    const uint32_t wny = k < 4 ? ny0 : ny1, wfy = k < 4 ? fy0 : fy1;
    const uint32_t wnz = k < 4 ? nz0 : nz1, wfz = k < 4 ? fz0 : fz1;
    const float q0 = RR_QEXACT ? 8388609.0f : 0.0f;
    const float tn = fmax3(__fmaf_rn(wbyte(wnx, k) - q0, ax, cx), __fmaf_rn(wbyte(wny, k) - q0, ay, cy),
                           __fmaf_rn(wbyte(wnz, k) - q0, az, cz));
    const float tf = fmin3(__fmaf_rn(wbyte(wfx, k) - q0, ax, cx), __fmaf_rn(wbyte(wfy, k) - q0, ay, cy),
                           __fmaf_rn(wbyte(wfz, k) - q0, az, cz));
    v.t[k] = tn;
    if (tn <= fminf(tf, tmax) && tf >= 0.0f) hit |= 1u << k;
  }
#endif
#undef RR_WFMA2
  if (RR_PIPE & 8) hit = ~hit;  // the misses gathered above
  v.hit = hit & bits & 0xffu & ~cull;
  v.imask = bits >> 24;
  v.child = mm.x;
  v.tri = mm.y;
  v.leafm = (bits & 0xffu) & ~v.imask;
  v.pairm = (bits >> 8) & 0xffu;
}

// ref of slot k: internal -> WNode index; leaf -> ~(first face | kPairBit if 2)
__device__ __forceinline__ int32_t wref(const WVisit& v, int k) {
  const uint32_t below = (1u << k) - 1u;
  if ((v.imask >> k) & 1u) return v.child + __popc(v.imask & below);
  const int32_t t = v.tri + __popc(v.leafm & below) + __popc(v.pairm & v.leafm & below);
  return ~(t | (((v.pairm >> k) & 1u) ? kPairBit : 0));
}

}  // namespace rr
