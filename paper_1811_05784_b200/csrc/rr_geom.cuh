// Device geometry shared by the tracer kernels.
//
// fp64 parts restate the reference operation order exactly; the library is
// compiled with -fmad=false so no FMA is contracted into them (the oracle is
// compiled for baseline x86-64 with -ffp-contract=off).  The fp32 box test is
// a conservative filter only: node boxes are rounded outward and expanded by
// eps = scale * 2^-20, which dominates the fp32 origin/slab rounding error,
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
constexpr int kStack = 32;

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
  double shift;  // the fp32 origin sits at o + shift*d (shift > 0 only for far origins)
};

__device__ __forceinline__ float inv_dir(double dk) {
  float f = __double2float_rn(dk);
  float a = fabsf(f);
  if (a < 1e-30f) f = copysignf(1e-30f, dk);
  return 1.0f / f;
}

// Origins farther than 4*scale from 0 are moved (in fp64) to the root box
// entry so that fp32 rounding of the origin stays below eps.
__device__ __forceinline__ bool make_rayf(const TravHeader& h, D3 o, D3 d, RayF& r) {
  const double scale = static_cast<double>(h.eps) * 0x1p20;
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
  const float x0 = (lx - r.ox) * r.ix, x1 = (hx - r.ox) * r.ix;
  const float y0 = (ly - r.oy) * r.iy, y1 = (hy - r.oy) * r.iy;
  const float z0 = (lz - r.oz) * r.iz, z1 = (hz - r.oz) * r.iz;
  const float tn = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fmaxf(fminf(z0, z1), 0.0f));
  const float tf = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fminf(fmaxf(z0, z1), tmax));
  return tn <= tf ? tn : __int_as_float(0x7f800000);
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

__device__ __forceinline__ HitResult closest_hit(const TravHeader& h, const TNode* __restrict__ nodes,
                                                 const TNode* smem, int32_t K, const FaceTri* __restrict__ tri,
                                                 D3 o, D3 d, int32_t* n_visit = nullptr) {
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
      const float tl = box_enter(r, nd.a.x, nd.a.y, nd.a.z, nd.a.w, nd.b.x, nd.b.y, tbest);
      const float tr = box_enter(r, nd.b.z, nd.b.w, nd.c.x, nd.c.y, nd.c.z, nd.c.w, tbest);
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
      const int32_t f = ~node;
      const double t = mt_delta(tri, f, o, d);
      if (t > 0.0 && (best.face < 0 || t < best.delta || (t == best.delta && f < best.face))) {
        best.delta = t;
        best.face = f;
        tbest = prune_bound(t, r.shift);
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
  if (n_visit) *n_visit = visits;
  return best;
}

}  // namespace rr
