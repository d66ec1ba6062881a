// K3w — cooperative tracer over the 8-wide compressed tree (rr_wide.cu).
//
// Included by rr_trace.cu.  Same contract as trace_kernel (tracer.cpp:19-149:
// step_ray per bounce, receiver captures, reflection, range / iteration
// termination, statistics), with the closest-hit query done by a GROUP of
// 8 lanes per ray, one lane per child slot of the node being visited:
//  * node visit: every lane of the group loads the same 80-B node (one L1
//    request per group) and tests its own slot's quantized box; hit slots
//    are found by a group ballot;
//  * leaf slots that are hit are tested at once, one lane per slot (1-2 fp64
//    Moller-Trumbore tests each), and the group takes the lexicographic
//    (delta, face) minimum by shuffles (accel_tree.cpp:148-153);
//  * internal slots that are hit and not beyond the pruning bound are ranked
//    by entry distance with 7 shuffles; rank 0 is visited next, the others
//    go to the group's stack in shared memory farthest first, written in
//    parallel (one store per lane).
// A warp traces 4 rays, so a bounce waits for the slowest of 4 traversals
// instead of 32, and the per-child box work is spread over the lanes instead
// of looping in one.  Shading (receiver tests, lane r tests receiver r;
// reflection; history) is computed redundantly by the 8 lanes (identical
// values), its stores done by one lane.
#pragma once

namespace rr {

template <int MINB, int STK, bool CNT = false>
__global__ void __launch_bounds__(128, MINB) trace_kernel_g8(const TraceParams p) {
  __shared__ int2 s_stk[16][STK];  // one stack per 8-lane group (16 groups per block)
  const int lane = threadIdx.x & 31;
  const int j = lane & 7;           // slot handled by this lane
  const int gl = lane & ~7;         // group's first lane
  const unsigned gmask = 0xffu << gl;
  int2* stk = s_stk[threadIdx.x >> 3];
  const uint32_t bsel = 0x7440u | static_cast<uint32_t>(j & 3);  // byte j&3 -> fp32 2^23 + b
  const uint32_t below = (1u << j) - 1u;
  const float kInf = __int_as_float(0x7f800000);

  int64_t ray = -1;
  bool exhausted = false;
  D3 o{}, d{};
  double path = 0.0;
  int32_t steps = 0, bounces = 0, rplane = -2;
  uint32_t st_bounce = 0, st_esc = 0, st_oor = 0, st_alive = 0;
  unsigned long long st_cnt[2] = {0, 0};
  int32_t st_max = 0;

  for (;;) {
    // ---- new rays for the groups that need one (their first lanes ask)
    const bool need = j == 0 && ray < 0 && !exhausted;
    const unsigned m = __ballot_sync(0xffffffffu, need);
    if (m) {
      const int leader = __ffs(m) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(p.ray_counter, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, leader);
      const long long c = static_cast<long long>(base) + __popc(m & ((1u << lane) - 1u));
      const long long cg = __shfl_sync(0xffffffffu, c, gl);
      const bool gneed = (m >> gl) & 1u;
      if (gneed) {
        if (cg < p.count) {
          const int64_t i = p.order ? static_cast<int64_t>(__ldg(p.order + cg)) : cg;
          ray = i;
          o = d3(p.src[0], p.src[1], p.src[2]);
          d = p.dirs ? d3(p.dirs[3 * i], p.dirs[3 * i + 1], p.dirs[3 * i + 2])
                     : fib_dir(global_ray(p, i), p.N, p.az_step);
          path = 0.0;
          steps = 0;
          bounces = 0;
          rplane = -2;
          if (p.max_iter <= 0) {  // trace() with a zero cap: nothing runs
            if (j == 0) st_alive++;
            ray = -1;
          }
        } else {
          exhausted = true;
        }
      }
    }
    if (__all_sync(0xffffffffu, ray < 0)) {
      if (__all_sync(0xffffffffu, exhausted)) break;
      continue;
    }
    if (ray < 0) continue;

    // ---- one step_ray (tracer.cpp:19-62): closest hit by the group
    ++steps;
    double bdelta = 0.0;
    int32_t bface = -1;
    RayF r;
    int32_t node = kDone;
    float tbest = FLT_MAX;
    if (make_rayf(p.hdr, o, d, r)) {
      const float t0 = box_enter(r, p.hdr.lo[0], p.hdr.hi[0], p.hdr.lo[1], p.hdr.hi[1], p.hdr.lo[2], p.hdr.hi[2],
                                 tbest);
      node = t0 == kInf ? kDone : 0;
    }
    const bool px = r.ix >= 0.0f, py = r.iy >= 0.0f, pz = r.iz >= 0.0f;
    int sp = 0;
    while (node != kDone) {  // uniform within the group
      if (CNT && j == 0) ++st_cnt[0];
      const float4* q = reinterpret_cast<const float4*>(p.wnodes + node);
      const float4 hh = __ldg(q);
      const int4 mm = __ldg(reinterpret_cast<const int4*>(q + 1));
      const uint4 qx = __ldg(reinterpret_cast<const uint4*>(q + 2));
      const uint4 qy = __ldg(reinterpret_cast<const uint4*>(q + 3));
      const uint4 qz = __ldg(reinterpret_cast<const uint4*>(q + 4));
      const uint32_t hw = __float_as_uint(hh.w);
      const uint32_t bits = static_cast<uint32_t>(mm.w);
      // this lane's slot: near / far plane bytes by the ray's octant
      const uint32_t lx = j < 4 ? qx.x : qx.y, ux = j < 4 ? qx.z : qx.w;
      const uint32_t ly = j < 4 ? qy.x : qy.y, uy = j < 4 ? qy.z : qy.w;
      const uint32_t lz = j < 4 ? qz.x : qz.y, uz = j < 4 ? qz.z : qz.w;
      const float fl_x = __uint_as_float(__byte_perm(lx, 0x4b000000u, bsel)) - 8388608.0f;
      const float fu_x = __uint_as_float(__byte_perm(ux, 0x4b000000u, bsel)) - 8388608.0f;
      const float fl_y = __uint_as_float(__byte_perm(ly, 0x4b000000u, bsel)) - 8388608.0f;
      const float fu_y = __uint_as_float(__byte_perm(uy, 0x4b000000u, bsel)) - 8388608.0f;
      const float fl_z = __uint_as_float(__byte_perm(lz, 0x4b000000u, bsel)) - 8388608.0f;
      const float fu_z = __uint_as_float(__byte_perm(uz, 0x4b000000u, bsel)) - 8388608.0f;
      const float ax = __uint_as_float((hw & 0xffu) << 23) * r.ix;
      const float ay = __uint_as_float(((hw >> 8) & 0xffu) << 23) * r.iy;
      const float az = __uint_as_float(((hw >> 16) & 0xffu) << 23) * r.iz;
      const float bx = __fmaf_rn(hh.x, r.ix, r.nx), by = __fmaf_rn(hh.y, r.iy, r.ny), bz = __fmaf_rn(hh.z, r.iz, r.nz);
      const float tnx = __fmaf_rn(px ? fl_x : fu_x, ax, bx), tfx = __fmaf_rn(px ? fu_x : fl_x, ax, bx);
      const float tny = __fmaf_rn(py ? fl_y : fu_y, ay, by), tfy = __fmaf_rn(py ? fu_y : fl_y, ay, by);
      const float tnz = __fmaf_rn(pz ? fl_z : fu_z, az, bz), tfz = __fmaf_rn(pz ? fu_z : fl_z, az, bz);
      const float tn = fmaxf(fmaxf(tnx, tny), fmaxf(tnz, 0.0f));
      const float tf = fminf(fminf(tfx, tfy), fminf(tfz, tbest));
      const bool culled = mm.z == rplane && ((bits >> (16 + j)) & 1u);
      const bool hit = ((bits >> j) & 1u) && !culled && tn <= tf;
      const uint32_t hm = (__ballot_sync(gmask, hit) >> gl) & 0xffu;
      const uint32_t imask = hw >> 24;
      const uint32_t lh = hm & ~imask;
      if (lh) {
        // leaf slots: test their faces now, one lane per slot
        double ld = 0.0;
        int32_t lf = -1;
        if ((lh >> j) & 1u) {
          const uint32_t leafm = (bits & 0xffu) & ~imask, pairm = (bits >> 8) & 0xffu;
          const int32_t t0 = mm.y + __popc(leafm & below) + __popc(pairm & leafm & below);
          const int nfc = ((pairm >> j) & 1u) ? 2 : 1;
          if (CNT) st_cnt[1] += nfc;
#pragma unroll 1
          for (int k = 0; k < nfc; ++k) {
            int32_t f;
            const double t = mt_delta_w(p.wtri, t0 + k, o, d, &f);
            if (t > 0.0 && (lf < 0 || t < ld || (t == ld && f < lf))) {
              ld = t;
              lf = f;
            }
          }
        }
        // group lexicographic minimum of (delta, face), then into the best
#pragma unroll
        for (int off = 4; off > 0; off >>= 1) {
          const double od = __shfl_xor_sync(gmask, ld, off, 8);
          const int32_t of = __shfl_xor_sync(gmask, lf, off, 8);
          if (of >= 0 && (lf < 0 || od < ld || (od == ld && of < lf))) {
            ld = od;
            lf = of;
          }
        }
        if (lf >= 0 && (bface < 0 || ld < bdelta || (ld == bdelta && lf < bface))) {
          bdelta = ld;
          bface = lf;
          tbest = prune_bound(bdelta, r.shift);
        }
      }
      // internal slots within the bound: nearest next, the rest pushed
      const bool mine = ((hm & imask) >> j) & 1u && tn <= tbest;
      const uint32_t im = (__ballot_sync(gmask, mine) >> gl) & 0xffu;
      if (im) {
        int rank = 0;
#pragma unroll
        for (int s = 1; s < 8; ++s) {
          const int oj = (j + s) & 7;
          const float to = __shfl_sync(gmask, tn, oj, 8);
          if ((im >> oj) & 1u) rank += (to < tn || (to == tn && oj < j)) ? 1 : 0;
        }
        const int32_t child = mm.x + __popc(imask & below);
        const int h = __popc(im);
        if (mine && rank > 0) stk[sp + h - 1 - rank] = make_int2(child, __float_as_int(tn));
        const uint32_t r0 = (__ballot_sync(gmask, mine && rank == 0) >> gl) & 0xffu;
        node = __shfl_sync(gmask, child, __ffs(r0) - 1, 8);
        sp += h - 1;
        __syncwarp(gmask);
      } else {
        node = kDone;
        while (sp > 0) {
          --sp;
          const int2 e = stk[sp];
          if (__int_as_float(e.y) <= tbest) {
            node = e.x;
            break;
          }
        }
      }
    }

    // ---- receivers: lane r tests receiver r (a receiver never alters a ray)
    const bool has_wall = bface >= 0;
    if (j < p.n_recv) {
      const double sd = sphere_delta(o, d, d3(p.rc[j][0], p.rc[j][1], p.rc[j][2]), p.rr[j]);
      bool cap = sd > 0.0 && (!has_wall || sd < bdelta);
      double L = 0.0;
      if (cap) {
        L = path + sd;
        cap = L <= p.rng[j];  // resolved_max_range of receiver j
      }
      const unsigned act = __activemask();
      const unsigned cm = __ballot_sync(act, cap);
      if (cm) {
        const int leader = __ffs(cm) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(p.cap_count, (unsigned long long)__popc(cm));
        base = __shfl_sync(act, base, leader);
        if (cap) {
          const unsigned long long slot = base + __popc(cm & ((1u << lane) - 1u));
          if (slot < static_cast<unsigned long long>(p.cap_capacity)) {
            Capture c;
            const D3 pt = o + sd * d;
            c.p[0] = pt.x; c.p[1] = pt.y; c.p[2] = pt.z;
            c.d[0] = d.x; c.d[1] = d.y; c.d[2] = d.z;
            c.path = L;
            c.ray = static_cast<int32_t>(ray);
            c.meta = (bounces << 8) | j;
            p.caps[slot] = c;
          }
        }
      }
    }
    __syncwarp(gmask);
    bool dead = false;
    if (!has_wall) {
      dead = true;
      if (j == 0) st_esc++;
    } else {
      const double* nn = p.normal + 3 * static_cast<int64_t>(bface);
      D3 n = d3(__ldg(nn), __ldg(nn + 1), __ldg(nn + 2));
      if (dot(n, d) > 0.0) n = d3(-n.x, -n.y, -n.z);
      const D3 pt = o + bdelta * d;
      const double s2 = 2.0 * dot(d, n);
      d = d - s2 * n;  // reflect, tracer.hpp:33-37
      o = pt;
      const int32_t pid = __ldg(p.face_plane + bface);
      if (pid >= 0) {
        const int k = pid >> 29;
        const double dk = k == 0 ? d.x : (k == 1 ? d.y : d.z);
        rplane = fabs(dk) > p.cull_min ? pid : -2;
      } else {
        rplane = -2;
      }
      path += bdelta;
      if (j == 0) p.hist[ray * p.H + bounces] = bface;
      ++bounces;
      if (path > p.max_range) {
        dead = true;
        if (j == 0) st_oor++;
      }
    }
    if (!dead && steps >= p.max_iter) {
      dead = true;
      if (j == 0) st_alive++;
    }
    if (dead) {
      if (j == 0) {
        st_bounce += steps;
        st_max = max(st_max, steps);
      }
      ray = -1;
    }
  }
  // ---- statistics
  for (int off = 16; off > 0; off >>= 1) {
    st_bounce += __shfl_xor_sync(0xffffffffu, st_bounce, off);
    st_esc += __shfl_xor_sync(0xffffffffu, st_esc, off);
    st_oor += __shfl_xor_sync(0xffffffffu, st_oor, off);
    st_alive += __shfl_xor_sync(0xffffffffu, st_alive, off);
    st_max = max(st_max, __shfl_xor_sync(0xffffffffu, st_max, off));
  }
  if (lane == 0) {
    atomicAdd(p.stats + 0, (unsigned long long)st_bounce);
    atomicAdd(p.stats + 1, (unsigned long long)st_esc);
    atomicAdd(p.stats + 2, (unsigned long long)st_oor);
    atomicAdd(p.stats + 3, (unsigned long long)st_alive);
    atomicMax(p.stats + 4, (unsigned long long)st_max);
  }
  if (CNT) {
    for (int off = 16; off > 0; off >>= 1) {
      st_cnt[0] += __shfl_xor_sync(0xffffffffu, st_cnt[0], off);
      st_cnt[1] += __shfl_xor_sync(0xffffffffu, st_cnt[1], off);
    }
    if (lane == 0) {
      atomicAdd(p.stats + 5, st_cnt[0]);
      atomicAdd(p.stats + 6, st_cnt[1]);
    }
  }
}

}  // namespace rr
