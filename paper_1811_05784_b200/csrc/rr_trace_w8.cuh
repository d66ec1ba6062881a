// K3w — the tracer over the 8-wide compressed tree (rr_wide.cu), for deep
// scenes (default from 2^18 faces: C3, C5).  Included by rr_trace.cu.
//
// Same contract as trace_kernel (tracer.cpp:19-149: step_ray per bounce,
// receiver captures, reflection, range / iteration termination, statistics),
// restructured so that lanes do not idle behind the slowest traversal of
// their warp:
//  * every lane owns one ray and keeps its traversal state (node, stack,
//    stashed leaf, best hit) across loop iterations;
//  * traversal phase: lanes still searching visit up to UNR 8-wide nodes
//    (visit_w8: 8 quantized slab tests; hit slots pushed farthest first, the
//    nearest continued), reached leaves are stashed and tested in warp-voted
//    batches (as in closest_hit_pl), until at least DONET lanes of the warp
//    have finished their closest-hit query (or none is searching);
//  * shading phase: the finished lanes together do the receiver tests and
//    the warp-aggregated capture append, reflect, write the face history,
//    terminate, take new rays from the global counter and start their next
//    query.
// Leaves are tested (one batch, all stashed faces spread over the warp,
// RR_COOP) once a quarter of the searching lanes are stuck behind their
// stashed leaf (STUCKD 4; HOLDD 1: or all of them hold one).
// Without the batching a warp's bounce lasts as long as its slowest lane's
// query: on C5 (17 node visits per ray-bounce on average) only ~7 of 32
// lanes were active per node visit.
#pragma once

namespace rr {

// 8-bit mask permutation by index xor: bit j of the result = bit (j ^ o) of m
__device__ __forceinline__ uint32_t xperm8(uint32_t m, uint32_t o) {
  if (o & 1u) m = ((m & 0x55u) << 1) | ((m >> 1) & 0x55u);
  if (o & 2u) m = ((m & 0x33u) << 2) | ((m >> 2) & 0x33u);
  if (o & 4u) m = ((m & 0x0fu) << 4) | ((m >> 4) & 0x0fu);
  return m;
}

// start fetching the faces of a leaf stashed for the next batched test
__device__ __forceinline__ void prefetch_leaf(const FaceTri* wtri, int32_t leaf) {
  if (RR_PF8 == 0) return;
  const char* a = reinterpret_cast<const char*>(wtri + leaf_face(leaf));
  const char* b = a + leaf_faces(leaf) * sizeof(FaceTri) - 1;
  if (RR_PF8 == 1) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(b));
  } else {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(b));
  }
}

// GRP: group traversal.  The stack holds one entry per visited node with
// more than one hit slot -- the node and the mask of its remaining hit slots
// -- instead of one entry per pushed child: the visit continues into the
// nearest hit slot (GNEAR; exact entry distance) and the rest are taken later
// in the ray octant's slot order (slot j ^ octant for j = 0..7; the builder
// places the children by direction, rr_wide.cu expand_kernel), with no sort,
// no per-child pushes and no distances on the stack.  C5: 547 -> 527 ms with
// 20.5 instead of 18.2 node visits per ray-bounce (popped children are not
// culled by their entry distance; carrying a group bound -- the exact minimum
// of the rest, 535 ms, or the nearest slot's distance, 535 ms -- cut visits
// less than it cost).  The stack bound is the tree depth.
template <int MINB, int DONET, int UNR, int STK, bool CNT = false, int SMS = 0, int STUCKD = 2, int HOLDD = 2,
          bool GRP = false, bool GNEAR = true>
__global__ void __launch_bounds__(128, MINB) trace_kernel_w8(const TraceParams p) {
  // the SMS oldest stack entries of each lane in shared memory (column tid:
  // lane i always in bank i, conflict-free), deeper ones in local memory
  __shared__ int2 s_st[SMS > 0 ? SMS * 128 : 1];
  int2* sst = s_st + threadIdx.x;
#if RR_GST
  // group entries: (first child, first face) in s_st / st, the node's slot
  // bits with the remaining-slot mask in bits 16-23 here
  __shared__ uint32_t s_st2[SMS > 0 ? SMS * 128 : 1];
  uint32_t* sst2 = s_st2 + threadIdx.x;
#endif
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const float kInf = __int_as_float(0x7f800000);
  // the fp64 ray state (origin, direction, best hit so far, path length, ray
  // index, step and bounce counts) lives in shared memory: the node visits,
  // the bulk of the work, need only the fp32 slab data in registers; the
  // leaf tests and the shading read it from shared memory.  Each register
  // moved out of the 64-register budget of 8 blocks per SM removed spill
  // traffic (C5: statistics 645 -> 628 ms, path / counters 610, origin /
  // direction / best hit 587; 9 or 10 blocks per SM spill more, 592 / 620).
  struct LaneState {
    D3 o, d;
    HitResult best;
    double path;
    int32_t ray, steps, bounces, pad;
  };
  __shared__ LaneState s_lane[128];
#if RR_RSM
  // the fp32 slab terms of the lane's ray (inv, -o * inv), column tid: read
  // at every node visit from shared memory instead of spill slots (local
  // memory, 22 % L1 hit rate under the node / face streams)
  __shared__ float s_ray[6 * 128];
  float* sry = s_ray + threadIdx.x;
#endif
#if RR_COOP
  __shared__ uint8_t s_item[128];  // per warp: lane (| 32 for a second face) of each stashed face
#endif
  LaneState& ls = s_lane[threadIdx.x];
#if RR_HBUF
  // face history: each lane's current 32-B sector of hist[] in shared memory
  // (column tid), written out as two 16-B stores when the sector fills and
  // lies inside the ray's own history, else word by word (the ray's first
  // and last sectors).  One 4-B store per bounce made every bounce a partial
  // sector in L2; with the L2 streaming triangles most were evicted before
  // the next bounce filled them (C5: 31.7 GB of DRAM writes per trace for a
  // 3.2 GB history).
  __shared__ int32_t s_hist[8 * 128];
  int32_t* shb = s_hist + threadIdx.x;
  auto hist_words = [&](int64_t from, int64_t to) {  // hist[from..to] from the sector buffer
    for (int64_t j = from; j <= to; ++j) p.hist[j] = shb[(j & 7) * 128];
  };
#endif
  D3& o = ls.o;
  D3& d = ls.d;
  HitResult& best = ls.best;
  bool has_ray = false;
  bool exhausted = false;
  int32_t rplane = -2;
  // traversal of the current step
  bool searching = false;  // a closest-hit query is in progress
  RayF r{};
  bool px = true, py = true, pz = true;
  float tbest = FLT_MAX;
  int32_t node = kDone, leaf = 0;
  int2 st[STK > SMS ? STK - SMS : 1];
#if RR_GST
  uint32_t st2[STK > SMS ? STK - SMS : 1];
#endif
  int sp = 0;
  int2 top[2] = {};
  int n_top = 0;
  // GRP: the current node group (node, its remaining hit slots by order
  // position, its child / face bases and slot masks) and the ray octant
  // (bit a: negative direction along axis a)
  int32_t g_node = 0, g_child = 0, g_tri = 0;
  uint32_t g_mask = 0, g_bits = 0, oct = 0;
  auto gperm = [&](uint32_t m) -> uint32_t { return xperm8(m, oct); };  // slot bits -> order-position bits
  auto gslot = [&](int j) -> int { return j ^ static_cast<int>(oct); };

  // termination statistics in shared memory (updated once per ray, rare),
  // which keeps five counters out of the register budget
  __shared__ unsigned long long s_stat[5];  // bounces, escaped, out of range, alive, max steps
  if (threadIdx.x < 5) s_stat[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long st_cnt[3] = {0, 0, 0};  // node visits, face tests, visits hitting no slot

  auto st_put = [&](int i, int2 e) {
    RR_DCHECK(i < STK);
    if (SMS > 0 && (SMS >= STK || i < SMS)) sst[i * 128] = e;
    else st[i - SMS] = e;
  };
  auto st_get = [&](int i) -> int2 { return (SMS > 0 && (SMS >= STK || i < SMS)) ? sst[i * 128] : st[i - SMS]; };
#if RR_GST
  auto st_put2 = [&](int i, uint32_t b) {
    if (SMS > 0 && (SMS >= STK || i < SMS)) sst2[i * 128] = b;
    else st2[i - SMS] = b;
  };
  auto st_get2 = [&](int i) -> uint32_t { return (SMS > 0 && (SMS >= STK || i < SMS)) ? sst2[i * 128] : st2[i - SMS]; };
#endif
  auto push = [&](int2 e) {
    if (n_top == 2) st_put(sp++, top[1]);
    top[1] = top[0];
    top[0] = e;
    n_top = min(n_top + 1, 2);
  };
  auto pop = [&]() {
    node = kDone;
    while (n_top > 0) {
      const int2 e = top[0];
      top[0] = top[1];
      --n_top;
      if (__int_as_float(e.y) <= tbest) {
        node = e.x;
        return;
      }
    }
    while (sp > 0) {
      --sp;
      const int2 e = st_get(sp);
      if (__int_as_float(e.y) <= tbest) {
        node = e.x;
        break;
      }
    }
  };
  // GRP: ref of slot k of the current group's node (wref from its header)
  auto gref = [&](int k) -> int32_t {
    const uint32_t below = (1u << k) - 1u;
    const uint32_t im = g_bits >> 24;
    if ((im >> k) & 1u) return g_child + __popc(im & below);
    const uint32_t lm = g_bits & 0xffu & ~im, pm = (g_bits >> 8) & lm;
    const int32_t t = g_tri + __popc(lm & below) + __popc(pm & below);
    return ~(t | (((pm >> k) & 1u) ? kPairBit : 0));
  };
  // GRP: next node from the current group, else from the stack's groups
  auto gtake = [&]() {
    if (g_mask == 0) {
      if (sp == 0) {
        node = kDone;
        return;
      }
#if RR_GST
      --sp;
      const int2 e = st_get(sp);
      g_child = e.x;
      g_tri = e.y;
      g_bits = st_get2(sp);
      g_mask = (g_bits >> 16) & 0xffu;
#else
      const int2 e = st_get(--sp);
      g_node = e.x;
      g_mask = static_cast<uint32_t>(e.y);
      const int4 mm = __ldg(reinterpret_cast<const int4*>(p.wnodes + g_node) + 1);
      g_child = mm.x;
      g_tri = mm.y;
      g_bits = static_cast<uint32_t>(mm.w);
#endif
    }
    const int j = __ffs(g_mask) - 1;
    g_mask &= g_mask - 1u;
    node = gref(gslot(j));
  };
  // start the closest-hit query of the next step_ray
  auto begin_query = [&]() {
    ++ls.steps;
    best = HitResult{0.0, -1};
    tbest = FLT_MAX;
    sp = 0;
    n_top = 0;
    leaf = 0;
    node = kDone;
    if (make_rayf(p.hdr, o, d, r)) {
      const float t0 = box_enter(r, p.hdr.lo[0], p.hdr.hi[0], p.hdr.lo[1], p.hdr.hi[1], p.hdr.lo[2], p.hdr.hi[2],
                                 tbest);
      node = t0 == kInf ? kDone : 0;
    }
#if RR_RSM
    sry[0] = r.ix;
    sry[128] = r.iy;
    sry[256] = r.iz;
    sry[384] = r.nx;
    sry[512] = r.ny;
    sry[640] = r.nz;
#endif
    px = r.ix >= 0.0f;
    py = r.iy >= 0.0f;
    pz = r.iz >= 0.0f;
    oct = (px ? 0u : 1u) | (py ? 0u : 2u) | (pz ? 0u : 4u);
    g_mask = 0;
    searching = true;
  };

  for (;;) {
    // ---------------- shading: rays whose query finished, and new rays
    const bool shade = has_ray && !searching;
    if (shade) {
      const bool has_wall = best.face >= 0;
      for (int rc = 0; rc < p.n_recv; ++rc) {
        const double sd = sphere_delta(o, d, d3(p.rc[rc][0], p.rc[rc][1], p.rc[rc][2]), p.rr[rc]);
        bool cap = sd > 0.0 && (!has_wall || sd < best.delta);
        double L = 0.0;
        if (cap) {
          L = ls.path + sd;
          cap = L <= p.rng[rc];  // resolved_max_range of receiver rc
        }
        const unsigned act = __activemask();
        const unsigned cm = __ballot_sync(act, cap);
        if (cm) {
          const int leader = __ffs(cm) - 1;
          unsigned long long base = 0;
          if (lane == leader) base = atomicAdd(p.cap_count, (unsigned long long)__popc(cm));
          base = __shfl_sync(act, base, leader);
          if (cap) {
            const unsigned long long slot = base + __popc(cm & lt_mask);
            if (slot < static_cast<unsigned long long>(p.cap_capacity)) {
              Capture c;
              const D3 pt = o + sd * d;
              c.p[0] = pt.x; c.p[1] = pt.y; c.p[2] = pt.z;
              c.d[0] = d.x; c.d[1] = d.y; c.d[2] = d.z;
              c.path = L;
              c.ray = ls.ray;
              c.meta = (ls.bounces << 8) | rc;
              p.caps[slot] = c;
            }
          }
        }
      }
      bool dead = false;
      if (!has_wall) {
        dead = true;
        atomicAdd(s_stat + 1, 1ull);
      } else {
        const double* nn = p.normal + 3 * static_cast<int64_t>(best.face);
        D3 n = d3(__ldg(nn), __ldg(nn + 1), __ldg(nn + 2));
        if (dot(n, d) > 0.0) n = d3(-n.x, -n.y, -n.z);
        const D3 pt = o + best.delta * d;
        const double s2 = 2.0 * dot(d, n);
        d = d - s2 * n;  // reflect, tracer.hpp:33-37
        o = pt;
        // the next segment leaves this face's plane: cull coplanar subtrees
        // (p.cull_min: see run_trace)
        const int32_t pid = __ldg(p.face_plane + best.face);
        if (pid >= 0) {
          const int k = pid >> 29;
          const double dk = k == 0 ? d.x : (k == 1 ? d.y : d.z);
          rplane = fabs(dk) > p.cull_min ? pid : -2;
        } else {
          rplane = -2;
        }
        ls.path += best.delta;
        RR_DCHECK(ls.ray < p.count && ls.bounces < p.H && best.face < p.nf);
        const int64_t g = static_cast<int64_t>(ls.ray) * p.H + ls.bounces;
#if RR_HBUF
        shb[(g & 7) * 128] = best.face;
        if ((g & 7) == 7) {
          const int64_t g0 = static_cast<int64_t>(ls.ray) * p.H;
          if (g - 7 >= g0) {
            int4* dst = reinterpret_cast<int4*>(p.hist + (g - 7));
            dst[0] = make_int4(shb[0], shb[128], shb[256], shb[384]);
            dst[1] = make_int4(shb[512], shb[640], shb[768], shb[896]);
          } else {
            hist_words(g0, g);
          }
        }
#elif RR_HCS
        __stcs(p.hist + g, best.face);
#else
        p.hist[g] = best.face;
#endif
        ++ls.bounces;
        if (ls.path > p.max_range) {
          dead = true;
          atomicAdd(s_stat + 2, 1ull);
        }
      }
      if (!dead && ls.steps >= p.max_iter) {
        dead = true;
        atomicAdd(s_stat + 3, 1ull);
      }
      if (dead) {
#if RR_HBUF
        if (ls.bounces > 0) {  // the ray's last, partial sector
          const int64_t g0 = static_cast<int64_t>(ls.ray) * p.H, gl = g0 + ls.bounces - 1;
          if ((gl & 7) != 7) hist_words(max(g0, gl & ~static_cast<int64_t>(7)), gl);
        }
#endif
        atomicAdd(s_stat + 0, static_cast<unsigned long long>(ls.steps));
        atomicMax(s_stat + 4, static_cast<unsigned long long>(ls.steps));
        has_ray = false;
      } else {
        begin_query();
      }
    }
    // new rays (warp-aggregated fetch from the global counter)
    const bool need = !has_ray && !exhausted;
    const unsigned m = __ballot_sync(0xffffffffu, need);
    if (m) {
      const int leader = __ffs(m) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(p.ray_counter, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (need) {
        const int64_t c = static_cast<int64_t>(base) + __popc(m & lt_mask);
        if (c < p.count) {
          const int64_t i = p.order ? static_cast<int64_t>(__ldg(p.order + c)) : c;
          has_ray = true;
          ls.ray = static_cast<int32_t>(i);
          o = d3(p.src[0], p.src[1], p.src[2]);
          d = p.dirs ? d3(p.dirs[3 * i], p.dirs[3 * i + 1], p.dirs[3 * i + 2])
                     : fib_dir(global_ray(p, i), p.N, p.az_step);
          ls.path = 0.0;
          ls.steps = 0;
          ls.bounces = 0;
          rplane = -2;
          if (p.max_iter <= 0) {  // trace() with a zero cap: nothing runs
            atomicAdd(s_stat + 3, 1ull);
            has_ray = false;
          } else {
            begin_query();
          }
        } else {
          exhausted = true;
        }
      }
    }
    if (__all_sync(0xffffffffu, !has_ray && exhausted)) break;

    // ---------------- traversal until DONET lanes wait for shading
    for (;;) {
      if (searching) {
#pragma unroll 1
        for (int u = 0; u < UNR && is_inner(node) && (u == 0 || leaf == 0); ++u) {
          if (CNT) ++st_cnt[0];
          WVisit v;
          RR_DCHECK(node < p.n_wnodes);
#if RR_OCT  // the octant flags from the one octant word (fewer live registers)
#if RR_RSM
          RayF rs;
          rs.ix = sry[0];
          rs.iy = sry[128];
          rs.iz = sry[256];
          rs.nx = sry[384];
          rs.ny = sry[512];
          rs.nz = sry[640];
          visit_w8(p.wnodes, node, rs, (oct & 1u) == 0u, (oct & 2u) == 0u, (oct & 4u) == 0u, tbest, rplane, v);
#else
          visit_w8(p.wnodes, node, r, (oct & 1u) == 0u, (oct & 2u) == 0u, (oct & 4u) == 0u, tbest, rplane, v);
#endif
#else
          visit_w8(p.wnodes, node, r, px, py, pz, tbest, rplane, v);
#endif
          const uint32_t hm = v.hit;
          if (CNT && hm == 0) ++st_cnt[2];
          if constexpr (GRP) {
            if (hm == 0) {
              gtake();
            } else {
              int k;
              uint32_t pm;
              if constexpr (GNEAR) {  // the nearest hit slot first (exact entry distance), the rest in octant order
                uint32_t mn = 0xffffffffu;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                  mn = min(mn, ((hm >> q) & 1u) ? ((__float_as_uint(RR_HIT2 ? v.t[q] : fmaxf(v.t[q], 0.0f)) & ~7u) | q)
                                                : 0xffffffffu);
                k = static_cast<int>(mn & 7u);
                pm = gperm(hm & ~(1u << k));
              } else {
                pm = gperm(hm);
                k = gslot(__ffs(pm) - 1);
                pm &= pm - 1u;
              }
              const int32_t next = wref(v, k);
              if (pm) {  // the node's other hit slots become the current group
#if RR_GST
                if (g_mask != 0) {
                  st_put2(sp, (g_bits & 0xff00ffffu) | (g_mask << 16));
                  st_put(sp++, make_int2(g_child, g_tri));
                }
#else
                if (g_mask != 0) st_put(sp++, make_int2(g_node, static_cast<int>(g_mask)));
#endif
                g_node = node;
                g_mask = pm;
                g_child = v.child;
                g_tri = v.tri;
                g_bits = (v.imask << 24) | (v.pairm << 8) | v.leafm | v.imask;
              }
              node = next;
            }
          } else if (hm == 0) {
            pop();
          } else {
            // continue into the nearest hit slot; push the others farthest
            // first.  Sort keys pack the entry distance (clamped at 0, low 3
            // mantissa bits replaced by the slot, top bit set so no hit key
            // is 0) into one u32: t >= 0 orders like its bits, so min / max
            // are integer min / max; a pushed entry keeps t rounded down by
            // < 8 ulps (pruning stays conservative).
            uint32_t key[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
              key[k] = ((hm >> k) & 1u) ? (0x80000000u | (__float_as_uint(fmaxf(v.t[k], 0.0f)) & ~7u) | k) : 0u;
            uint32_t mn = 0xffffffffu;
#pragma unroll
            for (int k = 0; k < 8; ++k) mn = min(mn, key[k] ? key[k] : 0xffffffffu);
            const int kmn = static_cast<int>(mn & 7u);
            if (hm & (hm - 1u)) {
#pragma unroll
              for (int k = 0; k < 8; ++k) key[k] = k == kmn ? 0u : key[k];
              for (;;) {
                uint32_t mx = 0;
#pragma unroll
                for (int k = 0; k < 8; ++k) mx = max(mx, key[k]);
                if (mx == 0) break;
                const int kmx = static_cast<int>(mx & 7u);
                push(make_int2(wref(v, kmx), static_cast<int>(mx & 0x7ffffff8u)));
#pragma unroll
                for (int k = 0; k < 8; ++k) key[k] = k == kmx ? 0u : key[k];
              }
            }
            node = wref(v, kmn);
          }
          if (node < 0 && leaf == 0) {  // stash a reached leaf and keep traversing
            leaf = node;
            prefetch_leaf(p.wtri, leaf);
            if constexpr (GRP) gtake(); else pop();
          }
        }
        if (node < 0 && leaf == 0) {  // a popped leaf with no node visit
          leaf = node;
          prefetch_leaf(p.wtri, leaf);
          if constexpr (GRP) gtake(); else pop();
        }
#if !RR_COOP
        // batched fp64 leaf tests (closest_hit_pl's vote)
        const unsigned act = __activemask();
        const unsigned hv = __ballot_sync(act, leaf != 0);
        if (hv != 0) {
          const bool can = is_inner(node);
          const bool must = leaf != 0 && !can;
          const unsigned mv = __ballot_sync(act, must);
          const unsigned cv = __ballot_sync(act, can);
          const int na = __popc(act);
          if (STUCKD * __popc(mv) >= na || cv == 0 || HOLDD * __popc(hv) >= na) {
            if (leaf != 0) {
              if (CNT) st_cnt[1] += leaf_faces(leaf);
              RR_DCHECK(leaf_face(leaf) + leaf_faces(leaf) <= p.nf);
              if (test_leaf_w(p.wtri, leaf, o, d, best)) tbest = prune_bound(best.delta, r.shift);
              leaf = 0;
              if (node < 0) {  // the leaf that waited for the slot
                leaf = node;
                prefetch_leaf(p.wtri, leaf);
                if constexpr (GRP) gtake(); else pop();
              }
            }
          }
        }
        if (node == kDone && leaf == 0) searching = false;  // query done: best holds the hit
#endif
      }
#if RR_COOP
      // batched fp64 leaf tests (closest_hit_pl's vote), spread over the
      // whole warp: the stashed leaves' faces are numbered (first faces of
      // the holding lanes in lane order, then the second faces of the pair
      // leaves), lane j tests face j against its owner's ray (read from
      // the owner's shared-memory lane state) and the owners collect their
      // results by shuffles, in the leaf's face order (test_leaf_w's rule).
      // Before, only the holding lanes ran the fp64 tests (a quarter to a
      // half of the warp, one loop trip per face of the largest leaf).
      {
        const unsigned hv = __ballot_sync(0xffffffffu, leaf != 0);
        if (hv != 0) {
          const bool can = searching && is_inner(node);
          const bool must = leaf != 0 && !can;
          const unsigned mv = __ballot_sync(0xffffffffu, must);
          const unsigned cv = __ballot_sync(0xffffffffu, can);
          const int na = __popc(__ballot_sync(0xffffffffu, searching));
          if (STUCKD * __popc(mv) >= na || cv == 0 || HOLDD * __popc(hv) >= na) {
            const bool two = leaf != 0 && leaf_faces(leaf) == 2;
            const unsigned h2 = __ballot_sync(0xffffffffu, two);
            const int c1 = __popc(hv), c2 = __popc(h2);
            const int ia = __popc(hv & lt_mask), ib = c1 + __popc(h2 & lt_mask);
            if (CNT && leaf != 0) st_cnt[1] += leaf_faces(leaf);
            if (c1 + c2 <= 32) {
              uint8_t* it = s_item + (threadIdx.x & ~31u);
              if (leaf != 0) it[ia] = static_cast<uint8_t>(lane);
              if (two) it[ib] = static_cast<uint8_t>(lane | 32);
              __syncwarp();
              const int own = lane < c1 + c2 ? it[lane] : 0;
              const int32_t ol = __shfl_sync(0xffffffffu, leaf, own & 31);
              double t = -1.0;
              int32_t f = -1;
              if (lane < c1 + c2) {
                const LaneState& os = s_lane[(threadIdx.x & ~31u) + (own & 31)];
                RR_DCHECK(leaf_face(ol) + leaf_faces(ol) <= p.nf);
                t = mt_delta_w(p.wtri, leaf_face(ol) + (own >> 5), os.o, os.d, &f);
              }
              const double ta = __shfl_sync(0xffffffffu, t, ia & 31), tb = __shfl_sync(0xffffffffu, t, ib & 31);
              const int32_t fa = __shfl_sync(0xffffffffu, f, ia & 31), fb = __shfl_sync(0xffffffffu, f, ib & 31);
              __syncwarp();
              if (leaf != 0) {
                bool better = false;
                if (ta > 0.0 && (best.face < 0 || ta < best.delta || (ta == best.delta && fa < best.face))) {
                  best.delta = ta;
                  best.face = fa;
                  better = true;
                }
                if (two && tb > 0.0 && (best.face < 0 || tb < best.delta || (tb == best.delta && fb < best.face))) {
                  best.delta = tb;
                  best.face = fb;
                  better = true;
                }
                if (better) tbest = prune_bound(best.delta, r.shift);
              }
            } else if (leaf != 0) {  // more than 32 faces: every lane its own leaf
              RR_DCHECK(leaf_face(leaf) + leaf_faces(leaf) <= p.nf);
              if (test_leaf_w(p.wtri, leaf, o, d, best)) tbest = prune_bound(best.delta, r.shift);
            }
            if (leaf != 0) {
              leaf = 0;
              if (node < 0) {  // the leaf that waited for the slot
                leaf = node;
                prefetch_leaf(p.wtri, leaf);
                if constexpr (GRP) gtake(); else pop();
              }
            }
          }
        }
        if (searching && node == kDone && leaf == 0) searching = false;  // query done: best holds the hit
      }
#endif
      const unsigned sv = __ballot_sync(0xffffffffu, searching);
      const unsigned wv = __ballot_sync(0xffffffffu, has_ray && !searching);
      if (sv == 0 || __popc(wv) >= DONET) break;
    }
  }
  // ---- statistics
  __syncthreads();
  if (threadIdx.x < 4) atomicAdd(p.stats + threadIdx.x, s_stat[threadIdx.x]);
  if (threadIdx.x == 4) atomicMax(p.stats + 4, s_stat[4]);
  if (CNT) {
    for (int off = 16; off > 0; off >>= 1) {
      st_cnt[0] += __shfl_xor_sync(0xffffffffu, st_cnt[0], off);
      st_cnt[1] += __shfl_xor_sync(0xffffffffu, st_cnt[1], off);
      st_cnt[2] += __shfl_xor_sync(0xffffffffu, st_cnt[2], off);
    }
    if (lane == 0) {
      atomicAdd(p.stats + 5, st_cnt[0]);
      atomicAdd(p.stats + 6, st_cnt[1]);
      atomicAdd(p.stats + 7, st_cnt[2]);
    }
  }
}

}  // namespace rr
