// Diagnostic tracer variant (built only with -DRR_DIAG, selected by RR_DF):
// the dynamic-fetch state machine of round 1, slower than trace_kernel once
// leaf batching was added there.  Kept for A/B timing, not in the product.
#pragma once
// ---------------------------------------------------------------- dynamic-fetch tracer
// Same contract as trace_kernel<1, *>, restructured for SIMT efficiency (the
// per-ray loop above runs each warp's traversal to its slowest lane, so ~60 %
// of lanes idle): every lane runs a small state machine inside one loop.
//  * traversal: one node per iteration; a leaf reached while another leaf is
//    still pending is not tested at once but stashed, and pending leaves are
//    tested together when enough lanes hold one (LEAFT) or a lane cannot go
//    on without it, so the fp64 Moller-Trumbore runs with most lanes active;
//  * when at least DONET lanes have finished their closest-hit query (or no
//    lane can continue) the finished lanes shade together: receiver tests,
//    capture append, reflection, history, termination, and either start their
//    next bounce's traversal or take a new ray from the global counter.
// Pruning uses the bound of the leaves tested so far; a postponed leaf only
// makes it looser, so the set of candidate faces still contains the
// reference's closest face and the fp64 (delta, face) minimum is unchanged.
struct LaneRay {
  D3 o, d;
  double path;
};

template <int DONET, int LEAFT, int MINB, bool SMS>
__global__ void __launch_bounds__(128, MINB) trace_kernel_df(const TraceParams p) {
  // SMS: the fp64 ray state lives in shared memory (SoA, one slot per
  // thread) so the traversal loop keeps only fp32 state in registers
  __shared__ double s_state[SMS ? 7 : 1][SMS ? 128 : 1];
  const int lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  const unsigned lt_mask = (1u << lane) - 1u;
  constexpr int32_t kNoLeaf = 0;  // leaves are encoded < 0
  const float kInf = __int_as_float(0x7f800000);
  const TravHeader& h = p.hdr;

  int64_t ray = -1;
  bool exhausted = false;
  LaneRay R{};
  int32_t steps = 0, bounces = 0, rplane = -2;
  RayF rf{};
  double best_delta = 0.0;
  int32_t best_face = -1;
  float tbest = FLT_MAX;
  int32_t node = kDone, leaf = kNoLeaf;
  int32_t st_n[kStack];
  float st_t[kStack];
  int sp = 0;
  unsigned long long st_bounce = 0, st_esc = 0, st_oor = 0, st_alive = 0;
  int32_t st_max = 0;

  auto load_ray = [&]() -> LaneRay {
    if constexpr (SMS) {
      return LaneRay{d3(s_state[0][tid], s_state[1][tid], s_state[2][tid]),
                     d3(s_state[3][tid], s_state[4][tid], s_state[5][tid]), s_state[6][tid]};
    } else {
      return R;
    }
  };
  auto store_ray = [&](const LaneRay& x) {
    if constexpr (SMS) {
      s_state[0][tid] = x.o.x; s_state[1][tid] = x.o.y; s_state[2][tid] = x.o.z;
      s_state[3][tid] = x.d.x; s_state[4][tid] = x.d.y; s_state[5][tid] = x.d.z;
      s_state[6][tid] = x.path;
    } else {
      R = x;
    }
  };
  // begin one closest-hit query from the lane's ray
  auto start_query = [&](const LaneRay& x) {
    best_face = -1;
    best_delta = 0.0;
    tbest = FLT_MAX;
    sp = 0;
    leaf = kNoLeaf;
    if (!make_rayf(h, x.o, x.d, rf)) {
      node = kDone;
    } else if (h.root_ref < 0) {
      node = h.root_ref;
    } else {
      const float t = box_enter(rf, h.lo[0], h.hi[0], h.lo[1], h.hi[1], h.lo[2], h.hi[2], tbest);
      node = (t == kInf) ? kDone : h.root_ref;
    }
  };
  auto pop = [&]() {
    node = kDone;
    while (sp > 0) {
      --sp;
      if (st_t[sp] <= tbest) {
        node = st_n[sp];
        break;
      }
    }
  };

  for (;;) {
    // ---- refill lanes without a ray (warp-aggregated atomic)
    const bool need = ray < 0 && !exhausted;
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
          ray = i;
          LaneRay x;
          x.o = d3(p.src[0], p.src[1], p.src[2]);
          x.d = p.dirs ? d3(p.dirs[3 * i], p.dirs[3 * i + 1], p.dirs[3 * i + 2])
                       : fib_dir(global_ray(p, i), p.N, p.az_step);
          x.path = 0.0;
          steps = 0;
          bounces = 0;
          rplane = -2;
          if (p.max_iter <= 0) {
            st_alive++;
            ray = -1;
            node = kDone;
          } else {
            store_ray(x);
            start_query(x);
          }
        } else {
          exhausted = true;
        }
      }
    }
    if (__all_sync(0xffffffffu, ray < 0 && exhausted)) break;

    // ---- traversal until DONET lanes have finished (or none can continue)
    for (;;) {
      const bool busy = ray >= 0 && (node != kDone || leaf != kNoLeaf);
      const unsigned bm = __ballot_sync(0xffffffffu, busy);
      const unsigned have = __ballot_sync(0xffffffffu, ray >= 0);
      if (bm == 0 || __popc(have & ~bm) >= DONET) break;
      if (busy && node != kDone && node >= 0) {
        // internal node: both children's fp32 boxes
        const float4* q = reinterpret_cast<const float4*>(p.nodes + node);
        const float4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
        const int4 dd = __ldg(reinterpret_cast<const int4*>(q + 3));
        float tl = box_enter(rf, a.x, a.y, a.z, a.w, b.x, b.y, tbest);
        float tr = box_enter(rf, b.z, b.w, c.x, c.y, c.z, c.w, tbest);
        if (dd.z == rplane) tl = kInf;
        if (dd.w == rplane) tr = kInf;
        const bool hl = tl != kInf, hr = tr != kInf;
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
          pop();
        }
      }
      // stash a reached leaf if the slot is free and keep traversing
      if (busy && node < 0 && leaf == kNoLeaf) {
        leaf = node;
        pop();
      }
      // test pending leaves together
      const bool stuck = busy && leaf != kNoLeaf && (node < 0 || node == kDone);
      const unsigned lm = __ballot_sync(0xffffffffu, busy && leaf != kNoLeaf);
      if (__any_sync(0xffffffffu, stuck) || __popc(lm) >= LEAFT) {
        if (busy && leaf != kNoLeaf) {
          const LaneRay x = load_ray();
          HitResult hb{best_delta, best_face};
          if (test_leaf(p.tri, leaf, x.o, x.d, hb)) {
            best_delta = hb.delta;
            best_face = hb.face;
            tbest = prune_bound(hb.delta, rf.shift);
          }
          leaf = kNoLeaf;
          if (node < 0) {  // the leaf that was waiting for the slot
            leaf = node;
            pop();
          }
        }
      }
    }

    // ---- finished lanes: one step_ray (tracer.cpp:19-62) each
    const bool fin = ray >= 0 && node == kDone && leaf == kNoLeaf;
    if (fin) {
      LaneRay x = load_ray();
      ++steps;
      const bool has_wall = best_face >= 0;
      for (int r = 0; r < p.n_recv; ++r) {
        const double sd = sphere_delta(x.o, x.d, d3(p.rc[r][0], p.rc[r][1], p.rc[r][2]), p.rr[r]);
        bool cap = sd > 0.0 && (!has_wall || sd < best_delta);
        double L = 0.0;
        if (cap) {
          L = x.path + sd;
          cap = L <= p.rng[r];
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
              const D3 pt = x.o + sd * x.d;
              c.p[0] = pt.x; c.p[1] = pt.y; c.p[2] = pt.z;
              c.d[0] = x.d.x; c.d[1] = x.d.y; c.d[2] = x.d.z;
              c.path = L;
              c.ray = static_cast<int32_t>(ray);
              c.meta = (bounces << 8) | r;
              p.caps[slot] = c;
            }
          }
        }
      }
      bool dead = false;
      if (!has_wall) {
        dead = true;
        st_esc++;
      } else {
        const double* nn = p.normal + 3 * static_cast<int64_t>(best_face);
        D3 n = d3(__ldg(nn), __ldg(nn + 1), __ldg(nn + 2));
        if (dot(n, x.d) > 0.0) n = d3(-n.x, -n.y, -n.z);
        const D3 pt = x.o + best_delta * x.d;
        const double s2 = 2.0 * dot(x.d, n);
        x.d = x.d - s2 * n;  // reflect, tracer.hpp:33-37
        x.o = pt;
        const int32_t pid = __ldg(p.face_plane + best_face);
        if (pid >= 0) {
          const int k = pid >> 29;
          const double dk = k == 0 ? x.d.x : (k == 1 ? x.d.y : x.d.z);
          rplane = fabs(dk) > p.cull_min ? pid : -2;
        } else {
          rplane = -2;
        }
        x.path += best_delta;
        p.hist[ray * p.H + bounces] = best_face;
        ++bounces;
        if (x.path > p.max_range) {
          dead = true;
          st_oor++;
        }
      }
      if (!dead && steps >= p.max_iter) {
        dead = true;
        st_alive++;
      }
      if (dead) {
        st_bounce += steps;
        st_max = max(st_max, steps);
        ray = -1;
        node = kDone;
      } else {
        store_ray(x);
        start_query(x);
      }
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    st_bounce += __shfl_xor_sync(0xffffffffu, st_bounce, off);
    st_esc += __shfl_xor_sync(0xffffffffu, st_esc, off);
    st_oor += __shfl_xor_sync(0xffffffffu, st_oor, off);
    st_alive += __shfl_xor_sync(0xffffffffu, st_alive, off);
    st_max = max(st_max, __shfl_xor_sync(0xffffffffu, st_max, off));
  }
  if (lane == 0) {
    atomicAdd(p.stats + 0, st_bounce);
    atomicAdd(p.stats + 1, st_esc);
    atomicAdd(p.stats + 2, st_oor);
    atomicAdd(p.stats + 3, st_alive);
    atomicMax(p.stats + 4, (unsigned long long)st_max);
  }
}

// RR_DF selector of the round-1 A/B variants (profiles/r1_trace_kernel_ncu.md):
// 0 per-ray loop, 1-6 dynamic-fetch state machine, 7 child prefetch, 8-17
// postponed-leaf thresholds, 30-32 shared-memory stack bottom, 33 56-register
// budget, 34-37 internal nodes per vote round, 46 fp32 leaf prefilter, 47-48
// register stack entries, 54 72-register budget, 59 no leaf prefetch (the
// product default), 23/24 the 4-wide collapse.
using TraceKernelFn = void (*)(const TraceParams);
inline TraceKernelFn diag_trace_kernel(int df, bool have4, TraceKernelFn dflt) {
  if (df < 0) return dflt;
  TraceKernelFn dfk = df == 2 ? trace_kernel_df<8, 16, 8, true> : df == 3 ? trace_kernel_df<8, 16, 10, true>
           : df == 4 ? trace_kernel_df<8, 16, 12, true> : df == 5 ? trace_kernel_df<16, 16, 10, true>
           : df == 6 ? trace_kernel_df<4, 16, 10, true> : df == 1 ? trace_kernel_df<8, 16, 8, false> : dflt;
  if (df == 0) dfk = trace_kernel<1, 8>;
  if (df == 7) dfk = trace_kernel<1, 8, true>;
  if (df == 8) dfk = trace_kernel<1, 8, false, 8>;    // postponed leaves, >= 8/32 lanes
  if (df == 9) dfk = trace_kernel<1, 8, false, 16>;   // >= 16/32
  if (df == 10) dfk = trace_kernel<1, 8, false, 24>;  // >= 24/32
  if (df == 11) dfk = trace_kernel<1, 8, false, 16, 4>;  // ... or >= 4 lanes stuck
  if (df == 12) dfk = trace_kernel<1, 8, false, 16, 8>;
  if (df == 13) dfk = trace_kernel<1, 8, false, 16, 16>;
  if (df == 14) dfk = trace_kernel<1, 8, false, 8, 4>;
  if (df == 15) dfk = trace_kernel<1, 8, false, 16, -4>;  // >= 1/4 of the loop's lanes stuck
  if (df == 16) dfk = trace_kernel<1, 8, false, 16, -2>;
  if (df == 17) dfk = trace_kernel<1, 8, false, 16, -8>;
  if (df == 33) dfk = trace_kernel<1, 9, false, 16, -2>;  // 56-register budget
  if (df == 34) dfk = trace_kernel<1, 8, false, 16, -2, false, 2>;  // 2 / 4 internal nodes per vote round
  if (df == 35) dfk = trace_kernel<1, 8, false, 16, -2, false, 4>;
  if (df == 36) dfk = trace_kernel<1, 8, false, 16, -2, false, 8>;
  if (df == 46) dfk = trace_kernel<1, 8, false, 16, -2, false, 16, 0, true>;  // fp32 leaf prefilter (C2 +3 %)
  if (df == 47) dfk = trace_kernel<1, 8, false, 16, -2, false, 16, 0, false, 1>;  // top entry in registers
  if (df == 48) dfk = trace_kernel<1, 8, false, 16, -2, false, 16, 0, false, 2>;  // two top entries
  if (df == 54) dfk = trace_kernel<1, 7, false, 16, -2, false, 16, 0, false, 2>;  // 72-register budget
  if (df == 59) dfk = trace_kernel<1, 7, false, 16, -2, false, 16, 0, false, 2, false>;  // no leaf prefetch
  if (df == 37) dfk = trace_kernel<1, 8, false, 16, -2, false, 16>;
  if (df == 30) dfk = trace_kernel<1, 8, false, 16, -2, false, 1, 4>;   // shared-memory stack bottom
  if (df == 31) dfk = trace_kernel<1, 8, false, 16, -2, false, 1, 8>;
  if (df == 32) dfk = trace_kernel<1, 8, false, 16, -2, false, 1, 16>;
  if (df == 23 && have4) dfk = trace_kernel<3, 8>;
  if (df == 24 && have4) dfk = trace_kernel<3, 6>;
  return dfk;
}
