// K2+K3+K4 — persistent specular tracer.
//
// Replaces trace/step/step_ray (tracer.cpp:19-149), emit/fibonacci_directions
// (emission.cpp:17-43) and nearest_hit/nearest_hit_brute
// (accel_tree.cpp:125-191).
//
// One persistent kernel per trace: each lane owns one ray from emission to
// death and pulls a new ray index from a global counter (warp-aggregated
// atomic) when its ray dies, so no ray state goes back to HBM between
// bounces.  Per bounce: closest hit (fp32 conservative box traversal over the
// 64-B TNode pairs, top levels from shared memory, short per-lane stack;
// fp64 Moller-Trumbore at leaves), receiver-sphere tests, capture append
// (warp-aggregated atomic into a compact buffer), reflection, path update and
// one 4-B face-history write.  Band multipliers are not carried per ray: they
// are the ordered product of (1 - alpha) over the face history and are
// rebuilt per capture afterwards (bit-identical to the running product of
// tracer.cpp:57-58).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "rr_sincos.cuh"
#include "rr_trace.cuh"

namespace rr {

constexpr int kStack8 = 96;  // 8-wide traversal stack (entries); the tree's bound must fit
constexpr int kStack8G = 32;  // 8-wide group traversal: one entry per level
// stack entries per lane in shared memory (8-wide tracers).  The shared
// memory per SM sets the L1 size (256 KB - the carveout the driver picks for
// 8 blocks): C5 with 12 entries (196 KB carveout, 60 KB L1) 516 ms, 8 (164 KB,
// 92 KB L1) 508, 4 (132 KB) 510, 0 (100 KB, the stack in local memory) 523;
// the face-history sector buffer (RR_HBUF, +4 KB per block) at 12 entries
// forced the 228 KB carveout (28 KB L1, L1 hit rate 34 -> 24 %): 728 ms; at
// equal carveouts it is neutral (8 entries 511, 4 entries 509).  Group
// entries with the child / face bases (RR_GST, 12 B): 5 entries (164 KB)
// 486.6 ms, 4 490, 2 503, 0 502, 8 (196 KB) 491; without, 8 entries 491.
// With the fp32 ray terms in shared memory too (RR_RSM, +3 KB per block):
// 5 entries (196 KB carveout) 415.3 ms, 3 (164 KB) 417.2; without RR_RSM 5
// entries 417.9, 3 entries 425.9.
#ifndef RR_SMS8
#define RR_SMS8 (RR_HBUF ? 4 : RR_GST ? 5 : 8)
#endif
constexpr int kSms8 = RR_SMS8;
#ifndef RR_MINB8
#define RR_MINB8 8  // blocks of 128 per SM (64 registers)
#endif
#ifndef RR_STUCKD8
#define RR_STUCKD8 4  // leaf batch when 1/STUCKD of the searching lanes wait on their stashed leaf
#endif
#ifndef RR_HOLDD8
#define RR_HOLDD8 1  // ... or 1/HOLDD of them hold one (with RR_COOP, STUCKD / HOLDD 4 / 1 427.5 ms,
                     // 4 / 2 428.8, 4 / 4 437.6, 2 / 2 435.9, 8 / 2 440.8, 3 / 1 431.3, 5 / 1 428.5, 6 / 1 431.2)
#endif
#ifndef RR_DONET8
#define RR_DONET8 8  // lanes done before a warp leaves traversal for shading (final kernel: 5 / 6 / 7 / 8 / 9 / 10:
                   // 409.8 / 406.4 / 404.8 / 404.4 / 404.7 / 405.7 ms)
#endif

__device__ __forceinline__ int64_t global_ray(const TraceParams& p, int64_t i) {
  if (p.block > 0) {
    // block-cyclic: rank = first, world = stride
    const int64_t blk = i / p.block, off = i - blk * p.block;
    return (blk * p.stride + p.first) * p.block + off;
  }
  return p.first + i * p.stride;
}

// fibonacci_directions, emission.cpp:17-29
__device__ __forceinline__ D3 fib_dir(int64_t k, int64_t n, double az_step) {
  const double z = 1.0 - (2.0 * static_cast<double>(k) + 1.0) / static_cast<double>(n);
  const double t = 1.0 - z * z;
  const double rho = sqrt(0.0 < t ? t : 0.0);
  const double phi = az_step * static_cast<double>(k);
  double s, c;
  sincos_emit(phi, &s, &c);
  return d3(rho * c, rho * s, z);
}

}  // namespace rr
#include "rr_trace_w8.cuh"
namespace rr {

// V = 0: binary nodes, fp32 leaf classification + fp64 resolution (diagnostic)
// V = 1: binary nodes, fp64 test at every leaf (default)
// V = 2: 4-wide nodes, fp64 test at every leaf (diagnostic)
template <int V, int MINB, bool PF = false, int PL = 0, int ST = 1, bool CNT = false, int UNR = 1, int SMS = 0,
          bool F32L = false, int TOS = 0, bool PFL = true>
__global__ void __launch_bounds__(128, MINB) trace_kernel(const TraceParams p) {
  constexpr bool WIDE = V == 2;
  __shared__ int2 s_stack[SMS > 0 ? SMS * 128 : 1];  // bottom of the traversal stacks (SMS > 0)
  extern __shared__ TNode smem_nodes[];
  QNode* smem_q = reinterpret_cast<QNode*>(smem_nodes);
  const int32_t K = (p.use_smem && V != 0) ? (WIDE ? p.hdr.K4 : p.hdr.K) : 0;
  if (WIDE) {
    for (int i = threadIdx.x; i < K; i += blockDim.x) smem_q[i] = p.qnodes[i];
  } else {
    for (int i = threadIdx.x; i < K; i += blockDim.x) smem_nodes[i] = p.nodes[i];
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  int64_t ray = -1;
  bool exhausted = false;
  D3 o{}, d{};
  double path = 0.0;
  int32_t steps = 0, bounces = 0, rplane = -2;
  uint32_t st_bounce = 0, st_esc = 0, st_oor = 0, st_alive = 0;  // per thread: fits 32 bits
  unsigned long long st_cnt[2] = {0, 0};  // node visits, leaf tests (CNT)
  int32_t st_max = 0;

  for (;;) {
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
          o = d3(p.src[0], p.src[1], p.src[2]);
          if (p.dirs) {
            d = d3(p.dirs[3 * i], p.dirs[3 * i + 1], p.dirs[3 * i + 2]);
          } else {
            d = fib_dir(global_ray(p, i), p.N, p.az_step);
          }
          path = 0.0;
          steps = 0;
          bounces = 0;
          rplane = -2;
          if (p.max_iter <= 0) {  // trace() with a zero cap: nothing runs
            st_alive++;
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

    // ---- one step_ray (tracer.cpp:19-62)
    ++steps;
    HitResult wall;
    if (V == 0) {
      wall = closest_hit_f(p.hdr, p.nodes, p.tri32, p.tri, o, d);
    } else if (V == 3) {
      wall = closest_hit4_pl<16, -2, RegRay, UNR, TOS, CNT>(p.hdr, p.q4, p.root4, p.tri, RegRay{o, d}, rplane, st_cnt);
    } else if (V == 1 && PL > 0) {
      wall = closest_hit_pl<PL, ST, RegRay, CNT, UNR, SMS, F32L, TOS, PFL>(p.hdr, p.nodes, p.tri, RegRay{o, d}, rplane,
                                                                  st_cnt, s_stack + threadIdx.x, p.tri32);
    } else if (V == 1) {
      wall = closest_hit<PF>(p.hdr, p.nodes, smem_nodes, K, p.tri, o, d, nullptr, rplane);
    } else {
      wall = closest_hit4(p.hdr, p.qnodes, smem_q, K, p.tri, o, d);
    }
    const bool has_wall = wall.face >= 0;
    for (int r = 0; r < p.n_recv; ++r) {
      const double sd = sphere_delta(o, d, d3(p.rc[r][0], p.rc[r][1], p.rc[r][2]), p.rr[r]);
      bool cap = sd > 0.0 && (!has_wall || sd < wall.delta);
      double L = 0.0;
      if (cap) {
        L = path + sd;
        cap = L <= p.rng[r];  // resolved_max_range of receiver r
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
      const double* nn = p.normal + 3 * static_cast<int64_t>(wall.face);
      D3 n = d3(__ldg(nn), __ldg(nn + 1), __ldg(nn + 2));
      if (dot(n, d) > 0.0) n = d3(-n.x, -n.y, -n.z);
      const D3 pt = o + wall.delta * d;
      const double s2 = 2.0 * dot(d, n);
      d = d - s2 * n;  // reflect, tracer.hpp:33-37
      o = pt;
      // the next segment leaves this face's plane: cull coplanar subtrees
      // (p.cull_min: the |d_axis| above which a re-hit of the plane cannot
      // reach the self-hit epsilon at this scene's coordinate magnitude)
      const int32_t pid = __ldg(p.face_plane + wall.face);
      if (pid >= 0) {
        const int k = pid >> 29;
        const double dk = k == 0 ? d.x : (k == 1 ? d.y : d.z);
        rplane = fabs(dk) > p.cull_min ? pid : -2;
      } else {
        rplane = -2;
      }
      path += wall.delta;
      RR_DCHECK(ray < p.count && bounces < p.H && wall.face < p.nf);
      p.hist[ray * p.H + bounces] = wall.face;
      ++bounces;
      if (path > p.max_range) {
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

#ifdef RR_DIAG
#include "rr_trace_diag.cuh"
#endif

// ---------------------------------------------------------------- ray order
// Warps take rays in a spatially coherent order: neighbours of a Fibonacci
// point are far apart in index (azimuth step = golden angle), so the lattice
// order puts 32 unrelated directions in a warp.  Sorting the rays by the
// Morton code of an approximate direction groups nearby directions; mirror
// reflection keeps such beams together for many bounces, so warps traverse
// similar nodes.  Only the processing order changes (captures are sorted by
// ray index afterwards), never a result.
__device__ __forceinline__ uint32_t part1by2(uint32_t x) {
  x &= 0x3ff;
  x = (x | (x << 16)) & 0x030000ff;
  x = (x | (x << 8)) & 0x0300f00f;
  x = (x | (x << 4)) & 0x030c30c3;
  x = (x | (x << 2)) & 0x09249249;
  return x;
}

__global__ void ray_order_key_kernel(const TraceParams p, uint32_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= p.count) return;
  float x, y, z;
  if (p.dirs) {
    x = static_cast<float>(p.dirs[3 * c]);
    y = static_cast<float>(p.dirs[3 * c + 1]);
    z = static_cast<float>(p.dirs[3 * c + 2]);
  } else {
    const int64_t k = global_ray(p, c);
    const double zz = 1.0 - (2.0 * static_cast<double>(k) + 1.0) / static_cast<double>(p.N);
    const double rho = sqrt(fmax(0.0, 1.0 - zz * zz));
    // azimuth modulo 2 pi from the fractional part of k * (1 - 1/golden)
    const double f = static_cast<double>(k) * 0.38196601125010515;
    const float phi = static_cast<float>(6.283185307179586 * (f - floor(f)));
    float s, co;
    sincosf(phi, &s, &co);
    x = static_cast<float>(rho) * co;
    y = static_cast<float>(rho) * s;
    z = static_cast<float>(zz);
  }
  const uint32_t qx = static_cast<uint32_t>(fminf(fmaxf((x + 1.0f) * 512.0f, 0.0f), 1023.0f));
  const uint32_t qy = static_cast<uint32_t>(fminf(fmaxf((y + 1.0f) * 512.0f, 0.0f), 1023.0f));
  const uint32_t qz = static_cast<uint32_t>(fminf(fmaxf((z + 1.0f) * 512.0f, 0.0f), 1023.0f));
  keys[c] = (part1by2(qx) << 2) | (part1by2(qy) << 1) | part1by2(qz);
  vals[c] = static_cast<int32_t>(c);
}

// ---------------------------------------------------------------- captures
// sort key (receiver, ray, order) packed into as few bits as the run needs
// (b_ray bits of the local ray index, monotone in the global one; b_ord bits
// of the order), so the radix sort makes only the passes it must
__global__ void capture_keys_kernel(const Capture* __restrict__ caps, int64_t n, int b_ray, int b_ord,
                                    unsigned long long* __restrict__ keys, int32_t* __restrict__ idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Capture c = caps[i];
  const uint64_t k = static_cast<uint64_t>(c.ray);
  const uint64_t order = static_cast<uint32_t>(c.meta) >> 8;
  const uint64_t recv = c.meta & 0xff;
  keys[i] = (((recv << b_ray) | k) << b_ord) | order;
  idx[i] = static_cast<int32_t>(i);
}

__global__ void capture_len_kernel(const Capture* __restrict__ caps, const int32_t* __restrict__ idx, int64_t n,
                                   int64_t* __restrict__ len) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) len[i] = static_cast<uint32_t>(caps[idx[i]].meta) >> 8;
  if (i == n) len[i] = 0;
}

// Sorted SoA captures + face paths + band multipliers (the ordered product
// of (1 - alpha), tracer.cpp:57-58).
// Materialise the sorted captures: 8 lanes per capture, lane b rebuilds band
// b's multiplier as the ordered product of (1 - alpha) over the face history
// (tracer.cpp:57-58, the same bits as the running product) and copies every
// 8th history entry; lane 0 writes the fixed fields.
__global__ void capture_out_kernel(const Capture* __restrict__ caps, const int32_t* __restrict__ idx, int64_t n,
                                   TraceParams p, const int32_t* __restrict__ mat, const double* __restrict__ oma,
                                   const int64_t* __restrict__ off, int32_t* __restrict__ o_recv,
                                   int32_t* __restrict__ o_ray, double* __restrict__ o_point,
                                   double* __restrict__ o_dir, double* __restrict__ o_path,
                                   double* __restrict__ o_mult, int32_t* __restrict__ o_hist) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i = g >> 3;
  const int b = static_cast<int>(g & 7);
  if (i >= n) return;
  const Capture& c = caps[idx[i]];
  const int32_t meta = c.meta;
  const int32_t order = static_cast<uint32_t>(meta) >> 8;
  const int32_t ray = c.ray;
  if (b == 0) {
    o_recv[i] = meta & 0xff;
    o_ray[i] = static_cast<int32_t>(global_ray(p, ray));
    o_path[i] = c.path;
  }
  if (b < 3) {
    o_point[3 * i + b] = c.p[b];
    o_dir[3 * i + b] = c.d[b];
  }
  const int32_t* h = p.hist + static_cast<int64_t>(ray) * p.H;
  const int64_t base = off[i];
  const int g0 = threadIdx.x & 24;              // first lane of this capture's group of 8
  const unsigned gm = 0xffu << g0;              // the group runs its loops in lockstep
  double m = 1.0;
  int j = 0;
  // up to four chunks of 8 faces per iteration: the history and material
  // loads of all of them are issued before the (ordered) products
  for (; j + 8 <= order; j += 32) {
    const int nc = min(4, (order - j) >> 3);  // full chunks in this round (uniform over the group)
    int32_t mt[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) mt[c] = c < nc ? h[j + 8 * c + b] : 0;  // each lane fetches one face per chunk
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c < nc) o_hist[base + j + 8 * c + b] = mt[c];
#pragma unroll
    for (int c = 0; c < 4; ++c) mt[c] = c < nc ? mat[mt[c]] : 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (c < nc) {
#pragma unroll
        for (int u = 0; u < 8; ++u) m *= oma[kBands * __shfl_sync(gm, mt[c], g0 + u) + b];
      }
    }
    if (nc < 4) {
      j += 8 * nc;
      break;
    }
  }
  const int rest = order - j;
  int32_t mt = 0;
  if (b < rest) {
    const int32_t f = h[j + b];
    o_hist[base + j + b] = f;
    mt = mat[f];
  }
  for (int u = 0; u < rest; ++u) m *= oma[kBands * __shfl_sync(gm, mt, g0 + u) + b];
  o_mult[kBands * i + b] = m;
}

// ---------------------------------------------------------------- queries
__global__ void nearest_hit_kernel(TravHeader h, const TNode* __restrict__ nodes, const QNode* __restrict__ qnodes,
                                   const float4* __restrict__ tri32, const FaceTri* __restrict__ tri,
                                   const double* __restrict__ o, const double* __restrict__ d, int64_t n,
                                   int32_t* __restrict__ face, double* __restrict__ delta,
                                   double* __restrict__ point) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const D3 oo = d3(o[3 * i], o[3 * i + 1], o[3 * i + 2]);
  const D3 dd = d3(d[3 * i], d[3 * i + 1], d[3 * i + 2]);
  const HitResult r = tri32 ? closest_hit_f(h, nodes, tri32, tri, oo, dd) : qnodes ? closest_hit4(h, qnodes, nullptr, 0, tri, oo, dd)
                             : closest_hit(h, nodes, nullptr, 0, tri, oo, dd);
  face[i] = r.face;
  delta[i] = r.face >= 0 ? r.delta : 0.0;
  const D3 pt = r.face >= 0 ? oo + r.delta * dd : d3(0, 0, 0);
  point[3 * i] = pt.x;
  point[3 * i + 1] = pt.y;
  point[3 * i + 2] = pt.z;
}

// nearest_hit_brute accel_tree.cpp:183-191 (strict <: lowest face on ties)
__global__ void brute_hit_kernel(const FaceTri* __restrict__ tri, int64_t nf, const double* __restrict__ o,
                                 const double* __restrict__ d, int64_t n, int32_t* __restrict__ face,
                                 double* __restrict__ delta, double* __restrict__ point) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const D3 oo = d3(o[3 * i], o[3 * i + 1], o[3 * i + 2]);
  const D3 dd = d3(d[3 * i], d[3 * i + 1], d[3 * i + 2]);
  int32_t bf = -1;
  double bd = 0.0;
  for (int64_t f = 0; f < nf; ++f) {
    const double t = mt_delta(tri, static_cast<int32_t>(f), oo, dd);
    if (t > 0.0 && (bf < 0 || t < bd)) {
      bd = t;
      bf = static_cast<int32_t>(f);
    }
  }
  face[i] = bf;
  delta[i] = bf >= 0 ? bd : 0.0;
  const D3 pt = bf >= 0 ? oo + bd * dd : d3(0, 0, 0);
  point[3 * i] = pt.x;
  point[3 * i + 1] = pt.y;
  point[3 * i + 2] = pt.z;
}

__global__ void fib_kernel(int64_t n, int64_t first, int64_t stride, int64_t count, double az_step,
                           double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const D3 d = fib_dir(first + i * stride, n, az_step);
  out[3 * i] = d.x;
  out[3 * i + 1] = d.y;
  out[3 * i + 2] = d.z;
}

void fibonacci_device(rr_ctx* ctx, int64_t n, int64_t first, int64_t stride, int64_t count, double* out) {
  if (count == 0) return;
  cudaStream_t st = ctx->stream;
  cudaPointerAttributes at{};
  RR_CUDA(cudaPointerGetAttributes(&at, out));
  const bool dev = at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
  DevBuf<double> tmp;
  double* d_out = out;
  if (!dev) {
    tmp.alloc(3 * count, st);
    d_out = tmp.p;
  }
  const double golden = (1.0 + std::sqrt(5.0)) / 2.0;  // emission.cpp:19-20, as run_trace
  fib_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, st>>>(n, first, stride, count,
                                                                        2.0 * M_PI * (1.0 - 1.0 / golden), d_out);
  RR_LAUNCH_CHECK();
  ctx->launches++;
  if (!dev) RR_CUDA(cudaMemcpyAsync(out, d_out, sizeof(double) * 3 * count, cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
}

void nearest_hit_batch(rr_scene* s, const double* d_o, const double* d_d, int64_t n, int brute, int32_t* d_face,
                       double* d_delta, double* d_point) {
  if (n <= 0) return;
  const unsigned g = static_cast<unsigned>((n + 127) / 128);
  // brute 0: the SAH tree; 2 / 3: diagnostics on the reference median tree
  // (fp32 leaf classification, 4-wide nodes)
  const bool sah = brute == 0 && s->snodes.p != nullptr;
  if (brute != 1 && !sah) ensure_reference_tree(s);
  if (brute == 1)
    brute_hit_kernel<<<g, 128, 0, s->ctx->stream>>>(s->tri.p, s->nf, d_o, d_d, n, d_face, d_delta, d_point);
  else
    nearest_hit_kernel<<<g, 128, 0, s->ctx->stream>>>(sah ? s->shdr : s->hdr, sah ? s->snodes.p : s->tnodes.p,
                                                       brute == 3 ? s->qnodes.p : nullptr,
                                                       brute == 2 ? s->tri32.p : nullptr, s->tri.p, d_o, d_d, n,
                                                       d_face, d_delta, d_point);
  RR_LAUNCH_CHECK();
  s->ctx->launches++;
}

}  // namespace rr

namespace rr {

rr_trace_result* run_trace(rr_scene* s, const rr_source* src, const rr_receiver* recv, int32_t n_recv,
                           const rr_trace_config* cfg, const double* d_dirs) {
  if (n_recv < 1 || n_recv > kMaxRecv) invalid("n_recv must be in [1, 8]");
  for (int r = 0; r < n_recv; ++r)
    if (!(recv[r].radius > 0.0)) invalid("receiver radius must be > 0");  // tracer.cpp:111-113
  if (src->ray_count < 1) invalid("source ray_count must be >= 1");       // emission.cpp:9-11
  if (cfg->max_iterations > (1 << 20) - 1) invalid("max_iterations must be < 2^20");
  if (src->ray_count >= (int64_t(1) << 36)) invalid("ray_count must be < 2^36");
  cudaStream_t st = s->ctx->stream;
  StageTimer tm(st);
  auto res = std::make_unique<rr_trace_result>();
  res->scene = s;
  TraceParams& p = res->params;
  // traversal tree: the SAH tree (RR_SAH=0: the reference median tree)
  static const int use_sah = [] {
    const char* e = std::getenv("RR_SAH");
    return e ? std::atoi(e) : 1;
  }();
  // (the fp32-leaf diagnostic classifies single-face leaves: reference tree)
  const bool sah = use_sah && s->snodes.p != nullptr && !(cfg->flags & RR_TRACE_F32_LEAVES);
  if (!sah || (cfg->flags & RR_TRACE_WIDE)) ensure_reference_tree(s);
  // kernel variant (RR_DF, see below); the 4-wide SAH collapse is built on
  // first use by the variants that traverse it
  static const int df_env0 = [] {
    const char* e = std::getenv("RR_DF");
    return e ? std::atoi(e) : -1;
  }();
  // Trees by scene size (measured): the binary SAH tree
  // below 2^18 faces; its 4-wide fp32 collapse from 2^18 (C3: 1.06 ms vs
  // 1.39 binary, 2.09 8-wide); the 8-wide compressed tree from 2^20, where
  // the binary node array (64 B per face) no longer fits the 126 MB L2
  // (C5: 657 ms vs 724 4-wide, 997 binary).  RR_WIDE moves the 8-wide threshold.
  static const int64_t wide_min = [] {
    const char* e = std::getenv("RR_WIDE");
    return e ? std::atoll(e) : int64_t(1) << 20;
  }();
  const bool want4 = sah && !(cfg->flags & (RR_TRACE_TREE2 | RR_TRACE_TREE8 | RR_TRACE_WIDE)) &&
                     ((df_env0 < 0 && s->nf >= (1 << 18) && s->nf < wide_min) || df_env0 == 23 || df_env0 == 24);
  if (want4) build_sah4(s);
  const bool want8 = sah && !(cfg->flags & RR_TRACE_TREE2) && !(cfg->flags & RR_TRACE_WIDE) &&
                     ((cfg->flags & RR_TRACE_TREE8) || (df_env0 < 0 && s->nf >= wide_min));
  if (want8) build_wide(s);
  p.wnodes = s->wnodes.p;
  p.wtri = s->wtri.p;
  p.n_wnodes = static_cast<int32_t>(s->wnodes.n);
  p.nf = s->nf;
  p.nodes = sah ? s->snodes.p : s->tnodes.p;
  p.qnodes = s->qnodes.p;
  // default: binary nodes, fp64 test at every leaf (fastest measured); diagnostics: fp32 leaf classification, 4-wide nodes
  const int variant = (cfg->flags & RR_TRACE_F32_LEAVES) ? 1 : (cfg->flags & RR_TRACE_WIDE) ? 2 : 0;
  p.wide = variant == 2 ? 1 : 0;
  p.tri32 = s->tri32.p;
  p.face_plane = s->face_plane.p;
  p.tri = s->tri.p;
  p.normal = s->normal.p;
  p.hdr = sah ? s->shdr : s->hdr;
  p.q4 = s->s4nodes.p;
  p.root4 = s->s4root;
  // shared-memory top-level cache: measured slower for the default kernel
  // (profiles/r1_ab_variants.md), kept for the diagnostic ones
  p.use_smem = (variant == 0 || (cfg->flags & RR_TRACE_NO_SMEM_CACHE)) ? 0 : 1;
  for (int k = 0; k < 3; ++k) p.src[k] = src->position[k];
  p.N = src->ray_count;
  // ray subset
  int64_t count;
  if (cfg->block > 0) {
    const int64_t world = std::max<int64_t>(cfg->stride, 1), rank = cfg->first;
    if (rank < 0 || rank >= world) invalid("block-cyclic rank out of range");
    const int64_t nblk = (p.N + cfg->block - 1) / cfg->block;
    const int64_t my_full = nblk / world + (rank < nblk % world ? 1 : 0);
    count = my_full * cfg->block;
    // trim the last (partial) global block if this rank owns it
    const int64_t last_blk = nblk - 1;
    if (last_blk % world == rank) count -= nblk * cfg->block - p.N;
    p.first = rank;
    p.stride = world;
    p.block = cfg->block;
  } else if (cfg->stride <= 0) {
    count = p.N;
    p.first = 0;
    p.stride = 1;
    p.block = 0;
  } else {
    if (cfg->first < 0 || cfg->first >= p.N) invalid("subset first out of range");
    count = (p.N - cfg->first + cfg->stride - 1) / cfg->stride;
    if (cfg->count > 0) count = std::min(count, cfg->count);
    p.first = cfg->first;
    p.stride = cfg->stride;
    p.block = 0;
  }
  p.count = count;
  const double golden = (1.0 + std::sqrt(5.0)) / 2.0;
  p.az_step = 2.0 * M_PI * (1.0 - 1.0 / golden);
  p.dirs = d_dirs;
  DevBuf<double> host_dirs;
  if (!d_dirs && cfg->directions) {
    host_dirs.alloc(3 * std::max<int64_t>(count, 1), st);
    RR_CUDA(cudaMemcpyAsync(host_dirs.p, cfg->directions, sizeof(double) * 3 * count, cudaMemcpyHostToDevice, st));
    p.dirs = host_dirs.p;
  }
  p.n_recv = n_recv;
  for (int r = 0; r < n_recv; ++r) {
    for (int k = 0; k < 3; ++k) p.rc[r][k] = recv[r].center[k];
    p.rr[r] = recv[r].radius;
    res->recv_center.insert(res->recv_center.end(), recv[r].center, recv[r].center + 3);
    res->recv_radius.push_back(recv[r].radius);
  }
  p.max_iter = cfg->max_iterations;
  // resolved_max_range (tracer.cpp:10-15) per receiver: the reference runs
  // one trace per receiver, each with its own range.  One trace here serves
  // all receivers on the same trajectories: receiver r captures while
  // L <= rng[r], and rays die past the largest range, so every receiver gets
  // exactly its own run's captures (a ray alive at path <= rng[r] in the
  // combined trace is alive in r's run, and conversely).  The escape /
  // out-of-range counters follow the largest range.
  p.max_range = 0.0;
  for (int r = 0; r < n_recv; ++r) {
    p.rng[r] = cfg->max_range > 0.0 ? cfg->max_range
                                    : 0.5 * recv[r].radius * std::sqrt(static_cast<double>(p.N));
    p.max_range = std::max(p.max_range, p.rng[r]);
  }
  // coplanar cull threshold.  After reflecting off a face in an
  // axis-aligned plane, the origin's axis coordinate is off the plane by the
  // rounding of o + delta*d and of delta (well below 80 eps_64 * B, B = the
  // largest |coordinate|), and a re-hit of the plane is computed at
  // delta' <~ 80 eps_64 B / |d_axis|; it can be accepted (> 1e-6,
  // kSelfHitEpsilon) only if |d_axis| < 1.8e-8 B.  The cull runs only above
  // 2^-40 B / 1e-6 = 9.1e-7 B (50x margin; 1e-6 at least): 2.7e-5 for the
  // 30 m C5 room, 2.7e-2 for a room moved 30 km off the origin.
  {
    const double scale = static_cast<double>(p.hdr.eps) * 0x1p19;  // eps = scale * 2^-19 (rr_geom.cuh)
    p.cull_min = std::max(1e-6, std::ldexp(scale, -40) / 1e-6);
  }
  p.H = std::max(cfg->max_iterations, 1);
  res->hist.alloc(static_cast<size_t>(std::max<int64_t>(count, 1)) * p.H, st);
  p.hist = res->hist.p;

  DevBuf<unsigned long long> counters;
  counters.alloc(10, st);
  p.cap_count = counters.p;
  p.ray_counter = counters.p + 1;
  p.stats = counters.p + 2;

  // capture buffer: 2 per ray and receiver, or 1.25x the rate of the last
  // trace of this scene; an overflow re-runs the kernel with the exact size
  const double per_ray = std::max(2.0, 1.25 * s->caps_per_ray);
  int64_t capacity = std::max<int64_t>(1 << 16, static_cast<int64_t>(per_ray * count * n_recv));
  DevBuf<Capture> caps;
  const size_t smem = (!p.use_smem || variant == 0) ? 0
                      : p.wide ? sizeof(QNode) * static_cast<size_t>(p.hdr.K4)
                               : sizeof(TNode) * static_cast<size_t>(p.hdr.K);
  // blocks per SM for the register budget (dev override RR_MINB)
  // Product kernels: the per-ray loop with postponed (batched) leaf tests
  // over the binary SAH tree, the two newest stack entries in registers, a
  // 72-register budget; deep trees (>= 2^18 faces) over the 4-wide collapse,
  // which halves the dependent node fetches (C3 -15 %, C5 -8 %; C2 +8 %, so
  // not there).  Optimisation log: DESIGN.md section 4.  The A/B variants of
  // round 1 (RR_DF) are compiled only with -DRR_DIAG.
  static const int df_env = [] {
    const char* e = std::getenv("RR_DF");
    return e ? std::atoi(e) : -1;
  }();
  const bool wide4 = want4 && s->s4nodes.p != nullptr && (df_env < 0 || df_env == 23);
  // 8-wide compressed tree: trace_kernel_w8 (rr_trace_w8.cuh), the group
  // traversal when the tree's depth fits its stack, else the sorted-push
  // traversal.  RR_W8V (A/B): 1 the sorted-push kernel, 2 the group kernel
  // in pure octant order (C5: 527 / 547 / 538 ms for 0 / 1 / 2).
  static const int w8v = [] {
    const char* e = std::getenv("RR_W8V");
    return e ? std::atoi(e) : 0;
  }();
  const bool wide8 = want8 && s->wnodes.p != nullptr && s->wstack <= kStack8 && s->wide_ok;
  const bool grp8 = wide8 && w8v != 1 && s->wdepth < kStack8G;
  const bool cnt = (cfg->flags & RR_TRACE_COUNT) != 0;
  using KFn = void (*)(const TraceParams);
  // A/B of the sorted-push kernel (C5, ms; before the ray state moved to
  // shared memory): MINB 8, DONET 8, UNR 1, sorted pushes 657; unsorted
  // pushes 667; 12 stack entries in shared memory 658; MINB 7 666; DONET 16 /
  // UNR 4 at MINB 6 716; UNR 8 810; no batching (the per-ray loop) 1074.
  // After: 587 (MINB 9 592; 10: 620; 12: 692).  Group kernel: DONET 4 / 8
  // 535 / 527, STUCKD 2 / 8 529 / 547, HOLDD 4 547, MINB 9 (56 registers)
  // 833, 16 stack entries all in shared memory (7 blocks per SM) 752.
  KFn w8k = cnt ? trace_kernel_w8<RR_MINB8, RR_DONET8, 1, kStack8, true, kSms8, RR_STUCKD8, RR_HOLDD8> : trace_kernel_w8<RR_MINB8, RR_DONET8, 1, kStack8, false, kSms8, RR_STUCKD8, RR_HOLDD8>;
  if (grp8)
    w8k = w8v == 2 ? (cnt ? trace_kernel_w8<RR_MINB8, RR_DONET8, 1, kStack8G, true, kSms8, RR_STUCKD8, RR_HOLDD8, true, false>
                          : trace_kernel_w8<RR_MINB8, RR_DONET8, 1, kStack8G, false, kSms8, RR_STUCKD8, RR_HOLDD8, true, false>)
                   : (cnt ? trace_kernel_w8<RR_MINB8, RR_DONET8, 1, kStack8G, true, kSms8, RR_STUCKD8, RR_HOLDD8, true, true>
                          : trace_kernel_w8<RR_MINB8, RR_DONET8, 1, kStack8G, false, kSms8, RR_STUCKD8, RR_HOLDD8, true, true>);
  auto dfk = wide8 ? w8k : wide4 ? trace_kernel<3, 8> : trace_kernel<1, 7, false, 16, -2, false, 16, 0, false, 2, false>;
#ifdef RR_DIAG
  dfk = diag_trace_kernel(df_env, s->s4nodes.p != nullptr, dfk);
#endif
  if (cnt && !wide8)  // counts of the default
    dfk = wide4 ? trace_kernel<3, 8, false, 0, 1, true> : trace_kernel<1, 7, false, 16, -2, true, 16, 0, false, 2, false>;
  // diagnostics: fp32 leaf classification / 4-wide nodes over the reference tree
  auto kernel = variant == 0 ? dfk : variant == 1 ? trace_kernel<0, 8> : trace_kernel<2, 1>;
  static thread_local int occ_cache_smem = -1, occ_cache_blocks = 0;
  static thread_local const void* occ_cache_fn = nullptr;
  if (occ_cache_smem != static_cast<int>(smem) || occ_cache_fn != reinterpret_cast<const void*>(kernel)) {
    // RR_CARVE (dev A/B): preferred shared-memory carveout in percent; -1
    // leaves the driver's choice
    static const int carve = [] {
      const char* e = std::getenv("RR_CARVE");
      return e ? std::atoi(e) : -1;
    }();
    if (carve >= 0) {
      RR_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
      if (smem > 0)
        RR_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    } else {
      cudaFuncAttributes fa{};
      RR_CUDA(cudaFuncGetAttributes(&fa, kernel));
      const int dyn = std::min<int>(200 * 1024, 227 * 1024 - static_cast<int>(fa.sharedSizeBytes));
      RR_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    }
    RR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_cache_blocks, kernel, 128, smem));
    occ_cache_smem = static_cast<int>(smem);
    occ_cache_fn = reinterpret_cast<const void*>(kernel);
  }
  const int blocks_per_sm = std::max(occ_cache_blocks, 1);
  const int64_t want = (count + 127) / 128;
  const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)s->ctx->sm_count * blocks_per_sm)));
  // spatially coherent work order (RR_ORDER=0 keeps the lattice order)
  static const int order_env = [] {
    const char* e = std::getenv("RR_ORDER");
    return e ? std::atoi(e) : 1;
  }();
  DevBuf<int32_t> order;
  p.order = nullptr;
  if (order_env && count > 1 && count < (int64_t(1) << 31)) {
    DevBuf<uint32_t> ok, ok_s;
    DevBuf<int32_t> ov;
    ok.alloc(count, st);
    ok_s.alloc(count, st);
    ov.alloc(count, st);
    order.alloc(count, st);
    ray_order_key_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, st>>>(p, ok.p, ov.p);
    RR_LAUNCH_CHECK();
    size_t tb = 0;
    RR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, ok.p, ok_s.p, ov.p, order.p, static_cast<int>(count), 0, 30,
                                            st));
    DevBuf<uint8_t> tmp;
    tmp.alloc(tb, st);
    RR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, ok.p, ok_s.p, ov.p, order.p, static_cast<int>(count), 0, 30,
                                            st));
    s->ctx->launches += 5;
    p.order = order.p;
  }
  tm.mark("trace: setup");
  cudaEvent_t e0, e1;
  RR_CUDA(cudaEventCreate(&e0));
  RR_CUDA(cudaEventCreate(&e1));
  unsigned long long hc[10];
  static const int l2p = [] {
    const char* e = std::getenv("RR_L2P");
    return e ? std::atoi(e) : 0;
  }();
  for (int attempt = 0; attempt < 2; ++attempt) {
    caps.alloc(capacity, st);
    p.caps = caps.p;
    p.cap_capacity = capacity;
    RR_CUDA(cudaMemsetAsync(counters.p, 0, sizeof(unsigned long long) * 10, st));
    RR_CUDA(cudaEventRecord(e0, st));
    if (l2p > 0 && wide8) {
      // A/B (RR_L2P): an L2 persisting window over the 8-wide nodes (1) or
      // the leaf-ordered faces (2) for this launch
      static bool limit_set = false;
      cudaDeviceProp prop;
      RR_CUDA(cudaGetDeviceProperties(&prop, s->ctx->device));
      if (!limit_set) {
        RR_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prop.persistingL2CacheMaxSize));
        limit_set = true;
      }
      const void* base = l2p == 1 ? static_cast<const void*>(s->wnodes.p) : static_cast<const void*>(s->wtri.p);
      const size_t bytes = l2p == 1 ? s->wnodes.n * sizeof(WNode) : s->wtri.n * sizeof(FaceTri);
      const size_t win = std::min<size_t>(bytes, static_cast<size_t>(prop.accessPolicyMaxWindowSize));
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeAccessPolicyWindow;
      at[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(base);
      at[0].val.accessPolicyWindow.num_bytes = win;
      at[0].val.accessPolicyWindow.hitRatio =
          std::min(1.0f, static_cast<float>(prop.persistingL2CacheMaxSize) / static_cast<float>(win));
      at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(grid);
      lc.blockDim = dim3(128);
      lc.dynamicSmemBytes = smem;
      lc.stream = st;
      lc.attrs = at;
      lc.numAttrs = 1;
      if (attempt == 0 && std::getenv("RR_TIMING"))
        std::fprintf(stderr, "[rr timing] L2 window %zu B (persisting max %d B, hit ratio %.3f)\n", win,
                     prop.persistingL2CacheMaxSize, at[0].val.accessPolicyWindow.hitRatio);
      RR_CUDA(cudaLaunchKernelEx(&lc, kernel, p));
    } else {
      kernel<<<grid, 128, smem, st>>>(p);
    }
    RR_LAUNCH_CHECK();
    RR_CUDA(cudaEventRecord(e1, st));
    s->ctx->launches++;
    RR_CUDA(cudaMemcpyAsync(hc, counters.p, sizeof hc, cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
    if (static_cast<int64_t>(hc[0]) <= capacity) break;
    capacity = static_cast<int64_t>(hc[0]);  // exact re-run with the measured size
  }
  tm.mark("trace: kernel");
  RR_CUDA(cudaEventElapsedTime(&res->kernel_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const int64_t nc = static_cast<int64_t>(hc[0]);
  rr_trace_stats& S = res->stats;
  S.ray_bounces = static_cast<int64_t>(hc[2]);
  S.escaped = static_cast<int64_t>(hc[3]);
  S.out_of_range = static_cast<int64_t>(hc[4]);
  S.truncated = hc[5] > 0 ? 1 : 0;
  S.iterations = cfg->max_iterations > 0 ? static_cast<int32_t>(hc[6]) : 0;
  S.max_range = p.max_range;
  S.n_captures = nc;
  S.n_rays = count;
  S.node_visits = (cfg->flags & RR_TRACE_COUNT) ? static_cast<int64_t>(hc[7]) : -1;
  S.leaf_tests = (cfg->flags & RR_TRACE_COUNT) ? static_cast<int64_t>(hc[8]) : -1;
  if ((cfg->flags & RR_TRACE_COUNT) && std::getenv("RR_TIMING"))
    std::fprintf(stderr, "[rr timing] node visits hitting no slot: %llu of %llu\n", hc[9], hc[7]);
  S.tree_width = wide8 ? 8 : (wide4 || variant == 2) ? 4 : 2;
  S.node_bytes = wide8 ? static_cast<int32_t>(sizeof(WNode)) : (wide4 || variant == 2) ? static_cast<int32_t>(sizeof(QNode))
                                                                                      : static_cast<int32_t>(sizeof(TNode));
  s->caps_per_ray = static_cast<double>(nc) / static_cast<double>(std::max<int64_t>(count, 1) * n_recv);

  // ---- sort captures by (receiver, ray, order) and materialise
  const bool sort = !(cfg->flags & RR_TRACE_KEEP_UNSORTED);
  DevBuf<unsigned long long> keys, keys_o;
  DevBuf<int32_t> idx, idx_o;
  keys.alloc(std::max<int64_t>(nc, 1), st);
  keys_o.alloc(std::max<int64_t>(nc, 1), st);
  idx.alloc(std::max<int64_t>(nc, 1), st);
  idx_o.alloc(std::max<int64_t>(nc, 1), st);
  res->c_off.alloc(nc + 1, st);
  if (nc > 0) {
    const unsigned g = static_cast<unsigned>((nc + 255) / 256);
    auto bits = [](int64_t v) {  // bits to hold 0..v
      int b = 0;
      while (b < 63 && (int64_t(1) << b) <= v) ++b;
      return b;
    };
    const int b_ray = bits(count - 1), b_ord = bits(std::max<int64_t>(cfg->max_iterations, 1)),
              b_rec = bits(n_recv - 1);
    const int end_bit = std::min(64, b_rec + b_ray + b_ord);
    capture_keys_kernel<<<g, 256, 0, st>>>(caps.p, nc, b_ray, b_ord, keys.p, idx.p);
    RR_LAUNCH_CHECK();
    s->ctx->launches++;
    int32_t* order_idx = idx.p;
    if (sort) {
      size_t tb = 0;
      RR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, keys_o.p, idx.p, idx_o.p, static_cast<int>(nc),
                                              0, end_bit, st));
      DevBuf<uint8_t> tmp;
      tmp.alloc(tb, st);
      RR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, keys_o.p, idx.p, idx_o.p, static_cast<int>(nc), 0,
                                              end_bit, st));
      s->ctx->launches += 4;
      order_idx = idx_o.p;
    }
    DevBuf<int64_t> len;
    len.alloc(nc + 1, st);
    capture_len_kernel<<<static_cast<unsigned>((nc + 256) / 256), 256, 0, st>>>(caps.p, order_idx, nc, len.p);
    RR_LAUNCH_CHECK();
    size_t tb = 0;
    RR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, len.p, res->c_off.p, static_cast<int>(nc + 1), st));
    DevBuf<uint8_t> tmp;
    tmp.alloc(tb, st);
    RR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, len.p, res->c_off.p, static_cast<int>(nc + 1), st));
    int64_t total = 0;
    RR_CUDA(cudaMemcpyAsync(&total, res->c_off.p + nc, sizeof total, cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
    S.total_history = total;
    res->c_recv.alloc(nc, st);
    res->c_ray.alloc(nc, st);
    res->c_point.alloc(3 * nc, st);
    res->c_dir.alloc(3 * nc, st);
    res->c_path.alloc(nc, st);
    res->c_mult.alloc(kBands * nc, st);
    res->c_hist.alloc(std::max<int64_t>(total, 1), st);
    capture_out_kernel<<<static_cast<unsigned>((8 * nc + 255) / 256), 256, 0, st>>>(
        caps.p, order_idx, nc, p, s->mat.p, s->oma.p, res->c_off.p,
                                           res->c_recv.p, res->c_ray.p, res->c_point.p, res->c_dir.p,
                                           res->c_path.p, res->c_mult.p, res->c_hist.p);
    RR_LAUNCH_CHECK();
    s->ctx->launches += 4;
  } else {
    RR_CUDA(cudaMemsetAsync(res->c_off.p, 0, sizeof(int64_t), st));
  }
  tm.mark("trace: captures");
  RR_CUDA(cudaStreamSynchronize(st));
  return res.release();
}

}  // namespace rr
