// Multi-GPU pipeline behind the C ABI: run_trace_pipeline's trace -> image
// sources -> impulse responses (pipeline.cpp:163-175) over the ranks of an
// NCCL communicator, one process or thread per GPU.
//
// The reference is single-process; its trace() chunks the rays over host
// threads (tracer.cpp:82-105).  Here each rank holds the replicated mesh and
// tree and traces a block-cyclic shard of the global Fibonacci lattice
// (4 096-ray blocks) with no communication.  The one exchange step:
//  1. order classes: each receiver's per-order capture histogram is summed
//     over the ranks (ncclAllReduce) and the (receiver, order class) units
//     are assigned to ranks jointly by a deterministic longest-processing-
//     time rule (C3: 5 receivers with ~4 populated orders each balance to
//     1.00 at 8 ranks, where per-receiver ownership left 2.8-3.3x).
//     Grouping (exact face path), group splitting and the coplanar merge
//     only ever combine captures / images of one order
//     (image_sources.cpp:87-90, 111-116), so a class is a closed unit and
//     its result does not depend on the number of ranks;
//  2. captures go to their class owner: a stable radix sort by destination,
//     a packing kernel (global ray index, order, point, direction, path,
//     multipliers, face history CSR), grouped ncclSend / ncclRecv of every
//     field (an all-to-all with uneven splits);
//  3. owners rebuild the reference capture order (rr_captures_import: radix
//     sort by (ray, order)) and build their image sources (K5, energy with
//     the global ray count);
//  4. impulse responses: the fixed-point scale of K6 is made global (max
//     amplitude max-reduced, image count sum-reduced), each rank bins its
//     images, the 64-bit integer histograms are summed exactly
//     (ncclAllReduce), converted, and every rank runs the FIR (K7): the
//     result is bit-identical to one GPU's;
//  5. image lists are gathered to rank 0 (ncclSend / ncclRecv) and stably
//     sorted by order class; within a class the owner's list already is in
//     the reference (order, distance, path) order (image_sources.cpp:163-168).
// A communicator of one rank runs the same exchange (tests); no communicator
// runs the plain single-GPU pipeline.  NCCL errors surface as RR_NCCL.
#include <cub/cub.cuh>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <tuple>
#include <numeric>
#include <vector>

#include "rr_trace.cuh"

// In-process loopback "communicator" for testing the multi-rank exchange on
// one GPU: every rank is a host thread with its own context (same device);
// the collectives rendezvous on the hub and move data with device copies.
// Only the NCCL calls themselves are bypassed (rr_comm_init_loopback).
struct rr_hub {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const void*> ptr;                                      // per rank: published buffer
  std::vector<std::vector<std::tuple<int, const void*, size_t>>> sends;  // per rank: (peer, buf, bytes)
  explicit rr_hub(int ranks) : n(ranks), ptr(ranks, nullptr), sends(ranks) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct rr_comm {
  rr_ctx* ctx = nullptr;
  ncclComm_t nccl = nullptr;
  rr_hub* hub = nullptr;  // loopback ranks (tests) instead of NCCL
  int rank = 0, nranks = 1;
  // a loopback group's pending point-to-point operations
  std::vector<std::tuple<int, const void*, size_t>> g_send;
  std::vector<std::tuple<int, void*, size_t>> g_recv;
};

struct rr_sharded {
  rr_scene* scene = nullptr;
  int32_t n_recv = 0;
  int64_t length = 0;
  int64_t ray_bounces = 0, n_rays = 0, local_images = 0;
  std::vector<rr_images*> images;  // per receiver; owned until taken
  rr::DevBuf<double> band_ir, broadband;
  float stage_ms[5] = {0, 0, 0, 0, 0};  // trace, exchange, images, ir, gather
};

#define RR_NCCL_CHECK(x)                                                                       \
  do {                                                                                         \
    ncclResult_t rr_n_ = (x);                                                                  \
    if (rr_n_ != ncclSuccess)                                                                  \
      throw ::rr::Error(RR_NCCL, std::string(#x) + ": " + ncclGetErrorString(rr_n_));          \
  } while (0)

namespace rr {
namespace {

inline unsigned grid(int64_t n, int b = 256) { return static_cast<unsigned>(std::max<int64_t>(1, (n + b - 1) / b)); }

// the trace's local ray index -> global lattice index (rr_trace.cu global_ray)
__device__ __forceinline__ int64_t lattice_index(int64_t first, int64_t stride, int64_t block, int64_t i) {
  if (block > 0) {
    const int64_t blk = i / block, off = i - blk * block;
    return (blk * stride + first) * block + off;
  }
  return first + i * stride;
}

__global__ void range_kernel(const int32_t* __restrict__ recv, int64_t n, int32_t r, int64_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || recv[i] != r) return;
  if (i == 0 || recv[i - 1] != r) out[0] = i;
  if (i == n - 1 || recv[i + 1] != r) out[1] = i + 1;
}

__global__ void order_hist_kernel(const int64_t* __restrict__ off, int64_t c0, int64_t n, int32_t max_order,
                                  unsigned long long* __restrict__ counts) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t o = off[c0 + i + 1] - off[c0 + i];
  atomicAdd(counts + (o < max_order ? o : static_cast<int64_t>(max_order)), 1ull);
}

__global__ void dest_kernel(const int64_t* __restrict__ off, int64_t c0, int64_t n, int32_t max_order,
                            const int32_t* __restrict__ owner, uint32_t* __restrict__ dest, int32_t* __restrict__ idx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t o = off[c0 + i + 1] - off[c0 + i];
  dest[i] = static_cast<uint32_t>(owner[(o < max_order ? o : static_cast<int64_t>(max_order))]);
  idx[i] = static_cast<int32_t>(i);
}

__global__ void send_counts_kernel(const uint32_t* __restrict__ dest_sorted, const int32_t* __restrict__ perm,
                                   const int64_t* __restrict__ off, int64_t c0, int64_t n,
                                   unsigned long long* __restrict__ cnt /* [world][2] */) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t s = c0 + perm[j];
  atomicAdd(cnt + 2 * dest_sorted[j], 1ull);
  atomicAdd(cnt + 2 * dest_sorted[j] + 1, static_cast<unsigned long long>(off[s + 1] - off[s]));
}

// pack receiver r's captures in destination order
__global__ void pack_kernel(const int32_t* __restrict__ perm, int64_t c0, int64_t n, const int32_t* __restrict__ ray,
                            const double* __restrict__ point, const double* __restrict__ dir,
                            const double* __restrict__ path, const double* __restrict__ mult,
                            const int64_t* __restrict__ off, int64_t first, int64_t stride, int64_t block,
                            int32_t* __restrict__ o_ray, int32_t* __restrict__ o_ord, double* __restrict__ o_point,
                            double* __restrict__ o_dir, double* __restrict__ o_path, double* __restrict__ o_mult,
                            int64_t* __restrict__ o_len) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) {
    if (j == n) o_len[n] = 0;
    return;
  }
  const int64_t s = c0 + perm[j];
  o_ray[j] = static_cast<int32_t>(lattice_index(first, stride, block, ray[s]));
  const int64_t o = off[s + 1] - off[s];
  o_ord[j] = static_cast<int32_t>(o);
  o_len[j] = o;
  for (int k = 0; k < 3; ++k) {
    o_point[3 * j + k] = point[3 * s + k];
    o_dir[3 * j + k] = dir[3 * s + k];
  }
  o_path[j] = path[s];
  for (int b = 0; b < kBands; ++b) o_mult[kBands * j + b] = mult[kBands * s + b];
}

__global__ void pack_hist_kernel(const int32_t* __restrict__ perm, int64_t c0, int64_t n,
                                 const int64_t* __restrict__ off, const int32_t* __restrict__ hist,
                                 const int64_t* __restrict__ new_off, int32_t* __restrict__ o_hist) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t s = c0 + perm[j];
  const int64_t a = off[s], len = off[s + 1] - a, d = new_off[j];
  for (int64_t k = 0; k < len; ++k) o_hist[d + k] = hist[a + k];
}

__global__ void ord_to_len_kernel(const int32_t* __restrict__ ord, int64_t n, int64_t* __restrict__ len) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) len[i] = ord[i];
  if (i == n) len[n] = 0;
}

// image gather: per-image path length, then rank 0's stable sort by order
__global__ void path_len_kernel(const int64_t* __restrict__ off, int64_t n, int64_t* __restrict__ len) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) len[i] = off[i + 1] - off[i];
  if (i == n) len[n] = 0;
}

__global__ void order_keys_kernel(const int32_t* __restrict__ order, int64_t n, uint32_t* __restrict__ key,
                                  int32_t* __restrict__ idx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  key[i] = static_cast<uint32_t>(order[i]);
  idx[i] = static_cast<int32_t>(i);
}

template <typename T>
__global__ void gather_rows_kernel(const int32_t* __restrict__ perm, int64_t n, int w, const T* __restrict__ in,
                                   T* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * w) return;
  const int64_t r = i / w, c = i - r * w;
  out[i] = in[static_cast<int64_t>(perm[r]) * w + c];
}

__global__ void gather_len_kernel(const int32_t* __restrict__ perm, int64_t n, const int64_t* __restrict__ len_in,
                                  int64_t* __restrict__ len_out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) len_out[i] = len_in[perm[i]];
  if (i == n) len_out[n] = 0;
}

__global__ void gather_path_kernel(const int32_t* __restrict__ perm, int64_t n, const int64_t* __restrict__ off_in,
                                   const int32_t* __restrict__ path_in, const int64_t* __restrict__ off_out,
                                   int32_t* __restrict__ path_out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t a = off_in[perm[i]], len = off_in[perm[i] + 1] - a, d = off_out[i];
  for (int64_t k = 0; k < len; ++k) path_out[d + k] = path_in[a + k];
}

template <typename F>
void cub_call(F&& f, DevBuf<uint8_t>& tmp, cudaStream_t st) {
  size_t need = 0;
  RR_CUDA(f(nullptr, need));
  if (need > tmp.n) tmp.alloc(need + 16, st);
  size_t have = tmp.n;
  RR_CUDA(f(tmp.p, have));
}

void exclusive_sum(const int64_t* in, int64_t* out, int64_t n, DevBuf<uint8_t>& tmp, cudaStream_t st) {
  cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, in, out, static_cast<int>(n), st); },
           tmp, st);
}

template <typename T>
ncclDataType_t nccl_type();
template <>
ncclDataType_t nccl_type<double>() { return ncclFloat64; }
template <>
ncclDataType_t nccl_type<int32_t>() { return ncclInt32; }
template <>
ncclDataType_t nccl_type<int64_t>() { return ncclInt64; }

// ---- collectives: NCCL, or the loopback hub (tests)
__global__ void u64_reduce_kernel(const unsigned long long* const* __restrict__ src, int n_src, int64_t count,
                                  int op_max, unsigned long long* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  unsigned long long v = src[0][i];
  for (int r = 1; r < n_src; ++r) v = op_max ? max(v, src[r][i]) : v + src[r][i];
  out[i] = v;
}

void allreduce_u64(rr_comm* cm, unsigned long long* buf, int64_t count, bool op_max, cudaStream_t st) {
  if (!cm->hub) {
    RR_NCCL_CHECK(ncclAllReduce(buf, buf, count, ncclUint64, op_max ? ncclMax : ncclSum, cm->nccl, st));
    return;
  }
  rr_hub* h = cm->hub;
  RR_CUDA(cudaStreamSynchronize(st));
  h->ptr[cm->rank] = buf;
  h->barrier();
  DevBuf<unsigned long long> tmp;
  DevBuf<const unsigned long long*> srcs;
  tmp.alloc(std::max<int64_t>(count, 1), st);
  srcs.alloc(h->n, st);
  std::vector<const unsigned long long*> hs(h->n);
  for (int r = 0; r < h->n; ++r) hs[r] = static_cast<const unsigned long long*>(h->ptr[r]);
  RR_CUDA(cudaMemcpyAsync(srcs.p, hs.data(), sizeof(void*) * h->n, cudaMemcpyHostToDevice, st));
  u64_reduce_kernel<<<grid(count), 256, 0, st>>>(srcs.p, h->n, count, op_max ? 1 : 0, tmp.p);
  RR_LAUNCH_CHECK();
  RR_CUDA(cudaStreamSynchronize(st));
  h->barrier();  // every rank has read every buffer
  RR_CUDA(cudaMemcpyAsync(buf, tmp.p, sizeof(unsigned long long) * count, cudaMemcpyDeviceToDevice, st));
  RR_CUDA(cudaStreamSynchronize(st));
  h->barrier();
}

void allgather_u64(rr_comm* cm, const unsigned long long* send, unsigned long long* recv, int64_t count,
                   cudaStream_t st) {
  if (!cm->hub) {
    RR_NCCL_CHECK(ncclAllGather(send, recv, count, ncclUint64, cm->nccl, st));
    return;
  }
  rr_hub* h = cm->hub;
  RR_CUDA(cudaStreamSynchronize(st));
  h->ptr[cm->rank] = send;
  h->barrier();
  for (int r = 0; r < h->n; ++r)
    RR_CUDA(cudaMemcpyAsync(recv + r * count, h->ptr[r], sizeof(unsigned long long) * count,
                            cudaMemcpyDeviceToDevice, st));
  RR_CUDA(cudaStreamSynchronize(st));
  h->barrier();
}

void group_start(rr_comm* cm) {
  if (!cm->hub) {
    RR_NCCL_CHECK(ncclGroupStart());
    return;
  }
  cm->g_send.clear();
  cm->g_recv.clear();
}

template <typename T>
void p2p_send(rr_comm* cm, const T* buf, size_t n, int peer, cudaStream_t st) {
  if (!cm->hub) {
    RR_NCCL_CHECK(ncclSend(buf, n, nccl_type<T>(), peer, cm->nccl, st));
    return;
  }
  cm->g_send.emplace_back(peer, buf, n * sizeof(T));
}

template <typename T>
void p2p_recv(rr_comm* cm, T* buf, size_t n, int peer, cudaStream_t st) {
  if (!cm->hub) {
    RR_NCCL_CHECK(ncclRecv(buf, n, nccl_type<T>(), peer, cm->nccl, st));
    return;
  }
  cm->g_recv.emplace_back(peer, buf, n * sizeof(T));
}

// the k-th receive from rank q matches q's k-th send to this rank
void group_end(rr_comm* cm, cudaStream_t st) {
  if (!cm->hub) {
    RR_NCCL_CHECK(ncclGroupEnd());
    return;
  }
  rr_hub* h = cm->hub;
  RR_CUDA(cudaStreamSynchronize(st));
  h->sends[cm->rank] = cm->g_send;
  h->barrier();
  std::vector<int> used(h->n, 0);
  for (const auto& rv : cm->g_recv) {
    const int q = std::get<0>(rv);
    int k = -1;
    for (int seen = 0, j = 0; j < static_cast<int>(h->sends[q].size()); ++j)
      if (std::get<0>(h->sends[q][j]) == cm->rank && seen++ == used[q]) {
        k = j;
        break;
      }
    if (k < 0) throw Error(RR_NCCL, "loopback: receive without a matching send");
    ++used[q];
    const auto& sd = h->sends[q][k];
    if (std::get<2>(sd) != std::get<2>(rv)) throw Error(RR_NCCL, "loopback: send / receive sizes differ");
    RR_CUDA(cudaMemcpyAsync(std::get<1>(rv), std::get<1>(sd), std::get<2>(rv), cudaMemcpyDeviceToDevice, st));
  }
  RR_CUDA(cudaStreamSynchronize(st));
  h->barrier();
}

// rows of `w` elements: send `sn[q]` rows to rank q from consecutive blocks,
// receive `rn[q]` rows from rank q into consecutive blocks (caller groups)
template <typename T>
void a2a_rows(rr_comm* cm, const T* send, const std::vector<int64_t>& sn, T* recv, const std::vector<int64_t>& rn,
              int64_t w, cudaStream_t st) {
  int64_t so = 0, ro = 0;
  for (int q = 0; q < cm->nranks; ++q) {
    if (q == cm->rank) {
      if (sn[q] != rn[q]) throw Error(RR_RUNTIME, "exchange: self counts disagree");
      if (sn[q])
        RR_CUDA(cudaMemcpyAsync(recv + ro * w, send + so * w, sizeof(T) * sn[q] * w, cudaMemcpyDeviceToDevice, st));
    } else {
      if (sn[q]) p2p_send<T>(cm, send + so * w, static_cast<size_t>(sn[q] * w), q, st);
      if (rn[q]) p2p_recv<T>(cm, recv + ro * w, static_cast<size_t>(rn[q] * w), q, st);
    }
    so += sn[q];
    ro += rn[q];
  }
}

// deterministic LPT: classes by decreasing count (ties: lower order first)
// to the least-loaded rank (ties: lower rank) -- shard.py assign_orders
std::vector<int32_t> assign_orders(const std::vector<unsigned long long>& counts, int world) {
  std::vector<int32_t> cls(counts.size());
  std::iota(cls.begin(), cls.end(), 0);
  std::stable_sort(cls.begin(), cls.end(), [&](int a, int b) { return counts[a] > counts[b]; });
  std::vector<unsigned long long> load(world, 0);
  std::vector<int32_t> owner(counts.size(), 0);
  for (int o : cls) {
    int r = 0;
    for (int q = 1; q < world; ++q)
      if (load[q] < load[r]) r = q;
    owner[o] = r;
    load[r] += counts[o];
  }
  return owner;
}

struct Timer {
  cudaStream_t st;
  std::vector<cudaEvent_t> ev;
  explicit Timer(cudaStream_t s) : st(s) { mark(); }
  void mark() {
    cudaEvent_t e;
    RR_CUDA(cudaEventCreate(&e));
    RR_CUDA(cudaEventRecord(e, st));
    ev.push_back(e);
  }
  ~Timer() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
};

// the exchange of receiver r's captures; returns the imported trace on
// this rank (its order classes, reference order)
// receiver r's range [c0, c0 + n) of the (receiver, ray, order)-sorted captures
void receiver_range(rr_trace_result* tr, int32_t r, int64_t* c0, int64_t* n) {
  cudaStream_t st = tr->scene->ctx->stream;
  const int64_t nc_all = tr->stats.n_captures;
  int64_t range[2] = {0, 0};
  if (nc_all) {
    DevBuf<int64_t> dr;
    dr.alloc(2, st);
    RR_CUDA(cudaMemsetAsync(dr.p, 0, 2 * sizeof(int64_t), st));
    range_kernel<<<grid(nc_all), 256, 0, st>>>(tr->c_recv.p, nc_all, r, dr.p);
    RR_LAUNCH_CHECK();
    RR_CUDA(cudaMemcpyAsync(range, dr.p, sizeof range, cudaMemcpyDeviceToHost, st));
    RR_CUDA(cudaStreamSynchronize(st));
  }
  *c0 = range[0];
  *n = range[1] - range[0];
}

// ownership of every (receiver, order class) unit: per-receiver order
// histograms summed over the ranks (one all-reduce), then the deterministic
// LPT rule over all units jointly -- several receivers' classes spread over
// the ranks even when each receiver has few populated orders (C3: 5
// receivers, orders 0-3) -- owner[r * (max_order + 1) + o]
std::vector<int32_t> assign_units(rr_comm* cm, rr_trace_result* tr, int32_t n_recv, int32_t max_order) {
  cudaStream_t st = tr->scene->ctx->stream;
  const int64_t per = max_order + 1;
  DevBuf<unsigned long long> counts;
  counts.alloc(n_recv * per, st);
  RR_CUDA(cudaMemsetAsync(counts.p, 0, counts.bytes(), st));
  for (int32_t r = 0; r < n_recv; ++r) {
    int64_t c0, n;
    receiver_range(tr, r, &c0, &n);
    if (n) order_hist_kernel<<<grid(n), 256, 0, st>>>(tr->c_off.p, c0, n, max_order, counts.p + r * per);
    RR_LAUNCH_CHECK();
  }
  allreduce_u64(cm, counts.p, n_recv * per, false, st);
  std::vector<unsigned long long> h(n_recv * per);
  RR_CUDA(cudaMemcpyAsync(h.data(), counts.p, counts.bytes(), cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  return assign_orders(h, cm->nranks);
}

std::unique_ptr<rr_trace_result> exchange_captures(rr_comm* cm, rr_trace_result* tr, int32_t r,
                                                   const rr_receiver& receiver, int32_t max_order,
                                                   const int32_t* owner_row) {
  rr_scene* s = tr->scene;
  cudaStream_t st = s->ctx->stream;
  const int world = cm->nranks;
  DevBuf<uint8_t> tmp;
  int64_t c0, n;
  receiver_range(tr, r, &c0, &n);
  DevBuf<int32_t> d_owner;
  d_owner.alloc(max_order + 1, st);
  RR_CUDA(cudaMemcpyAsync(d_owner.p, owner_row, sizeof(int32_t) * (max_order + 1), cudaMemcpyHostToDevice, st));
  // 2. destination order (stable), counts, packing
  DevBuf<uint32_t> dest, dest_s;
  DevBuf<int32_t> idx, perm;
  dest.alloc(std::max<int64_t>(n, 1), st);
  dest_s.alloc(std::max<int64_t>(n, 1), st);
  idx.alloc(std::max<int64_t>(n, 1), st);
  perm.alloc(std::max<int64_t>(n, 1), st);
  DevBuf<unsigned long long> sc;
  sc.alloc(2 * world, st);
  RR_CUDA(cudaMemsetAsync(sc.p, 0, sc.bytes(), st));
  if (n) {
    dest_kernel<<<grid(n), 256, 0, st>>>(tr->c_off.p, c0, n, max_order, d_owner.p, dest.p, idx.p);
    RR_LAUNCH_CHECK();
    int bits = 1;
    while ((1 << bits) < world) ++bits;
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, dest.p, dest_s.p, idx.p, perm.p, static_cast<int>(n), 0, bits, st);
    }, tmp, st);
    send_counts_kernel<<<grid(n), 256, 0, st>>>(dest_s.p, perm.p, tr->c_off.p, c0, n, sc.p);
    RR_LAUNCH_CHECK();
  }
  // counts of every rank to every rank
  DevBuf<unsigned long long> all_sc;
  all_sc.alloc(2 * world * world, st);
  allgather_u64(cm, sc.p, all_sc.p, 2 * world, st);
  std::vector<unsigned long long> h_all(2 * world * world);
  RR_CUDA(cudaMemcpyAsync(h_all.data(), all_sc.p, all_sc.bytes(), cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> sn(world), sh(world), rn(world), rh(world);
  for (int q = 0; q < world; ++q) {
    sn[q] = static_cast<int64_t>(h_all[2 * world * cm->rank + 2 * q]);
    sh[q] = static_cast<int64_t>(h_all[2 * world * cm->rank + 2 * q + 1]);
    rn[q] = static_cast<int64_t>(h_all[2 * world * q + 2 * cm->rank]);
    rh[q] = static_cast<int64_t>(h_all[2 * world * q + 2 * cm->rank + 1]);
  }
  const int64_t total_h = std::accumulate(sh.begin(), sh.end(), int64_t(0));
  DevBuf<int32_t> s_ray, s_ord, s_hist;
  DevBuf<double> s_point, s_dir, s_path, s_mult;
  DevBuf<int64_t> s_len, s_off;
  s_ray.alloc(std::max<int64_t>(n, 1), st);
  s_ord.alloc(std::max<int64_t>(n, 1), st);
  s_point.alloc(3 * std::max<int64_t>(n, 1), st);
  s_dir.alloc(3 * std::max<int64_t>(n, 1), st);
  s_path.alloc(std::max<int64_t>(n, 1), st);
  s_mult.alloc(kBands * std::max<int64_t>(n, 1), st);
  s_len.alloc(n + 1, st);
  s_off.alloc(n + 1, st);
  s_hist.alloc(std::max<int64_t>(total_h, 1), st);
  const TraceParams& P = tr->params;
  pack_kernel<<<grid(n + 1), 256, 0, st>>>(perm.p, c0, n, tr->c_ray.p, tr->c_point.p, tr->c_dir.p, tr->c_path.p,
                                            tr->c_mult.p, tr->c_off.p, P.first, P.stride, P.block, s_ray.p, s_ord.p,
                                            s_point.p, s_dir.p, s_path.p, s_mult.p, s_len.p);
  RR_LAUNCH_CHECK();
  exclusive_sum(s_len.p, s_off.p, n + 1, tmp, st);
  if (n) pack_hist_kernel<<<grid(n), 256, 0, st>>>(perm.p, c0, n, tr->c_off.p, tr->c_hist.p, s_off.p, s_hist.p);
  RR_LAUNCH_CHECK();
  s->ctx->launches += 8;
  // 3. all-to-all of every field (one NCCL group)
  const int64_t m = std::accumulate(rn.begin(), rn.end(), int64_t(0));
  const int64_t mh = std::accumulate(rh.begin(), rh.end(), int64_t(0));
  DevBuf<int32_t> r_ray, r_ord, r_hist;
  DevBuf<double> r_point, r_dir, r_path, r_mult;
  r_ray.alloc(std::max<int64_t>(m, 1), st);
  r_ord.alloc(std::max<int64_t>(m, 1), st);
  r_point.alloc(3 * std::max<int64_t>(m, 1), st);
  r_dir.alloc(3 * std::max<int64_t>(m, 1), st);
  r_path.alloc(std::max<int64_t>(m, 1), st);
  r_mult.alloc(kBands * std::max<int64_t>(m, 1), st);
  r_hist.alloc(std::max<int64_t>(mh, 1), st);
  group_start(cm);
  a2a_rows<int32_t>(cm, s_ray.p, sn, r_ray.p, rn, 1, st);
  a2a_rows<int32_t>(cm, s_ord.p, sn, r_ord.p, rn, 1, st);
  a2a_rows<double>(cm, s_point.p, sn, r_point.p, rn, 3, st);
  a2a_rows<double>(cm, s_dir.p, sn, r_dir.p, rn, 3, st);
  a2a_rows<double>(cm, s_path.p, sn, r_path.p, rn, 1, st);
  a2a_rows<double>(cm, s_mult.p, sn, r_mult.p, rn, kBands, st);
  a2a_rows<int32_t>(cm, s_hist.p, sh, r_hist.p, rh, 1, st);
  group_end(cm, st);
  // 4. history offsets of the received records, then the reference order
  DevBuf<int64_t> r_len, r_off;
  r_len.alloc(m + 1, st);
  r_off.alloc(m + 1, st);
  ord_to_len_kernel<<<grid(m + 1), 256, 0, st>>>(r_ord.p, m, r_len.p);
  RR_LAUNCH_CHECK();
  exclusive_sum(r_len.p, r_off.p, m + 1, tmp, st);
  s->ctx->launches += 2;
  rr_trace_result* im = import_captures(s, m, nullptr, r_ray.p, r_point.p, r_dir.p, r_path.p, r_mult.p, r_off.p,
                                        r_hist.p, &receiver, 1);
  return std::unique_ptr<rr_trace_result>(im);
}

// receiver's images of every rank to rank 0, stably ordered by order class
rr_images* gather_images(rr_comm* cm, rr_images* local) {
  rr_scene* s = local->scene;
  cudaStream_t st = s->ctx->stream;
  const int world = cm->nranks;
  const int64_t n = local->n;
  DevBuf<uint8_t> tmp;
  DevBuf<int64_t> plen;
  plen.alloc(n + 1, st);
  path_len_kernel<<<grid(n + 1), 256, 0, st>>>(local->path_off.p, n, plen.p);
  RR_LAUNCH_CHECK();
  DevBuf<unsigned long long> mine, all;
  mine.alloc(2, st);
  all.alloc(2 * world, st);
  const unsigned long long h_mine[2] = {static_cast<unsigned long long>(n),
                                        static_cast<unsigned long long>(local->total_path)};
  RR_CUDA(cudaMemcpyAsync(mine.p, h_mine, sizeof h_mine, cudaMemcpyHostToDevice, st));
  allgather_u64(cm, mine.p, all.p, 2, st);
  std::vector<unsigned long long> h_all(2 * world);
  RR_CUDA(cudaMemcpyAsync(h_all.data(), all.p, all.bytes(), cudaMemcpyDeviceToHost, st));
  RR_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> sn(world, 0), sh(world, 0), rn(world, 0), rh(world, 0);
  sn[0] = n;
  sh[0] = local->total_path;
  if (cm->rank == 0)
    for (int q = 0; q < world; ++q) {
      rn[q] = static_cast<int64_t>(h_all[2 * q]);
      rh[q] = static_cast<int64_t>(h_all[2 * q + 1]);
    }
  const int64_t m = std::accumulate(rn.begin(), rn.end(), int64_t(0));
  const int64_t mh = std::accumulate(rh.begin(), rh.end(), int64_t(0));
  DevBuf<double> pos, dist, energy, mult, proj;
  DevBuf<int32_t> ray_count, order, has_proj, path;
  DevBuf<int64_t> len;
  const int64_t m1 = std::max<int64_t>(m, 1);
  pos.alloc(3 * m1, st);
  dist.alloc(m1, st);
  energy.alloc(kBands * m1, st);
  mult.alloc(kBands * m1, st);
  proj.alloc(3 * m1, st);
  ray_count.alloc(m1, st);
  order.alloc(m1, st);
  has_proj.alloc(m1, st);
  len.alloc(m1, st);
  path.alloc(std::max<int64_t>(mh, 1), st);
  group_start(cm);
  a2a_rows<double>(cm, local->pos.p, sn, pos.p, rn, 3, st);
  a2a_rows<double>(cm, local->dist.p, sn, dist.p, rn, 1, st);
  a2a_rows<double>(cm, local->energy.p, sn, energy.p, rn, kBands, st);
  a2a_rows<double>(cm, local->mult.p, sn, mult.p, rn, kBands, st);
  a2a_rows<double>(cm, local->proj.p, sn, proj.p, rn, 3, st);
  a2a_rows<int32_t>(cm, local->ray_count.p, sn, ray_count.p, rn, 1, st);
  a2a_rows<int32_t>(cm, local->order.p, sn, order.p, rn, 1, st);
  a2a_rows<int32_t>(cm, local->has_proj.p, sn, has_proj.p, rn, 1, st);
  a2a_rows<int64_t>(cm, plen.p, sn, len.p, rn, 1, st);
  a2a_rows<int32_t>(cm, local->path.p, sh, path.p, rh, 1, st);
  group_end(cm, st);
  if (cm->rank != 0) {
    RR_CUDA(cudaStreamSynchronize(st));
    return nullptr;
  }
  // rank 0: stable sort by order class, then gather every field
  DevBuf<uint32_t> key, key_s;
  DevBuf<int32_t> idx, perm;
  key.alloc(m1, st);
  key_s.alloc(m1, st);
  idx.alloc(m1, st);
  perm.alloc(m1, st);
  DevBuf<int64_t> off_in, len_s;
  off_in.alloc(m + 1, st);
  len_s.alloc(m + 1, st);
  // offsets of the received paths (len has m entries; a trailing 0 for the scan)
  {
    DevBuf<int64_t> len1;
    len1.alloc(m + 1, st);
    RR_CUDA(cudaMemsetAsync(len1.p, 0, sizeof(int64_t) * (m + 1), st));
    if (m) RR_CUDA(cudaMemcpyAsync(len1.p, len.p, sizeof(int64_t) * m, cudaMemcpyDeviceToDevice, st));
    exclusive_sum(len1.p, off_in.p, m + 1, tmp, st);
  }
  auto out = std::make_unique<rr_images>();
  out->scene = s;
  out->n = m;
  out->total_path = mh;
  out->pos.alloc(3 * m1, st);
  out->dist.alloc(m1, st);
  out->energy.alloc(kBands * m1, st);
  out->mult.alloc(kBands * m1, st);
  out->proj.alloc(3 * m1, st);
  out->ray_count.alloc(m1, st);
  out->order.alloc(m1, st);
  out->has_proj.alloc(m1, st);
  out->path_off.alloc(m + 1, st);
  out->path.alloc(std::max<int64_t>(mh, 1), st);
  if (m) {
    order_keys_kernel<<<grid(m), 256, 0, st>>>(order.p, m, key.p, idx.p);
    RR_LAUNCH_CHECK();
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, key.p, key_s.p, idx.p, perm.p, static_cast<int>(m), 0, 21, st);
    }, tmp, st);
    gather_rows_kernel<double><<<grid(3 * m), 256, 0, st>>>(perm.p, m, 3, pos.p, out->pos.p);
    gather_rows_kernel<double><<<grid(m), 256, 0, st>>>(perm.p, m, 1, dist.p, out->dist.p);
    gather_rows_kernel<double><<<grid(kBands * m), 256, 0, st>>>(perm.p, m, kBands, energy.p, out->energy.p);
    gather_rows_kernel<double><<<grid(kBands * m), 256, 0, st>>>(perm.p, m, kBands, mult.p, out->mult.p);
    gather_rows_kernel<double><<<grid(3 * m), 256, 0, st>>>(perm.p, m, 3, proj.p, out->proj.p);
    gather_rows_kernel<int32_t><<<grid(m), 256, 0, st>>>(perm.p, m, 1, ray_count.p, out->ray_count.p);
    gather_rows_kernel<int32_t><<<grid(m), 256, 0, st>>>(perm.p, m, 1, order.p, out->order.p);
    gather_rows_kernel<int32_t><<<grid(m), 256, 0, st>>>(perm.p, m, 1, has_proj.p, out->has_proj.p);
    gather_len_kernel<<<grid(m + 1), 256, 0, st>>>(perm.p, m, len.p, len_s.p);
    RR_LAUNCH_CHECK();
    exclusive_sum(len_s.p, out->path_off.p, m + 1, tmp, st);
    gather_path_kernel<<<grid(m), 256, 0, st>>>(perm.p, m, off_in.p, path.p, out->path_off.p, out->path.p);
    RR_LAUNCH_CHECK();
    s->ctx->launches += 14;
  } else {
    RR_CUDA(cudaMemsetAsync(out->path_off.p, 0, sizeof(int64_t), st));
  }
  RR_CUDA(cudaStreamSynchronize(st));
  return out.release();
}

}  // namespace

rr_sharded* pipeline_sharded(rr_scene* s, rr_comm* cm, const rr_source* src, const rr_receiver* recv, int32_t n_recv,
                             const rr_trace_config* cfg, const rr_air& air, const rr_cluster_options& opt, double fs,
                             int64_t length, int32_t taps, int32_t block) {
  if (length <= 0) invalid("length must be > 0");
  if (taps < 1) invalid("taps must be >= 1");
  if (block < 1) invalid("block must be >= 1");
  if (cm && cm->ctx != s->ctx) invalid("communicator and scene belong to different contexts");
  rr_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  const int world = cm ? cm->nranks : 1;
  const int rank = cm ? cm->rank : 0;
  auto out = std::make_unique<rr_sharded>();
  out->scene = s;
  out->n_recv = n_recv;
  out->length = length;
  Timer tm(st);
  // trace this rank's block-cyclic shard
  rr_trace_config c = *cfg;
  c.directions = nullptr;
  if (world > 1) {
    c.first = rank;
    c.stride = world;
    c.block = block;
    c.count = 0;
  }
  std::unique_ptr<rr_trace_result> tr(run_trace(s, src, recv, n_recv, &c, nullptr));
  out->ray_bounces = tr->stats.ray_bounces;
  out->n_rays = tr->stats.n_rays;
  tm.mark();
  const int64_t lh = length + taps;
  out->band_ir.alloc(static_cast<size_t>(n_recv) * kBands * length, st);
  out->broadband.alloc(static_cast<size_t>(n_recv) * length, st);
  // exchange every receiver's captures (owners of (receiver, order) units),
  // then build every image list, then reduce / gather per receiver: the image
  // work between the collectives is what the joint ownership balances
  const int32_t max_order = std::max(cfg->max_iterations, 1);
  std::vector<std::unique_ptr<rr_trace_result>> mine(n_recv);
  if (cm) {
    const std::vector<int32_t> owner = assign_units(cm, tr.get(), n_recv, max_order);
    for (int32_t r = 0; r < n_recv; ++r)
      mine[r] = exchange_captures(cm, tr.get(), r, recv[r], max_order, owner.data() + r * (max_order + 1));
  }
  tm.mark();
  std::vector<std::unique_ptr<rr_images>> local(n_recv);
  for (int32_t r = 0; r < n_recv; ++r) {
    local[r].reset(cm ? build_image_sources(mine[r].get(), 0, src->ray_count, air, opt)
                      : build_image_sources(tr.get(), r, src->ray_count, air, opt));
    out->local_images += local[r]->n;
    mine[r].reset();
  }
  tm.mark();
  for (int32_t r = 0; r < n_recv; ++r) {
    // impulse responses: global fixed-point scale, exact integer sum
    DevBuf<unsigned long long> mx, acc;
    mx.alloc(1, st);
    acc.alloc(kBands * lh, st);
    RR_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(unsigned long long), st));
    RR_CUDA(cudaMemsetAsync(acc.p, 0, acc.bytes(), st));
    ir_max_amp(ctx, local[r]->n, local[r]->energy.p, mx.p);
    int64_t n_all = local[r]->n;
    if (cm) {
      DevBuf<unsigned long long> dn;
      dn.alloc(1, st);
      const unsigned long long hn = static_cast<unsigned long long>(local[r]->n);
      RR_CUDA(cudaMemcpyAsync(dn.p, &hn, sizeof hn, cudaMemcpyHostToDevice, st));
      allreduce_u64(cm, mx.p, 1, true, st);
      allreduce_u64(cm, dn.p, 1, false, st);
      unsigned long long h = 0;
      RR_CUDA(cudaMemcpyAsync(&h, dn.p, sizeof h, cudaMemcpyDeviceToHost, st));
      RR_CUDA(cudaStreamSynchronize(st));
      n_all = static_cast<int64_t>(h);
    }
    const int64_t n_scale = std::max<int64_t>(n_all, 1);
    ir_bin_fixed(ctx, local[r]->n, local[r]->dist.p, local[r]->energy.p, cfg->speed_of_sound, fs, lh, mx.p, n_scale,
                 acc.p);
    if (cm) allreduce_u64(cm, acc.p, kBands * lh, false, st);
    DevBuf<double> hist;
    hist.alloc(kBands * lh, st);
    ir_unfix(ctx, acc.p, kBands * lh, n_scale, mx.p, hist.p);
    ir_filter(ctx, hist.p, lh, fs, taps, length, out->band_ir.p + static_cast<size_t>(r) * kBands * length,
              out->broadband.p + static_cast<size_t>(r) * length);
  }
  tm.mark();
  for (int32_t r = 0; r < n_recv; ++r) {
    rr_images* merged = cm ? gather_images(cm, local[r].get()) : local[r].release();
    if (!merged) {  // ranks other than 0 hold an empty list
      merged = new rr_images();
      merged->scene = s;
      merged->path_off.alloc(1, st);
      RR_CUDA(cudaMemsetAsync(merged->path_off.p, 0, sizeof(int64_t), st));
    }
    out->images.push_back(merged);
  }
  tm.mark();
  RR_CUDA(cudaStreamSynchronize(st));
  // stage times: trace, exchange, images, ir, gather (all receivers)
  for (size_t i = 1; i < tm.ev.size() && i <= 5; ++i) {
    float ms = 0.f;
    RR_CUDA(cudaEventElapsedTime(&ms, tm.ev[i - 1], tm.ev[i]));
    out->stage_ms[i - 1] = ms;
  }
  return out.release();
}

}  // namespace rr

// ---------------------------------------------------------------- C ABI
namespace rr {
rr_status abi_guard_nccl(const std::function<void()>& f);
void scene_retain(rr_scene* s);
void scene_drop(rr_scene* s);
}  // namespace rr

extern "C" {

rr_status rr_comm_unique_id(uint8_t* id) {
  return rr::abi_guard_nccl([&] {
    if (!id) rr::invalid("id must not be null");
    static_assert(sizeof(ncclUniqueId) == RR_NCCL_ID_BYTES, "NCCL unique id size");
    ncclUniqueId u;
    RR_NCCL_CHECK(ncclGetUniqueId(&u));
    std::memcpy(id, &u, sizeof u);
  });
}

rr_status rr_comm_init(rr_ctx* ctx, const uint8_t* id, int32_t nranks, int32_t rank, rr_comm** out) {
  return rr::abi_guard_nccl([&] {
    if (!ctx || !id || !out) rr::invalid("ctx, id and out must not be null");
    if (nranks < 1 || rank < 0 || rank >= nranks) rr::invalid("rank out of range");
    RR_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    auto c = std::make_unique<rr_comm>();
    c->ctx = ctx;
    c->rank = rank;
    c->nranks = nranks;
    RR_NCCL_CHECK(ncclCommInitRank(&c->nccl, nranks, u, rank));
    ctx->refs++;
    *out = c.release();
  });
}

rr_status rr_hub_create(int32_t nranks, rr_hub** out) {
  return rr::abi_guard_nccl([&] {
    if (!out || nranks < 1) rr::invalid("nranks must be >= 1");
    *out = new rr_hub(nranks);
  });
}

rr_status rr_hub_destroy(rr_hub* hub) {
  return rr::abi_guard_nccl([&] { delete hub; });
}

rr_status rr_comm_init_loopback(rr_ctx* ctx, rr_hub* hub, int32_t rank, rr_comm** out) {
  return rr::abi_guard_nccl([&] {
    if (!ctx || !hub || !out) rr::invalid("ctx, hub and out must not be null");
    if (rank < 0 || rank >= hub->n) rr::invalid("rank out of range");
    auto c = std::make_unique<rr_comm>();
    c->ctx = ctx;
    c->hub = hub;
    c->rank = rank;
    c->nranks = hub->n;
    ctx->refs++;
    *out = c.release();
  });
}

rr_status rr_comm_info(rr_comm* comm, int32_t* rank, int32_t* nranks) {
  return rr::abi_guard_nccl([&] {
    if (!comm) rr::invalid("comm must not be null");
    if (rank) *rank = comm->rank;
    if (nranks) *nranks = comm->nranks;
  });
}

rr_status rr_comm_destroy(rr_comm* comm) {
  return rr::abi_guard_nccl([&] {
    if (!comm) return;
    rr_ctx* ctx = comm->ctx;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    const ncclResult_t r = comm->nccl ? ncclCommDestroy(comm->nccl) : ncclSuccess;
    delete comm;
    rr_ctx_destroy(ctx);  // drops the reference taken by rr_comm_init
    if (r != ncclSuccess) throw rr::Error(RR_NCCL, std::string("ncclCommDestroy: ") + ncclGetErrorString(r));
  });
}

rr_status rr_pipeline_sharded(rr_scene* scene, rr_comm* comm, const rr_source* source, const rr_receiver* receivers,
                              int32_t n_recv, const rr_trace_config* cfg, const rr_air* air,
                              const rr_cluster_options* opt, double fs, int64_t length, int32_t taps, int32_t block,
                              rr_sharded** out) {
  return rr::abi_guard_nccl([&] {
    if (!scene || !source || !receivers || !cfg || !air || !out) rr::invalid("null argument");
    rr_cluster_options o{1e-6, 0};
    if (opt) o = *opt;
    RR_CUDA(cudaSetDevice(scene->ctx->device));
    rr_sharded* sh = rr::pipeline_sharded(scene, comm, source, receivers, n_recv, cfg, *air, o, fs, length, taps,
                                          block);
    rr::scene_retain(scene);
    for (size_t i = 0; i < sh->images.size(); ++i) rr::scene_retain(scene);  // each image list holds the scene
    *out = sh;
  });
}

rr_status rr_sharded_info(rr_sharded* sh, int64_t* ray_bounces, int64_t* n_rays, int64_t* local_images,
                          float* stage_ms) {
  return rr::abi_guard_nccl([&] {
    if (!sh) rr::invalid("result must not be null");
    if (ray_bounces) *ray_bounces = sh->ray_bounces;
    if (n_rays) *n_rays = sh->n_rays;
    if (local_images) *local_images = sh->local_images;
    if (stage_ms) std::memcpy(stage_ms, sh->stage_ms, sizeof sh->stage_ms);
  });
}

rr_status rr_sharded_take_images(rr_sharded* sh, int32_t recv, rr_images** out) {
  return rr::abi_guard_nccl([&] {
    if (!sh || !out) rr::invalid("null argument");
    if (recv < 0 || recv >= sh->n_recv) rr::invalid("receiver index out of range");
    if (!sh->images[recv]) rr::invalid("image list already taken");
    *out = sh->images[recv];
    sh->images[recv] = nullptr;
  });
}

rr_status rr_sharded_ir(rr_sharded* sh, int32_t recv, double* band_ir, double* broadband) {
  return rr::abi_guard_nccl([&] {
    if (!sh) rr::invalid("result must not be null");
    if (recv < 0 || recv >= sh->n_recv) rr::invalid("receiver index out of range");
    cudaStream_t st = sh->scene->ctx->stream;
    const size_t L = static_cast<size_t>(sh->length);
    if (band_ir)
      RR_CUDA(cudaMemcpyAsync(band_ir, sh->band_ir.p + recv * rr::kBands * L, sizeof(double) * rr::kBands * L,
                              cudaMemcpyDefault, st));
    if (broadband)
      RR_CUDA(cudaMemcpyAsync(broadband, sh->broadband.p + recv * L, sizeof(double) * L, cudaMemcpyDefault, st));
    RR_CUDA(cudaStreamSynchronize(st));
  });
}

rr_status rr_sharded_destroy(rr_sharded* sh) {
  return rr::abi_guard_nccl([&] {
    if (!sh) return;
    rr_scene* s = sh->scene;
    cudaSetDevice(s->ctx->device);
    for (rr_images* im : sh->images)
      if (im) {
        delete im;
        rr::scene_drop(s);
      }
    delete sh;
    cudaStreamSynchronize(s->ctx->stream);
    rr::scene_drop(s);
  });
}

}  // extern "C"
