// Trace-result layout shared by rr_trace.cu, rr_images.cu and rr_api.cu.
#pragma once

#include "rr_geom.cuh"

namespace rr {

constexpr int kMaxRecv = 8;

struct Capture {
  double p[3];
  double d[3];
  double path;
  int32_t ray;   // local ray index (row of the history table)
  int32_t meta;  // order << 8 | receiver
};
static_assert(sizeof(Capture) == 64, "capture record");

struct TraceParams {
  const TNode* nodes;
  const QNode* qnodes;
  const QNode* q4;   // 4-wide collapse of the SAH tree
  int32_t root4;
  const WNode* wnodes;  // 8-wide compressed collapse of the SAH tree (rr_wide.cu)
  const FaceTri* wtri;  // faces in its leaf order
  int32_t n_wnodes;     // (bounds checks of the checked build)
  int64_t nf;
  int32_t wide;  // 1: traverse the 4-wide QNodes, 0: the binary TNodes
  const FaceTri* tri;
  const float4* tri32;
  const int32_t* face_plane;
  const double* normal;
  TravHeader hdr;
  int32_t use_smem;
  // lattice: local ray i -> global index via (first, stride, block)
  double src[3];
  int64_t N;
  int64_t count;
  int64_t first, stride, block;
  double az_step;  // 2*pi*(1 - 1/golden) evaluated on the host
  const double* dirs;  // optional explicit directions (count*3), else lattice
  const int32_t* order;  // optional work order: the c-th ray taken is order[c] (spatially coherent warps)
  int32_t n_recv;
  double rc[kMaxRecv][3];
  double rr[kMaxRecv];
  int32_t max_iter;
  double rng[kMaxRecv];  // capture range per receiver: resolved_max_range (tracer.cpp:10-15) of each
  double max_range;      // kill range: the largest of rng (a receiver never alters a ray)
  double cull_min;       // coplanar-subtree cull only when |d_axis| exceeds this (see run_trace)
  int32_t* hist;  // count * H
  int64_t H;
  Capture* caps;
  unsigned long long* cap_count;
  int64_t cap_capacity;
  unsigned long long* ray_counter;
  unsigned long long* stats;  // 0 bounces, 1 escaped, 2 out_of_range, 3 alive, 4 max steps, 5 visits, 6 leaves
};

}  // namespace rr

struct rr_trace_result {
  rr_scene* scene = nullptr;
  rr_trace_stats stats{};
  float kernel_ms = 0.f;
  rr::TraceParams params{};
  rr::DevBuf<int32_t> hist;
  rr::DevBuf<int32_t> c_recv, c_ray, c_hist;
  rr::DevBuf<double> c_point, c_dir, c_path, c_mult;
  rr::DevBuf<int64_t> c_off;
  std::vector<double> recv_center, recv_radius;
};


namespace rr {
rr_trace_result* run_trace(rr_scene* s, const rr_source* src, const rr_receiver* recv, int32_t n_recv,
                           const rr_trace_config* cfg, const double* d_dirs);
// rr_step.cu
rr_trace_result* step_rays(rr_scene* s, int64_t n, double* origin, double* dir, double* mult, double* path,
                           int32_t* alive, int32_t* hist, int32_t* n_hist, int32_t hist_cap, const rr_receiver* recv,
                           const rr_trace_config* cfg, int32_t brute, float* kernel_ms);
// rr_import.cu
rr_trace_result* import_captures(rr_scene* s, int64_t n, const int32_t* recv, const int32_t* ray, const double* point,
                                 const double* dir, const double* path, const double* mult, const int64_t* hist_off,
                                 const int32_t* hist, const rr_receiver* receivers, int32_t n_recv);
}  // namespace rr

// Device image-source set (rr_images.cu), sorted by (order, distance, path).
struct rr_images {
  rr_scene* scene = nullptr;
  int64_t n = 0, total_path = 0;
  rr::DevBuf<double> pos, dist, energy, mult, proj;
  rr::DevBuf<int32_t> ray_count, order, has_proj, path;
  rr::DevBuf<int64_t> path_off;
  cudaEvent_t copies_done = nullptr;  // last rr_images_get_async on a caller stream
};

namespace rr {
rr_images* build_image_sources(rr_trace_result* tr, int32_t recv, int64_t total_rays, const rr_air& air,
                               const rr_cluster_options& opt);
}  // namespace rr

// Shoebox mirror-lattice oracle and matcher (rr_shoebox.cu).
struct rr_lattice {
  rr_ctx* ctx = nullptr;
  int64_t n = 0;
  rr::DevBuf<double> pos, dist, energy;
  rr::DevBuf<int32_t> order, hits;
};

struct rr_match {
  rr_ctx* ctx = nullptr;
  int64_t n_matched = 0, n_members = 0, n_unmatched_oracle = 0, n_unmatched_traced = 0;
  double max_position_error = 0.0, pos_tol = 0.0, energy_tol_db = 0.0;
  double rms_db[rr::kBands] = {};
  rr::DevBuf<int32_t> oracle_index, order, members, unmatched_oracle, unmatched_traced;
  rr::DevBuf<int64_t> member_off;
  rr::DevBuf<double> pos_err, delta_db;
};

namespace rr {
rr_lattice* enumerate_lattice(rr_ctx* ctx, const double* dims, const double* walls_alpha, const double* source,
                              const double* receiver, double max_distance, double receiver_radius, const rr_air& air);
rr_match* compare_lattice(rr_ctx* ctx, int64_t no, const double* opos, const double* oenergy, const int32_t* oorder,
                          int64_t nt, const double* tpos, const double* tenergy, double pos_tol, double energy_tol_db);
void air_beta_bands(const rr_air& a, double* beta);
}  // namespace rr

namespace rr {
// rr_trace.cu: the tracer's own lattice evaluation, for rr_fibonacci_directions
void fibonacci_device(rr_ctx* ctx, int64_t n, int64_t first, int64_t stride, int64_t count, double* out);
double air_alpha(const rr_air& a, double f);
void air_validate(const rr_air& a);
// rr_metrics.cu
void band_schroeder(rr_ctx* ctx, const int64_t* band_off, const double* amplitude, double* level);
}  // namespace rr
