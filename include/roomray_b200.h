/* roomray_b200 — C ABI of the B200-native specular ray / image-source engine.
 *
 * Drop-in boundary for the reference's hot path (reference = roomray, C++20,
 * /root/reference/proj).  Every entry point names the reference interface it
 * replaces.  Plain pointers and sizes only; all host buffers are caller-owned.
 * Calls are synchronous with respect to the host unless the name ends in
 * _async; a context owns one CUDA stream and is not thread-safe (use one
 * context per thread/GPU).  Errors: every call returns an rr_status; the
 * message of the last failure on the calling thread is rr_last_error().
 * RR_INVALID_ARGUMENT corresponds to the reference's std::invalid_argument.
 */
#ifndef ROOMRAY_B200_H
#define ROOMRAY_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RR_NUM_BANDS 8

typedef enum {
  RR_OK = 0,
  RR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  RR_RUNTIME = 2,          /* reference: other std::exception */
  RR_CUDA = 3,
  RR_NCCL = 4
} rr_status;

typedef struct rr_ctx rr_ctx;
typedef struct rr_scene rr_scene;
typedef struct rr_trace_result rr_trace_result;
typedef struct rr_images rr_images;
typedef struct rr_lattice rr_lattice;
typedef struct rr_match rr_match;
typedef struct rr_comm rr_comm;
typedef struct rr_sharded rr_sharded;
typedef struct rr_hub rr_hub;

/* Reference-layout tree node (TreeNode, accel_tree.hpp:15-22): post-order,
 * root last, leaves hold one face. */
typedef struct {
  double lo[3], hi[3];
  int32_t left, right, face_index, pad;
} rr_tree_node;

/* SourceConfig (emission.hpp:14-20). */
typedef struct {
  double position[3];
  int64_t ray_count;
} rr_source;

/* Receiver (tracer_types.hpp:21-24). */
typedef struct {
  double center[3];
  double radius;
} rr_receiver;

/* TraceConfig (tracer.hpp:13-20) plus the ray-subset selector used for
 * multi-GPU sharding: rays k = first + i*stride (i < count) of the N-ray
 * lattice; stride <= 0 selects all N.  block > 0 selects block-cyclic
 * sharding instead: blocks of `block` consecutive rays, block b owned by
 * rank b % world; `first` is then the rank and `stride` the world size. */
typedef struct {
  int32_t max_iterations;  /* reference default 1000 */
  double speed_of_sound;   /* reference default 343 */
  double max_range;        /* <= 0: (r/2) sqrt(N) of receiver 0 */
  int64_t first, stride, count, block;
  int32_t flags;           /* RR_TRACE_* */
  /* Optional host array (count x 3) of initial directions for the selected
   * rays, the Ray span of step() (tracer.hpp:43); NULL = the Fibonacci
   * lattice evaluated on the device (emission.cpp:17-29, correctly rounded
   * sin/cos). */
  const double* directions;
} rr_trace_config;

#define RR_TRACE_NO_SMEM_CACHE 1 /* traverse without the shared-memory top-level cache */
#define RR_TRACE_KEEP_UNSORTED 2 /* skip the capture sort (timing only) */
#define RR_TRACE_F32_LEAVES 4    /* diagnostic: fp32 leaf classification + fp64 resolution */
#define RR_TRACE_WIDE 8          /* diagnostic: traverse the 4-wide collapse */
#define RR_TRACE_COUNT 16        /* instrumented kernel: count node visits and leaf tests */
#define RR_TRACE_TREE8 32        /* traverse the 8-wide compressed tree at any scene size
                                    (the default from 2^20 faces up) */
#define RR_TRACE_TREE2 64        /* traverse the binary SAH tree at any scene size (the default
                                    below 2^18 faces; 2^18..2^20: its 4-wide collapse) */

/* Statistics of a trace (TraceResult, tracer.hpp:22-29). */
typedef struct {
  int32_t iterations;
  int32_t truncated;
  int64_t escaped;
  int64_t out_of_range;
  double max_range;
  int64_t n_captures;
  int64_t total_history; /* sum of capture face-path lengths */
  int64_t ray_bounces;   /* nearest-hit queries executed on live rays */
  int64_t n_rays;        /* rays traced by this call */
  int64_t node_visits;   /* internal-node visits (RR_TRACE_COUNT), else -1 */
  int64_t leaf_tests;    /* fp64 triangle tests (RR_TRACE_COUNT), else -1 */
  int32_t tree_width;    /* children per node of the traversed tree: 2, 4 or 8 */
  int32_t node_bytes;    /* bytes per node of that tree: 64 (binary), 128 (4-wide), 80 (8-wide) */
} rr_trace_stats;

/* AirModel (air_absorption.hpp:10-23). */
typedef struct {
  int32_t enabled;
  double temperature_c, relative_humidity, pressure_kpa;
} rr_air;

/* ClusterOptions (image_sources.hpp:25-31). */
typedef struct {
  double tol_scale;       /* reference default 1e-6 */
  int32_t merge_coplanar; /* ClusterOptions default 0; RunConfig default 1 */
} rr_cluster_options;

const char* rr_last_error(void);
const char* rr_version(void);

/* ---------------------------------------------------------------- context */
rr_status rr_ctx_create(int device, rr_ctx** out);
rr_status rr_ctx_destroy(rr_ctx* ctx);
/* The context's CUDA stream (cudaStream_t), for event timing by callers. */
void* rr_ctx_stream(rr_ctx* ctx);
/* Number of this library's kernels launched on the context so far. */
int64_t rr_ctx_launches(rr_ctx* ctx);

/* Page-locked host memory (cudaMallocHost) for staging buffers a caller
 * reuses across calls: the copies of rr_scene_create, rr_trace_captures,
 * rr_images_get and rr_images_pulse_trains run at full host-link speed from /
 * into it, where pageable buffers go through the driver's bounce buffer.
 * Not a reference interface (the reference has no device); the C++ façade
 * keeps one grow-only buffer per thread.  bytes == 0 returns NULL. */
rr_status rr_host_alloc(int64_t bytes, void** out);
rr_status rr_host_free(void* p);

/* ---------------------------------------------------------------- scene
 * TriangleMesh (geometry.hpp:60-77) + build_tree (accel_tree.hpp:38).
 * verts: nv*3 f64; tris: nf*4 i32 (a, b, c, material); alpha: nmat*8 f64.
 * Uploads the mesh, validates it on the device (TriangleMesh::validate,
 * geometry.cpp:47-75) when validate != 0, and builds the median-split tree on
 * the device.  nf == 0 fails like build_tree (accel_tree.cpp:71-73). */
rr_status rr_scene_create(rr_ctx* ctx, const double* verts, int64_t nv,
                          const int32_t* tris, int64_t nf, const double* alpha,
                          int32_t nmat, int32_t validate, rr_scene** out);
rr_status rr_scene_destroy(rr_scene* scene);
/* AccelTree::node_count / depth / root (accel_tree.hpp:26-34). */
rr_status rr_scene_tree_info(rr_scene* scene, int64_t* n_nodes, int32_t* root,
                             int32_t* depth);
/* Download the reference-layout tree: 2*nf-1 nodes. */
rr_status rr_scene_tree(rr_scene* scene, rr_tree_node* nodes);
/* Face normals (TriangleMesh::face_normal, geometry.cpp:9-14), nf*3 f64. */
rr_status rr_scene_normals(rr_scene* scene, double* normals);
/* Seconds spent in the device tree build of this scene (CUDA events). */
double rr_scene_build_ms(rr_scene* scene);

/* ---------------------------------------------------------------- queries
 * nearest_hit (accel_tree.hpp:50-51) for n rays; brute == 1 selects
 * nearest_hit_brute (accel_tree.hpp:54-55); 2 / 3 select the diagnostic
 * fp32-leaf / 4-wide traversals.  face[i] = -1 for no hit. */
rr_status rr_nearest_hit_batch(rr_scene* scene, const double* origins,
                               const double* dirs, int64_t n, int32_t brute,
                               int32_t* face, double* delta, double* point);

/* ---------------------------------------------------------------- trace
 * trace (tracer.hpp:50-52) with n_recv receivers traced on the same
 * trajectories (a receiver is transparent, tracer.cpp:27-29).  Captures stay
 * on the device until fetched. */
rr_status rr_trace(rr_scene* scene, const rr_source* source,
                   const rr_receiver* receivers, int32_t n_recv,
                   const rr_trace_config* config, rr_trace_result** out);
rr_status rr_trace_stats_get(rr_trace_result* res, rr_trace_stats* stats);
/* Captures sorted by (receiver, ray, path) (tracer.cpp:143-147).  Host or
 * device destination pointers (UVA).  Arrays:
 * recv/ray n, point/dir n*3, path n, mult n*8, hist_off n+1, hist
 * total_history.  Any pointer may be NULL to skip that field. */
rr_status rr_trace_captures(rr_trace_result* res, int32_t* recv, int32_t* ray,
                            double* point, double* dir, double* path,
                            double* mult, int64_t* hist_off, int32_t* hist);
/* Import caller-held capture records (host or device pointers, UVA) as a
 * trace result, e.g. the captures an owner rank received in the multi-GPU
 * exchange, or the std::vector<Capture> argument of build_image_sources
 * (image_sources.hpp:58-61).  Records are re-sorted into the reference order
 * (receiver, ray, path) (tracer.cpp:143-147).  recv may be NULL (all 0);
 * mult may be NULL (rebuilt from the face history as the ordered product of
 * 1 - alpha, tracer.cpp:57-58).  hist_off has n+1 entries starting at 0. */
rr_status rr_captures_import(rr_scene* scene, int64_t n, const int32_t* recv,
                             const int32_t* ray, const double* point,
                             const double* dir, const double* path,
                             const double* mult, const int64_t* hist_off,
                             const int32_t* hist, const rr_receiver* receivers,
                             int32_t n_recv, rr_trace_result** out);
/* fibonacci_directions (emission.cpp:17-29) as the tracer evaluates it on
 * the device (correctly rounded fp64 sin/cos): directions of lattice
 * indices first + i * stride, i < count, of an n-point lattice, into out
 * (count*3, host or device).  n < 1 -> RR_INVALID_ARGUMENT. */
rr_status rr_fibonacci_directions(rr_ctx* ctx, int64_t n, int64_t first, int64_t stride,
                                  int64_t count, double* out);
/* step (tracer.hpp:43-45): one iteration over n caller rays, in place —
 * the Ray span of the reference (tracer_types.hpp:11-18) as SoA arrays:
 * origin/dir n*3, mult n*8 (band multipliers), path n, alive n, hist
 * n*hist_cap face history with n_hist n entries used.  Host or device
 * arrays (device ones are updated without copies).  brute != 0 selects
 * nearest_hit_brute (the reference's step(tree = nullptr)).  max_range of
 * config (<= 0: (r/2) sqrt(n), tracer.cpp:70-71).  The captures of this
 * iteration, in ray order, come back as a trace result (receiver 0);
 * rr_trace_kernel_ms gives the step kernel's device time. */
rr_status rr_step(rr_scene* scene, int64_t n, double* origin, double* dir,
                  double* mult, double* path, int32_t* alive, int32_t* hist,
                  int32_t* n_hist, int32_t hist_cap,
                  const rr_receiver* receiver, const rr_trace_config* config,
                  int32_t brute, rr_trace_result** out);
/* Device time of the trace kernel itself (ms, CUDA events). */
double rr_trace_kernel_ms(rr_trace_result* res);
rr_status rr_trace_destroy(rr_trace_result* res);

/* ---------------------------------------------------------------- images
 * build_image_sources (image_sources.hpp:58-61) on the device for receiver
 * `recv` of a trace.  total_rays = N of the lattice (energy n/N,
 * image_sources.cpp:138). */
rr_status rr_build_image_sources(rr_trace_result* res, int32_t recv,
                                 int64_t total_rays, const rr_air* air,
                                 const rr_cluster_options* opt,
                                 rr_images** out);
rr_status rr_images_info(rr_images* im, int64_t* n, int64_t* total_path);
/* Sorted by (order, distance, face path) (image_sources.cpp:163-168). */
rr_status rr_images_get(rr_images* im, double* pos, double* dist,
                        double* energy, double* mult, int32_t* ray_count,
                        int32_t* order, int32_t* has_proj, double* proj,
                        int64_t* path_off, int32_t* path);
/* rr_images_get without the host synchronization: the copies are enqueued on
 * `stream` (a cudaStream_t; 0 = the legacy default stream) after the work
 * enqueued so far on the context's stream, so a D2H into pinned memory can
 * overlap later device work (the IR stage).  The caller synchronizes
 * `stream` before reading the outputs; rr_images_destroy may come earlier
 * (its stream-ordered frees wait for the copies). */
rr_status rr_images_get_async(rr_images* im, void* stream, double* pos,
                              double* dist, double* energy, double* mult,
                              int32_t* ray_count, int32_t* order,
                              int32_t* has_proj, double* proj,
                              int64_t* path_off, int32_t* path);
rr_status rr_images_destroy(rr_images* im);

/* ---------------------------------------------------------------- shoebox
 * The analytic mirror-lattice check of a rectangular room (shoebox.hpp).
 * rr_shoebox_images = enumerate_images (shoebox.hpp:38-43,
 * shoebox.cpp:43-116): box [0,L]^3 with walls x0,x1,y0,y1,z0,z1
 * (BoxWall, shoebox.hpp:13), walls_alpha 6*8; every lattice image within
 * max_distance of the receiver, sorted by (distance, lattice cell).  Errors
 * as the reference: dimensions <= 0, source/receiver not strictly inside,
 * max_distance or radius <= 0 -> RR_INVALID_ARGUMENT. */
rr_status rr_shoebox_images(rr_ctx* ctx, const double* dims, const double* walls_alpha,
                            const double* source, const double* receiver,
                            double max_distance, double receiver_radius,
                            const rr_air* air, rr_lattice** out);
rr_status rr_lattice_info(rr_lattice* lat, int64_t* n);
/* Any output may be NULL.  wall_hits 6 per image, energy 8 per image. */
rr_status rr_lattice_get(rr_lattice* lat, double* pos, double* dist, int32_t* order,
                         int32_t* wall_hits, double* energy);
rr_status rr_lattice_destroy(rr_lattice* lat);

/* compare (shoebox.hpp:67-70, shoebox.cpp:126-182): each traced image goes
 * to the nearest oracle image within pos_tol (largest oracle index on
 * ties); per matched oracle image the member list (traced order), the max
 * position error and 10 log10(sum traced E / oracle E) per band.  Arrays are
 * host or device memory; oracle order may be NULL (reported as 0). */
rr_status rr_shoebox_compare(rr_ctx* ctx, int64_t n_oracle, const double* oracle_pos,
                             const double* oracle_energy, const int32_t* oracle_order,
                             int64_t n_traced, const double* traced_pos,
                             const double* traced_energy, double pos_tol,
                             double energy_tol_db, rr_match** out);
/* The same on device-resident sets: a lattice against an image set. */
rr_status rr_lattice_compare_images(rr_lattice* lat, rr_images* traced, double pos_tol,
                                    double energy_tol_db, rr_match** out);
/* MatchReport (shoebox.hpp:56-66): counts, max_position_error and the 8
 * per-band rms energy errors (dB). */
rr_status rr_match_info(rr_match* m, int64_t* n_matched, int64_t* n_members,
                        int64_t* n_unmatched_oracle, int64_t* n_unmatched_traced,
                        double* max_position_error, double* rms_energy_error_db);
/* MatchedImage list in oracle order; member_off has n_matched+1 entries.
 * Any output may be NULL. */
rr_status rr_match_get(rr_match* m, int32_t* oracle_index, double* position_error,
                       int32_t* order, double* energy_delta_db, int64_t* member_off,
                       int32_t* members, int32_t* unmatched_oracle,
                       int32_t* unmatched_traced);
rr_status rr_match_destroy(rr_match* m);

/* Measurement helper (no reference counterpart): sustained L2 read
 * bandwidth (GB/s) streaming an L2-resident buffer of `bytes`, `iters`
 * passes in one launch; the L2 roofline denominator of bench.py. */
rr_status rr_l2_read_gbs(rr_ctx* ctx, int64_t bytes, int32_t iters, double* gbs);

/* air_beta_bands (air_absorption.cpp:59-65), 8 values. */
rr_status rr_air_beta_bands(const rr_air* air, double* beta);
/* air_alpha_db_per_m (air_absorption.cpp:21-53): ISO 9613-1 level
 * attenuation in dB/m at frequency f (0 when disabled). */
rr_status rr_air_alpha_db_per_m(const rr_air* air, double f, double* alpha);
/* AirModel::validate (air_absorption.cpp:8-19): RR_INVALID_ARGUMENT outside
 * [-20, 50] C, [10, 100] %, [80, 120] kPa (an enabled model only). */
rr_status rr_air_validate(const rr_air* air);

/* ---------------------------------------------------------------- IR
 * build_pulse_trains + synthesize (rir.hpp:33-45), per band: events at
 * sample lround(d/c*fs) with amplitude sqrt(E_b), binned into 8 histograms of
 * `length` samples, then convolved with the 8 band filters of `taps` taps
 * (design_band_filter, rir.cpp:32-58; reference: 1023).  Output: per-band
 * responses band_ir (8*length, may be NULL) and their sum broadband (length,
 * may be NULL).  Host buffers.  images from n arrays (dist n, energy n*8). */
rr_status rr_synthesize(rr_ctx* ctx, int64_t n, const double* dist,
                        const double* energy, double c, double fs,
                        int32_t taps, int64_t length, double* band_ir,
                        double* broadband);
/* Same, from device-resident arrays; outputs stay in caller-provided device
 * buffers (for multi-GPU reduction).  hist (8*length f64) receives the
 * binned pulse trains; band_ir may be NULL to stop after binning. */
rr_status rr_ir_bin_device(rr_ctx* ctx, int64_t n, const double* d_dist,
                           const double* d_energy, double c, double fs,
                           int64_t length, double* d_hist);
rr_status rr_ir_filter_device(rr_ctx* ctx, const double* d_hist, double fs,
                              int32_t taps, int64_t length, double* d_band_ir,
                              double* d_broadband);
/* synthesize (rir.hpp:45) from explicit pulse trains (PulseTrains,
 * rir.hpp:12-23): band b owns events [band_off[b], band_off[b+1]) of
 * time (s) and amplitude; band_off has 9 entries.  Host buffers. */
rr_status rr_synthesize_trains(rr_ctx* ctx, const int64_t* band_off,
                               const double* time, const double* amplitude,
                               double fs, int32_t taps, int64_t length,
                               double* band_ir, double* broadband);
/* ---------------------------------------------------------------- metrics
 * PerceptiveFactors / MetricValue (metrics.hpp:30-48): per band EDT, T30
 * (least-squares decay fits of the Schroeder curve), SPL, C80, D50, Ts. */
typedef struct {
  double value;
  int32_t reliable;
} rr_metric;

typedef struct {
  rr_metric edt_s, t30_s, spl_db, c80_db, d50_pct, ts_ms;
} rr_factors;

/* factors(const PulseTrains&) (metrics.hpp:56-60) on the device; out[0..7]
 * per band, out[8] the 500 Hz / 1 kHz average ("mid").  Trains as in
 * rr_synthesize_trains (host arrays, band_off 9 entries). */
rr_status rr_band_factors(rr_ctx* ctx, const int64_t* band_off,
                          const double* time, const double* amplitude,
                          rr_factors* out);
/* The same for the trains of an image set (build_pulse_trains: t = d / c,
 * amplitude sqrt(E_b)); dist / energy host or device arrays (UVA). */
rr_status rr_factors_from_images(rr_ctx* ctx, int64_t n, const double* dist,
                                 const double* energy, double c,
                                 rr_factors* out);
rr_status rr_images_factors(rr_images* im, double c, rr_factors* out);
/* schroeder(const BandPulseTrain&) (metrics.cpp:125-134) for the 8 trains
 * (band_off 9 entries, amplitudes in train order, host or device): level in
 * dB per event, 10 log10(remaining / total energy).  A band whose events
 * carry no energy -> RR_INVALID_ARGUMENT (metrics.cpp:17-19). */
rr_status rr_band_schroeder(rr_ctx* ctx, const int64_t* band_off,
                            const double* amplitude, double* level_db);

/* Length of the reference's response (rir.cpp:78-80): llround(t_last*fs) +
 * (taps-1)/2 + 1, or 0 without events. */
rr_status rr_ir_reference_length(int64_t n, const double* dist, double c,
                                 double fs, int32_t taps, int64_t* length);
/* design_band_filter restated with a tap count. */
rr_status rr_band_filter(int32_t band, double fs, int32_t taps, double* out);
/* Image arrays of a device image set (for rr_ir_bin_device). */
rr_status rr_images_device(rr_images* im, const double** d_dist,
                           const double** d_energy, int64_t* n);

/* build_pulse_trains (rir.cpp:9-30) of a device image set: band b's events
 * (t = d / c, amplitude sqrt(E_b)) sorted by (time, amplitude) at
 * [band_off[b], band_off[b+1]) of time / amplitude (8 * n each, host or
 * device; band_off 9 entries, may be NULL).  No host sort. */
rr_status rr_images_pulse_trains(rr_images* im, double c, int64_t* band_off,
                                 double* time, double* amplitude);
/* build_pulse_trains (rir.cpp:9-30) of host (or device) image data: dist n
 * f64 (ImageSource::distance), energy n*8 f64 (band_energy rows); outputs as
 * rr_images_pulse_trains, sorted on the device (the façade's
 * build_pulse_trains(images, c) calls this instead of a host sort). */
rr_status rr_pulse_trains(rr_ctx* ctx, int64_t n, const double* dist, const double* energy, double c,
                          int64_t* band_off, double* time, double* amplitude);
/* synthesize (rir.cpp:60-96) of a device image set.  With band_ir and
 * broadband both NULL: *length = the reference length llround(t_last*fs) +
 * (taps-1)/2 + 1 (0 without images).  Otherwise fills band_ir (8 x *length)
 * and / or broadband (*length), host or device buffers. */
rr_status rr_images_synthesize(rr_images* im, double c, double fs, int32_t taps,
                               int64_t* length, double* band_ir, double* broadband);

/* ---------------------------------------------------------------- multi-GPU
 * run_trace_pipeline's trace -> image sources -> impulse responses
 * (pipeline.cpp:163-175) over the ranks of an NCCL communicator, one process
 * or thread per GPU.  Each rank traces a block-cyclic shard of the lattice
 * (`block` rays per block) on its replicated scene; captures go to the owner
 * of their order class (ncclSend/ncclRecv), owners build the image sources,
 * the 8-band pulse histograms are summed exactly (64-bit fixed point,
 * ncclAllReduce) and every rank runs the FIR; image lists are gathered to
 * rank 0.  Results equal the single-GPU pipeline's bit for bit.  With comm ==
 * NULL the plain single-GPU pipeline runs, still device resident.  NCCL
 * failures return RR_NCCL.  (The reference has no multi-process path; its
 * trace() splits rays over host threads, tracer.cpp:82-105.) */
#define RR_NCCL_ID_BYTES 128
rr_status rr_comm_unique_id(uint8_t* id); /* ncclGetUniqueId, RR_NCCL_ID_BYTES bytes, rank 0 */
rr_status rr_comm_init(rr_ctx* ctx, const uint8_t* id, int32_t nranks, int32_t rank,
                       rr_comm** out); /* ncclCommInitRank on ctx's device */
rr_status rr_comm_info(rr_comm* comm, int32_t* rank, int32_t* nranks);
/* Testing aid: an in-process loopback hub of nranks ranks on ONE GPU, each
 * rank a host thread with its own rr_ctx; rr_pipeline_sharded's collectives
 * then rendezvous on the hub and move data by device copies instead of NCCL,
 * so the multi-rank exchange (sharding, ownership, packing, all-to-all,
 * exact IR reduction, gather) runs where only one GPU exists. */
rr_status rr_hub_create(int32_t nranks, rr_hub** out);
rr_status rr_hub_destroy(rr_hub* hub);
rr_status rr_comm_init_loopback(rr_ctx* ctx, rr_hub* hub, int32_t rank, rr_comm** out);
rr_status rr_comm_destroy(rr_comm* comm);
rr_status rr_pipeline_sharded(rr_scene* scene, rr_comm* comm, const rr_source* source,
                              const rr_receiver* receivers, int32_t n_recv,
                              const rr_trace_config* cfg, const rr_air* air,
                              const rr_cluster_options* opt, double fs, int64_t length,
                              int32_t taps, int32_t block, rr_sharded** out);
/* this rank's ray*bounces / rays, image sources built here (all receivers),
 * and stage times in ms [trace, exchange, images, ir, gather] (may be NULL) */
rr_status rr_sharded_info(rr_sharded* sh, int64_t* ray_bounces, int64_t* n_rays,
                          int64_t* local_images, float* stage_ms);
/* hands out receiver recv's image list (rank 0: all ranks' images in the
 * reference order; other ranks: empty); destroy it with rr_images_destroy */
rr_status rr_sharded_take_images(rr_sharded* sh, int32_t recv, rr_images** out);
/* receiver recv's band IRs (8 x length) and broadband IR (length); host or
 * device pointers, either may be NULL */
rr_status rr_sharded_ir(rr_sharded* sh, int32_t recv, double* band_ir, double* broadband);
rr_status rr_sharded_destroy(rr_sharded* sh);

#ifdef __cplusplus
}
#endif

#endif /* ROOMRAY_B200_H */
