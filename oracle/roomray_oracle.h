/* Plain-C restatement of the reference hot path — TEST INFRASTRUCTURE ONLY.
 *
 * This is the parity oracle for the CUDA path (see roomray_oracle.c for the
 * file:line each function restates).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it; the product library never
 * links or calls it.
 */
#ifndef ROOMRAY_ORACLE_H
#define ROOMRAY_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RO_BANDS 8

typedef struct ro_scene ro_scene;
typedef struct ro_trace ro_trace;
typedef struct ro_images ro_images;

const char* ro_last_error(void);

/* mesh + build_tree (accel_tree.cpp:70-87); validate => geometry.cpp:47-75 */
ro_scene* ro_scene_create(const double* verts, int64_t nv, const int32_t* tris,
                          int64_t nf, const double* alpha, int32_t nmat,
                          int validate);
void ro_scene_destroy(ro_scene* s);
int64_t ro_tree_size(const ro_scene* s, int32_t* root, int32_t* depth);
void ro_tree_nodes(const ro_scene* s, int32_t* left, int32_t* right,
                   int32_t* face, double* lo, double* hi);
void ro_face_normals(const ro_scene* s, double* normals);
void ro_scene_bounds(const ro_scene* s, double* lo, double* hi);

/* nearest_hit / nearest_hit_brute for n rays; n_int/n_leaf (optional, may be
 * NULL) count internal-node expansions and leaf tests that survive the prune
 * (accel_tree.cpp:141-179), per ray. */
int ro_nearest_hit(const ro_scene* s, const double* o, const double* d,
                   int64_t n, int brute, int32_t* face, double* delta,
                   double* point, int32_t* n_int, int32_t* n_leaf);

int ro_intersect_sphere(const double* o, const double* d, const double* c,
                        double r, double* out);
void ro_fibonacci(int64_t n, int64_t first, int64_t stride, int64_t count,
                  double* out);

/* trace (tracer.cpp:108-149) over the lattice subset k = first + i*stride,
 * i < count (stride <= 0: all rays).  n_recv receivers are traced with the
 * same trajectories (a receiver never alters a ray, tracer.cpp:27-29); each
 * capture records its receiver index. */
ro_trace* ro_trace_run(const ro_scene* s, const double* src, int64_t ray_count,
                       const double* recv_centers, const double* recv_radii,
                       int32_t n_recv, int32_t max_iterations, double max_range,
                       int32_t threads, int64_t first, int64_t stride,
                       int64_t count);
ro_trace* ro_trace_run_dirs(const ro_scene* s, const double* src, int64_t ray_count,
                            const double* recv_centers, const double* recv_radii,
                            int32_t n_recv, int32_t max_iterations, double max_range,
                            int32_t threads, int64_t first, int64_t stride,
                            int64_t count, const double* dirs);
void ro_trace_info(const ro_trace* t, int32_t* iterations, int32_t* truncated,
                   int64_t* escaped, int64_t* out_of_range, double* max_range,
                   int64_t* n_captures, int64_t* total_hist,
                   int64_t* ray_bounces, int64_t* sum_n_int,
                   int64_t* sum_n_leaf);
void ro_trace_captures(const ro_trace* t, int32_t* recv, int32_t* ray,
                       double* point, double* dir, double* path, double* mult,
                       int64_t* hist_off, int32_t* hist);
void ro_trace_free(ro_trace* t);

/* build_image_sources (image_sources.cpp:154-170) */
ro_images* ro_image_sources(const ro_scene* s, int64_t n, const int32_t* ray,
                            const double* point, const double* dir,
                            const double* path, const double* mult,
                            const int64_t* hist_off, const int32_t* hist,
                            int64_t total_rays, const double* air4,
                            const double* recv, double tol_scale,
                            int merge_coplanar);
void ro_images_info(const ro_images* r, int64_t* n, int64_t* total_path);
void ro_images_get(const ro_images* r, double* pos, double* dist,
                   double* energy, double* mult, int32_t* ray_count,
                   int32_t* order, int32_t* has_proj, double* proj,
                   int64_t* path_off, int32_t* path);
void ro_images_free(ro_images* r);

/* air_absorption.cpp:21-65; air4 = {enabled, T_c, RH_%, P_kPa} */
int ro_air_beta_bands(const double* air4, double* beta);
double ro_air_alpha(const double* air4, double f);

/* design_band_filter (rir.cpp:32-58) with the tap count as a parameter */
int ro_band_filter(int band, double fs, int taps, double* out);

/* build_pulse_trains + synthesize (rir.cpp:9-96), tap count as a parameter.
 * band_mask selects the populated trains.  Returns the response length
 * (llround(t_last*fs)+delay+1) and writes min(length, cap) samples. */
int64_t ro_synthesize(int64_t n, const double* dist, const double* energy,
                      double c, double fs, int taps, int32_t band_mask,
                      double* out, int64_t cap);

#ifdef __cplusplus
}
#endif

#endif
