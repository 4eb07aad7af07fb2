/* voxrf CPU oracle — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C (FP64) restatement of the reference's per-ray hot path
 * (/root/reference/proj/src/{voxel_grid,renderer,gradients,mapping,tracking}.cpp).
 * It is the checker the parity tests, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg compare the CUDA path against; it is never linked into or
 * called by the product library (paper_2307_03404_b200/).
 *
 * Pinning: oracle/Makefile also compiles the reference's own translation units
 * verbatim (against oracle/shim, an Eigen-subset + doctest + json_fwd shim)
 * into oracle/_ref/. The reference's 45 unit tests run against that build, and
 * tests/test_oracle_pinning.py checks this restatement against it
 * (render_image, sample_ray, mapping_step, pose_gradient, track_frame) on seeded
 * inputs, plus the golden fixtures under tests/golden/ generated from it.
 *
 * Layouts follow the reference: vertex payload AoS double[V][28] x-fastest
 * (voxel_grid.hpp:13-16,57-62), occupancy uint8 per cell, images row-major
 * double (image.hpp:10-26), poses as (w,x,y,z) quaternion + translation. */
#ifndef VOXRF_ORACLE_H
#define VOXRF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_OK = 0, OR_INVALID_ARGUMENT = 1, OR_OUT_OF_RANGE = 2, OR_RUNTIME = 3 };

typedef struct {
  int32_t res[3];
  double origin[3];
  double voxel_size;
} or_geometry;

typedef struct {
  or_geometry geom;
  double* data;           /* V*28 */
  const uint8_t* active;  /* (rx-1)(ry-1)(rz-1) */
} or_grid;

typedef struct {
  double fx, fy, cx, cy;
  int32_t width, height;
  double depth_scale;
} or_intrinsics;

typedef struct {
  double q[4]; /* w, x, y, z */
  double t[3];
} or_pose;

typedef struct {
  double step, t_near, t_far, termination_eps;
} or_render_params;

typedef struct {
  const double* color; /* H*W*3 */
  const double* depth; /* H*W   */
  or_pose pose;
} or_frame;

typedef struct {
  double color[3];
  double depth;
  double transmittance_terminal;
  int32_t count;
  int32_t hit;
  int32_t terminated_early;
} or_ray_result;

typedef struct {
  double lambda_d, lr_sigma, lr_sh, rmsprop_decay, rmsprop_eps;
  or_render_params render;
} or_mapping_config;

typedef struct {
  double loss_photometric, loss_geometric, loss_total;
  int32_t rays_color, rays_depth;
  double psnr_estimate;
  int64_t samples;
  int32_t bad_ray; /* -1 or the first ray index with a non-finite loss */
} or_map_stats;

typedef struct {
  double lambda_p, lambda_d;
  or_render_params render;
} or_tracking_loss;

typedef struct {
  double d_omega[3], d_tau[3];
  double loss;
  int32_t rays_used;
} or_pose_grad;

typedef struct {
  double jtj[21]; /* upper triangle, row-major over [omega; tau] */
  double jtr[6];
  double loss;    /* sum over hit rays of lambda_p|cres|^2 + lambda_d dres^2 (not /m) */
  int32_t rays_used;
} or_normal_eqs;

typedef struct {
  int32_t rays_per_iteration, iterations;
  double lr_omega, lr_tau, beta1, beta2, adam_eps, lambda_p, lambda_d;
  double convergence_step, divergence_factor;
  int32_t divergence_patience, max_redraws;
  uint64_t seed;
  or_render_params render;
} or_tracking_config;

typedef struct {
  or_pose pose;
  int32_t failed, iterations_run;
  double final_loss;
} or_track_result;

/* camera.hpp:33-41 */
int or_generate_ray(const or_intrinsics* intr, const or_pose* pose, double u, double v,
                    double o[3], double d[3]);
/* renderer.cpp:51-80; writes up to cap samples; returns the schedule length */
int or_sample_ray(const or_grid* g, const double o[3], const double d[3],
                  const or_render_params* p, int cap, double* t, double* delta,
                  uint32_t* cell);
/* renderer.cpp:142-147 */
int or_render_ray(const or_grid* g, const double o[3], const double d[3],
                  const or_render_params* p, or_ray_result* out);
/* renderer.cpp:149-174 */
int or_render_image(const or_grid* g, const or_intrinsics* intr, const or_pose* pose,
                    const or_render_params* p, int stride, double* color, double* depth);
/* mapping.cpp:114-233 with a pre-drawn batch (frame, px, py triples).
 * grad_out (V*28, optional) receives the merged gradient; if apply != 0 the
 * sparse RMSProp update is applied to g->data using rms_v (V*28). */
int or_mapping_step(or_grid* g, const or_frame* frames, int n_frames,
                    const or_intrinsics* intr, const or_mapping_config* cfg,
                    const int32_t* batch, int n_rays, double* rms_v, double* grad_out,
                    int apply, or_map_stats* stats);
/* One rank's share of a ray-sharded step: this batch's gradient with the upstream
 * normalised by the global hit counts (no update). */
int or_mapping_grad_global(or_grid* g, const or_frame* frames, int n_frames,
                           const or_intrinsics* intr, const or_mapping_config* cfg,
                           const int32_t* batch, int n_rays, int m_color, int m_depth,
                           double* grad_out, or_map_stats* stats);
/* tracking.cpp:76-143 */
int or_pose_gradient(const or_grid* g, const or_frame* frame, const or_intrinsics* intr,
                     const or_pose* pose, const int32_t* pixels, int n,
                     const or_tracking_loss* cfg, or_pose_grad* out);
/* New normal-equation path: per ray, grad_wrt_ray with unit
 * upstreams e_r, e_g, e_b (depth 0) and depth 1 (colour 0), chart-mapped as
 * tracking.cpp:125-128 and weighted by sqrt(lambda). */
int or_pose_normal_eqs(const or_grid* g, const or_frame* frame, const or_intrinsics* intr,
                       const or_pose* pose, const int32_t* pixels, int n,
                       const or_tracking_loss* cfg, or_normal_eqs* out);
/* tracking.cpp:147-166 */
int or_draw_valid_pixels(const double* depth, int w, int h, int count, int max_redraws,
                         uint64_t rng_state[4], int32_t* pixels_out);
/* tracking.cpp:170-252 */
int or_track_frame(const or_grid* g, const or_frame* frame, const or_intrinsics* intr,
                   const or_pose* init, const or_tracking_config* cfg, or_track_result* out,
                   double* loss_trace);
/* rng.hpp:13-81 */
void or_rng_seed(uint64_t seed, uint64_t state[4]);
uint64_t or_rng_next(uint64_t state[4]);
uint64_t or_rng_uniform_index(uint64_t state[4], uint64_t n);
double or_rng_uniform(uint64_t state[4]);
/* mapping.cpp:121-128 batch draw: 3 x uniform_index per ray */
void or_draw_batch(uint64_t state[4], int n_frames, int width, int height, int n_rays,
                   int32_t* batch);
/* pose.hpp:32-41 + tracking.hpp:21-26 */
void or_apply_perturbation(const double omega[3], const double tau[3], const or_pose* in,
                           or_pose* out);
/* voxel_grid.cpp:34-47 */
int or_sh_eval(const double d[3], double basis[9]);

int or_upsample(const or_grid* g, int max_resolution, int clamp_outside, or_geometry* fine,
                double* out, uint8_t* active_out);

#ifdef __cplusplus
}
#endif
#endif
