/* voxrf_b200 — C-ABI of the B200-native per-ray hot path.
 *
 * This is the drop-in boundary for the reference library's batch entry points
 * (/root/reference/proj/include/voxrf/*.hpp). Every function below names the
 * reference interface it replaces. The reference API is exception-based and
 * Eigen-typed; this boundary is plain C: POD structs, raw pointers, sizes and
 * an int status. The C++ binding that re-exposes the reference signatures on
 * top of it (integration/voxrf_gpu_backend.cpp) maps the status back to the
 * same exception types and messages.
 *
 * Status codes map to the reference's exception classes:
 *   VRF_ERR_INVALID_ARGUMENT -> std::invalid_argument
 *   VRF_ERR_OUT_OF_RANGE     -> std::out_of_range
 *   VRF_ERR_RUNTIME          -> std::runtime_error (same message text)
 *   VRF_ERR_CUDA             -> std::runtime_error ("cuda: ...")
 * vrf_last_error(ctx) returns the message of the last failing call.
 *
 * Device state lives in a vrf_context (one per GPU): the fp32 vertex payload
 * [V][28] (sigma_raw, r0..r8, g0..g8, b0..b8 — the .vxgf payload order,
 * voxel_grid.cpp:230-233), a 1-bit-per-cell occupancy mask, the fp32
 * gradient accumulator and RMSProp state, and the keyframe set. All calls are
 * synchronous at return unless stated otherwise; no call ever falls back to a
 * CPU implementation — without a usable CUDA device vrf_context_create fails.
 */
#ifndef VOXRF_B200_H
#define VOXRF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VRF_ABI_VERSION 1

enum {
  VRF_OK = 0,
  VRF_ERR_INVALID_ARGUMENT = 1,
  VRF_ERR_OUT_OF_RANGE = 2,
  VRF_ERR_RUNTIME = 3,
  VRF_ERR_CUDA = 4
};

typedef struct vrf_context vrf_context;

/* GridGeometry — voxel_grid.hpp:20-63 (res counts vertices per axis). */
typedef struct {
  int32_t res[3];
  double origin[3];
  double voxel_size;
} vrf_grid_geometry;

/* CameraIntrinsics — camera.hpp:11-24. */
typedef struct {
  double fx, fy, cx, cy;
  int32_t width, height;
  double depth_scale;
} vrf_intrinsics;

/* Pose — pose.hpp:11-24; q = (w, x, y, z), x_world = q * x_cam + t. */
typedef struct {
  double q[4];
  double t[3];
} vrf_pose;

/* RenderParams — renderer.hpp:12-24 (<= 0 selects the reference defaults). */
typedef struct {
  double step, t_near, t_far, termination_eps;
} vrf_render_params;

/* The MappingConfig fields mapping_step reads — mapping.hpp:19-41. */
typedef struct {
  double lambda_d, lr_sigma, lr_sh, rmsprop_decay, rmsprop_eps;
  int32_t deterministic; /* 1: sorted/segmented fp64 gradient reduce (bit-reproducible) */
  int32_t reserved;
  vrf_render_params render;
} vrf_mapping_config;

/* MapStepStats — mapping.hpp:68-75, plus the composited-sample count. */
typedef struct {
  double loss_photometric, loss_geometric, loss_total;
  int32_t rays_color, rays_depth;
  double psnr_estimate;
  int64_t samples;     /* sum over hit rays of RayWorkspace::count */
  int32_t bad_ray;     /* -1, or the first batch index with a non-finite loss */
  int32_t reserved;
} vrf_map_step_stats;

/* Loss weights + render params of TrackingConfig — tracking.hpp:29-51. */
typedef struct {
  double lambda_p, lambda_d;
  vrf_render_params render;
} vrf_tracking_loss;

/* PoseGradient — tracking.hpp:60-65. */
typedef struct {
  double d_omega[3], d_tau[3];
  double loss;
  int32_t rays_used;
  int32_t reserved;
  int64_t samples;
} vrf_pose_gradient_result;

/* Gauss-Newton normal equations over residuals r = [sqrt(lp) (C-C*); sqrt(ld) (D-D*)]
 * per hit ray, parameters [omega; tau] (the PosePerturbation chart,
 * tracking.hpp:15-26). jtj: upper triangle, row-major (21). loss is the
 * un-normalised sum; pose_gradient == (2/m) * jtr. */
typedef struct {
  double jtj[21];
  double jtr[6];
  double loss;
  int32_t rays_used;
  int32_t reserved;
  int64_t samples;
} vrf_normal_equations;

/* TrackingConfig — tracking.hpp:29-51 (init policy handled by the caller). */
typedef struct {
  int32_t rays_per_iteration, iterations;
  double lr_omega, lr_tau, beta1, beta2, adam_eps, lambda_p, lambda_d;
  double convergence_step, divergence_factor;
  int32_t divergence_patience, max_redraws;
  uint64_t seed;
  vrf_render_params render;
} vrf_tracking_config;

/* TrackFrameResult — tracking.hpp:75-80 (loss_trace returned separately). */
typedef struct {
  vrf_pose pose;
  int32_t failed, iterations_run;
  double final_loss;
} vrf_track_frame_result;

/* Pose kernels (K5). PARITY: FP64 SH and Jacobian partials, the reference-parity
 * path of pose_gradient / track_frame. GN: the Gauss-Newton tracker's kernel (fp32
 * SH contraction and lane Jacobian partials; FP64 march, sigma replay, T and
 * compositing). GN_CHECK: a second implementation of GN's arithmetic with
 * group-independent control flow, bit-identical to GN by test. */
#define VRF_POSE_KERNEL_PARITY 0
#define VRF_POSE_KERNEL_GN 1
#define VRF_POSE_KERNEL_GN_CHECK 2

/* Gauss-Newton / Levenberg-Marquardt tracker (new; the reference only has Adam).
 * Every iteration draws exactly rays_per_iteration pixels, stratified over a
 * 2^L x 2^L tile grid with 4^L <= rays_per_iteration. */
typedef struct {
  int32_t rays_per_iteration, iterations;
  double lambda_p, lambda_d;
  double damping;        /* LM: (JtJ + damping*diag(JtJ) + 1e-12 I) delta = -Jtr */
  int32_t max_redraws;
  int32_t kernel;        /* VRF_POSE_KERNEL_GN (default) or VRF_POSE_KERNEL_GN_CHECK */
  uint64_t seed;         /* device counter-based stream for the valid-depth pixel draws */
  vrf_render_params render;
} vrf_gn_config;

/* Device buffers owned by a context (for NCCL collectives issued by the caller). */
typedef struct {
  float* payload;        /* [num_vertices][28] */
  float* grad;           /* [padded_vertices][28] */
  float* rms_v;          /* [padded_vertices][28] */
  int64_t num_vertices;
  int64_t padded_vertices;
  void* stream;          /* cudaStream_t every call of this context runs on */
} vrf_device_buffers;

/* Per-rank partial results of the mapping forward pass. */
typedef struct {
  int32_t rays_color, rays_depth;
  double sum_photometric, sum_geometric;
  int64_t samples;
  int32_t bad_ray;
  int32_t reserved;
} vrf_map_partials;

/* ---- context */
int vrf_context_create(int device, vrf_context** out);
void vrf_context_destroy(vrf_context* ctx);
const char* vrf_last_error(const vrf_context* ctx);
int vrf_abi_version(void);
/* Pads the gradient/RMSProp buffers to a multiple of world_size vertices so
 * NCCL reduce-scatter shards are equal; call before vrf_grid_*. */
int vrf_set_shard_multiple(vrf_context* ctx, int world_size);
/* Run on an external stream (e.g. torch.cuda.current_stream()); NULL = the context's
 * own non-blocking stream. For the legacy default stream pass cudaStreamLegacy
 * ((void*)1), not NULL. */
int vrf_set_stream(vrf_context* ctx, void* stream);
int vrf_get_device_buffers(vrf_context* ctx, vrf_device_buffers* out);
/* Sample records of the fast mapping path (K0 writes up to K per ray, K2 walks
 * them; rays with more samples take the recompute-march backward). budget_gb <= 0:
 * 30 % of free HBM; max_k < 0: K from the longest ray seen (<= 1024); max_k == 0:
 * no records (every ray takes the recompute-march backward); max_k >= 4: at most
 * max_k records per ray. */
int vrf_set_record_limits(vrf_context* ctx, double budget_gb, int max_k);
/* Number of this library's own kernels the context launched since creation
 * (bench evidence; cub sorts and memsets are not counted). */
int64_t vrf_kernel_launch_count(const vrf_context* ctx);
/* Per-kernel CUDA-event timing on the context stream (resets the counters).
 * Slots: 0 map forward, 1 map backward (scatter), 2 RMSProp, 3 misc,
 *        4 pose forward, 5 pose backward, 6 render, 7 deterministic reduce. */
int vrf_profile_enable(vrf_context* ctx, int on);
int vrf_profile_read(vrf_context* ctx, int slot, double* ms, int64_t* launches);
/* float4 parameter groups RMSProp updated since vrf_profile_enable (96 B each). */
int64_t vrf_profile_touched_groups(vrf_context* ctx);
/* Composited samples of the Gauss-Newton tracking frames since vrf_profile_enable. */
int64_t vrf_profile_track_samples(vrf_context* ctx);

/* ---- grid: VoxelGrid (voxel_grid.hpp:112-175) */
/* VoxelGrid(geom, sigma_init) — voxel_grid.cpp:74-81 (all cells active). */
int vrf_grid_init(vrf_context* ctx, const vrf_grid_geometry* geom, double sigma_init);
/* Reset the payload to VoxelGrid(geom, sigma_init)'s (voxel_grid.cpp:74-81) keeping the
 * current occupancy; gradient and RMSProp state restart at zero. */
int vrf_grid_fill(vrf_context* ctx, double sigma_init);
/* Upload VoxelGrid::data() (double [V][28]) and occupancy() (uint8 per cell). */
int vrf_grid_upload(vrf_context* ctx, const vrf_grid_geometry* geom, const double* payload,
                    const uint8_t* occupancy);
/* Upload a .vxgf-style fp32 payload and LSB-first occupancy bitmask
 * (voxel_grid.cpp:222-239). */
int vrf_grid_upload_f32(vrf_context* ctx, const vrf_grid_geometry* geom, const float* payload,
                        const uint8_t* occupancy_bits);
int vrf_grid_download(vrf_context* ctx, double* payload, uint8_t* occupancy);
int vrf_grid_download_f32(vrf_context* ctx, float* payload);
int vrf_grid_get_geometry(const vrf_context* ctx, vrf_grid_geometry* out);
/* VoxelGrid::upsampled(max_resolution) — voxel_grid.cpp:190-220, in place: res -> 2 res - 1,
 * voxel / 2, same bounds; gradient and RMSProp state restart at zero. */
int vrf_grid_upsample(vrf_context* ctx, int max_resolution);
/* VoxelGrid::save / VoxelGrid::load — voxel_grid.cpp:222-278 (.vxgf v1: "VXGF", u32
 * version, u32 res[3], f64 origin[3], f64 voxel, f32 [V][28], LSB-first cell bits).
 * Same runtime_error messages; a failed load leaves the context without a grid. */
int vrf_grid_save(vrf_context* ctx, const char* path);
int vrf_grid_load(vrf_context* ctx, const char* path);
/* VoxelGrid::prune(tau) — voxel_grid.cpp:169-188. */
int vrf_grid_prune(vrf_context* ctx, double tau, int64_t* deactivated);
/* Device-side integrity digest of the grid (geometry, fp32 payload, occupancy
 * bits): an order-independent 64-bit hash computed in one pass over HBM. Used to
 * check that tracking and rendering never mutate the grid without
 * a download; VoxelGrid::checksum (voxel_grid.cpp:280-292, FNV-1a over the fp64
 * bytes) stays a host computation on a downloaded grid. */
int vrf_grid_digest(vrf_context* ctx, uint64_t* out);

/* ---- drop-in residency (integration/voxrf_gpu_backend.cpp keeps the device grid in
 * step with a caller's VoxelGrid without whole-grid copies per call):
 * partial writes of host-modified vertex ranges, an occupancy refresh, and the log
 * of the float4 groups the last RMSProp pass updated (mapping.cpp:218-231's
 * touched set) for a sparse write-back of the in-place result. */
int vrf_grid_write_vertices(vrf_context* ctx, int64_t first, int64_t count, const double* data);
int vrf_rmsprop_write_vertices(vrf_context* ctx, int64_t first, int64_t count, const double* v);
int vrf_grid_set_occupancy(vrf_context* ctx, const uint8_t* occupancy);
/* on: every later mapping step logs its updated groups (ids = vertex * 7 + group,
 * new theta and v as 4 floats each); the log holds the last step only. */
int vrf_track_updates(vrf_context* ctx, int on);
int vrf_updates_count(vrf_context* ctx, int64_t* n);
int vrf_updates_read(vrf_context* ctx, int64_t n, uint32_t* ids, float* theta, float* v);
/* Entries [first, first + count) of the log; sorted != 0: in ascending id order
 * (the first such call after a logged step sorts the log on the device). */
int vrf_updates_read_range(vrf_context* ctx, int64_t first, int64_t count, int sorted,
                           uint32_t* ids, float* theta, float* v);
/* fp32 device state to host, floats [first, first + count) of which = 0 the payload
 * [V][28], 1 the RMSProp v [V][28] (the drop-in's chunked dense write-back). */
int vrf_state_read_f32(vrf_context* ctx, int which, int64_t first, int64_t count, float* dst);
/* Page-locked host memory for staging buffers (cudaMallocHost; NULL on failure):
 * device <-> host copies into it run at full PCIe / C2C speed. */
void* vrf_host_alloc(size_t bytes);
void vrf_host_free(void* p);

/* ---- frames: Frame (frame.hpp:10-19); colour H*W*3, depth H*W along-ray metres */
int vrf_frames_upload(vrf_context* ctx, const vrf_intrinsics* intr, int n,
                      const double* const* colors, const double* const* depths,
                      const vrf_pose* poses);
int vrf_frames_count(const vrf_context* ctx);
/* Slot-addressed frame store for online use (the SLAM driver): reserve capacity
 * slots of intr's size, then write one slot at a time (keyframes appended as they
 * are selected, a tracking slot overwritten per frame). vrf_frames_count is the
 * high-water mark of written slots; mapping batches address slots by index. */
int vrf_frames_reserve(vrf_context* ctx, const vrf_intrinsics* intr, int capacity);
int vrf_frame_set(vrf_context* ctx, int slot, const double* color, const double* depth,
                  const vrf_pose* pose);
int vrf_frame_set_pose(vrf_context* ctx, int slot, const vrf_pose* pose);
/* vrf_frame_set from the sensor format the reference's dataset stores (8-bit RGB
 * H*W*3, 16-bit depth units H*W; image.cpp:53-55, 79): converted on the device as
 * colour / 255.0 and depth / intrinsics.depth_scale — 5 B/pixel over PCIe
 * instead of 32. */
int vrf_frame_set_u8u16(vrf_context* ctx, int slot, const uint8_t* rgb, const uint16_t* depth,
                        const vrf_pose* pose);

/* ---- renderer: render_image — renderer.hpp:83-84 (renderer.cpp:149-174).
 * color: ceil(H/stride)*ceil(W/stride)*3, depth: ceil(H/stride)*ceil(W/stride). */
int vrf_render_image(vrf_context* ctx, const vrf_intrinsics* intr, const vrf_pose* pose,
                     const vrf_render_params* params, int stride, double* color,
                     double* depth);

/* ---- mapping: mapping_step — mapping.hpp:80-82 (mapping.cpp:114-233) with the
 * batch drawn by the caller (the reference draws it from its Rng,
 * mapping.cpp:121-128): batch = n_rays (frame, px, py) int32 triples, host memory.
 * Mutates the device grid and RMSProp state in place, like the reference. */
int vrf_mapping_step(vrf_context* ctx, const vrf_mapping_config* cfg, const int32_t* batch,
                     int n_rays, vrf_map_step_stats* out);
/* map_scene's inner loop (mapping.cpp:302-312): n_steps mapping_step calls, batch i
 * drawn from the reference Rng stream `rng_state` (advanced in place) over the first
 * n_keyframes frame slots. The host draw of batch i+1 overlaps the device work of
 * step i (pinned double buffer). out: n_steps stats; stops at the first error. */
int vrf_mapping_steps(vrf_context* ctx, const vrf_mapping_config* cfg, uint64_t rng_state[4],
                      int n_keyframes, int n_rays, int n_steps, vrf_map_step_stats* out);
/* vrf_mapping_step with the batch already in device memory. */
int vrf_mapping_step_device(vrf_context* ctx, const vrf_mapping_config* cfg,
                            const int32_t* batch_dev, int n_rays, vrf_map_step_stats* out);
/* The merged grid gradient of one batch (no update): double [V][28] host. */
int vrf_mapping_gradient(vrf_context* ctx, const vrf_mapping_config* cfg, const int32_t* batch,
                         int n_rays, double* grad_out, vrf_map_step_stats* out);
/* RmspropState — mapping.hpp:48-52. */
int vrf_rmsprop_reset(vrf_context* ctx);
int vrf_rmsprop_download(vrf_context* ctx, double* v);
int vrf_rmsprop_upload(vrf_context* ctx, const double* v);
/* Multi-GPU phases (ray-sharded data parallel):
 *   forward (local partials) -> caller all-reduces partials ->
 *   backward with the GLOBAL hit counts -> caller reduce-scatters grad ->
 *   apply (RMSProp on the owned vertex shard, clears grad) -> caller all-gathers payload. */
int vrf_map_forward(vrf_context* ctx, const vrf_mapping_config* cfg, const int32_t* batch_dev,
                    int n_rays, vrf_map_partials* out);
int vrf_map_backward(vrf_context* ctx, const vrf_mapping_config* cfg, int32_t rays_color,
                     int32_t rays_depth);
int vrf_map_apply(vrf_context* ctx, const vrf_mapping_config* cfg, int64_t vertex_begin,
                  int64_t vertex_end);
/* Block-sparse variant of the exchange (distributed.py): the backward marks the
 * touched 8^3-vertex blocks; the caller max-all-reduces the per-block flags,
 * packs the touched blocks' gradients into [n][512][28] fp32 (ids_dev: int32
 * block ids, < 0 = padding; which 0 = gradient, 1 = payload), reduce-scatters
 * them by block owner, applies RMSProp to its own blocks, packs and all-gathers
 * the updated payload blocks, unpacks them and clears the gradient. */
int vrf_blocks_count(vrf_context* ctx, int32_t* n_blocks);
int vrf_blocks_touched(vrf_context* ctx, uint8_t* flags_dev);
int vrf_blocks_pack(vrf_context* ctx, const int32_t* ids_dev, int n, int which, float* out_dev);
int vrf_blocks_unpack_payload(vrf_context* ctx, const int32_t* ids_dev, int n,
                              const float* in_dev);
int vrf_blocks_apply(vrf_context* ctx, const vrf_mapping_config* cfg, const int32_t* ids_dev,
                     int n, const float* grad_packed_dev);
int vrf_grad_clear(vrf_context* ctx);

/* Fused exchange over peer memory (NVLink / NVSwitch), replacing the NCCL
 * block-sparse exchange above with ONE kernel: the owner of each touched
 * 8^3-vertex block (static owner id % world) reads every rank's gradient for the
 * block over peer memory, sums them in rank order, applies RMSProp
 * (mapping.cpp:218-231) to its payload and RMSProp state, and stores the updated
 * payload block into every rank's payload. Ordering is the caller's: call it
 * after a stream-ordered barrier that follows every rank's vrf_map_backward
 * (e.g. a one-element NCCL all-reduce on the same stream), then barrier again
 * before any rank reads its payload or clears its gradient (vrf_grad_clear).
 * Peer pointers are device pointers valid on this context's device: the other
 * contexts' buffers of the same process (vrf_peer_buffers_get), or IPC-opened
 * buffers of other processes (vrf_ipc_export on every rank, exchange the bytes,
 * vrf_peers_open_ipc). The table is dropped when the grid is re-allocated. */
#define VRF_MAX_PEERS 8
#define VRF_IPC_HANDLE_BYTES 192 /* 3 x cudaIpcMemHandle_t: gradient, payload, touched bitmap */
typedef struct {
  uint64_t grad, payload, tb; /* device addresses */
} vrf_peer_buffers;
int vrf_peer_buffers_get(vrf_context* ctx, vrf_peer_buffers* out);
int vrf_peers_set(vrf_context* ctx, int world, int rank, const vrf_peer_buffers* peers);
int vrf_ipc_export(vrf_context* ctx, uint8_t* handles);
int vrf_peers_open_ipc(vrf_context* ctx, int world, int rank, const uint8_t* handles);
int vrf_exchange_p2p(vrf_context* ctx, const vrf_mapping_config* cfg);

/* ---- tracking */
/* pose_gradient — tracking.hpp:70-73 (tracking.cpp:76-143); pixels: n (px, py). */
int vrf_pose_gradient(vrf_context* ctx, int frame, const vrf_intrinsics* intr,
                      const vrf_pose* pose, const int32_t* pixels, int n,
                      const vrf_tracking_loss* cfg, vrf_pose_gradient_result* out);
int vrf_pose_normal_equations(vrf_context* ctx, int frame, const vrf_intrinsics* intr,
                              const vrf_pose* pose, const int32_t* pixels, int n,
                              const vrf_tracking_loss* cfg, vrf_normal_equations* out);
/* The same normal equations through a chosen pose kernel (VRF_POSE_KERNEL_*):
 * the parity tests evaluate the Gauss-Newton kernel on fixed pixels with it. */
int vrf_pose_normal_equations_ex(vrf_context* ctx, int frame, const vrf_intrinsics* intr,
                                 const vrf_pose* pose, const int32_t* pixels, int n,
                                 const vrf_tracking_loss* cfg, int kernel,
                                 vrf_normal_equations* out);
/* track_frame — tracking.hpp:82-84 (tracking.cpp:170-252): Adam, pixel draws from
 * the reference Rng stream (xoshiro256**, seed cfg->seed). loss_trace: iterations. */
int vrf_track_frame(vrf_context* ctx, int frame, const vrf_intrinsics* intr,
                    const vrf_pose* init, const vrf_tracking_config* cfg,
                    vrf_track_frame_result* out, double* loss_trace);
/* Gauss-Newton/LM tracking with the whole iteration loop on the device (one CUDA
 * graph: draw -> render+Jacobian -> reduce -> 6x6 solve -> pose update). */
int vrf_track_frame_gn(vrf_context* ctx, int frame, const vrf_intrinsics* intr,
                       const vrf_pose* init, const vrf_gn_config* cfg,
                       vrf_track_frame_result* out);
/* Per-iteration record of the last vrf_track_frame_gn call: hist[3 i .. 3 i + 2] =
 * (loss / m, m, composited samples) of iteration i, as evaluated before its step.
 * Copies min(cap, 3 * iterations) doubles; returns the iteration count. */
int vrf_track_frame_gn_history(vrf_context* ctx, double* hist, int cap);

/* ---- evaluation: evaluate_map_quality (eval.cpp:210-240) with the views rendered
 * and scored on the device. n_views views at poses[v] against the reference images
 * colors[v] (H*W*3) / depths[v] (H*W), host memory. samples: n_samples (view, x, y)
 * triples — the PSNR pixel draws (vrf_rng_draw_eval_samples). Sums over the pixels
 * the render hit (rendered depth > 0): squared colour error over the samples
 * (psnr, eval.cpp:64-97) and |D - D*| over valid reference depth (depth_l1,
 * eval.cpp:99-122). */
typedef struct {
  double sum_sq_color;   /* sum over hit samples of sum_ch (C - C*)^2 */
  int64_t color_samples;
  double sum_abs_depth;  /* sum over hit pixels with D* > 0 of |D - D*| */
  int64_t depth_pixels;
} vrf_view_metrics;
int vrf_evaluate_views(vrf_context* ctx, const vrf_intrinsics* intr, int n_views,
                       const vrf_pose* poses, const double* const* colors,
                       const double* const* depths, const vrf_render_params* params,
                       const int32_t* samples, int n_samples, vrf_view_metrics* out);
/* eval.cpp:72-83's draws: per image draw, image = U[n_images), then pixels_per_image
 * (x = U[width), y = U[height)); out: images * pixels_per_image (image, x, y). */
void vrf_rng_draw_eval_samples(uint64_t state[4], int n_images, int width, int height,
                               int images, int pixels_per_image, int32_t* out);

/* ---- host helpers: the reference's Rng stream (rng.hpp:13-81, xoshiro256**) */
void vrf_rng_seed(uint64_t seed, uint64_t state[4]);
uint64_t vrf_rng_next(uint64_t state[4]);
/* mapping.cpp:121-128: per ray frame = U[n_frames), px = U[width), py = U[height) */
void vrf_rng_draw_batch(uint64_t state[4], int n_frames, int width, int height, int n,
                        int32_t* batch);
/* tracking.cpp:147-166; returns the number of pixels written (<= count) */
int vrf_rng_draw_valid_pixels(uint64_t state[4], const double* depth, int width, int height,
                              int count, int max_redraws, int32_t* pixels);

/* ---- inspection (parity tests): sample_ray / render_ray per explicit ray.
 * rays: n * (ox, oy, oz, dx, dy, dz). */
int vrf_debug_sample_rays(vrf_context* ctx, const double* rays, int n,
                          const vrf_render_params* params, int cap, int32_t* counts,
                          double* t, double* delta, uint32_t* cells);
/* out: n * 8 doubles (r, g, b, depth, T_terminal, count, hit, terminated_early). */
int vrf_debug_render_rays(vrf_context* ctx, const double* rays, int n,
                          const vrf_render_params* params, double* out);

#ifdef __cplusplus
}
#endif
#endif /* VOXRF_B200_H */
