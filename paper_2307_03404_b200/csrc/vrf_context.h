// Internal: the vrf_context definition and host helpers shared by the C-ABI
// translation units (vrf_capi.cu, vrf_map.cu, vrf_pose.cu).
#pragma once

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/voxrf_b200.h"
#include "vrf_internal.h"

namespace vrf_host {

struct DeviceScratch {
  void* ptr = nullptr;
  size_t bytes = 0;
};

}  // namespace vrf_host

using vrf::DevPose;
using vrf::MapStats;
using vrf::PosePartial;

struct vrf_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  std::string err;
  int shard_multiple = 1;
  long long launches = 0;

  // grid
  bool has_grid = false;
  vrf_grid_geometry geom{};
  long long V = 0, Vpad = 0, C = 0;
  float* payload = nullptr;
  float4* payload_soa = nullptr;  // A/B only (VRF_GATHER_SOA): [7][V] copy for K0's gathers
  float* grad = nullptr;
  float* rms = nullptr;
  uint32_t* occ = nullptr;
  uint32_t* bocc = nullptr;  // 8^3-cell block occupancy (empty-space skipping)
  int bdim[3] = {0, 0, 0};
  uint32_t* socc = nullptr;  // 64^3-cell superblock occupancy
  int sdim[3] = {0, 0, 0};
  uint32_t* tb = nullptr;    // touched 8^3-vertex blocks of the pending gradient
  uint32_t* tc = nullptr;    // touched 8^3-cell blocks marked by the scatter (-> tb)
  // fused peer-memory exchange (vrf_peers_set / vrf_peers_open_ipc / vrf_exchange_p2p)
  vrf::PeerTable peers{};
  bool peers_set = false;
  void* ipc_open[vrf::kMaxPeers][3] = {};  // IPC-opened peer buffers (closed with the grid)
  int tdim[3] = {0, 0, 0};
  bool touched_valid = false;  // every nonzero gradient group lies in a marked block
  bool all_blocks_active = false;
  unsigned int* d_nblocks = nullptr;

  // frames
  int n_frames = 0;         // slots in use (high-water mark of vrf_frame_set)
  int frame_capacity = 0;   // allocated slots
  vrf_intrinsics fintr{};
  double4* rgbd = nullptr;
  DevPose* poses = nullptr;
  std::vector<std::vector<double>> host_depth;

  // persistent small device state
  int* d_err = nullptr;
  MapStats* d_stats = nullptr;
  int* d_counts = nullptr;
  PosePartial* d_pose_out = nullptr;
  DevPose* d_pose = nullptr;
  // pinned host staging
  void* h_pinned = nullptr;
  size_t h_pinned_bytes = 0;
  // pinned double buffer of the pipelined mapping loop (vrf_mapping_steps)
  void* h_pipe = nullptr;
  size_t h_pipe_bytes = 0;
  // vrf_mapping_steps: the next batch's H2D runs on its own stream during the
  // current step (created on first use)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t copy_ev[2] = {nullptr, nullptr};

  // grow-only scratch
  vrf_host::DeviceScratch s_batch, s_raycd, s_flags, s_partials, s_count, s_offsets, s_keys, s_keys2,
      s_ids, s_ids2, s_values, s_grad64, s_cub, s_stage, s_out, s_batch2, s_rec, s_reccount;
  // fast-path sample records of the last forward (0 = recompute-march backward)
  int rec_K = 0;
  size_t rec_slots = 0;  // records per plane of s_rec (nn32 * rec_K; rec_planes)
  int max_ray_samples = 0;  // longest ray seen by a mapping forward (sizes rec_K)
  long long rec_need_tried = 0;  // last record depth the budget was evaluated for
  // RMSProp update log for the drop-in's sparse write-back (vrf_track_updates)
  bool log_updates = false;
  vrf_host::DeviceScratch s_upd_ids, s_upd_theta, s_upd_v;
  unsigned long long* d_upd_count = nullptr;
  // sorted view of the log (vrf_updates_read_range): ids, log positions, scratch
  vrf_host::DeviceScratch s_upd_sids, s_upd_perm, s_upd_iota, s_upd_tmp, s_upd_gth, s_upd_gv;
  bool upd_sorted = false;  // the sorted view matches the current log
  unsigned long long* d_digest = nullptr;
  double rec_budget_gb = -1.0;   // vrf_set_record_limits: <= 0 automatic (30 % of free HBM)
  int rec_max_k = -1;            // vrf_set_record_limits: < 0 automatic, 0 no records

  // multi-GPU phase state
  const int* last_batch = nullptr;
  int last_n = 0;

  // profiling: CUDA events around kernels on the context stream (vrf_profile_*)
  bool profiling = false;
  double prof_ms[8] = {0};
  long long prof_launches[8] = {0};
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  unsigned long long* d_touched = nullptr;  // RMSProp float4 groups updated
  long long prof_track_samples = 0;          // composited samples of GN tracking frames

  // coherent ray order (vrf_order.cu): keys, ids, sorted order, cub scratch
  vrf_host::DeviceScratch s_order, s_okeys, s_okeys2, s_oids, s_otmp;

  // tracking device state: frame index, Gauss-Newton pose / seed / history, and the
  // CUDA graph of one GN frame (re-captured when its key changes)
  int* d_frame = nullptr;
  DevPose* d_gn_pose = nullptr;
  unsigned long long* d_gn_seed = nullptr;
  double* d_gn_hist = nullptr;
  int gn_hist_cap = 0;
  std::vector<double> gn_last_hist;  // (loss/m, m, samples) per iteration of the last GN frame
  long long grid_generation = 0;
  cudaGraphExec_t gn_graph = nullptr;
  std::vector<unsigned char> gn_key;
};

namespace vrf_host {
using namespace vrf;

inline int set_err(vrf_context* c, int code, const std::string& m) {
  c->err = m;
  return code;
}

#define CU(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      return set_err(ctx, VRF_ERR_CUDA, std::string("cuda: ") + cudaGetErrorString(e_) + \
                                            " (" #x ")");                               \
  } while (0)

#define LAUNCHED(n) (ctx->launches += (n))

// Grow-only scratch. Work already queued on the context stream may still be
// using the old buffer (the multi-GPU phases return without a host sync), and
// cudaFree does not order itself after it: drain the stream before freeing.
inline int ensure(vrf_context* ctx, DeviceScratch& s, size_t bytes) {
  if (s.bytes >= bytes) return VRF_OK;
  if (s.ptr) {
    CU(cudaStreamSynchronize(ctx->stream));
    CU(cudaFree(s.ptr));
  }
  s.ptr = nullptr;
  s.bytes = 0;
  // 25 % headroom against regrowth, but none on multi-GB buffers
  const size_t want = bytes < 256 ? 256 : (bytes > (1ull << 30) ? bytes : bytes + bytes / 4);
  CU(cudaMalloc(&s.ptr, want));
  s.bytes = want;
  return VRF_OK;
}

// Like ensure, but an out-of-memory result is not an error: returns false (and
// clears the sticky CUDA error) so the caller can shrink the request.
inline bool try_ensure(cudaStream_t stream, DeviceScratch& s, size_t bytes) {
  if (s.bytes >= bytes) return true;
  if (s.ptr) {
    cudaStreamSynchronize(stream);
    cudaFree(s.ptr);
  }
  s.ptr = nullptr;
  s.bytes = 0;
  if (cudaMalloc(&s.ptr, bytes) != cudaSuccess) {
    cudaGetLastError();
    s.ptr = nullptr;
    return false;
  }
  s.bytes = bytes;
  return true;
}

inline int ensure_pinned(vrf_context* ctx, size_t bytes) {
  if (ctx->h_pinned_bytes >= bytes) return VRF_OK;
  if (ctx->h_pinned) {
    CU(cudaStreamSynchronize(ctx->stream));
    CU(cudaFreeHost(ctx->h_pinned));
  }
  ctx->h_pinned = nullptr;
  const size_t want = bytes < 4096 ? 4096 : bytes + bytes / 4;
  CU(cudaMallocHost(&ctx->h_pinned, want));
  ctx->h_pinned_bytes = want;
  return VRF_OK;
}

inline void close_peers(vrf_context* ctx) {
  for (auto& row : ctx->ipc_open)
    for (void*& p : row) {
      if (p) cudaIpcCloseMemHandle(p);
      p = nullptr;
    }
  ctx->peers = PeerTable{};
  ctx->peers_set = false;
}

inline void free_grid(vrf_context* ctx) {
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);  // queued work may still use them
  close_peers(ctx);  // the peer table points at this grid's buffers
  cudaFree(ctx->payload);
  cudaFree(ctx->grad);
  cudaFree(ctx->rms);
  cudaFree(ctx->occ);
  cudaFree(ctx->bocc);
  cudaFree(ctx->socc);
  cudaFree(ctx->tb);
  cudaFree(ctx->tc);
  ctx->tc = nullptr;
  ctx->payload = ctx->grad = ctx->rms = nullptr;
  ctx->occ = nullptr;
  ctx->bocc = nullptr;
  ctx->socc = nullptr;
  ctx->tb = nullptr;
  ctx->touched_valid = false;
  ctx->has_grid = false;
}

inline int validate_geometry(vrf_context* ctx, const vrf_grid_geometry* g) {
  // GridGeometry::validate — voxel_grid.hpp:25-28
  if (!g) return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "grid: null geometry");
  if (std::min(g->res[0], std::min(g->res[1], g->res[2])) < 2)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "grid: resolution must be >= 2 per axis");
  if (!(g->voxel_size > 0.0))
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "grid: voxel_size must be > 0");
  const long long V = (long long)g->res[0] * g->res[1] * g->res[2];
  if (V > 0xFFFFFFFFLL)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "grid: more than 2^32 vertices");
  return VRF_OK;
}

inline int alloc_grid(vrf_context* ctx, const vrf_grid_geometry* g) {
  int rc = validate_geometry(ctx, g);
  if (rc) return rc;
  free_grid(ctx);
  ctx->geom = *g;
  ctx->V = (long long)g->res[0] * g->res[1] * g->res[2];
  ctx->C = (long long)(g->res[0] - 1) * (g->res[1] - 1) * (g->res[2] - 1);
  const long long m = ctx->shard_multiple;
  ctx->Vpad = (ctx->V + m - 1) / m * m;
  ++ctx->grid_generation;  // invalidates captured graphs that baked the old pointers
  CU(cudaMalloc(&ctx->payload, sizeof(float) * 28 * ctx->Vpad));
  CU(cudaMalloc(&ctx->grad, sizeof(float) * 28 * ctx->Vpad));
  CU(cudaMalloc(&ctx->rms, sizeof(float) * 28 * ctx->Vpad));
  CU(cudaMalloc(&ctx->occ, sizeof(uint32_t) * ((ctx->C + 31) / 32 + 1)));
  for (int a = 0; a < 3; ++a)
    ctx->bdim[a] = (g->res[a] - 1 + (1 << kBlockLog2) - 1) >> kBlockLog2;
  const long long nblk = (long long)ctx->bdim[0] * ctx->bdim[1] * ctx->bdim[2];
  CU(cudaMalloc(&ctx->bocc, sizeof(uint32_t) * ((nblk + 31) / 32 + 1)));
  CU(cudaMalloc(&ctx->tc, sizeof(uint32_t) * ((nblk + 31) / 32 + 1)));
  CU(cudaMemsetAsync(ctx->tc, 0, sizeof(uint32_t) * ((nblk + 31) / 32 + 1), ctx->stream));
  constexpr int kS = kSuperLog2 - kBlockLog2;
  for (int a = 0; a < 3; ++a) ctx->sdim[a] = (ctx->bdim[a] + (1 << kS) - 1) >> kS;
  const long long nsup = (long long)ctx->sdim[0] * ctx->sdim[1] * ctx->sdim[2];
  CU(cudaMalloc(&ctx->socc, sizeof(uint32_t) * ((nsup + 31) / 32 + 1)));
  for (int a = 0; a < 3; ++a) ctx->tdim[a] = (g->res[a] + (1 << kTouchLog2) - 1) >> kTouchLog2;
  const long long ntb = (long long)ctx->tdim[0] * ctx->tdim[1] * ctx->tdim[2];
  CU(cudaMalloc(&ctx->tb, sizeof(uint32_t) * ((ntb + 31) / 32 + 1)));
  CU(cudaMemsetAsync(ctx->tb, 0, sizeof(uint32_t) * ((ntb + 31) / 32 + 1), ctx->stream));
  ctx->touched_valid = false;
  CU(cudaMemsetAsync(ctx->payload, 0, sizeof(float) * 28 * ctx->Vpad, ctx->stream));
  CU(cudaMemsetAsync(ctx->grad, 0, sizeof(float) * 28 * ctx->Vpad, ctx->stream));
  CU(cudaMemsetAsync(ctx->rms, 0, sizeof(float) * 28 * ctx->Vpad, ctx->stream));
  ctx->has_grid = true;
  return VRF_OK;
}

inline int need_grid(vrf_context* ctx) {
  if (!ctx->has_grid) return set_err(ctx, VRF_ERR_RUNTIME, "voxrf_b200: no grid loaded");
  return VRF_OK;
}

inline DevGrid dev_grid(const vrf_context* ctx) {
  DevGrid g;
  const vrf_grid_geometry& q = ctx->geom;
  g.rx = q.res[0];
  g.ry = q.res[1];
  g.rz = q.res[2];
  g.rxy = (uint32_t)q.res[0] * (uint32_t)q.res[1];
  g.ox = q.origin[0];
  g.oy = q.origin[1];
  g.oz = q.origin[2];
  g.hx = q.origin[0] + ((double)q.res[0] - 1.0) * q.voxel_size;
  g.hy = q.origin[1] + ((double)q.res[1] - 1.0) * q.voxel_size;
  g.hz = q.origin[2] + ((double)q.res[2] - 1.0) * q.voxel_size;
  g.voxel = q.voxel_size;
  g.inv_voxel = 1.0 / q.voxel_size;
  g.rcp_voxel = 1.0 / q.voxel_size;
  g.payload = reinterpret_cast<const float4*>(ctx->payload);
  g.soa = ctx->payload_soa;
  g.soa_stride = (long long)ctx->V;
  g.occ = ctx->occ;
  g.bocc = ctx->bocc;
  g.bx = ctx->bdim[0];
  g.by = ctx->bdim[1];
  g.bz = ctx->bdim[2];
  g.socc = ctx->socc;
  g.sx = ctx->sdim[0];
  g.sy = ctx->sdim[1];
  g.sz = ctx->sdim[2];
  g.tb = ctx->tb;
  g.tc = ctx->tc;
  g.tbx = ctx->tdim[0];
  g.tby = ctx->tdim[1];
  g.tbz = ctx->tdim[2];
  g.all_blocks_active = ctx->all_blocks_active ? 1 : 0;
  return g;
}

// Rebuild the 8^3-cell block occupancy after any change of the cell occupancy
// (synchronous: occupancy changes are per upload / prune, not per step).
inline int update_blocks(vrf_context* ctx) {
  if (!ctx->d_nblocks) CU(cudaMalloc(&ctx->d_nblocks, sizeof(unsigned int)));
  launch_block_occupancy(ctx->occ, ctx->geom.res[0], ctx->geom.res[1], ctx->geom.res[2],
                         ctx->bdim[0], ctx->bdim[1], ctx->bdim[2], ctx->bocc, ctx->d_nblocks,
                         ctx->stream);
  launch_super_occupancy(ctx->bocc, ctx->bdim[0], ctx->bdim[1], ctx->bdim[2], ctx->sdim[0],
                         ctx->sdim[1], ctx->sdim[2], ctx->socc, ctx->stream);
  ctx->launches += 1;
  unsigned int n = 0;
  CU(cudaMemcpyAsync(&n, ctx->d_nblocks, sizeof(n), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->all_blocks_active = (long long)n == (long long)ctx->bdim[0] * ctx->bdim[1] * ctx->bdim[2];
  return VRF_OK;
}

// RenderParams::effective_step/effective_t_far (renderer.hpp:18-24) and the
// sample_ray argument checks (renderer.cpp:56-58).
inline int resolve_params(vrf_context* ctx, const vrf_render_params* rp, DevParams* out) {
  const vrf_grid_geometry& q = ctx->geom;
  const double step = rp->step > 0.0 ? rp->step : 0.5 * q.voxel_size;
  double e[3];
  for (int a = 0; a < 3; ++a)
    e[a] = (q.origin[a] + ((double)q.res[a] - 1.0) * q.voxel_size) - q.origin[a];
  const double diag = std::sqrt((e[0] * e[0] + e[1] * e[1]) + e[2] * e[2]);
  const double t_far = rp->t_far > 0.0 ? rp->t_far : diag;
  if (!(step > 0.0)) return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "sample_ray: step must be > 0");
  if (!(rp->t_near >= 0.0) || t_far <= rp->t_near)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "sample_ray: need 0 <= t_near < t_far");
  out->step = step;
  out->t_near = rp->t_near;
  out->t_far = t_far;
  out->eps = rp->termination_eps;
  return VRF_OK;
}

inline DevCam dev_cam(const vrf_intrinsics* in) {
  DevCam c;
  c.fx = in->fx;
  c.fy = in->fy;
  c.cx = in->cx;
  c.cy = in->cy;
  c.width = in->width;
  c.height = in->height;
  return c;
}

inline DevPose dev_pose(const vrf_pose* p) {
  DevPose d;
  for (int i = 0; i < 4; ++i) d.q[i] = p->q[i];
  for (int i = 0; i < 3; ++i) d.t[i] = p->t[i];
  d.pad = 0.0;
  return d;
}

// Device error flags -> the reference's exception classes.
inline int err_from_flag(vrf_context* ctx, int flag) {
  if (flag & 2) return set_err(ctx, VRF_ERR_OUT_OF_RANGE, "generate_ray: pixel outside image");
  if (flag & 1)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "sh_eval: direction must be unit length");
  return VRF_OK;
}

inline int check_err_flag(vrf_context* ctx) {
  int flag = 0;
  CU(cudaMemcpyAsync(&flag, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (flag & 2) return set_err(ctx, VRF_ERR_OUT_OF_RANGE, "generate_ray: pixel outside image");
  if (flag & 1)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "sh_eval: direction must be unit length");
  return VRF_OK;
}

inline int check_frames(vrf_context* ctx, const vrf_intrinsics* intr) {
  if (ctx->n_frames == 0) return VRF_OK;
  if (intr->width != ctx->fintr.width || intr->height != ctx->fintr.height)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT,
                   "voxrf_b200: intrinsics size differs from the uploaded frames");
  return VRF_OK;
}

// Kernel-time slots reported by vrf_profile_read.
enum ProfSlot { kProfMapForward = 0, kProfMapBackward = 1, kProfRmsprop = 2, kProfMapMisc = 3,
                kProfPoseForward = 4, kProfPoseBackward = 5, kProfRender = 6, kProfDet = 7 };

inline cudaEvent_t prof_begin(vrf_context* ctx) {
  if (!ctx->profiling) return nullptr;
  cudaEvent_t b;
  cudaEventCreate(&b);
  cudaEventRecord(b, ctx->stream);
  return b;
}
inline void prof_end(vrf_context* ctx, int slot, cudaEvent_t b) {
  if (!ctx->profiling || !b) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, ctx->stream);
  ctx->pending.push_back({slot, {b, e}});
}
// After a stream sync: fold the recorded intervals into the per-slot totals.
inline void prof_collect(vrf_context* ctx) {
  for (auto& p : ctx->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.second.first, p.second.second) == cudaSuccess) {
      ctx->prof_ms[p.first] += ms;
      ctx->prof_launches[p.first] += 1;
    }
    cudaEventDestroy(p.second.first);
    cudaEventDestroy(p.second.second);
  }
  ctx->pending.clear();
}

inline double psnr_from_lp(double lp) {  // mapping.cpp:107-110
  if (lp <= 0.0) return 99.0;
  return std::min(99.0, 10.0 * std::log10(3.0 / lp));
}

// ----------------------------------------------------------------- mapping internals
// Forward + fixed-order reduce for a device batch; leaves ray_cd/flags/stats on device.
inline int map_forward_dev(vrf_context* ctx, const vrf_mapping_config* cfg, const int* batch_dev,
                           int n, bool fast, int* ray_count = nullptr) {
#ifdef VRF_GATHER_SOA
  if (fast) {  // A/B: refresh the planar copy K0 gathers from (misc slot, not K0)
    if (!ctx->payload_soa) CU(cudaMalloc(&ctx->payload_soa, sizeof(float4) * 7 * ctx->V));
    cudaEvent_t pt = prof_begin(ctx);
    launch_aos_to_soa((const float4*)ctx->payload, ctx->payload_soa, ctx->V, ctx->stream);
    prof_end(ctx, kProfMapMisc, pt);
  }
#endif
  const DevGrid g = dev_grid(ctx);
  DevParams p;
  int rc = resolve_params(ctx, &cfg->render, &p);
  if (rc) return rc;
  // (the record path may run the 8-lanes-per-ray K0g: size the partials for it)
  const int nb = std::max(map_forward_blocks(n > 0 ? n : 1),
                          fast ? map_forward_rec_blocks(n > 0 ? n : 1) : 0);
  const size_t nn = (size_t)(n > 0 ? n : 1);
  if ((rc = ensure(ctx, ctx->s_raycd, sizeof(double4) * nn))) return rc;
  if ((rc = ensure(ctx, ctx->s_flags, nn))) return rc;
  if ((rc = ensure(ctx, ctx->s_partials, sizeof(MapPartial) * nb))) return rc;
  CU(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
  if (n > 0 && fast) {
    // (keyframe, Morton tile) ray order for L2 locality.
    const size_t tmp = ray_order_tmp_bytes(n);
    if ((rc = ensure(ctx, ctx->s_order, sizeof(uint32_t) * nn))) return rc;
    if ((rc = ensure(ctx, ctx->s_okeys, sizeof(uint32_t) * nn))) return rc;
    if ((rc = ensure(ctx, ctx->s_okeys2, sizeof(uint32_t) * nn))) return rc;
    if ((rc = ensure(ctx, ctx->s_oids, sizeof(uint32_t) * nn))) return rc;
    if ((rc = ensure(ctx, ctx->s_otmp, tmp))) return rc;
    cudaEvent_t po = prof_begin(ctx);
    launch_ray_order(batch_dev, n, (uint32_t*)ctx->s_okeys.ptr, (uint32_t*)ctx->s_oids.ptr,
                     (uint32_t*)ctx->s_okeys2.ptr, (uint32_t*)ctx->s_order.ptr, ctx->s_otmp.ptr,
                     tmp, ctx->stream);
    prof_end(ctx, kProfMapMisc, po);
    LAUNCHED(1);  // k_ray_keys (the cub radix sort behind it is a library launch)
    // Sample records for the backward: up to K per ray. K covers the longest
    // ray seen so far (x1.25, rounded up to a power of two; 1024 before the first
    // step), within a memory budget (VRF_REC_GB; default 30 % of the free HBM
    // plus the record buffer already held). The buffer regrows only when that
    // at least doubles K, so steps do not reallocate. Longer rays overflow to
    // the recompute-march backward.
    ctx->rec_K = 0;
    // records carry 10-bit cell coordinates: larger grids take the recompute-march
    // backward (no records)
    const bool rec_fits = ctx->geom.res[0] - 1 <= kRecMaxCells &&
                          ctx->geom.res[1] - 1 <= kRecMaxCells &&
                          ctx->geom.res[2] - 1 <= kRecMaxCells;
    if (ctx->rec_max_k != 0 && rec_fits) {
      const double env_gb = ctx->rec_budget_gb > 0.0 ? ctx->rec_budget_gb : -1.0;
      long long need = 1024;
      if (ctx->max_ray_samples > 0) {
        need = 64;
        while (need < ctx->max_ray_samples * 5LL / 4 && need < 1024) need *= 2;
      }
      const size_t nn32 = (nn + 31) & ~(size_t)31;  // warp-tiled record layout
      const double per_level = (double)nn32 * (double)kRecBytes;
      // K the held buffer already covers; regrow only for a real shortfall
      // (2x), so a budget-limited cap does not reallocate every step
      const long long held_K = (long long)((double)ctx->s_rec.bytes / per_level);
      long long K = std::min(need, held_K);
      // (the budget is re-derived once per new `need`, not every step: a
      // budget-capped buffer would otherwise query cudaMemGetInfo each step)
      if (held_K < 16 || (need >= 2 * held_K && need != ctx->rec_need_tried)) {
        ctx->rec_need_tried = need;
        double budget = env_gb * 1e9;
        if (env_gb < 0.0) {
          size_t free_b = 0, total_b = 0;
          CU(cudaMemGetInfo(&free_b, &total_b));
          budget = 0.30 * (double)free_b + (double)ctx->s_rec.bytes;
        }
        const long long cand = std::min(need, (long long)(budget / per_level));
        if (held_K < 16 || cand >= 2 * held_K) K = cand;  // grow only by a real factor
      }
      // an explicit cap (tests force the overflow backward with a small K)
      const long long kmin = ctx->rec_max_k > 0 ? 4 : 16;
      if (ctx->rec_max_k > 0) K = std::min<long long>(std::max(K, kmin), ctx->rec_max_k);
      K &= ~3LL;
      // other allocators (e.g. torch's caching allocator in the multi-GPU
      // driver) may hold memory the budget counted: halve on out-of-memory
      while (K >= kmin &&
             !try_ensure(ctx->stream, ctx->s_rec, kRecBytes * nn32 * (size_t)K))
        K /= 2;
      if (K >= kmin) {
        if ((rc = ensure(ctx, ctx->s_reccount, sizeof(int2) * nn))) return rc;
        ctx->rec_K = (int)(K & ~3LL);
        ctx->rec_slots = nn32 * (size_t)ctx->rec_K;
      }
    }
    cudaEvent_t pb = prof_begin(ctx);
    if (ctx->rec_K > 0)
      launch_map_forward_rec(g, p, dev_cam(&ctx->fintr), ctx->rgbd, ctx->poses, ctx->n_frames,
                             batch_dev, n, (double4*)ctx->s_raycd.ptr, (uint8_t*)ctx->s_flags.ptr,
                             (MapPartial*)ctx->s_partials.ptr, ctx->d_err,
                             (const uint32_t*)ctx->s_order.ptr,
                             rec_planes(ctx->s_rec.ptr, ctx->rec_slots),
                             ctx->rec_K, (int2*)ctx->s_reccount.ptr, ctx->stream);
    else
      launch_map_forward(g, p, dev_cam(&ctx->fintr), ctx->rgbd, ctx->poses, ctx->n_frames,
                         batch_dev, n, (double4*)ctx->s_raycd.ptr, (uint8_t*)ctx->s_flags.ptr,
                         (MapPartial*)ctx->s_partials.ptr, nullptr, ctx->d_err, true,
                         (const uint32_t*)ctx->s_order.ptr, ctx->stream);
    prof_end(ctx, kProfMapForward, pb);
    LAUNCHED(1);
  } else if (n > 0) {
    ctx->rec_K = 0;
    cudaEvent_t pb = prof_begin(ctx);
    launch_map_forward(g, p, dev_cam(&ctx->fintr), ctx->rgbd, ctx->poses, ctx->n_frames,
                       batch_dev, n, (double4*)ctx->s_raycd.ptr, (uint8_t*)ctx->s_flags.ptr,
                       (MapPartial*)ctx->s_partials.ptr, ray_count, ctx->d_err, false, nullptr,
                       ctx->stream);
    prof_end(ctx, kProfMapForward, pb);
    LAUNCHED(1);
  } else {
    CU(cudaMemsetAsync(ctx->s_partials.ptr, 0, sizeof(MapPartial), ctx->stream));
  }
  // partials the launched forward wrote (K0g: 16 rays per CTA)
  const int nparts = (n > 0 && fast && ctx->rec_K > 0) ? map_forward_rec_blocks(n)
                                                       : map_forward_blocks(n > 0 ? n : 1);
  launch_map_reduce((const MapPartial*)ctx->s_partials.ptr, n > 0 ? nparts : 0, ctx->d_stats,
                    ctx->stream);
  LAUNCHED(1);
  CU(cudaGetLastError());
  return VRF_OK;
}

}  // namespace vrf_host

