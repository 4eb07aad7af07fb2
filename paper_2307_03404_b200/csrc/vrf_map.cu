// Mapping entry points of the C-ABI: mapping_step (mapping.cpp:114-233) on the
// device, its deterministic sorted/segmented-reduce variant, and the phases the
// multi-GPU driver composes with NCCL collectives.
#include <cstring>
#include <string>

#include <cub/cub.cuh>

#include "vrf_context.h"

using namespace vrf;
using namespace vrf_host;

namespace {

int validate_batch(vrf_context* ctx, const int32_t* batch, int n) {
  // mapping.cpp:121-128 draws frame < K, px < W, py < H; anything else would make
  // generate_ray throw std::out_of_range (camera.hpp:38-39).
  for (int i = 0; i < n; ++i) {
    const int32_t f = batch[3 * i], x = batch[3 * i + 1], y = batch[3 * i + 2];
    if (f < 0 || f >= ctx->n_frames)
      return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "mapping_step: keyframe index out of range");
    if (x < 0 || x >= ctx->fintr.width || y < 0 || y >= ctx->fintr.height)
      return set_err(ctx, VRF_ERR_OUT_OF_RANGE, "generate_ray: pixel outside image");
  }
  return VRF_OK;
}

int upload_batch(vrf_context* ctx, const int32_t* batch, int n, const int** dev) {
  int rc = validate_batch(ctx, batch, n);
  if (rc) return rc;
  const size_t bytes = sizeof(int32_t) * 3 * (size_t)(n > 0 ? n : 1);
  if ((rc = ensure(ctx, ctx->s_batch, bytes))) return rc;
  if ((rc = ensure_pinned(ctx, bytes))) return rc;
  if (n > 0) {
    std::memcpy(ctx->h_pinned, batch, sizeof(int32_t) * 3 * (size_t)n);
    CU(cudaMemcpyAsync(ctx->s_batch.ptr, ctx->h_pinned, sizeof(int32_t) * 3 * (size_t)n,
                       cudaMemcpyHostToDevice, ctx->stream));
  }
  *dev = (const int*)ctx->s_batch.ptr;
  return VRF_OK;
}

int read_stats(vrf_context* ctx, MapStats* st) {
  CU(cudaMemcpyAsync(st, ctx->d_stats, sizeof(MapStats), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->max_ray_samples = std::max(ctx->max_ray_samples, st->max_count);
  return VRF_OK;
}

// MapStepStats + the reference's exceptions (mapping.cpp:117, 152, 198-203, 213-216).
int finish_stats(vrf_context* ctx, const vrf_mapping_config* cfg, const MapStats& st,
                 const int* batch_host, vrf_map_step_stats* out) {
  vrf_map_step_stats s{};
  s.rays_color = st.m_c;
  s.rays_depth = st.m_d;
  s.samples = st.samples;
  s.bad_ray = st.bad == INT_MAX ? -1 : st.bad;
  if (out) *out = s;
  if (st.m_c == 0) return set_err(ctx, VRF_ERR_RUNTIME, "mapping_step: no ray hit the grid");
  if (st.bad != INT_MAX) {
    std::string msg = "mapping_step: non-finite loss";
    if (batch_host) {
      const int* b = batch_host + 3 * st.bad;
      msg += " at keyframe " + std::to_string(b[0]) + " pixel (" + std::to_string(b[1]) + "," +
             std::to_string(b[2]) + ")";
    }
    return set_err(ctx, VRF_ERR_RUNTIME, msg);
  }
  s.loss_photometric = st.lp / double(st.m_c);
  s.loss_geometric = st.m_d > 0 ? st.lg / double(st.m_d) : 0.0;
  s.loss_total = s.loss_photometric + cfg->lambda_d * s.loss_geometric;
  s.psnr_estimate = psnr_from_lp(s.loss_photometric);
  if (out) *out = s;
  return VRF_OK;
}

// K3: deterministic fp64 gradient into s_grad64 [V][28], summed per vertex in
// the reference's order (ray, sample, corner) — GradientBuffer::add with one
// worker (gradients.cpp:28-41, mapping.cpp:205-207). Needs the forward state
// (ray_cd, flags, per-ray counts in s_count) and the host copy of the stats.
int grad_deterministic(vrf_context* ctx, const vrf_mapping_config* cfg, const int* batch_dev,
                       int n, const MapStats& st) {
  ctx->touched_valid = false;  // the fp64 -> fp32 copy writes every vertex
  DevParams p;
  int rc = resolve_params(ctx, &cfg->render, &p);
  if (rc) return rc;
  if ((rc = ensure(ctx, ctx->s_grad64, sizeof(double) * 28 * (size_t)ctx->V))) return rc;
  CU(cudaMemsetAsync(ctx->s_grad64.ptr, 0, sizeof(double) * 28 * (size_t)ctx->V, ctx->stream));
  if (st.m_c == 0 || st.bad != INT_MAX || st.samples == 0) return VRF_OK;
  if ((rc = ensure(ctx, ctx->s_offsets, sizeof(long long) * (n + 1)))) return rc;
  long long* offsets = (long long*)ctx->s_offsets.ptr;
  size_t tmp_scan = 0;
  CU(cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, (const int*)ctx->s_count.ptr, offsets, n,
                                   ctx->stream));
  if ((rc = ensure(ctx, ctx->s_cub, tmp_scan))) return rc;
  CU(cub::DeviceScan::ExclusiveSum(ctx->s_cub.ptr, tmp_scan, (const int*)ctx->s_count.ptr,
                                   offsets, n, ctx->stream));
  // (cub kernels are library launches: not counted in vrf_kernel_launch_count)
  // Chunk the batch by rays so the records (36 doubles per sample + 8 keys/ids)
  // stay bounded; every chunk continues each vertex's running fp64 sum.
  std::vector<int> counts((size_t)n);
  CU(cudaMemcpyAsync(counts.data(), ctx->s_count.ptr, sizeof(int) * (size_t)n,
                     cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  const char* chunk_env = std::getenv("VRF_DET_CHUNK");  // tests force small chunks
  const long long kChunkSamples = chunk_env ? std::max(1LL, std::atoll(chunk_env))
                                            : (1LL << 22);  // 4M samples: 1.2 GB of records
  long long sid_base = 0;
  for (int r0 = 0; r0 < n;) {
    int r1 = r0;
    long long S = 0;
    while (r1 < n && (S == 0 || S + counts[r1] <= kChunkSamples)) S += counts[r1++];
    if (S > 0) {
      const long long R = 8 * S;
      if (R >= 0x7FFFFFFFLL)
        return set_err(ctx, VRF_ERR_RUNTIME, "deterministic mapping: one ray has too many samples");
      size_t tmp_sort = 0;
      CU(cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, (const uint32_t*)nullptr,
                                         (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                         (uint32_t*)nullptr, (int)R, 0, 32, ctx->stream));
      if ((rc = ensure(ctx, ctx->s_cub, tmp_sort))) return rc;
      if ((rc = ensure(ctx, ctx->s_keys, sizeof(uint32_t) * R))) return rc;
      if ((rc = ensure(ctx, ctx->s_keys2, sizeof(uint32_t) * R))) return rc;
      if ((rc = ensure(ctx, ctx->s_ids, sizeof(uint32_t) * R))) return rc;
      if ((rc = ensure(ctx, ctx->s_ids2, sizeof(uint32_t) * R))) return rc;
      if ((rc = ensure(ctx, ctx->s_values, sizeof(double) * 36 * S))) return rc;
      launch_map_backward_records(dev_grid(ctx), p, dev_cam(&ctx->fintr), ctx->rgbd, ctx->poses,
                                  batch_dev, n, (const double4*)ctx->s_raycd.ptr,
                                  (const uint8_t*)ctx->s_flags.ptr, ctx->d_stats, cfg->lambda_d,
                                  offsets, (uint32_t*)ctx->s_keys.ptr, (uint32_t*)ctx->s_ids.ptr,
                                  (double*)ctx->s_values.ptr, r0, r1, sid_base, ctx->stream);
      // LSD radix sort is stable: equal vertices keep (ray, sample, corner) order.
      CU(cub::DeviceRadixSort::SortPairs(
          ctx->s_cub.ptr, tmp_sort, (const uint32_t*)ctx->s_keys.ptr,
          (uint32_t*)ctx->s_keys2.ptr, (const uint32_t*)ctx->s_ids.ptr,
          (uint32_t*)ctx->s_ids2.ptr, (int)R, 0, 32, ctx->stream));
      launch_segmented_reduce((const uint32_t*)ctx->s_keys2.ptr, (const uint32_t*)ctx->s_ids2.ptr,
                              (const double*)ctx->s_values.ptr, R, (double*)ctx->s_grad64.ptr,
                              ctx->stream);
      LAUNCHED(2);  // k_map_records + k_segmented_reduce (the cub sort is not ours)
      CU(cudaGetLastError());
    }
    sid_base += S;
    r0 = r1;
  }
  return VRF_OK;
}

// K2 on the coherent ray order of the preceding forward pass.
void launch_backward_fast(vrf_context* ctx, const vrf_mapping_config* cfg, const DevParams& p,
                          const int* batch_dev, int n, const int* global_counts) {
  cudaEvent_t pb = prof_begin(ctx);
  {
    if (ctx->rec_K > 0) {
      launch_map_backward_rec(dev_grid(ctx), p, dev_cam(&ctx->fintr), ctx->rgbd, ctx->poses,
                              batch_dev, n, (const double4*)ctx->s_raycd.ptr,
                              (const uint8_t*)ctx->s_flags.ptr, ctx->d_stats, global_counts,
                              (float4*)ctx->grad, cfg->lambda_d,
                              (const uint32_t*)ctx->s_order.ptr,
                              rec_planes(ctx->s_rec.ptr, ctx->rec_slots), ctx->rec_K,
                              (const int2*)ctx->s_reccount.ptr, ctx->stream);
      LAUNCHED(1);
    }
    // without records: every ray; with records: only the rays that overflowed K
    launch_map_backward(dev_grid(ctx), p, dev_cam(&ctx->fintr), ctx->rgbd, ctx->poses,
                        batch_dev, n, (const double4*)ctx->s_raycd.ptr,
                        (const uint8_t*)ctx->s_flags.ptr, ctx->d_stats, global_counts,
                        (float4*)ctx->grad, cfg->lambda_d, /*overflow_only=*/ctx->rec_K > 0,
                        (const uint32_t*)ctx->s_order.ptr, ctx->stream);
  }
  launch_touched_dilate(ctx->tc, ctx->bdim[0], ctx->bdim[1], ctx->bdim[2], ctx->tb, ctx->tdim[0],
                        ctx->tdim[1], ctx->tdim[2], ctx->stream);
  LAUNCHED(1);
  prof_end(ctx, kProfMapBackward, pb);
  LAUNCHED(1);
}

// K4 over the whole grid, or block-sparse when the fast scatter marked every
// touched block of this gradient (ctx->touched_valid).
// The update log (drop-in write-back): one slot per float4 group of the grid.
int update_log(vrf_context* ctx, UpdateLog* log) {
  *log = UpdateLog{};
  if (!ctx->log_updates) return VRF_OK;
  const size_t groups = (size_t)ctx->V * kVec4PerVertex;
  int rc;
  if ((rc = ensure(ctx, ctx->s_upd_ids, sizeof(uint32_t) * groups))) return rc;
  if ((rc = ensure(ctx, ctx->s_upd_theta, sizeof(float4) * groups))) return rc;
  if ((rc = ensure(ctx, ctx->s_upd_v, sizeof(float4) * groups))) return rc;
  if (!ctx->d_upd_count) CU(cudaMalloc(&ctx->d_upd_count, sizeof(unsigned long long)));
  CU(cudaMemsetAsync(ctx->d_upd_count, 0, sizeof(unsigned long long), ctx->stream));
  ctx->upd_sorted = false;
  log->ids = (uint32_t*)ctx->s_upd_ids.ptr;
  log->theta = (float4*)ctx->s_upd_theta.ptr;
  log->v = (float4*)ctx->s_upd_v.ptr;
  log->count = ctx->d_upd_count;
  log->cap = (long long)groups;
  return VRF_OK;
}

int launch_rmsprop_step(vrf_context* ctx, const vrf_mapping_config* cfg) {
  UpdateLog log;
  int rc = update_log(ctx, &log);
  if (rc) return rc;
  cudaEvent_t pr = prof_begin(ctx);
  static const bool force_full = std::getenv("VRF_RMSPROP_FULL") != nullptr;  // A/B, tests
  if (ctx->touched_valid && !force_full) {
    launch_rmsprop_blocks((float4*)ctx->payload, (float4*)ctx->grad, (float4*)ctx->rms, ctx->tb,
                          ctx->geom.res[0], ctx->geom.res[1], ctx->geom.res[2], ctx->tdim[0],
                          ctx->tdim[1], ctx->tdim[2], cfg->rmsprop_decay, cfg->lr_sigma,
                          cfg->lr_sh, cfg->rmsprop_eps, ctx->d_stats,
                          ctx->profiling ? ctx->d_touched : nullptr, ctx->stream, log);
  } else {
    launch_rmsprop((float4*)ctx->payload, (float4*)ctx->grad, (float4*)ctx->rms, 0, ctx->V,
                   cfg->rmsprop_decay, cfg->lr_sigma, cfg->lr_sh, cfg->rmsprop_eps, ctx->d_stats,
                   ctx->profiling ? ctx->d_touched : nullptr, ctx->stream, log);
    const long long ntb = (long long)ctx->tdim[0] * ctx->tdim[1] * ctx->tdim[2];
    cudaMemsetAsync(ctx->tb, 0, sizeof(uint32_t) * ((ntb + 31) / 32 + 1), ctx->stream);
  }
  ctx->touched_valid = false;
  prof_end(ctx, kProfRmsprop, pr);
  LAUNCHED(1);
  return VRF_OK;
}

// Fills ctx->grad (fp32) with this batch's gradient. Deterministic mode goes
// through the sorted fp64 reduce, then rounds once to fp32.
int map_gradient(vrf_context* ctx, const vrf_mapping_config* cfg, const int* batch_dev, int n,
                 MapStats* st_out, bool need_host_stats) {
  int rc = map_forward_dev(ctx, cfg, batch_dev, n, /*fast=*/true);
  if (rc) return rc;
  DevParams p;
  if ((rc = resolve_params(ctx, &cfg->render, &p))) return rc;
  if (n > 0) launch_backward_fast(ctx, cfg, p, batch_dev, n, nullptr);
  // the scatter kernels mark every touched 8^3-vertex block (K4 runs block-sparse)
  ctx->touched_valid = true;
  CU(cudaGetLastError());
  if (need_host_stats && (rc = read_stats(ctx, st_out))) return rc;
  return VRF_OK;
}

int check_ready(vrf_context* ctx) {
  int rc = need_grid(ctx);
  if (rc) return rc;
  if (ctx->n_frames == 0) return set_err(ctx, VRF_ERR_RUNTIME, "mapping_step: no keyframes");
  return VRF_OK;
}

// Deterministic forward: also records per-ray counts (s_count) for the offsets.
int det_forward(vrf_context* ctx, const vrf_mapping_config* cfg, const int* batch_dev, int n,
                MapStats* st) {
  int rc = ensure(ctx, ctx->s_count, sizeof(int) * (size_t)(n > 0 ? n : 1));
  if (rc) return rc;
  if ((rc = map_forward_dev(ctx, cfg, batch_dev, n, /*fast=*/false, (int*)ctx->s_count.ptr)))
    return rc;
  if ((rc = check_err_flag(ctx))) return rc;
  return read_stats(ctx, st);
}

int step_impl(vrf_context* ctx, const vrf_mapping_config* cfg, const int* batch_dev,
              const int32_t* batch_host, int n, vrf_map_step_stats* out) {
  cudaSetDevice(ctx->device);
  int rc;
  MapStats st;
  if (cfg->deterministic) {
    cudaEvent_t pb = prof_begin(ctx);
    if ((rc = det_forward(ctx, cfg, batch_dev, n, &st))) return rc;
    if ((rc = grad_deterministic(ctx, cfg, batch_dev, n, st))) return rc;
    launch_f64_to_f32((const double*)ctx->s_grad64.ptr, ctx->grad, ctx->V * 28, ctx->stream);
    prof_end(ctx, kProfDet, pb);
    LAUNCHED(1);
  } else {
    if ((rc = map_gradient(ctx, cfg, batch_dev, n, &st, false))) return rc;
  }
  // K4: RMSProp over the touched groups (g != 0 == the reference's touched set).
  if ((rc = launch_rmsprop_step(ctx, cfg))) return rc;
  CU(cudaGetLastError());
  if ((rc = check_err_flag(ctx))) return rc;
  if ((rc = read_stats(ctx, &st))) return rc;
  prof_collect(ctx);
  if (st.m_c == 0 || st.bad != INT_MAX) {
    // No update happened (k_rmsprop gated on the stats) — clear the gradient.
    CU(cudaMemsetAsync(ctx->grad, 0, sizeof(float) * 28 * (size_t)ctx->Vpad, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  return finish_stats(ctx, cfg, st, batch_host, out);
}

}  // namespace

extern "C" {

int vrf_mapping_step(vrf_context* ctx, const vrf_mapping_config* cfg, const int32_t* batch,
                     int n_rays, vrf_map_step_stats* out) {
  cudaSetDevice(ctx->device);
  int rc = check_ready(ctx);
  if (rc) return rc;
  const int* dev = nullptr;
  if ((rc = upload_batch(ctx, batch, n_rays, &dev))) return rc;
  return step_impl(ctx, cfg, dev, batch, n_rays, out);
}

// map_scene's inner loop (mapping.cpp:302-312): n_steps mapping_step calls whose
// batches come from the reference Rng stream (mapping.cpp:121-128). The host
// draws batch i+1 into the other half of a pinned double buffer while the device
// runs step i, so the single-threaded draw is off the critical path; each step
// still uploads its batch and reads its stats back.
int vrf_mapping_steps(vrf_context* ctx, const vrf_mapping_config* cfg, uint64_t rng_state[4],
                      int n_keyframes, int n_rays, int n_steps, vrf_map_step_stats* out) {
  cudaSetDevice(ctx->device);
  int rc = check_ready(ctx);
  if (rc) return rc;
  if (n_keyframes < 1 || n_keyframes > ctx->n_frames)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "mapping_step: keyframe index out of range");
  if (n_rays < 0 || n_steps < 0)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "mapping_step: negative batch size");
  const int W = ctx->fintr.width, H = ctx->fintr.height;
  if (cfg->deterministic || n_rays == 0) {  // sequential: the sorted reduce syncs anyway
    std::vector<int32_t> b((size_t)3 * (n_rays > 0 ? n_rays : 1));
    for (int i = 0; i < n_steps; ++i) {
      vrf_rng_draw_batch(rng_state, n_keyframes, W, H, n_rays, b.data());
      if ((rc = vrf_mapping_step(ctx, cfg, b.data(), n_rays, out ? out + i : nullptr))) return rc;
    }
    return VRF_OK;
  }
  const size_t bbytes = sizeof(int32_t) * 3 * (size_t)n_rays;
  const size_t half = (bbytes + 255) / 256 * 256;
  const size_t need = 2 * half + 2 * 256;
  if (ctx->h_pipe_bytes < need) {
    CU(cudaStreamSynchronize(ctx->stream));
    if (ctx->h_pipe) CU(cudaFreeHost(ctx->h_pipe));
    ctx->h_pipe = nullptr;
    ctx->h_pipe_bytes = 0;
    CU(cudaMallocHost(&ctx->h_pipe, need));
    ctx->h_pipe_bytes = need;
  }
  if ((rc = ensure(ctx, ctx->s_batch, bbytes))) return rc;
  if ((rc = ensure(ctx, ctx->s_batch2, bbytes))) return rc;
  char* hp = (char*)ctx->h_pipe;
  int32_t* hb[2] = {(int32_t*)hp, (int32_t*)(hp + half)};
  MapStats* h_st = (MapStats*)(hp + 2 * half);
  int* h_err = (int*)(hp + 2 * half + 256);
  const int* db[2] = {(const int*)ctx->s_batch.ptr, (const int*)ctx->s_batch2.ptr};
  DevParams p;
  if ((rc = resolve_params(ctx, &cfg->render, &p))) return rc;
  if (!ctx->copy_stream) {
    CU(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (cudaEvent_t& e : ctx->copy_ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // batch i+1 is drawn on the host and copied to the device (copy stream) while
  // the device runs step i; step i+1 waits on the copy's event
  vrf_rng_draw_batch(rng_state, n_keyframes, W, H, n_rays, hb[0]);
  CU(cudaMemcpyAsync((void*)db[0], hb[0], bbytes, cudaMemcpyHostToDevice, ctx->copy_stream));
  CU(cudaEventRecord(ctx->copy_ev[0], ctx->copy_stream));
  for (int i = 0; i < n_steps; ++i) {
    const int c = i & 1;
    CU(cudaStreamWaitEvent(ctx->stream, ctx->copy_ev[c], 0));
    if ((rc = map_gradient(ctx, cfg, db[c], n_rays, nullptr, false))) return rc;
    if ((rc = launch_rmsprop_step(ctx, cfg))) return rc;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(h_st, ctx->d_stats, sizeof(MapStats), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(h_err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    if (i + 1 < n_steps) {  // overlaps the device work of step i
      // (db[c ^ 1] was last read by step i - 1, which the previous iteration's
      // synchronize retired)
      vrf_rng_draw_batch(rng_state, n_keyframes, W, H, n_rays, hb[c ^ 1]);
      CU(cudaMemcpyAsync((void*)db[c ^ 1], hb[c ^ 1], bbytes, cudaMemcpyHostToDevice,
                         ctx->copy_stream));
      CU(cudaEventRecord(ctx->copy_ev[c ^ 1], ctx->copy_stream));
    }
    CU(cudaStreamSynchronize(ctx->stream));
    prof_collect(ctx);
    if (*h_err & 2) return set_err(ctx, VRF_ERR_OUT_OF_RANGE, "generate_ray: pixel outside image");
    if (*h_err & 1)
      return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "sh_eval: direction must be unit length");
    const MapStats st = *h_st;
    ctx->max_ray_samples = std::max(ctx->max_ray_samples, st.max_count);
    if (st.m_c == 0 || st.bad != INT_MAX) {
      CU(cudaMemsetAsync(ctx->grad, 0, sizeof(float) * 28 * (size_t)ctx->Vpad, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
    }
    if ((rc = finish_stats(ctx, cfg, st, hb[c], out ? out + i : nullptr))) return rc;
  }
  return VRF_OK;
}

int vrf_mapping_step_device(vrf_context* ctx, const vrf_mapping_config* cfg,
                            const int32_t* batch_dev, int n_rays, vrf_map_step_stats* out) {
  cudaSetDevice(ctx->device);
  int rc = check_ready(ctx);
  if (rc) return rc;
  return step_impl(ctx, cfg, batch_dev, nullptr, n_rays, out);
}

int vrf_mapping_gradient(vrf_context* ctx, const vrf_mapping_config* cfg, const int32_t* batch,
                         int n_rays, double* grad_out, vrf_map_step_stats* out) {
  cudaSetDevice(ctx->device);
  int rc = check_ready(ctx);
  if (rc) return rc;
  const int* dev = nullptr;
  if ((rc = upload_batch(ctx, batch, n_rays, &dev))) return rc;
  MapStats st;
  if (cfg->deterministic) {
    if ((rc = det_forward(ctx, cfg, dev, n_rays, &st))) return rc;
    if ((rc = grad_deterministic(ctx, cfg, dev, n_rays, st))) return rc;
  } else {
    if ((rc = map_gradient(ctx, cfg, dev, n_rays, &st, false))) return rc;
    if ((rc = ensure(ctx, ctx->s_grad64, sizeof(double) * 28 * (size_t)ctx->V))) return rc;
    launch_f32_to_f64(ctx->grad, (double*)ctx->s_grad64.ptr, ctx->V * 28, ctx->stream);
    LAUNCHED(1);
    CU(cudaMemsetAsync(ctx->grad, 0, sizeof(float) * 28 * (size_t)ctx->Vpad, ctx->stream));
  }
  if ((rc = check_err_flag(ctx))) return rc;
  if ((rc = read_stats(ctx, &st))) return rc;
  if ((rc = finish_stats(ctx, cfg, st, batch, out))) return rc;
  CU(cudaMemcpyAsync(grad_out, ctx->s_grad64.ptr, sizeof(double) * 28 * (size_t)ctx->V,
                     cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

int vrf_rmsprop_reset(vrf_context* ctx) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  CU(cudaMemsetAsync(ctx->rms, 0, sizeof(float) * 28 * (size_t)ctx->Vpad, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

int vrf_rmsprop_download(vrf_context* ctx, double* v) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  if ((rc = ensure(ctx, ctx->s_grad64, sizeof(double) * 28 * (size_t)ctx->V))) return rc;
  launch_f32_to_f64(ctx->rms, (double*)ctx->s_grad64.ptr, ctx->V * 28, ctx->stream);
  LAUNCHED(1);
  CU(cudaMemcpyAsync(v, ctx->s_grad64.ptr, sizeof(double) * 28 * (size_t)ctx->V,
                     cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

int vrf_rmsprop_upload(vrf_context* ctx, const double* v) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  const long long total = ctx->V * 28, chunk = 4LL << 20;
  if ((rc = ensure(ctx, ctx->s_out, sizeof(double) * chunk))) return rc;
  for (long long off = 0; off < total; off += chunk) {
    const long long n = std::min(chunk, total - off);
    CU(cudaMemcpyAsync(ctx->s_out.ptr, v + off, sizeof(double) * n, cudaMemcpyHostToDevice,
                       ctx->stream));
    launch_f64_to_f32((const double*)ctx->s_out.ptr, ctx->rms + off, n, ctx->stream);
    LAUNCHED(1);
  }
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

// ---- multi-GPU phases (the caller owns the collectives)
int vrf_map_forward(vrf_context* ctx, const vrf_mapping_config* cfg, const int32_t* batch_dev,
                    int n_rays, vrf_map_partials* out) {
  cudaSetDevice(ctx->device);
  int rc = check_ready(ctx);
  if (rc) return rc;
  if ((rc = map_forward_dev(ctx, cfg, batch_dev, n_rays, /*fast=*/true))) return rc;
  if ((rc = check_err_flag(ctx))) return rc;
  MapStats st;
  if ((rc = read_stats(ctx, &st))) return rc;
  ctx->last_batch = batch_dev;
  ctx->last_n = n_rays;
  out->rays_color = st.m_c;
  out->rays_depth = st.m_d;
  out->sum_photometric = st.lp;
  out->sum_geometric = st.lg;
  out->samples = st.samples;
  out->bad_ray = st.bad == INT_MAX ? -1 : st.bad;
  out->reserved = 0;
  return VRF_OK;
}

int vrf_map_backward(vrf_context* ctx, const vrf_mapping_config* cfg, int32_t rays_color,
                     int32_t rays_depth) {
  cudaSetDevice(ctx->device);
  int rc = check_ready(ctx);
  if (rc) return rc;
  if (!ctx->last_batch) return set_err(ctx, VRF_ERR_RUNTIME, "vrf_map_backward: no forward pass");
  DevParams p;
  if ((rc = resolve_params(ctx, &cfg->render, &p))) return rc;
  const int counts[2] = {rays_color, rays_depth};
  CU(cudaMemcpyAsync(ctx->d_counts, counts, sizeof(counts), cudaMemcpyHostToDevice, ctx->stream));
  if (ctx->last_n > 0)
    launch_backward_fast(ctx, cfg, p, ctx->last_batch, ctx->last_n, ctx->d_counts);
  CU(cudaGetLastError());
  // the reduce-scatter brings other ranks' gradients: vrf_map_apply scans its shard
  ctx->touched_valid = false;
  return VRF_OK;
}

// ---- block-sparse exchange (distributed.py): 8^3-vertex blocks, packed
// [n][512][28] fp32 device buffers owned by the caller (the NCCL tensors).
int vrf_blocks_count(vrf_context* ctx, int32_t* n_blocks) {
  int rc = need_grid(ctx);
  if (rc) return rc;
  *n_blocks = ctx->tdim[0] * ctx->tdim[1] * ctx->tdim[2];
  return VRF_OK;
}

int vrf_blocks_touched(vrf_context* ctx, uint8_t* flags_dev) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  launch_touched_flags(ctx->tb, ctx->tdim[0] * ctx->tdim[1] * ctx->tdim[2], flags_dev,
                       ctx->stream);
  LAUNCHED(1);
  CU(cudaGetLastError());
  return VRF_OK;
}

int vrf_blocks_pack(vrf_context* ctx, const int32_t* ids_dev, int n, int which, float* out_dev) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  if (which != 0 && which != 1)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "vrf_blocks_pack: which must be 0 or 1");
  launch_blocks_pack((const float4*)(which == 0 ? ctx->grad : ctx->payload), ids_dev, n,
                     ctx->geom.res[0], ctx->geom.res[1], ctx->geom.res[2], ctx->tdim[0],
                     ctx->tdim[1], (float4*)out_dev, ctx->stream);
  LAUNCHED(1);
  CU(cudaGetLastError());
  return VRF_OK;
}

int vrf_blocks_unpack_payload(vrf_context* ctx, const int32_t* ids_dev, int n,
                              const float* in_dev) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  launch_blocks_unpack((float4*)ctx->payload, ids_dev, n, ctx->geom.res[0], ctx->geom.res[1],
                       ctx->geom.res[2], ctx->tdim[0], ctx->tdim[1], (const float4*)in_dev,
                       ctx->stream);
  LAUNCHED(1);
  CU(cudaGetLastError());
  return VRF_OK;
}

int vrf_blocks_apply(vrf_context* ctx, const vrf_mapping_config* cfg, const int32_t* ids_dev,
                     int n, const float* grad_packed_dev) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  launch_blocks_apply((float4*)ctx->payload, (float4*)ctx->rms, ids_dev, n, ctx->geom.res[0],
                      ctx->geom.res[1], ctx->geom.res[2], ctx->tdim[0], ctx->tdim[1],
                      (const float4*)grad_packed_dev, cfg->rmsprop_decay, cfg->lr_sigma,
                      cfg->lr_sh, cfg->rmsprop_eps, ctx->stream);
  LAUNCHED(1);
  CU(cudaGetLastError());
  return VRF_OK;
}

int vrf_grad_clear(vrf_context* ctx) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  CU(cudaMemsetAsync(ctx->grad, 0, sizeof(float) * 28 * (size_t)ctx->Vpad, ctx->stream));
  const long long ntb = (long long)ctx->tdim[0] * ctx->tdim[1] * ctx->tdim[2];
  CU(cudaMemsetAsync(ctx->tb, 0, sizeof(uint32_t) * ((ntb + 31) / 32 + 1), ctx->stream));
  ctx->touched_valid = false;
  return VRF_OK;
}

int vrf_map_apply(vrf_context* ctx, const vrf_mapping_config* cfg, int64_t vertex_begin,
                  int64_t vertex_end) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  if (vertex_begin < 0 || vertex_end > ctx->Vpad || vertex_begin > vertex_end)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "vrf_map_apply: bad vertex range");
  const int64_t end = std::min<int64_t>(vertex_end, ctx->V);
  launch_rmsprop((float4*)ctx->payload, (float4*)ctx->grad, (float4*)ctx->rms, vertex_begin,
                 end, cfg->rmsprop_decay, cfg->lr_sigma, cfg->lr_sh, cfg->rmsprop_eps, nullptr,
                 ctx->profiling ? ctx->d_touched : nullptr, ctx->stream);
  LAUNCHED(1);
  CU(cudaGetLastError());
  return VRF_OK;
}

// ---- drop-in residency: partial uploads and the update log (integration/)
void* vrf_host_alloc(size_t bytes) {
  void* p = nullptr;
  return cudaMallocHost(&p, bytes) == cudaSuccess ? p : nullptr;
}

void vrf_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int vrf_track_updates(vrf_context* ctx, int on) {
  ctx->log_updates = on != 0;
  return VRF_OK;
}

int vrf_updates_count(vrf_context* ctx, int64_t* n) {
  cudaSetDevice(ctx->device);
  unsigned long long c = 0;
  if (ctx->log_updates && ctx->d_upd_count) {
    CU(cudaMemcpyAsync(&c, ctx->d_upd_count, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  *n = (int64_t)c;
  return VRF_OK;
}

int vrf_updates_read(vrf_context* ctx, int64_t n, uint32_t* ids, float* theta, float* v) {
  cudaSetDevice(ctx->device);
  if (!ctx->log_updates || n <= 0) return VRF_OK;
  if (n > (int64_t)(ctx->V * kVec4PerVertex))
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "vrf_updates_read: count exceeds the grid");
  CU(cudaMemcpyAsync(ids, ctx->s_upd_ids.ptr, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaMemcpyAsync(theta, ctx->s_upd_theta.ptr, sizeof(float4) * n, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaMemcpyAsync(v, ctx->s_upd_v.ptr, sizeof(float4) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

int vrf_updates_read_range(vrf_context* ctx, int64_t first, int64_t count, int sorted,
                           uint32_t* ids, float* theta, float* v) {
  cudaSetDevice(ctx->device);
  if (!ctx->log_updates || count <= 0) return VRF_OK;
  int64_t n = 0;
  int rc = vrf_updates_count(ctx, &n);
  if (rc) return rc;
  if (first < 0 || first + count > n)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "vrf_updates_read_range: range exceeds the log");
  if (!sorted) {
    CU(cudaMemcpyAsync(ids, (const uint32_t*)ctx->s_upd_ids.ptr + first, sizeof(uint32_t) * count,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(theta, (const float4*)ctx->s_upd_theta.ptr + first, sizeof(float4) * count,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(v, (const float4*)ctx->s_upd_v.ptr + first, sizeof(float4) * count,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return VRF_OK;
  }
  if (!ctx->upd_sorted) {  // once per logged step: sort the whole log by id
    const size_t tb = update_sort_tmp_bytes(n);
    if ((rc = ensure(ctx, ctx->s_upd_sids, sizeof(uint32_t) * n))) return rc;
    if ((rc = ensure(ctx, ctx->s_upd_perm, sizeof(uint32_t) * n))) return rc;
    if ((rc = ensure(ctx, ctx->s_upd_iota, sizeof(uint32_t) * n))) return rc;
    if ((rc = ensure(ctx, ctx->s_upd_tmp, tb))) return rc;
    launch_update_sort((const uint32_t*)ctx->s_upd_ids.ptr, n, (uint32_t*)ctx->s_upd_sids.ptr,
                       (uint32_t*)ctx->s_upd_iota.ptr, (uint32_t*)ctx->s_upd_perm.ptr,
                       ctx->s_upd_tmp.ptr, tb, ctx->stream);
    CU(cudaGetLastError());
    ctx->upd_sorted = true;
  }
  if ((rc = ensure(ctx, ctx->s_upd_gth, sizeof(float4) * count))) return rc;
  if ((rc = ensure(ctx, ctx->s_upd_gv, sizeof(float4) * count))) return rc;
  launch_update_gather((const uint32_t*)ctx->s_upd_perm.ptr, first, count,
                       (const float4*)ctx->s_upd_theta.ptr, (const float4*)ctx->s_upd_v.ptr,
                       (float4*)ctx->s_upd_gth.ptr, (float4*)ctx->s_upd_gv.ptr, ctx->stream);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(ids, (const uint32_t*)ctx->s_upd_sids.ptr + first, sizeof(uint32_t) * count,
                     cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(theta, ctx->s_upd_gth.ptr, sizeof(float4) * count, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaMemcpyAsync(v, ctx->s_upd_gv.ptr, sizeof(float4) * count, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

int vrf_state_read_f32(vrf_context* ctx, int which, int64_t first, int64_t count, float* dst) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  const float* src = which == 0 ? ctx->payload : which == 1 ? ctx->rms : nullptr;
  if (!src) return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "vrf_state_read_f32: which");
  if (first < 0 || count < 0 || first + count > (int64_t)ctx->V * 28)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "vrf_state_read_f32: range");
  CU(cudaMemcpyAsync(dst, src + first, sizeof(float) * count, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

namespace {
int write_vertices(vrf_context* ctx, float* dst, int64_t first, int64_t count, const double* src,
                   const char* what) {
  int rc = need_grid(ctx);
  if (rc) return rc;
  if (first < 0 || count < 0 || first + count > ctx->V)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, std::string(what) + ": vertex range");
  const long long total = count * 28, chunk = 4LL << 20;
  if ((rc = ensure(ctx, ctx->s_out, sizeof(double) * chunk))) return rc;
  for (long long off = 0; off < total; off += chunk) {
    const long long n = std::min(chunk, total - off);
    CU(cudaMemcpyAsync(ctx->s_out.ptr, src + off, sizeof(double) * n, cudaMemcpyHostToDevice,
                       ctx->stream));
    launch_f64_to_f32((const double*)ctx->s_out.ptr, dst + first * 28 + off, n, ctx->stream);
    LAUNCHED(1);
  }
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}
}  // namespace

int vrf_grid_write_vertices(vrf_context* ctx, int64_t first, int64_t count, const double* data) {
  cudaSetDevice(ctx->device);
  return write_vertices(ctx, ctx->payload, first, count, data, "vrf_grid_write_vertices");
}

int vrf_rmsprop_write_vertices(vrf_context* ctx, int64_t first, int64_t count, const double* v) {
  cudaSetDevice(ctx->device);
  return write_vertices(ctx, ctx->rms, first, count, v, "vrf_rmsprop_write_vertices");
}

}  // extern "C"

// ---- fused peer-memory exchange (distributed.py exchange="p2p")
int vrf_peer_buffers_get(vrf_context* ctx, vrf_peer_buffers* out) {
  int rc = need_grid(ctx);
  if (rc) return rc;
  out->grad = (uint64_t)(uintptr_t)ctx->grad;
  out->payload = (uint64_t)(uintptr_t)ctx->payload;
  out->tb = (uint64_t)(uintptr_t)ctx->tb;
  return VRF_OK;
}

namespace {
// Validates and installs the peer table (does not touch IPC mappings).
int set_peer_table(vrf_context* ctx, int world, int rank, const vrf_peer_buffers* peers) {
  if (world < 1 || world > VRF_MAX_PEERS || rank < 0 || rank >= world || !peers)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "vrf_peers_set: bad world/rank/peers");
  if (peers[rank].grad != (uint64_t)(uintptr_t)ctx->grad ||
      peers[rank].payload != (uint64_t)(uintptr_t)ctx->payload ||
      peers[rank].tb != (uint64_t)(uintptr_t)ctx->tb)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT,
                   "vrf_peers_set: entry [rank] must be this context's own buffers");
  PeerTable pt{};
  for (int r = 0; r < world; ++r) {
    pt.grad[r] = reinterpret_cast<float4*>((uintptr_t)peers[r].grad);
    pt.payload[r] = reinterpret_cast<float4*>((uintptr_t)peers[r].payload);
    pt.tb[r] = reinterpret_cast<const uint32_t*>((uintptr_t)peers[r].tb);
    if (!pt.grad[r] || !pt.payload[r] || !pt.tb[r])
      return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "vrf_peers_set: null peer buffer");
  }
  pt.world = world;
  pt.rank = rank;
  ctx->peers = pt;
  ctx->peers_set = true;
  return VRF_OK;
}
}  // namespace

int vrf_peers_set(vrf_context* ctx, int world, int rank, const vrf_peer_buffers* peers) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  close_peers(ctx);
  return set_peer_table(ctx, world, rank, peers);
}

int vrf_ipc_export(vrf_context* ctx, uint8_t* handles) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  void* bufs[3] = {ctx->grad, ctx->payload, ctx->tb};
  for (int k = 0; k < 3; ++k) {
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, bufs[k]));
    std::memcpy(handles + k * sizeof(cudaIpcMemHandle_t), &h, sizeof(h));
  }
  return VRF_OK;
}

int vrf_peers_open_ipc(vrf_context* ctx, int world, int rank, const uint8_t* handles) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  static_assert(3 * sizeof(cudaIpcMemHandle_t) == VRF_IPC_HANDLE_BYTES, "IPC handle size");
  if (world < 1 || world > VRF_MAX_PEERS || rank < 0 || rank >= world || !handles)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "vrf_peers_open_ipc: bad world/rank/handles");
  close_peers(ctx);
  vrf_peer_buffers peers[VRF_MAX_PEERS];
  for (int r = 0; r < world; ++r) {
    if (r == rank) {
      vrf_peer_buffers_get(ctx, &peers[r]);
      continue;
    }
    uint64_t* dst[3] = {&peers[r].grad, &peers[r].payload, &peers[r].tb};
    for (int k = 0; k < 3; ++k) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + (size_t)r * VRF_IPC_HANDLE_BYTES + k * sizeof(h), sizeof(h));
      void* p = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        close_peers(ctx);
        return set_err(ctx, VRF_ERR_CUDA,
                       std::string("vrf_peers_open_ipc: cudaIpcOpenMemHandle: ") +
                           cudaGetErrorString(e));
      }
      ctx->ipc_open[r][k] = p;
      *dst[k] = (uint64_t)(uintptr_t)p;
    }
  }
  rc = set_peer_table(ctx, world, rank, peers);
  if (rc) close_peers(ctx);
  return rc;
}

int vrf_exchange_p2p(vrf_context* ctx, const vrf_mapping_config* cfg) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  if (!ctx->peers_set)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT,
                   "vrf_exchange_p2p: no peer table (vrf_peers_set / vrf_peers_open_ipc)");
  const int nb = ctx->tdim[0] * ctx->tdim[1] * ctx->tdim[2];
  cudaEvent_t pr = prof_begin(ctx);
  launch_exchange_p2p(ctx->peers, (float4*)ctx->rms, nb, ctx->geom.res[0], ctx->geom.res[1],
                      ctx->geom.res[2], ctx->tdim[0], ctx->tdim[1], cfg->rmsprop_decay,
                      cfg->lr_sigma, cfg->lr_sh, cfg->rmsprop_eps, nullptr, ctx->stream);
  prof_end(ctx, kProfRmsprop, pr);
  LAUNCHED(1);
  CU(cudaGetLastError());
  return VRF_OK;
}
