// C-ABI of libvoxrf_b200 (include/voxrf_b200.h): device context, memory,
// orchestration of the kernels and the reference's error contract.
#include "vrf_context.h"

using namespace vrf;
using namespace vrf_host;

// =================================================================== C-ABI
extern "C" {

int vrf_abi_version(void) { return VRF_ABI_VERSION; }

int vrf_context_create(int device, vrf_context** out) {
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) return VRF_ERR_CUDA;
  if (device < 0 || device >= count) return VRF_ERR_INVALID_ARGUMENT;
  if (cudaSetDevice(device) != cudaSuccess) return VRF_ERR_CUDA;
  auto* ctx = new vrf_context;
  ctx->device = device;
  if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&ctx->d_err, sizeof(int)) != cudaSuccess ||
      cudaMalloc(&ctx->d_stats, sizeof(MapStats)) != cudaSuccess ||
      cudaMalloc(&ctx->d_counts, sizeof(int) * 2) != cudaSuccess ||
      cudaMalloc(&ctx->d_pose_out, sizeof(PosePartial)) != cudaSuccess ||
      cudaMalloc(&ctx->d_pose, sizeof(DevPose)) != cudaSuccess) {
    delete ctx;
    return VRF_ERR_CUDA;
  }
  ctx->stream = ctx->own_stream;
  *out = ctx;
  return VRF_OK;
}

void vrf_context_destroy(vrf_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  free_grid(ctx);
  cudaFree(ctx->rgbd);
  cudaFree(ctx->poses);
  cudaFree(ctx->d_err);
  cudaFree(ctx->d_stats);
  cudaFree(ctx->d_counts);
  cudaFree(ctx->d_pose_out);
  cudaFree(ctx->d_pose);
  cudaFree(ctx->d_touched);
  cudaFree(ctx->d_upd_count);
  cudaFree(ctx->d_digest);
  cudaFree(ctx->payload_soa);
  cudaFree(ctx->d_nblocks);
  cudaFree(ctx->d_frame);
  cudaFree(ctx->d_gn_pose);
  cudaFree(ctx->d_gn_seed);
  cudaFree(ctx->d_gn_hist);
  if (ctx->gn_graph) cudaGraphExecDestroy(ctx->gn_graph);
  prof_collect(ctx);
  for (DeviceScratch* s : {&ctx->s_order, &ctx->s_okeys, &ctx->s_okeys2, &ctx->s_oids,
                           &ctx->s_otmp, &ctx->s_batch, &ctx->s_raycd, &ctx->s_flags, &ctx->s_partials,
                           &ctx->s_count, &ctx->s_offsets, &ctx->s_keys, &ctx->s_keys2,
                           &ctx->s_ids, &ctx->s_ids2, &ctx->s_values, &ctx->s_grad64, &ctx->s_cub,
                           &ctx->s_stage, &ctx->s_out, &ctx->s_batch2, &ctx->s_rec,
                           &ctx->s_upd_ids, &ctx->s_upd_theta, &ctx->s_upd_v,
                           &ctx->s_upd_sids, &ctx->s_upd_perm, &ctx->s_upd_iota,
                           &ctx->s_upd_tmp, &ctx->s_upd_gth, &ctx->s_upd_gv,
                           &ctx->s_reccount})
    cudaFree(s->ptr);
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  if (ctx->h_pipe) cudaFreeHost(ctx->h_pipe);
  for (cudaEvent_t e : ctx->copy_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

const char* vrf_last_error(const vrf_context* ctx) { return ctx ? ctx->err.c_str() : ""; }

int vrf_set_shard_multiple(vrf_context* ctx, int world_size) {
  if (world_size < 1) return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "world_size must be >= 1");
  ctx->shard_multiple = world_size;
  return VRF_OK;
}

int vrf_set_record_limits(vrf_context* ctx, double budget_gb, int max_k) {
  if (max_k > 0 && max_k < 4)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "vrf_set_record_limits: max_k must be 0 or >= 4");
  ctx->rec_budget_gb = budget_gb;
  ctx->rec_max_k = max_k;
  ctx->rec_need_tried = 0;
  return VRF_OK;
}

int vrf_set_stream(vrf_context* ctx, void* stream) {
  ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
  return VRF_OK;
}

int vrf_get_device_buffers(vrf_context* ctx, vrf_device_buffers* out) {
  int rc = need_grid(ctx);
  if (rc) return rc;
  out->payload = ctx->payload;
  out->grad = ctx->grad;
  out->rms_v = ctx->rms;
  out->num_vertices = ctx->V;
  out->padded_vertices = ctx->Vpad;
  out->stream = ctx->stream;
  return VRF_OK;
}

int64_t vrf_kernel_launch_count(const vrf_context* ctx) { return ctx->launches; }

int vrf_profile_enable(vrf_context* ctx, int on) {
  cudaSetDevice(ctx->device);
  CU(cudaStreamSynchronize(ctx->stream));
  prof_collect(ctx);
  for (int i = 0; i < 8; ++i) {
    ctx->prof_ms[i] = 0.0;
    ctx->prof_launches[i] = 0;
  }
  if (!ctx->d_touched) CU(cudaMalloc(&ctx->d_touched, sizeof(unsigned long long)));
  CU(cudaMemsetAsync(ctx->d_touched, 0, sizeof(unsigned long long), ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->profiling = on != 0;
  ctx->prof_track_samples = 0;
  return VRF_OK;
}

int64_t vrf_profile_track_samples(vrf_context* ctx) { return ctx->prof_track_samples; }

int vrf_profile_read(vrf_context* ctx, int slot, double* ms, int64_t* launches) {
  if (slot < 0 || slot >= 8) return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "profile slot");
  cudaSetDevice(ctx->device);
  CU(cudaStreamSynchronize(ctx->stream));
  prof_collect(ctx);
  *ms = ctx->prof_ms[slot];
  *launches = ctx->prof_launches[slot];
  return VRF_OK;
}

int64_t vrf_profile_touched_groups(vrf_context* ctx) {
  unsigned long long n = 0;
  if (!ctx->d_touched) return 0;
  cudaSetDevice(ctx->device);
  if (cudaMemcpy(&n, ctx->d_touched, sizeof(n), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return (int64_t)n;
}

// ----------------------------------------------------------------- grid
int vrf_grid_init(vrf_context* ctx, const vrf_grid_geometry* geom, double sigma_init) {
  cudaSetDevice(ctx->device);
  int rc = alloc_grid(ctx, geom);
  if (rc) return rc;
  launch_fill_payload(ctx->payload, ctx->V, (float)sigma_init, ctx->stream);
  LAUNCHED(1);
  CU(cudaMemsetAsync(ctx->occ, 0xFF, sizeof(uint32_t) * ((ctx->C + 31) / 32 + 1), ctx->stream));
  update_blocks(ctx);
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

// VoxelGrid(geom, sigma_init) payload (voxel_grid.cpp:74-81) over the current
// geometry, keeping the occupancy (e.g. a pruned shell); gradient and RMSProp
// state restart at zero.
int vrf_grid_fill(vrf_context* ctx, double sigma_init) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  launch_fill_payload(ctx->payload, ctx->V, (float)sigma_init, ctx->stream);
  LAUNCHED(1);
  CU(cudaMemsetAsync(ctx->grad, 0, sizeof(float) * 28 * ctx->Vpad, ctx->stream));
  CU(cudaMemsetAsync(ctx->rms, 0, sizeof(float) * 28 * ctx->Vpad, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

static int upload_occupancy_u8(vrf_context* ctx, const uint8_t* occupancy) {
  if (!occupancy) {
    CU(cudaMemsetAsync(ctx->occ, 0xFF, sizeof(uint32_t) * ((ctx->C + 31) / 32 + 1), ctx->stream));
    return VRF_OK;
  }
  int rc = ensure(ctx, ctx->s_stage, (size_t)ctx->C);
  if (rc) return rc;
  CU(cudaMemcpyAsync(ctx->s_stage.ptr, occupancy, (size_t)ctx->C, cudaMemcpyHostToDevice,
                     ctx->stream));
  launch_pack_occupancy((const uint8_t*)ctx->s_stage.ptr, ctx->occ, ctx->C, ctx->stream);
  LAUNCHED(1);
  return VRF_OK;
}

int vrf_grid_upload(vrf_context* ctx, const vrf_grid_geometry* geom, const double* payload,
                    const uint8_t* occupancy) {
  cudaSetDevice(ctx->device);
  int rc = alloc_grid(ctx, geom);
  if (rc) return rc;
  // fp64 -> fp32 in 32 MB chunks through a device staging buffer.
  const long long total = ctx->V * 28;
  const long long chunk = 4LL << 20;
  if ((rc = ensure(ctx, ctx->s_out, sizeof(double) * chunk))) return rc;
  for (long long off = 0; off < total; off += chunk) {
    const long long n = std::min(chunk, total - off);
    CU(cudaMemcpyAsync(ctx->s_out.ptr, payload + off, sizeof(double) * n, cudaMemcpyHostToDevice,
                       ctx->stream));
    launch_f64_to_f32((const double*)ctx->s_out.ptr, ctx->payload + off, n, ctx->stream);
    LAUNCHED(1);
  }
  if ((rc = upload_occupancy_u8(ctx, occupancy))) return rc;
  update_blocks(ctx);
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

// A cheap device-side grid-integrity check (tracking never mutates
// the grid; voxel_grid.cpp:280-292's FNV-1a checksum is sequential over the fp64
// bytes and stays host-side). Covers the geometry, the fp32 payload and the
// occupancy bits.
int vrf_grid_digest(vrf_context* ctx, uint64_t* out) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  if (!ctx->d_digest) CU(cudaMalloc(&ctx->d_digest, sizeof(unsigned long long)));
  CU(cudaMemsetAsync(ctx->d_digest, 0, sizeof(unsigned long long), ctx->stream));
  launch_digest((const uint32_t*)ctx->payload, ctx->V * 28, 0x5041594c4f4144ULL, ctx->d_digest,
                ctx->stream);
  launch_digest(ctx->occ, (ctx->C + 31) / 32, 0x4f43435550ULL, ctx->d_digest, ctx->stream);
  LAUNCHED(2);
  unsigned long long h = 0;
  CU(cudaMemcpyAsync(&h, ctx->d_digest, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  // fold in the geometry
  const vrf_grid_geometry& gm = ctx->geom;
  uint64_t x = h;
  const unsigned char* p = reinterpret_cast<const unsigned char*>(&gm);
  for (size_t k = 0; k < sizeof(gm); ++k) x = (x ^ p[k]) * 0x100000001b3ULL;
  *out = x;
  return VRF_OK;
}

int vrf_grid_set_occupancy(vrf_context* ctx, const uint8_t* occupancy) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  if ((rc = upload_occupancy_u8(ctx, occupancy))) return rc;
  update_blocks(ctx);
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

int vrf_grid_upload_f32(vrf_context* ctx, const vrf_grid_geometry* geom, const float* payload,
                        const uint8_t* occupancy_bits) {
  cudaSetDevice(ctx->device);
  int rc = alloc_grid(ctx, geom);
  if (rc) return rc;
  CU(cudaMemcpyAsync(ctx->payload, payload, sizeof(float) * 28 * ctx->V, cudaMemcpyHostToDevice,
                     ctx->stream));
  if (occupancy_bits) {
    // LSB-first byte mask (voxel_grid.cpp:234-236) == little-endian uint32 words.
    CU(cudaMemsetAsync(ctx->occ, 0, sizeof(uint32_t) * ((ctx->C + 31) / 32 + 1), ctx->stream));
    CU(cudaMemcpyAsync(ctx->occ, occupancy_bits, (size_t)((ctx->C + 7) / 8),
                       cudaMemcpyHostToDevice, ctx->stream));
  } else {
    CU(cudaMemsetAsync(ctx->occ, 0xFF, sizeof(uint32_t) * ((ctx->C + 31) / 32 + 1), ctx->stream));
  }
  update_blocks(ctx);
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

int vrf_grid_download(vrf_context* ctx, double* payload, uint8_t* occupancy) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  if (payload) {
    const long long total = ctx->V * 28;
    const long long chunk = 4LL << 20;
    if ((rc = ensure(ctx, ctx->s_out, sizeof(double) * chunk))) return rc;
    for (long long off = 0; off < total; off += chunk) {
      const long long n = std::min(chunk, total - off);
      launch_f32_to_f64(ctx->payload + off, (double*)ctx->s_out.ptr, n, ctx->stream);
      LAUNCHED(1);
      CU(cudaMemcpyAsync(payload + off, ctx->s_out.ptr, sizeof(double) * n,
                         cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
    }
  }
  if (occupancy) {
    if ((rc = ensure(ctx, ctx->s_stage, (size_t)ctx->C))) return rc;
    launch_unpack_occupancy(ctx->occ, (uint8_t*)ctx->s_stage.ptr, ctx->C, ctx->stream);
    LAUNCHED(1);
    CU(cudaMemcpyAsync(occupancy, ctx->s_stage.ptr, (size_t)ctx->C, cudaMemcpyDeviceToHost,
                       ctx->stream));
  }
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

int vrf_grid_download_f32(vrf_context* ctx, float* payload) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  CU(cudaMemcpyAsync(payload, ctx->payload, sizeof(float) * 28 * ctx->V, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

int vrf_grid_get_geometry(const vrf_context* ctx, vrf_grid_geometry* out) {
  if (!ctx->has_grid) return VRF_ERR_RUNTIME;
  *out = ctx->geom;
  return VRF_OK;
}

int vrf_grid_prune(vrf_context* ctx, double tau, int64_t* deactivated) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  if ((rc = ensure(ctx, ctx->s_out, sizeof(unsigned long long)))) return rc;
  CU(cudaMemsetAsync(ctx->s_out.ptr, 0, sizeof(unsigned long long), ctx->stream));
  launch_prune(dev_grid(ctx), ctx->occ, tau, (unsigned long long*)ctx->s_out.ptr, ctx->stream);
  LAUNCHED(1);
  update_blocks(ctx);
  unsigned long long n = 0;
  CU(cudaMemcpyAsync(&n, ctx->s_out.ptr, sizeof(n), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (deactivated) *deactivated = (int64_t)n;
  return VRF_OK;
}

// VoxelGrid::upsampled(max_resolution) — voxel_grid.cpp:190-220, in place on the
// device; gradient and RMSProp state restart at zero (map_scene resets RMSProp
// on every stage, mapping.cpp:297-300).
int vrf_grid_upsample(vrf_context* ctx, int max_resolution) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  vrf_grid_geometry ng = ctx->geom;
  for (int a = 0; a < 3; ++a) ng.res[a] = 2 * ctx->geom.res[a] - 1;
  ng.voxel_size = ctx->geom.voxel_size * 0.5;
  if (std::max(ng.res[0], std::max(ng.res[1], ng.res[2])) > max_resolution)
    return set_err(ctx, VRF_ERR_RUNTIME, "upsample: resolution would exceed configured maximum");
  const DevGrid coarse = dev_grid(ctx);
  float* old_payload = ctx->payload;
  uint32_t* old_occ = ctx->occ;
  ctx->payload = nullptr;  // keep the coarse payload/occupancy alive through alloc_grid
  ctx->occ = nullptr;
  if ((rc = alloc_grid(ctx, &ng))) {
    cudaFree(old_payload);
    cudaFree(old_occ);
    return rc;
  }
  launch_upsample(coarse, ng.res[0], ng.res[1], ng.res[2], ctx->payload, ctx->occ, ctx->stream);
  LAUNCHED(2);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(ctx->stream));
  cudaFree(old_payload);
  cudaFree(old_occ);
  return update_blocks(ctx);
}

// .vxgf I/O — VoxelGrid::save / load (voxel_grid.cpp:222-278). The device payload
// is already the file's fp32 [V][28] AoS and the occupancy words are the file's
// LSB-first bitmask, so both directions stream straight through pinned staging.
namespace {
constexpr char kVxgfMagic[4] = {'V', 'X', 'G', 'F'};
constexpr uint32_t kVxgfVersion = 1;
constexpr size_t kVxgfHeader = 4 + 4 + 3 * 4 + 3 * 8 + 8;
constexpr size_t kIoChunk = 64u << 20;

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};
}  // namespace

int vrf_grid_save(vrf_context* ctx, const char* path) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  const std::string p = path ? path : "";
  File out;
  out.f = fopen(p.c_str(), "wb");
  if (!out.f) return set_err(ctx, VRF_ERR_RUNTIME, "grid save: cannot open " + p);
  bool ok = fwrite(kVxgfMagic, 1, 4, out.f) == 4 &&
            fwrite(&kVxgfVersion, sizeof(uint32_t), 1, out.f) == 1;
  for (int a = 0; a < 3 && ok; ++a) {
    const uint32_t r = (uint32_t)ctx->geom.res[a];
    ok = fwrite(&r, sizeof(r), 1, out.f) == 1;
  }
  ok = ok && fwrite(ctx->geom.origin, sizeof(double), 3, out.f) == 3 &&
       fwrite(&ctx->geom.voxel_size, sizeof(double), 1, out.f) == 1;
  if ((rc = ensure_pinned(ctx, kIoChunk))) return rc;
  char* stage = (char*)ctx->h_pinned;
  const size_t payload_bytes = sizeof(float) * 28 * (size_t)ctx->V;
  for (size_t off = 0; off < payload_bytes && ok; off += kIoChunk) {
    const size_t n = std::min(kIoChunk, payload_bytes - off);
    CU(cudaMemcpyAsync(stage, (const char*)ctx->payload + off, n, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    ok = fwrite(stage, 1, n, out.f) == n;
  }
  const size_t bit_bytes = (size_t)((ctx->C + 7) / 8);
  for (size_t off = 0; off < bit_bytes && ok; off += kIoChunk) {
    const size_t n = std::min(kIoChunk, bit_bytes - off);
    CU(cudaMemcpyAsync(stage, (const char*)ctx->occ + off, n, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    ok = fwrite(stage, 1, n, out.f) == n;
  }
  ok = ok && fflush(out.f) == 0;
  if (!ok) return set_err(ctx, VRF_ERR_RUNTIME, "grid save: write failed for " + p);
  return VRF_OK;
}

int vrf_grid_load(vrf_context* ctx, const char* path) {
  cudaSetDevice(ctx->device);
  const std::string p = path ? path : "";
  File in;
  in.f = fopen(p.c_str(), "rb");
  if (!in.f) return set_err(ctx, VRF_ERR_RUNTIME, "grid load: cannot open " + p);
  char magic[4];
  if (fread(magic, 1, 4, in.f) != 4 || std::memcmp(magic, kVxgfMagic, 4) != 0)
    return set_err(ctx, VRF_ERR_RUNTIME, "grid load: bad magic in " + p);
  uint32_t version = 0;
  if (fread(&version, sizeof(version), 1, in.f) != 1 || version != kVxgfVersion)
    return set_err(ctx, VRF_ERR_RUNTIME, "grid load: unsupported version in " + p);
  vrf_grid_geometry g{};
  bool ok = true;
  for (int a = 0; a < 3 && ok; ++a) {
    uint32_t r = 0;
    ok = fread(&r, sizeof(r), 1, in.f) == 1;
    g.res[a] = (int32_t)r;
  }
  ok = ok && fread(g.origin, sizeof(double), 3, in.f) == 3 &&
       fread(&g.voxel_size, sizeof(double), 1, in.f) == 1;
  if (!ok) return set_err(ctx, VRF_ERR_RUNTIME, "grid load: truncated header in " + p);
  int rc = validate_geometry(ctx, &g);
  if (rc) return rc;
  const size_t V = (size_t)g.res[0] * g.res[1] * g.res[2];
  const size_t C = (size_t)(g.res[0] - 1) * (g.res[1] - 1) * (g.res[2] - 1);
  const size_t payload_bytes = sizeof(float) * 28 * V, bit_bytes = (C + 7) / 8;
  // The reference reads payload + bits before checking either (voxel_grid.cpp:262-267):
  // truncation is reported ahead of non-finite values.
  if (fseeko(in.f, 0, SEEK_END) != 0 ||
      (size_t)ftello(in.f) < kVxgfHeader + payload_bytes + bit_bytes ||
      fseeko(in.f, (off_t)kVxgfHeader, SEEK_SET) != 0)
    return set_err(ctx, VRF_ERR_RUNTIME, "grid load: truncated payload in " + p);
  if ((rc = ensure_pinned(ctx, kIoChunk))) return rc;
  if ((rc = alloc_grid(ctx, &g))) return rc;
  char* stage = (char*)ctx->h_pinned;
  for (size_t off = 0; off < payload_bytes; off += kIoChunk) {
    const size_t n = std::min(kIoChunk, payload_bytes - off);
    CU(cudaStreamSynchronize(ctx->stream));  // the previous chunk has left the stage
    if (fread(stage, 1, n, in.f) != n) {
      free_grid(ctx);
      return set_err(ctx, VRF_ERR_RUNTIME, "grid load: truncated payload in " + p);
    }
    const float* f = (const float*)stage;
    for (size_t i = 0; i < n / sizeof(float); ++i)
      if (!std::isfinite(f[i])) {
        free_grid(ctx);
        return set_err(ctx, VRF_ERR_RUNTIME, "grid load: non-finite payload in " + p);
      }
    CU(cudaMemcpyAsync((char*)ctx->payload + off, stage, n, cudaMemcpyHostToDevice, ctx->stream));
  }
  CU(cudaStreamSynchronize(ctx->stream));
  CU(cudaMemsetAsync(ctx->occ, 0, sizeof(uint32_t) * ((ctx->C + 31) / 32 + 1), ctx->stream));
  for (size_t off = 0; off < bit_bytes; off += kIoChunk) {
    const size_t n = std::min(kIoChunk, bit_bytes - off);
    CU(cudaStreamSynchronize(ctx->stream));
    if (fread(stage, 1, n, in.f) != n) {
      free_grid(ctx);
      return set_err(ctx, VRF_ERR_RUNTIME, "grid load: truncated payload in " + p);
    }
    CU(cudaMemcpyAsync((char*)ctx->occ + off, stage, n, cudaMemcpyHostToDevice, ctx->stream));
  }
  // bits past the last cell are never read (cell_active / block occupancy stop at C)
  CU(cudaStreamSynchronize(ctx->stream));
  return update_blocks(ctx);
}

// ----------------------------------------------------------------- frames
int vrf_frames_upload(vrf_context* ctx, const vrf_intrinsics* intr, int n,
                      const double* const* colors, const double* const* depths,
                      const vrf_pose* poses) {
  cudaSetDevice(ctx->device);
  if (n < 0 || !intr || intr->width <= 0 || intr->height <= 0)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "intrinsics: empty image size");
  CU(cudaStreamSynchronize(ctx->stream));
  cudaFree(ctx->rgbd);
  cudaFree(ctx->poses);
  ctx->rgbd = nullptr;
  ctx->poses = nullptr;
  ctx->n_frames = 0;
  ctx->host_depth.clear();
  const long long npix = (long long)intr->width * intr->height;
  if (n > 0) {
    CU(cudaMalloc(&ctx->rgbd, sizeof(double4) * npix * n));
    CU(cudaMalloc(&ctx->poses, sizeof(DevPose) * n));
    int rc = ensure(ctx, ctx->s_stage, sizeof(double) * npix * 4);
    if (rc) return rc;
    std::vector<DevPose> hp(n);
    for (int f = 0; f < n; ++f) {
      double* st = (double*)ctx->s_stage.ptr;
      CU(cudaMemcpyAsync(st, colors[f], sizeof(double) * npix * 3, cudaMemcpyHostToDevice,
                         ctx->stream));
      CU(cudaMemcpyAsync(st + npix * 3, depths[f], sizeof(double) * npix, cudaMemcpyHostToDevice,
                         ctx->stream));
      launch_pack_frames(st, st + npix * 3, ctx->rgbd + npix * f, npix, ctx->stream);
      LAUNCHED(1);
      CU(cudaStreamSynchronize(ctx->stream));
      hp[f] = dev_pose(&poses[f]);
      ctx->host_depth.emplace_back(depths[f], depths[f] + npix);
    }
    CU(cudaMemcpyAsync(ctx->poses, hp.data(), sizeof(DevPose) * n, cudaMemcpyHostToDevice,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  ctx->fintr = *intr;
  ctx->n_frames = n;
  ctx->frame_capacity = n;
  return VRF_OK;
}

int vrf_frames_count(const vrf_context* ctx) { return ctx->n_frames; }

int vrf_frames_reserve(vrf_context* ctx, const vrf_intrinsics* intr, int capacity) {
  cudaSetDevice(ctx->device);
  if (capacity < 0 || !intr || intr->width <= 0 || intr->height <= 0)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "intrinsics: empty image size");
  CU(cudaStreamSynchronize(ctx->stream));
  cudaFree(ctx->rgbd);
  cudaFree(ctx->poses);
  ctx->rgbd = nullptr;
  ctx->poses = nullptr;
  ctx->n_frames = 0;
  ctx->frame_capacity = 0;
  ctx->host_depth.assign(capacity, {});
  const long long npix = (long long)intr->width * intr->height;
  if (capacity > 0) {
    CU(cudaMalloc(&ctx->rgbd, sizeof(double4) * npix * capacity));
    CU(cudaMalloc(&ctx->poses, sizeof(DevPose) * capacity));
  }
  ctx->fintr = *intr;
  ctx->frame_capacity = capacity;
  return VRF_OK;
}

int vrf_frame_set(vrf_context* ctx, int slot, const double* color, const double* depth,
                  const vrf_pose* pose) {
  cudaSetDevice(ctx->device);
  if (slot < 0 || slot >= ctx->frame_capacity)
    return set_err(ctx, VRF_ERR_OUT_OF_RANGE, "frames: slot out of range");
  const long long npix = (long long)ctx->fintr.width * ctx->fintr.height;
  int rc = ensure(ctx, ctx->s_stage, sizeof(double) * npix * 4);
  if (rc) return rc;
  if ((rc = ensure_pinned(ctx, sizeof(DevPose)))) return rc;
  double* st = (double*)ctx->s_stage.ptr;
  CU(cudaMemcpyAsync(st, color, sizeof(double) * npix * 3, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(st + npix * 3, depth, sizeof(double) * npix, cudaMemcpyHostToDevice,
                     ctx->stream));
  launch_pack_frames(st, st + npix * 3, ctx->rgbd + npix * slot, npix, ctx->stream);
  LAUNCHED(1);
  const DevPose dp = dev_pose(pose);
  std::memcpy(ctx->h_pinned, &dp, sizeof(dp));
  CU(cudaMemcpyAsync(ctx->poses + slot, ctx->h_pinned, sizeof(DevPose), cudaMemcpyHostToDevice,
                     ctx->stream));
  ctx->host_depth[slot].assign(depth, depth + npix);
  ctx->n_frames = std::max(ctx->n_frames, slot + 1);
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

int vrf_frame_set_u8u16(vrf_context* ctx, int slot, const uint8_t* rgb, const uint16_t* depth,
                        const vrf_pose* pose) {
  cudaSetDevice(ctx->device);
  if (slot < 0 || slot >= ctx->frame_capacity)
    return set_err(ctx, VRF_ERR_OUT_OF_RANGE, "frames: slot out of range");
  const long long npix = (long long)ctx->fintr.width * ctx->fintr.height;
  const size_t doff = ((size_t)npix * 3 + 15) & ~(size_t)15;  // aligned depth block
  const size_t bytes = doff + (size_t)npix * 2;
  int rc = ensure(ctx, ctx->s_stage, bytes + 16);
  if (rc) return rc;
  if ((rc = ensure_pinned(ctx, sizeof(DevPose)))) return rc;
  char* h = (char*)ctx->h_pinned;
  char* st = (char*)ctx->s_stage.ptr;
  // The sensor buffers go H2D straight from the caller's pageable memory (the
  // driver pipelines its own staging: r02, config-2 e2e ~510 frames/s against
  // ~494 with a memcpy into our page-locked stage first), then the decode, the
  // pose copy and one synchronize.
  CU(cudaMemcpyAsync(st, rgb, (size_t)npix * 3, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(st + doff, depth, (size_t)npix * 2, cudaMemcpyHostToDevice, ctx->stream));
  const DevPose dp = dev_pose(pose);
  std::memcpy(h, &dp, sizeof(dp));
  launch_pack_frames_u8((const uint8_t*)st, (const uint16_t*)(st + doff), ctx->fintr.depth_scale,
                        ctx->rgbd + npix * slot, npix, ctx->stream);
  LAUNCHED(1);
  CU(cudaMemcpyAsync(ctx->poses + slot, h, sizeof(DevPose), cudaMemcpyHostToDevice,
                     ctx->stream));
  ctx->host_depth[slot].clear();  // rebuilt from the device on demand (Adam tracking)
  ctx->n_frames = std::max(ctx->n_frames, slot + 1);
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

int vrf_frame_set_pose(vrf_context* ctx, int slot, const vrf_pose* pose) {
  cudaSetDevice(ctx->device);
  if (slot < 0 || slot >= ctx->n_frames)
    return set_err(ctx, VRF_ERR_OUT_OF_RANGE, "frames: slot out of range");
  int rc = ensure_pinned(ctx, sizeof(DevPose));
  if (rc) return rc;
  const DevPose dp = dev_pose(pose);
  std::memcpy(ctx->h_pinned, &dp, sizeof(dp));
  CU(cudaMemcpyAsync(ctx->poses + slot, ctx->h_pinned, sizeof(DevPose), cudaMemcpyHostToDevice,
                     ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

// ----------------------------------------------------------------- render_image
int vrf_render_image(vrf_context* ctx, const vrf_intrinsics* intr, const vrf_pose* pose,
                     const vrf_render_params* params, int stride, double* color, double* depth) {
  cudaSetDevice(ctx->device);
  if (stride < 1)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "render_image: stride must be >= 1");
  int rc = need_grid(ctx);
  if (rc) return rc;
  DevParams p;
  if ((rc = resolve_params(ctx, params, &p))) return rc;
  const int out_w = (intr->width + stride - 1) / stride;
  const int out_h = (intr->height + stride - 1) / stride;
  const long long n = (long long)out_w * out_h;
  if (n <= 0) return VRF_OK;
  if ((rc = ensure(ctx, ctx->s_out, sizeof(double) * 4 * n))) return rc;
  double* dc = (double*)ctx->s_out.ptr;
  CU(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
  launch_render_image(dev_grid(ctx), p, dev_cam(intr), dev_pose(pose), stride, out_w, out_h, dc,
                      dc + 3 * n, ctx->d_err, ctx->stream);
  LAUNCHED(1);
  CU(cudaGetLastError());
  if ((rc = check_err_flag(ctx))) return rc;
  CU(cudaMemcpyAsync(color, dc, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(depth, dc + 3 * n, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

// ----------------------------------------------------------------- inspection
int vrf_debug_sample_rays(vrf_context* ctx, const double* rays, int n,
                          const vrf_render_params* params, int cap, int32_t* counts, double* t,
                          double* delta, uint32_t* cells) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  DevParams p;
  if ((rc = resolve_params(ctx, params, &p))) return rc;
  if (n <= 0) return VRF_OK;
  const size_t need = sizeof(double) * 6 * n + sizeof(int) * n + (size_t)n * cap * 20 + 64;
  if ((rc = ensure(ctx, ctx->s_out, need))) return rc;
  char* base = (char*)ctx->s_out.ptr;
  double* d_rays = (double*)base;
  double* d_t = d_rays + 6 * n;
  double* d_delta = d_t + (size_t)n * cap;
  uint32_t* d_cells = (uint32_t*)(d_delta + (size_t)n * cap);
  int* d_counts = (int*)(d_cells + (size_t)n * cap);
  CU(cudaMemcpyAsync(d_rays, rays, sizeof(double) * 6 * n, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
  launch_debug_rays(dev_grid(ctx), p, d_rays, n, cap, d_counts, d_t, d_delta, d_cells, nullptr,
                    ctx->d_err, ctx->stream);
  LAUNCHED(1);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(counts, d_counts, sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->stream));
  if (cap > 0) {
    CU(cudaMemcpyAsync(t, d_t, sizeof(double) * n * cap, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(delta, d_delta, sizeof(double) * n * cap, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaMemcpyAsync(cells, d_cells, sizeof(uint32_t) * n * cap, cudaMemcpyDeviceToHost,
                       ctx->stream));
  }
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

int vrf_debug_render_rays(vrf_context* ctx, const double* rays, int n,
                          const vrf_render_params* params, double* out) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  DevParams p;
  if ((rc = resolve_params(ctx, params, &p))) return rc;
  if (n <= 0) return VRF_OK;
  if ((rc = ensure(ctx, ctx->s_out, sizeof(double) * 14 * n))) return rc;
  double* d_rays = (double*)ctx->s_out.ptr;
  double* d_out = d_rays + 6 * n;
  CU(cudaMemcpyAsync(d_rays, rays, sizeof(double) * 6 * n, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
  launch_debug_rays(dev_grid(ctx), p, d_rays, n, 0, nullptr, nullptr, nullptr, nullptr, d_out,
                    ctx->d_err, ctx->stream);
  LAUNCHED(1);
  CU(cudaGetLastError());
  if ((rc = check_err_flag(ctx))) return rc;
  CU(cudaMemcpyAsync(out, d_out, sizeof(double) * 8 * n, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return VRF_OK;
}

}  // extern "C"
