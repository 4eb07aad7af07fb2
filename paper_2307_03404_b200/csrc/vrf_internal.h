// Internal host<->kernel interface of libvoxrf_b200 (not part of the C-ABI).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "vrf_device.cuh"

namespace vrf {

// Per-block partial and reduced statistics of a mapping forward pass.
struct MapPartial {
  double lp, lg;
  long long samples;
  int m_c, m_d, bad;
  int max_count;  // longest composited sample run of one ray (record-cap sizing)
};
using MapStats = MapPartial;  // reduced: bad = first bad ray (INT_MAX if none)

// Per-block partial / reduced normal equations of a pose pass.
struct PosePartial {
  double jtj[21];
  double jtr[6];
  double loss;
  long long samples;
  int m;
  int bad;
};

enum FlagBits : uint8_t { kHit = 1, kDepthValid = 2, kOverflow = 4 };

// Per-sample record of the fast mapping forward (24 B in two planes), consumed by
// the reverse-order backward. Plane a (float4): w_i and the clamped colour, each
// channel negated when its clamp fired (sign bit = clamp flag). Plane b (uint2):
// the sample's cell (cx | cy << 10 | cz << 20, located in FP64 by the forward)
// with sigma_raw > 0 in bit 30, and its segment midpoint t (fp32). T_{i+1} is not
// stored: the walk rebuilds it from the ray's final T (rec_count[t].y) as
// T_i = T_{i+1} + w_i. The backward re-derives only the trilinear weights, in
// fp32. Both planes share the slot index rec_index(t, c, K). (r01 stored 24 B
// and re-located the cell in FP64; r02's first record was 32 B with T and the
// flags in separate words: K0 9.15 ms against 8.70 here.)
struct RecBuf {
  float4* a;
  uint2* b;
};
constexpr size_t kRecBytes = sizeof(float4) + sizeof(uint2);
// The two planes of a record buffer of `slots` records at `base`.
inline RecBuf rec_planes(void* base, size_t slots) {
  return RecBuf{(float4*)base, (uint2*)((char*)base + slots * sizeof(float4))};
}
constexpr uint32_t kRecSigmaPos = 1u << 30;  // in the cell word
constexpr int kRecMaxCells = 1024;  // per axis (10-bit cell coordinates in the record)
__host__ __device__ __forceinline__ uint32_t pack_cell(int cx, int cy, int cz) {
  return (uint32_t)cx | ((uint32_t)cy << 10) | ((uint32_t)cz << 20);
}

// Launchers (vrf_kernels.cu). All take the context stream.
void launch_render_image(const DevGrid& g, const DevParams& p, const DevCam& cam,
                         const DevPose& pose, int stride, int out_w, int out_h, double* color,
                         double* depth, int* err_flag, cudaStream_t s);
void launch_debug_rays(const DevGrid& g, const DevParams& p, const double* rays, int n, int cap,
                       int* counts, double* t, double* delta, uint32_t* cells, double* out,
                       int* err_flag, cudaStream_t s);
void launch_map_forward(const DevGrid& g, const DevParams& p, const DevCam& cam,
                        const double4* rgbd, const DevPose* poses, int n_frames,
                        const int* batch, int n, double4* ray_cd, uint8_t* flags,
                        MapPartial* partials, int* ray_count, int* err_flag, bool fast,
                        const uint32_t* order, cudaStream_t s);
int map_forward_blocks(int n);
void launch_map_reduce(const MapPartial* partials, int nparts, MapStats* out, cudaStream_t s);
// Fast forward that also stores up to K sample records per ray, warp-tiled sample-major
// (rec_index(slot, c, K), slot = coherent order index); rays with more samples get
// kOverflow. rec_count[slot] = (samples stored, final T as float bits).
// CTAs of the K0 launch for n rays (the small-batch K0g has 16 rays per CTA).
int map_forward_rec_blocks(int n);
void launch_map_forward_rec(const DevGrid& g, const DevParams& p, const DevCam& cam,
                            const double4* rgbd, const DevPose* poses, int n_frames,
                            const int* batch, int n, double4* ray_cd, uint8_t* flags,
                            MapPartial* partials, int* err, const uint32_t* order, RecBuf rec,
                            int K, int2* rec_count, cudaStream_t s);
// Backward over the records (no payload gathers); kOverflow rays are
// left to launch_map_backward(..., overflow_only = true).
void launch_map_backward_rec(const DevGrid& g, const DevParams& p, const DevCam& cam,
                             const double4* rgbd, const DevPose* poses, const int* batch, int n,
                             const double4* ray_cd, const uint8_t* flags, const MapStats* stats,
                             const int* global_counts, float4* grad, double lambda_d,
                             const uint32_t* order, const RecBuf rec, int K,
                             const int2* rec_count, cudaStream_t s);
void launch_map_backward(const DevGrid& g, const DevParams& p, const DevCam& cam,
                         const double4* rgbd, const DevPose* poses, const int* batch, int n,
                         const double4* ray_cd, const uint8_t* flags, const MapStats* stats,
                         const int* global_counts, float4* grad, double lambda_d, bool overflow_only,
                         const uint32_t* order, cudaStream_t s);
void launch_map_backward_records(const DevGrid& g, const DevParams& p, const DevCam& cam,
                                 const double4* rgbd, const DevPose* poses, const int* batch,
                                 int n, const double4* ray_cd, const uint8_t* flags,
                                 const MapStats* stats, double lambda_d,
                                 const long long* ray_offsets, uint32_t* keys, uint32_t* ids,
                                 double* values, int r0, int r1, long long sid_base,
                                 cudaStream_t s);
void launch_segmented_reduce(const uint32_t* sorted_keys, const uint32_t* perm,
                             const double* values, long long nrec, double* grad_out_f64,
                             cudaStream_t s);
// The update log sorted by group id (perm: log position of each sorted entry),
// and a contiguous gather of a range of it (vrf_order.cu).
void launch_update_sort(const uint32_t* ids, long long n, uint32_t* ids_sorted, uint32_t* iota,
                        uint32_t* perm, void* tmp, size_t tmp_bytes, cudaStream_t s);
size_t update_sort_tmp_bytes(long long n);
void launch_update_gather(const uint32_t* perm, long long first, long long count,
                          const float4* theta, const float4* v, float4* theta_out, float4* v_out,
                          cudaStream_t s);
// Log of the float4 groups an RMSProp pass updated (index, new theta, new v): the
// drop-in's sparse write-back (vrf_updates_read). count == nullptr: off.
struct UpdateLog {
  uint32_t* ids = nullptr;
  float4* theta = nullptr;
  float4* v = nullptr;
  unsigned long long* count = nullptr;
  long long cap = 0;
};
// Block-sparse RMSProp over the touched 8^3-vertex blocks; clears the bitmap.
void launch_rmsprop_blocks(float4* theta, float4* grad, float4* v, uint32_t* tb, int rx, int ry,
                           int rz, int tbx, int tby, int tbz, double rho, double lr_sigma,
                           double lr_sh, double eps, const MapStats* stats,
                           unsigned long long* touched, cudaStream_t s,
                           const UpdateLog& log = UpdateLog{});
// Block-sparse multi-GPU exchange (8^3-vertex blocks, packed [n][512][28] fp32; id < 0 = pad).
void launch_touched_flags(const uint32_t* tb, int nb, uint8_t* flags, cudaStream_t s);
// Touched cell blocks (marked by the scatter) -> touched vertex blocks (ORed into
// tb); clears tc.
void launch_touched_dilate(uint32_t* tc, int bx, int by, int bz, uint32_t* tb, int tbx, int tby,
                           int tbz, cudaStream_t s);
void launch_blocks_pack(const float4* src, const int* ids, int n, int rx, int ry, int rz, int tbx,
                        int tby, float4* out, cudaStream_t s);
void launch_blocks_unpack(float4* dst, const int* ids, int n, int rx, int ry, int rz, int tbx,
                          int tby, const float4* in, cudaStream_t s);
// Fused peer-memory exchange (vrf_exchange_p2p): per-rank device pointers as seen
// from the launching device (UVA; IPC-opened for other processes' buffers).
constexpr int kMaxPeers = 8;
struct PeerTable {
  float4* grad[kMaxPeers];
  float4* payload[kMaxPeers];
  const uint32_t* tb[kMaxPeers];
  int world, rank;
};
void launch_exchange_p2p(const PeerTable& pt, float4* v, int nb, int rx, int ry, int rz, int tbx,
                         int tby, double rho, double lr_sigma, double lr_sh, double eps,
                         const MapStats* stats, cudaStream_t s);
void launch_blocks_apply(float4* theta, float4* v, const int* ids, int n, int rx, int ry, int rz,
                         int tbx, int tby, const float4* packed, double rho, double lr_sigma,
                         double lr_sh, double eps, cudaStream_t s);
void launch_rmsprop(float4* theta, float4* grad, float4* v, long long v_begin, long long v_end,
                    double rho, double lr_sigma, double lr_sh, double eps,
                    const MapStats* stats, unsigned long long* touched, cudaStream_t s,
                    const UpdateLog& log = UpdateLog{});
// Tracking (vrf_track.cu).

// kParityFp64: k_pose_group<double> (FP64 SH + Jacobian partials; pose_gradient,
// track_frame). kGnUniform: k_pose_group_u (fp32 partials; the Gauss-Newton
// tracker). kGroupFp32: k_pose_group<float>, the GN kernel's checker (tests).
enum class PoseKernel : int { kParityFp64 = 0, kGnUniform = 1, kGroupFp32 = 2 };
// CTAs (= partials) of a pose-kernel launch over n rays
int pose_fused_blocks(int n, PoseKernel which = PoseKernel::kParityFp64);
void launch_pose_fused(PoseKernel which, const DevGrid& g, const DevParams& p, const DevCam& cam,
                       const double4* rgbd_base, const int* frame_idx, long long npix,
                       const DevPose* pose, const int* pixels, const uint32_t* order, int n,
                       double lambda_p, double lambda_d, PosePartial* partials, int* err,
                       cudaStream_t s);
void launch_pose_reduce2(const PosePartial* partials, int nparts, PosePartial* out,
                         cudaStream_t s);
void launch_draw_strat(const double4* rgbd_base, const int* frame_idx, long long npix, int width,
                       int height, int tiles_log2, int max_redraws,
                       const unsigned long long* seed, int iteration, int* pixels, int n,
                       cudaStream_t s);
void launch_gn_step(const PosePartial* ne, DevPose* pose, double damping, double* hist,
                    int iteration, cudaStream_t s);

// Coherent ray order (vrf_order.cu).
size_t ray_order_tmp_bytes(int n);
void launch_ray_order(const int* batch, int n, uint32_t* keys, uint32_t* ids, uint32_t* keys2,
                      uint32_t* order, void* tmp, size_t tmp_bytes, cudaStream_t s);
void launch_pixel_order(const int* pixels, int n, uint32_t* keys, uint32_t* ids, uint32_t* keys2,
                        uint32_t* order, void* tmp, size_t tmp_bytes, cudaStream_t s);

// Utilities.
void launch_fill_payload(float* payload, long long n_vertices, float sigma, cudaStream_t s);
// Order-independent 64-bit digest of n 32-bit words, added into *out.
void launch_digest(const uint32_t* words, long long n, uint64_t salt, unsigned long long* out,
                   cudaStream_t s);
// A/B only: payload [V][7] float4 -> [7][V] (tools/ab/soa.sh)
void launch_aos_to_soa(const float4* aos, float4* soa, long long nv, cudaStream_t s);
void launch_f64_to_f32(const double* in, float* out, long long n, cudaStream_t s);
void launch_f32_to_f64(const float* in, double* out, long long n, cudaStream_t s);
void launch_pack_occupancy(const uint8_t* occ_u8, uint32_t* bits, long long n_cells,
                           cudaStream_t s);
void launch_unpack_occupancy(const uint32_t* bits, uint8_t* occ_u8, long long n_cells,
                             cudaStream_t s);
void launch_pack_frames(const double* color, const double* depth, double4* rgbd, long long npix,
                        cudaStream_t s);
void launch_prune(const DevGrid& g, uint32_t* occ_bits, double tau, unsigned long long* count,
                  cudaStream_t s);
void launch_pack_frames_u8(const uint8_t* rgb, const uint16_t* depth, double depth_scale,
                           double4* rgbd, long long npix, cudaStream_t s);
void launch_extract_depth(const double4* rgbd, double* out, long long npix, cudaStream_t s);
void launch_upsample(const DevGrid& coarse, int frx, int fry, int frz, float* fine,
                     uint32_t* fine_occ, cudaStream_t s);
// Superblock bit = OR of its (up to) 8^3 block bits.
void launch_super_occupancy(const uint32_t* bocc, int bx, int by, int bz, int sx, int sy, int sz,
                            uint32_t* socc, cudaStream_t s);
void launch_block_occupancy(const uint32_t* occ, int rx, int ry, int rz, int bx, int by, int bz,
                            uint32_t* bocc, unsigned int* n_active, cudaStream_t s);

}  // namespace vrf
