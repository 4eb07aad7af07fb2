// Coherent ray order for the per-ray kernels: rays sorted by (keyframe, Morton
// order of the pixel), so the 32 rays of a warp march nearly the same
// cells and the grid / gradient lines of the rays in flight stay in L2 (r01:
// 1.18e9 -> 3.41e9 mapping samples/s over draw order).
#include <algorithm>

#include <cub/cub.cuh>

#include "vrf_internal.h"

namespace vrf {

namespace {

// ------------------------------------------------------------------ ray ordering
__device__ __forceinline__ uint32_t spread_bits(uint32_t x) {  // 10 bits -> 20 (every other)
  x &= 0x3ff;
  x = (x | (x << 8)) & 0x00ff00ff;
  x = (x | (x << 4)) & 0x0f0f0f0f;
  x = (x | (x << 2)) & 0x33333333;
  x = (x | (x << 1)) & 0x55555555;
  return x;
}

#ifndef VRF_RAY_TILE_LOG2
#define VRF_RAY_TILE_LOG2 0  // Morton tile edge 2^T pixels: single pixels (r02 A/B,
                             // tools/ab/tile.sh: 1.118e10 vs 1.114e10 samples/s for 4x4)
#endif
__device__ __forceinline__ uint32_t spread_bits11(uint32_t x) {  // 11 bits -> 22
  x &= 0x7ff;
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}
__global__ void k_ray_keys(const int* __restrict__ batch, int n, uint32_t* keys, uint32_t* ids) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
#if VRF_RAY_TILE_LOG2 == 2
  const uint32_t f = (uint32_t)batch[3 * i], x = (uint32_t)batch[3 * i + 1] >> 2,
                 y = (uint32_t)batch[3 * i + 2] >> 2;
  // keyframe in the high bits, Morton order of 4x4-pixel tiles below
  keys[i] = (f << 20) | spread_bits(x) | (spread_bits(y) << 1);
#else
  const uint32_t f = (uint32_t)batch[3 * i], x = (uint32_t)batch[3 * i + 1] >> VRF_RAY_TILE_LOG2,
                 y = (uint32_t)batch[3 * i + 2] >> VRF_RAY_TILE_LOG2;
  keys[i] = (f << 22) | spread_bits11(x) | (spread_bits11(y) << 1);
#endif
  ids[i] = (uint32_t)i;
}

// Tracking pixels (px, py): Morton order of 4x4-pixel tiles.
__global__ void k_pixel_keys(const int* __restrict__ px, int n, uint32_t* keys, uint32_t* ids) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t x = (uint32_t)px[2 * i] >> 2, y = (uint32_t)px[2 * i + 1] >> 2;
  keys[i] = spread_bits(x) | (spread_bits(y) << 1);
  ids[i] = (uint32_t)i;
}

__global__ void k_iota(uint32_t* out, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (uint32_t)i;
}

}  // namespace

void launch_pixel_order(const int* pixels, int n, uint32_t* keys, uint32_t* ids, uint32_t* keys2,
                        uint32_t* order, void* tmp, size_t tmp_bytes, cudaStream_t s) {
  k_pixel_keys<<<(n + 255) / 256, 256, 0, s>>>(pixels, n, keys, ids);
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, ids, order, n, 0, 32, s);
}

void launch_ray_order(const int* batch, int n, uint32_t* keys, uint32_t* ids, uint32_t* keys2,
                      uint32_t* order, void* tmp, size_t tmp_bytes, cudaStream_t s) {
  k_ray_keys<<<(n + 255) / 256, 256, 0, s>>>(batch, n, keys, ids);
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, ids, order, n, 0, 32, s);
}

// The RMSProp update log in vertex order (the drop-in's host scatter then walks
// the caller's fp64 arrays forward): sort (id, position) pairs by id.
void launch_update_sort(const uint32_t* ids, long long n, uint32_t* ids_sorted, uint32_t* iota,
                        uint32_t* perm, void* tmp, size_t tmp_bytes, cudaStream_t s) {
  k_iota<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(iota, n);
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, ids, ids_sorted, iota, perm, (int)n, 0, 32, s);
}
size_t update_sort_tmp_bytes(long long n) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 32);
  return b;
}
// Entries [first, first + count) of the sorted log, gathered contiguously.
__global__ void k_update_gather(const uint32_t* __restrict__ perm, long long first, long long count,
                                const float4* __restrict__ theta, const float4* __restrict__ v,
                                float4* __restrict__ theta_out, float4* __restrict__ v_out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const uint32_t p = perm[first + i];
    theta_out[i] = theta[p];
    v_out[i] = v[p];
  }
}
void launch_update_gather(const uint32_t* perm, long long first, long long count,
                          const float4* theta, const float4* v, float4* theta_out, float4* v_out,
                          cudaStream_t s) {
  const long long blocks = std::min<long long>((count + 255) / 256, 148LL * 16);
  k_update_gather<<<(unsigned)std::max(1LL, blocks), 256, 0, s>>>(perm, first, count, theta, v,
                                                                  theta_out, v_out);
}

size_t ray_order_tmp_bytes(int n) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, n, 0, 32);
  return b;
}

}  // namespace vrf
