// Microbenchmark: scatter of 112-B vertex gradients with 7 x red.global.add.v4.f32
// per thread vs one cp.reduce.async.bulk (UBLKRED) per thread. Addresses follow
// a coherent-ray-like pattern: warp lanes hit nearby vertices, 4 corners per event.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_red(float4* g, int nv, int events, unsigned seed) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned x = seed ^ (t * 2654435761u);
  int base = (int)((t / 32) * 97u % (unsigned)(nv - 4096)) + (t % 32) * 3;
  for (int e = 0; e < events; ++e) {
    x = x * 1664525u + 1013904223u;
    const int v = base + e * 5 + (x >> 28);
    float4* d = g + (size_t)(v % nv) * 7;
    const float a = (float)(x & 255) * 1e-3f;
#pragma unroll
    for (int j = 0; j < 7; ++j) atomicAdd(d + j, make_float4(a, a, a, a));
  }
}

__global__ void k_bulk(float4* g, int nv, int events, unsigned seed) {
  __shared__ __align__(16) float4 s[128][2][7];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned x = seed ^ (t * 2654435761u);
  int base = (int)((t / 32) * 97u % (unsigned)(nv - 4096)) + (t % 32) * 3;
  for (int e = 0; e < events; ++e) {
    x = x * 1664525u + 1013904223u;
    const int v = base + e * 5 + (x >> 28);
    const float a = (float)(x & 255) * 1e-3f;
    float4* my = s[threadIdx.x][e & 1];
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 7; ++j) my[j] = make_float4(a, a, a, a);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(my);
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 112;"
                 :: "l"(g + (size_t)(v % nv) * 7), "r"(sa) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const int nv = 17000000, events = 64, threads = 1 << 20;
  float4* g;
  cudaMalloc(&g, (size_t)nv * 112);
  cudaMemset(g, 0, (size_t)nv * 112);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    for (int mode = 0; mode < 2; ++mode) {
      cudaEventRecord(a);
      if (mode == 0) k_red<<<threads / 128, 128>>>(g, nv, events, rep);
      else k_bulk<<<threads / 128, 128>>>(g, nv, events, rep);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double flushes = (double)threads * events;
      printf("%s: %.3f ms, %.2f G vertex-flushes/s (%s)\n", mode ? "bulk UBLKRED" : "7x red.v4",
             ms, flushes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
