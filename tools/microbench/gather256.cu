// Microbenchmark: trilinear corner gathers of coherent rays from a [V][28] fp32
// payload with 7 x LDG.128 per corner (112-B vertices) against 4 x LDG.256 per
// corner (vertices padded to 128 B). Rays of a warp start in neighbouring cells
// and march one half-cell per sample along a shared direction.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int R = 257;

template <int STRIDE_F4, bool WIDE>
__global__ void k(const float4* __restrict__ p, float* out, int samples) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int w = t >> 5, l = t & 31;
  float ox = 20.f + (w % 200) + (l & 7) * 0.13f, oy = 20.f + ((w / 200) % 200) + (l >> 3) * 0.13f,
        oz = 5.f + (w % 7);
  const float dx = 0.55f, dy = 0.35f, dz = 0.75f;
  float acc = 0.f;
  for (int s = 0; s < samples; ++s) {
    const float x = ox + dx * 0.5f * s, y = oy + dy * 0.5f * s, z = oz + dz * 0.5f * s;
    const int cx = min((int)x, R - 2), cy = min((int)y, R - 2), cz = min((int)z, R - 2);
    const int base = cx + R * (cy + R * cz);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int v = base + (k & 1) + ((k >> 1) & 1) * R + ((k >> 2) & 1) * R * R;
      const float4* vp = p + (size_t)v * STRIDE_F4;
      if (WIDE) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float a0, a1, a2, a3, a4, a5, a6, a7;
          asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3), "=f"(a4), "=f"(a5), "=f"(a6),
                         "=f"(a7)
                       : "l"(vp + 2 * j));
          acc += a0 * 0.1f + a1 + a2 + a3 + a4 + a5 + a6 + a7;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 7; ++j) {
          const float4 a = __ldg(vp + j);
          acc += a.x * 0.1f + a.y + a.z + a.w;
        }
      }
    }
  }
  out[t] = acc;
}

int main() {
  const size_t V = (size_t)R * R * R;
  float4* p;
  cudaMalloc(&p, V * 128);
  cudaMemset(p, 0, V * 128);
  float* out;
  const int n = 1 << 20, samples = 200;
  cudaMalloc(&out, n * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep)
    for (int mode = 0; mode < 2; ++mode) {
      cudaEventRecord(a);
      if (mode == 0) k<7, false><<<n / 128, 128>>>(p, out, samples);
      else k<8, true><<<n / 128, 128>>>(p, out, samples);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("%s: %.3f ms (%.2f G samples/s) %s\n", mode ? "4 x LDG.256 (128 B)" : "7 x LDG.128 (112 B)",
             ms, (double)n * samples / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
