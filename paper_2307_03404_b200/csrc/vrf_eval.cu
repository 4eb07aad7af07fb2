// evaluate_map_quality (eval.cpp:210-240) on the device: the evaluation views are
// rendered by K1 into HBM and scored there, so neither image leaves the GPU.
//   depth_l1 (eval.cpp:99-122): sum |D - D*| over the pixels with valid reference
//     depth (D* > 0) that the render hit (D > 0, the rendered-depth mask);
//   psnr (eval.cpp:64-97): the squared colour error summed over the sampled
//     pixels (the reference's Rng stream, drawn on the host by
//     vrf_rng_draw_eval_samples) that the render hit.
// Each view's sums are per-block partials reduced in a fixed order, so the
// result is deterministic (it differs from the reference's sequential sums at
// the rounding level only).
#include "vrf_context.h"

using namespace vrf;
using namespace vrf_host;

namespace {

constexpr int kEvT = 256;

struct EvPartial {
  double sum;
  long long count;
};

template <typename T>
__device__ __forceinline__ T ev_block_sum(T v, T* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  T r = T(0);
  if (threadIdx.x == 0)
    for (int w = 0; w < kEvT / 32; ++w) r += smem[w];  // fixed order
  return r;
}

__global__ void __launch_bounds__(kEvT) k_eval_depth(const double* __restrict__ depth,
                                                     const double* __restrict__ ref_depth,
                                                     long long npix, EvPartial* out) {
  __shared__ double s_d[kEvT / 32];
  __shared__ long long s_c[kEvT / 32];
  double acc = 0.0;
  long long cnt = 0;
  for (long long i = (long long)blockIdx.x * kEvT + threadIdx.x; i < npix;
       i += (long long)gridDim.x * kEvT) {
    const double b = ref_depth[i], a = depth[i];
    if (b > 0.0 && a > 0.0) {
      acc += fabs(a - b);
      ++cnt;
    }
  }
  const double s = ev_block_sum(acc, s_d);
  const long long c = ev_block_sum(cnt, s_c);
  if (threadIdx.x == 0) out[blockIdx.x] = EvPartial{s, c};
}

// samples: (x, y) pairs of this view
__global__ void __launch_bounds__(kEvT) k_eval_color(const double* __restrict__ color,
                                                     const double* __restrict__ depth,
                                                     const double* __restrict__ ref_color,
                                                     int width, const int* __restrict__ xy, int n,
                                                     EvPartial* out) {
  __shared__ double s_d[kEvT / 32];
  __shared__ long long s_c[kEvT / 32];
  double acc = 0.0;
  long long cnt = 0;
  for (int i = blockIdx.x * kEvT + threadIdx.x; i < n; i += gridDim.x * kEvT) {
    const long long p = (long long)xy[2 * i + 1] * width + xy[2 * i];
    if (depth[p] > 0.0) {
      double e = 0.0;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const double d = color[3 * p + ch] - ref_color[3 * p + ch];
        e += d * d;
      }
      acc += e;
      ++cnt;
    }
  }
  const double s = ev_block_sum(acc, s_d);
  const long long c = ev_block_sum(cnt, s_c);
  if (threadIdx.x == 0) out[blockIdx.x] = EvPartial{s, c};
}

constexpr int kEvBlocks = 148 * 2;  // per view and metric: a fixed, SM-count multiple

}  // namespace

extern "C" {

// eval.cpp:72-83's draw order: for each of `images` draws an image index, then
// pixels_per_image (x, y) pairs; out: images * pixels_per_image (image, x, y).
void vrf_rng_draw_eval_samples(uint64_t state[4], int n_images, int width, int height,
                               int images, int pixels_per_image, int32_t* out) {
  size_t k = 0;
  for (int i = 0; i < images; ++i) {
    // Rng::uniform_index (rng.hpp): the high 64 bits of next() * n
    const int32_t img =
        (int32_t)(((unsigned __int128)vrf_rng_next(state) * (uint64_t)n_images) >> 64);
    for (int s = 0; s < pixels_per_image; ++s) {
      const int32_t x = (int32_t)(((unsigned __int128)vrf_rng_next(state) * (uint64_t)width) >> 64);
      const int32_t y = (int32_t)(((unsigned __int128)vrf_rng_next(state) * (uint64_t)height) >> 64);
      out[3 * k] = img;
      out[3 * k + 1] = x;
      out[3 * k + 2] = y;
      ++k;
    }
  }
}

int vrf_evaluate_views(vrf_context* ctx, const vrf_intrinsics* intr, int n_views,
                       const vrf_pose* poses, const double* const* colors,
                       const double* const* depths, const vrf_render_params* params,
                       const int32_t* samples, int n_samples, vrf_view_metrics* out) {
  cudaSetDevice(ctx->device);
  int rc = need_grid(ctx);
  if (rc) return rc;
  if (n_views <= 0)
    return set_err(ctx, VRF_ERR_RUNTIME, "evaluate_map_quality: no frames");
  DevParams p;
  if ((rc = resolve_params(ctx, params, &p))) return rc;
  const int w = intr->width, h = intr->height;
  const long long npix = (long long)w * h;
  // per view: samples grouped by view (their order within a view is kept)
  std::vector<std::vector<int32_t>> xy((size_t)n_views);
  for (int i = 0; i < n_samples; ++i) {
    const int v = samples[3 * i], x = samples[3 * i + 1], y = samples[3 * i + 2];
    if (v < 0 || v >= n_views || x < 0 || x >= w || y < 0 || y >= h)
      return set_err(ctx, VRF_ERR_OUT_OF_RANGE, "evaluate_map_quality: sample outside image");
    xy[(size_t)v].push_back(x);
    xy[(size_t)v].push_back(y);
  }
  size_t max_xy = 2;
  for (const auto& v : xy) max_xy = std::max(max_xy, v.size());
  // scratch: render colour + depth, reference colour + depth, sample list, partials
  const size_t img_b = sizeof(double) * 4 * (size_t)npix;
  if ((rc = ensure(ctx, ctx->s_out, 2 * img_b + sizeof(int32_t) * max_xy))) return rc;
  const size_t parts_n = (size_t)n_views * 2 * kEvBlocks;
  if ((rc = ensure(ctx, ctx->s_partials, sizeof(EvPartial) * parts_n))) return rc;
  double* rc_col = (double*)ctx->s_out.ptr;
  double* rc_dep = rc_col + 3 * npix;
  double* ref_col = rc_dep + npix;
  double* ref_dep = ref_col + 3 * npix;
  int32_t* d_xy = (int32_t*)(ref_dep + npix);
  EvPartial* parts = (EvPartial*)ctx->s_partials.ptr;
  CU(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
  const DevGrid g = dev_grid(ctx);
  const DevCam cam = dev_cam(intr);
  for (int v = 0; v < n_views; ++v) {
    launch_render_image(g, p, cam, dev_pose(&poses[v]), 1, w, h, rc_col, rc_dep, ctx->d_err,
                        ctx->stream);
    CU(cudaMemcpyAsync(ref_col, colors[v], sizeof(double) * 3 * npix, cudaMemcpyHostToDevice,
                       ctx->stream));
    CU(cudaMemcpyAsync(ref_dep, depths[v], sizeof(double) * npix, cudaMemcpyHostToDevice,
                       ctx->stream));
    EvPartial* pd = parts + (size_t)v * 2 * kEvBlocks;
    k_eval_depth<<<kEvBlocks, kEvT, 0, ctx->stream>>>(rc_dep, ref_dep, npix, pd);
    const int ns = (int)(xy[(size_t)v].size() / 2);
    if (ns > 0)
      CU(cudaMemcpyAsync(d_xy, xy[(size_t)v].data(), sizeof(int32_t) * 2 * ns,
                         cudaMemcpyHostToDevice, ctx->stream));
    k_eval_color<<<kEvBlocks, kEvT, 0, ctx->stream>>>(rc_col, rc_dep, ref_col, w, d_xy, ns,
                                                      pd + kEvBlocks);
    LAUNCHED(3);
    // the host vectors and the next view's uploads reuse the buffers: order them
    CU(cudaStreamSynchronize(ctx->stream));
  }
  // fixed-order totals over the views' block partials
  std::vector<EvPartial> hp(parts_n);
  CU(cudaMemcpyAsync(hp.data(), parts, sizeof(EvPartial) * hp.size(), cudaMemcpyDeviceToHost,
                     ctx->stream));
  if ((rc = check_err_flag(ctx))) return rc;
  vrf_view_metrics m{};
  for (int v = 0; v < n_views; ++v) {
    for (int b = 0; b < kEvBlocks; ++b) {
      const EvPartial& d = hp[(size_t)v * 2 * kEvBlocks + b];
      const EvPartial& c = hp[(size_t)v * 2 * kEvBlocks + kEvBlocks + b];
      m.sum_abs_depth += d.sum;
      m.depth_pixels += d.count;
      m.sum_sq_color += c.sum;
      m.color_samples += c.count;
    }
  }
  *out = m;
  return VRF_OK;
}

}  // extern "C"
