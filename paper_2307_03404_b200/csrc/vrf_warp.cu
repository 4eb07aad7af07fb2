// Warp-per-ray mapping kernels (the fast path of mapping_step).
//
// One warp owns one ray at a time; lane c (< 28) owns payload slot c
// (sigma, r0..r8, g0..g8, b0..b8 — voxel_grid.hpp:104). Consequences:
//  * every corner gather is one coalesced 112-B load (28 lanes x 4 B) and
//    every gradient scatter one coalesced 112-B red.global.add.f32;
//  * each lane's trilinear sum runs over the 8 corners in the reference's
//    order in FP64, so sigma_raw, the SH coefficients, the SH colour
//    (summed by lanes 0-2 from shared memory in reference order) and hence T
//    and the termination decision are bit-identical to the CPU reference;
//  * the schedule is located 32 segments at a time, one per lane (FP64,
//    reference order), and walked in order with a ballot;
//  * the backward keeps the 8 corner accumulators of the current cell in
//    registers (8 per lane) and flushes them only when the ray leaves the cell,
//    so consecutive samples in one cell cost one scatter;
//  * rays are taken from a device work queue in (keyframe, Morton tile) order
//    so the whole GPU works on a spatially coherent window of rays at any time,
//    which keeps the grid and gradient lines of that window resident in L2.
#include <climits>
#include <cub/cub.cuh>

#include "vrf_internal.h"

namespace vrf {

namespace {

constexpr int kWarpThreads = 256;  // 8 warps per CTA
constexpr unsigned kFull = 0xffffffffu;

struct WarpRay {
  double o[3], d[3];
  double lo, hi, step;
  long long nseg;
};

// Segment k of the uniform schedule (renderer.cpp:66-79) located in the grid.
__device__ __forceinline__ bool segment_sample(const DevGrid& g, const WarpRay& r, long long k,
                                               Sample& s) {
  const double s0 = dadd(r.lo, dmul((double)k, r.step));
  const double s0s = dadd(s0, r.step);
  const double s1 = (r.hi < s0s) ? r.hi : s0s;
  const double len = dsub(s1, s0);
  if (len < 1e-12) return false;
  const double tm = dmul(0.5, dadd(s0, s1));
  const double p[3] = {dadd(r.o[0], dmul(tm, r.d[0])), dadd(r.o[1], dmul(tm, r.d[1])),
                       dadd(r.o[2], dmul(tm, r.d[2]))};
  if (!locate(g, p, s)) return false;
  if (!cell_active(g, s.cell)) return false;
  s.t = tm;
  s.delta = len;
  return true;
}

struct Bcast {
  double t, delta, fx, fy, fz;
  uint32_t base;
};

__device__ __forceinline__ Bcast bcast(const Sample& s, int src) {
  Bcast b;
  b.t = __shfl_sync(kFull, s.t, src);
  b.delta = __shfl_sync(kFull, s.delta, src);
  b.fx = __shfl_sync(kFull, s.fx, src);
  b.fy = __shfl_sync(kFull, s.fy, src);
  b.fz = __shfl_sync(kFull, s.fz, src);
  b.base = __shfl_sync(kFull, s.base, src);
  return b;
}

__device__ __forceinline__ void weights8(const Bcast& b, double w[8]) {
  const double wx[2] = {dsub(1.0, b.fx), b.fx};
  const double wy[2] = {dsub(1.0, b.fy), b.fy};
  const double wz[2] = {dsub(1.0, b.fz), b.fz};
#pragma unroll
  for (int k = 0; k < 8; ++k) w[k] = dmul(dmul(wx[k & 1], wy[(k >> 1) & 1]), wz[(k >> 2) & 1]);
}

// Slot-parallel trilerp + SH colour of one sample. Returns sigma_raw (all lanes);
// c[3] and the clamp mask (bit ch) are warp-uniform on return.
__device__ __forceinline__ double shade_warp(const DevGrid& g, const float* __restrict__ pay,
                                             const Bcast& b, const double w[8], double basis_l,
                                             int lane, double* sm, double c[3], unsigned& clamp,
                                             double& acc_out) {
  float v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    v[k] = lane < kPayload ? __ldg(pay + (size_t)corner_index(g, b.base, k) * kPayload + lane) : 0.f;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc = dadd(acc, dmul(w[k], (double)v[k]));
  acc_out = acc;
  sm[lane] = (lane >= 1 && lane < kPayload) ? dmul(acc, basis_l) : 0.0;
  __syncwarp();
  double col = 0.0;
  bool cl = false;
  if (lane < 3) {
    double s = 0.5;
#pragma unroll
    for (int m = 0; m < 9; ++m) s = dadd(s, sm[1 + 9 * lane + m]);
    cl = (s <= 0.0 || s >= 1.0);
    col = (s < 0.0) ? 0.0 : ((1.0 < s) ? 1.0 : s);
  }
  clamp = __ballot_sync(kFull, cl) & 7u;
  c[0] = __shfl_sync(kFull, col, 0);
  c[1] = __shfl_sync(kFull, col, 1);
  c[2] = __shfl_sync(kFull, col, 2);
  __syncwarp();
  return __shfl_sync(kFull, acc, 0);
}

__device__ __forceinline__ bool warp_ray_begin(const DevGrid& g, const DevParams& p,
                                               const DevCam& cam, const DevPose& pose, int px,
                                               int py, WarpRay& r, double& basis_l, int lane,
                                               bool& basis_ok) {
  March m;
  generate_dir(cam, pose, (double)px, (double)py, m.d);
  m.o[0] = pose.t[0];
  m.o[1] = pose.t[1];
  m.o[2] = pose.t[2];
  double basis[9];
  basis_ok = sh_basis(m.d, basis);
  basis_l = 0.0;
  if (lane >= 1 && lane < kPayload) {
    const int mm = (lane - 1) % 9;
#pragma unroll
    for (int q = 0; q < 9; ++q)
      if (q == mm) basis_l = basis[q];
  }
  for (int a = 0; a < 3; ++a) {
    r.o[a] = m.o[a];
    r.d[a] = m.d[a];
  }
  if (!march_begin(g, p, m)) return false;
  r.lo = m.lo;
  r.hi = m.hi;
  r.step = m.step;
  r.nseg = m.nseg;
  return true;
}

__device__ __forceinline__ int next_ray(int* queue, int lane) {
  int i = 0;
  if (lane == 0) i = atomicAdd(queue, 1);
  return __shfl_sync(kFull, i, 0);
}

// ------------------------------------------------------------------ forward
__global__ void __launch_bounds__(kWarpThreads) k_map_forward_w(
    DevGrid g, DevParams p, DevCam cam, const double4* __restrict__ rgbd,
    const DevPose* __restrict__ poses, int n_frames, const int* __restrict__ batch,
    const uint32_t* __restrict__ order, int n, double4* __restrict__ ray_cd,
    uint8_t* __restrict__ flags, MapPartial* __restrict__ partials, int* queue, int* err) {
  __shared__ double s_prod[kWarpThreads / 32][32];
  __shared__ double s_d[kWarpThreads / 32][2];
  __shared__ long long s_l[kWarpThreads / 32];
  __shared__ int s_i[kWarpThreads / 32][3];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* sm = s_prod[wid];
  const float* pay = reinterpret_cast<const float*>(g.payload);
  double lp = 0.0, lg = 0.0;
  long long samples = 0;
  int mc = 0, md = 0, bad = INT_MAX;
  for (int q = next_ray(queue, lane); q < n; q = next_ray(queue, lane)) {
    const int i = (int)order[q];
    const int f = batch[3 * i], px = batch[3 * i + 1], py = batch[3 * i + 2];
    if (f < 0 || f >= n_frames || px < 0 || px >= cam.width || py < 0 || py >= cam.height) {
      if (lane == 0) {
        atomicOr(err, 2);
        flags[i] = 0;
      }
      continue;
    }
    WarpRay r;
    double basis_l;
    bool basis_ok;
    const bool any = warp_ray_begin(g, p, cam, poses[f], px, py, r, basis_l, lane, basis_ok);
    if (!basis_ok && lane == 0) atomicOr(err, 1);
    double T = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0, D = 0.0;
    int count = 0;
    bool done = !any;
    for (long long k0 = 0; k0 < (any ? r.nseg : 0) && !done; k0 += 32) {
      Sample s;
      const long long k = k0 + lane;
      const bool valid = k < r.nseg && segment_sample(g, r, k, s);
      unsigned mask = __ballot_sync(kFull, valid);
      while (mask) {
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        const Bcast b = bcast(s, src);
        double w[8];
        weights8(b, w);
        double c[3], acc;
        unsigned clamp;
        const double sraw = shade_warp(g, pay, b, w, basis_l, lane, sm, c, clamp, acc);
        const double sigma = (sraw < 0.0) ? 0.0 : sraw;
        const double decay = exp(dmul(-sigma, b.delta));
        const double wgt = dmul(T, dsub(1.0, decay));
        C0 = dadd(C0, dmul(wgt, c[0]));
        C1 = dadd(C1, dmul(wgt, c[1]));
        C2 = dadd(C2, dmul(wgt, c[2]));
        D = dadd(D, dmul(wgt, b.t));
        T = dmul(T, decay);
        ++count;
        if (T < p.eps) {
          done = true;
          break;
        }
      }
    }
    if (lane == 0) {
      uint8_t fl = 0;
      if (count == 0) C0 = C1 = C2 = D = 0.0;
      const double4 tg =
          rgbd[(long long)f * cam.width * cam.height + (long long)py * cam.width + px];
      if (count > 0) {
        fl |= kHit;
        ++mc;
        samples += count;
        const double r0 = dsub(C0, tg.x), r1 = dsub(C1, tg.y), r2 = dsub(C2, tg.z);
        const double sq = dadd(dadd(dmul(r0, r0), dmul(r1, r1)), dmul(r2, r2));
        if (!isfinite(sq) || !isfinite(D)) {
          bad = min(bad, i);
        } else {
          lp += sq;
          if (tg.w > 0.0) {
            fl |= kDepthValid;
            ++md;
            const double dr = dsub(D, tg.w);
            lg += dmul(dr, dr);
          }
        }
      }
      ray_cd[i] = make_double4(C0, C1, C2, D);
      flags[i] = fl;
    }
  }
  // per-CTA partial (lane 0 of each warp holds the warp's sums)
  if (lane == 0) {
    s_d[wid][0] = lp;
    s_d[wid][1] = lg;
    s_l[wid] = samples;
    s_i[wid][0] = mc;
    s_i[wid][1] = md;
    s_i[wid][2] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    MapPartial out{0.0, 0.0, 0, 0, 0, INT_MAX, 0};
    for (int w = 0; w < kWarpThreads / 32; ++w) {
      out.lp += s_d[w][0];
      out.lg += s_d[w][1];
      out.samples += s_l[w];
      out.m_c += s_i[w][0];
      out.m_d += s_i[w][1];
      out.bad = min(out.bad, s_i[w][2]);
    }
    partials[blockIdx.x] = out;
  }
}

// ------------------------------------------------------------------ backward
__device__ __forceinline__ void flush_cell(const DevGrid& g, float* __restrict__ grad,
                                           uint32_t base, float acc[8], int lane) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const bool nz = __any_sync(kFull, acc[k] != 0.f);
    if (nz && lane < kPayload)
      atomicAdd(grad + (size_t)corner_index(g, base, k) * kPayload + lane, acc[k]);
    acc[k] = 0.f;
  }
}

__global__ void __launch_bounds__(kWarpThreads) k_map_backward_w(
    DevGrid g, DevParams p, DevCam cam, const double4* __restrict__ rgbd,
    const DevPose* __restrict__ poses, const int* __restrict__ batch,
    const uint32_t* __restrict__ order, int n, const double4* __restrict__ ray_cd,
    const uint8_t* __restrict__ flags, const MapStats* __restrict__ stats,
    const int* __restrict__ global_counts, float* __restrict__ grad, double lambda_d,
    int* queue) {
  __shared__ double s_prod[kWarpThreads / 32][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* sm = s_prod[wid];
  const float* pay = reinterpret_cast<const float*>(g.payload);
  const MapStats st = *stats;
  if (st.bad != INT_MAX) return;
  const int mcount = global_counts ? global_counts[0] : st.m_c;
  const int dcount = global_counts ? global_counts[1] : st.m_d;
  if (mcount == 0) return;
  for (int q = next_ray(queue, lane); q < n; q = next_ray(queue, lane)) {
    const int i = (int)order[q];
    const uint8_t fl = flags[i];
    if (!(fl & kHit)) continue;
    const int f = batch[3 * i], px = batch[3 * i + 1], py = batch[3 * i + 2];
    const double4 tg = rgbd[(long long)f * cam.width * cam.height + (long long)py * cam.width + px];
    const double4 cd = ray_cd[i];
    // upstream (mapping.cpp:172-193)
    const double upc0 = ddiv(dmul(2.0, dsub(cd.x, tg.x)), (double)mcount);
    const double upc1 = ddiv(dmul(2.0, dsub(cd.y, tg.y)), (double)mcount);
    const double upc2 = ddiv(dmul(2.0, dsub(cd.z, tg.z)), (double)mcount);
    const bool depth_ok = (fl & kDepthValid) && dcount > 0;
    const double upd =
        depth_ok ? ddiv(dmul(dmul(lambda_d, 2.0), dsub(cd.w, tg.w)), (double)dcount) : 0.0;
    const bool use_depth = depth_ok && upd != 0.0;
    WarpRay r;
    double basis_l;
    bool basis_ok;
    if (!warp_ray_begin(g, p, cam, poses[f], px, py, r, basis_l, lane, basis_ok) || !basis_ok)
      continue;
    // this lane's upstream channel: slot 0 -> sigma, 1..27 -> SH channel (slot-1)/9
    const int ch = lane >= 1 && lane < kPayload ? (lane - 1) / 9 : 0;
    double T = 1.0, pre0 = 0.0, pre1 = 0.0, pre2 = 0.0, pre_d = 0.0;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    uint32_t cur = 0xffffffffu;
    bool done = false;
    for (long long k0 = 0; k0 < r.nseg && !done; k0 += 32) {
      Sample s;
      const long long k = k0 + lane;
      const bool valid = k < r.nseg && segment_sample(g, r, k, s);
      unsigned mask = __ballot_sync(kFull, valid);
      while (mask) {
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        const Bcast b = bcast(s, src);
        double w[8];
        weights8(b, w);
        double c[3], sh_acc;
        unsigned clamp;
        const double sraw = shade_warp(g, pay, b, w, basis_l, lane, sm, c, clamp, sh_acc);
        const double sigma = (sraw < 0.0) ? 0.0 : sraw;
        const double decay = exp(dmul(-sigma, b.delta));
        const double wgt = dmul(T, dsub(1.0, decay));
        const double Tn = dmul(T, decay);
        // prefix form, gradients.cpp:69-97
        pre0 = dadd(pre0, dmul(c[0], wgt));
        pre1 = dadd(pre1, dmul(c[1], wgt));
        pre2 = dadd(pre2, dmul(c[2], wgt));
        double ds = 0.0;
        ds = dadd(ds, dmul(dmul(upc0, b.delta), dadd(dsub(dmul(c[0], Tn), cd.x), pre0)));
        ds = dadd(ds, dmul(dmul(upc1, b.delta), dadd(dsub(dmul(c[1], Tn), cd.y), pre1)));
        ds = dadd(ds, dmul(dmul(upc2, b.delta), dadd(dsub(dmul(c[2], Tn), cd.z), pre2)));
        if (use_depth) {
          pre_d = dadd(pre_d, dmul(b.t, wgt));
          ds = dadd(ds, dmul(dmul(upd, b.delta), dadd(dsub(dmul(b.t, Tn), cd.w), pre_d)));
        }
        // backprop_to_vertices (gradients.cpp:99-114): this lane's slot
        double up;
        if (lane == 0) {
          up = sraw > 0.0 ? ds : 0.0;
        } else {
          const double upc = ch == 0 ? upc0 : (ch == 1 ? upc1 : upc2);
          const bool cl = (clamp >> ch) & 1u;
          up = cl ? 0.0 : dmul(dmul(upc, wgt), basis_l);
        }
        if (b.base != cur) {
          if (cur != 0xffffffffu) flush_cell(g, grad, cur, acc, lane);
          cur = b.base;
        }
        const float upf = (float)up;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) acc[kk] = fmaf((float)w[kk], upf, acc[kk]);
        T = Tn;
        if (T < p.eps) {
          done = true;
          break;
        }
      }
    }
    if (cur != 0xffffffffu) flush_cell(g, grad, cur, acc, lane);
  }
}

// ------------------------------------------------------------------ ray ordering
__device__ __forceinline__ uint32_t spread_bits(uint32_t x) {  // 10 bits -> 20 (every other)
  x &= 0x3ff;
  x = (x | (x << 8)) & 0x00ff00ff;
  x = (x | (x << 4)) & 0x0f0f0f0f;
  x = (x | (x << 2)) & 0x33333333;
  x = (x | (x << 1)) & 0x55555555;
  return x;
}

__global__ void k_ray_keys(const int* __restrict__ batch, int n, uint32_t* keys, uint32_t* ids) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t f = (uint32_t)batch[3 * i], x = (uint32_t)batch[3 * i + 1] >> 2,
                 y = (uint32_t)batch[3 * i + 2] >> 2;
  // keyframe in the high bits, Morton order of 4x4-pixel tiles below
  keys[i] = (f << 20) | spread_bits(x) | (spread_bits(y) << 1);
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

}  // namespace

void launch_pixel_order(const int* pixels, int n, uint32_t* keys, uint32_t* ids, uint32_t* keys2,
                        uint32_t* order, void* tmp, size_t tmp_bytes, cudaStream_t s) {
  k_pixel_keys<<<(n + 255) / 256, 256, 0, s>>>(pixels, n, keys, ids);
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, ids, order, n, 0, 32, s);
}

int warp_kernel_blocks() { return 148 * 8; }

void launch_ray_order(const int* batch, int n, uint32_t* keys, uint32_t* ids, uint32_t* keys2,
                      uint32_t* order, void* tmp, size_t tmp_bytes, cudaStream_t s) {
  k_ray_keys<<<(n + 255) / 256, 256, 0, s>>>(batch, n, keys, ids);
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, ids, order, n, 0, 32, s);
}

size_t ray_order_tmp_bytes(int n) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, n, 0, 32);
  return b;
}

void launch_map_forward_w(const DevGrid& g, const DevParams& p, const DevCam& cam,
                          const double4* rgbd, const DevPose* poses, int n_frames,
                          const int* batch, const uint32_t* order, int n, double4* ray_cd,
                          uint8_t* flags, MapPartial* partials, int* queue, int* err,
                          cudaStream_t s) {
  k_map_forward_w<<<warp_kernel_blocks(), kWarpThreads, 0, s>>>(
      g, p, cam, rgbd, poses, n_frames, batch, order, n, ray_cd, flags, partials, queue, err);
}

void launch_map_backward_w(const DevGrid& g, const DevParams& p, const DevCam& cam,
                           const double4* rgbd, const DevPose* poses, const int* batch,
                           const uint32_t* order, int n, const double4* ray_cd,
                           const uint8_t* flags, const MapStats* stats, const int* global_counts,
                           float* grad, double lambda_d, int* queue, cudaStream_t s) {
  k_map_backward_w<<<warp_kernel_blocks(), kWarpThreads, 0, s>>>(
      g, p, cam, rgbd, poses, batch, order, n, ray_cd, flags, stats, global_counts, grad,
      lambda_d, queue);
}

}  // namespace vrf
