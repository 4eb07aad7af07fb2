// Tracking kernels.
//
//   k_pose_fused   one pass per ray: forward render (Ĉ, D̂) then the recompute
//                  march that builds the ray's 4x6 Jacobian of [C; D] w.r.t. the
//                  pose chart [omega; tau] (gradients.cpp:116-143 with unit
//                  upstreams, chart as tracking.cpp:125-128) -> per-CTA partial
//                  J^T J (21) + J^T r (6) + loss + hit count. The reference's
//                  1/m normalisation (tracking.cpp:118-120) is a host-side scale,
//                  so the forward and backward need no global sync between them.
//   k_draw_strat   device pixel draws for the Gauss-Newton tracker: stratified
//                  over a tile grid in Morton order (coherent warps by
//                  construction), redraws inside the tile on invalid depth
//                  (tracking.cpp:147-166 semantics, counter-based RNG).
//   k_pose_reduce2 fixed-order reduction of the CTA partials.
//   k_gn_step      1 thread: damped 6x6 Cholesky (LM) + PosePerturbation update
//                  (pose.hpp:32-41, tracking.hpp:21-26) on the device pose.
// A whole Gauss-Newton frame (iterations x [draw, fused, reduce, step]) is one
// CUDA graph replayed per frame (vrf_pose.cu).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <string>

#include "vrf_internal.h"

namespace vrf {

namespace {

constexpr int kT = 128;

template <typename ShT>
__global__ void __launch_bounds__(kT) k_pose_fused(
    DevGrid g, DevParams p, DevCam cam, const double4* __restrict__ rgbd_base,
    const int* __restrict__ frame_idx, long long npix, const DevPose* __restrict__ pose_ptr,
    const int* __restrict__ pixels, const uint32_t* __restrict__ order, int n, double lambda_p,
    double lambda_d, PosePartial* __restrict__ partials, int* err) {
  __shared__ double s_d[kT / 32][32];
  __shared__ long long s_l[kT / 32];
  __shared__ int s_i[kT / 32];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = (order && t < n) ? (int)order[t] : t;
  const double4* rgbd = rgbd_base + npix * (long long)(*frame_idx);
  double jtj[21], jtr[6], loss = 0.0;
#pragma unroll
  for (int k = 0; k < 21; ++k) jtj[k] = 0.0;
#pragma unroll
  for (int k = 0; k < 6; ++k) jtr[k] = 0.0;
  int hit = 0;
  long long samples = 0;
  const int px = t < n ? pixels[2 * i] : -1, py = t < n ? pixels[2 * i + 1] : -1;
  if (t < n && px >= 0) {
    if (px >= cam.width || py < 0 || py >= cam.height) {
      atomicOr(err, 2);
    } else {
      const DevPose pose = *pose_ptr;
      March m;
      ray_from_pixel(cam, pose, (double)px, (double)py, m);
      double basis[9];
      // One march: compositing and the Jacobian together. dC/dsigma_i =
      // delta_i (c_i T_{i+1} - C + prefix_i) (gradients.cpp:69-97) is linear in
      // the not-yet-known totals C, D, so the per-axis sums split into
      //   J = sum_i [delta_i (c_i T_{i+1} + prefix_i) g_i + w_i Gc_i] - C sum_i delta_i g_i
      // (g_i = gated spatial gradient of sigma) and C is applied after the ray.
      double Jo[4][3], Jd[4][3], Bo[3] = {0, 0, 0}, Bd[3] = {0, 0, 0};
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int a = 0; a < 3; ++a) Jo[r][a] = Jd[r][a] = 0.0;
      double T = 1.0, prefix[3] = {0, 0, 0}, prefix_d = 0.0;
      int count = 0;
      if (!sh_basis(m.d, basis)) {
        atomicOr(err, 1);
      } else if (march_begin(g, p, m)) {
        const double sgn[2] = {-1.0, 1.0};
        ShT bs[9];
#pragma unroll
        for (int mm = 0; mm < 9; ++mm) bs[mm] = ShT(basis[mm]);
        Sample s;
        while (march_next(g, m, s)) {
          // trilerp + SH colour (renderer.cpp:98-112) and the spatial gradients
          // of sigma and the basis-contracted SH channels (voxel_grid.cpp:130-151)
          // from the same 8 corner loads
          const double wx[2] = {dsub(1.0, s.fx), s.fx}, wy[2] = {dsub(1.0, s.fy), s.fy},
                       wz[2] = {dsub(1.0, s.fz), s.fz};
          double sraw = 0.0;
          ShT csh[3] = {ShT(0), ShT(0), ShT(0)};
          double Gs[3] = {0, 0, 0}, Gc[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll 1
          for (int k = 0; k < 8; ++k) {
            const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
            const double wk = dmul(dmul(wx[dx], wy[dy]), wz[dz]);
            const double dw[3] = {sgn[dx] * wy[dy] * wz[dz] * g.inv_voxel,
                                  wx[dx] * sgn[dy] * wz[dz] * g.inv_voxel,
                                  wx[dx] * wy[dy] * sgn[dz] * g.inv_voxel};
            const float4* vp4 = g.payload + (size_t)corner_index(g, s.base, k) * kVec4PerVertex;
            float v[28];
#pragma unroll
            for (int j = 0; j < kVec4PerVertex; ++j) {
              const float4 a = __ldg(vp4 + j);
              v[4 * j] = a.x;
              v[4 * j + 1] = a.y;
              v[4 * j + 2] = a.z;
              v[4 * j + 3] = a.w;
            }
            sraw = dadd(sraw, dmul(wk, (double)v[0]));
            double shd[3];
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
              ShT acc = ShT(0);
#pragma unroll
              for (int mm = 0; mm < 9; ++mm) acc = fma(bs[mm], (ShT)v[1 + ch * 9 + mm], acc);
              shd[ch] = (double)acc;
              csh[ch] = fma(ShT(wk), acc, csh[ch]);
            }
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              Gs[a] = fma(dw[a], (double)v[0], Gs[a]);
#pragma unroll
              for (int ch = 0; ch < 3; ++ch) Gc[ch][a] = fma(dw[a], shd[ch], Gc[ch][a]);
            }
          }
          double c[3];
          bool clamped[3];
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const double v = 0.5 + (double)csh[ch];
            clamped[ch] = (v <= 0.0 || v >= 1.0);
            c[ch] = (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v);
          }
          const double sigma = (sraw < 0.0) ? 0.0 : sraw;
          const double decay = exp(dmul(-sigma, s.delta));
          const double wgt = dmul(T, dsub(1.0, decay));
          const double T_next = dmul(T, decay);
          ++count;
          double dsig[4];
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            prefix[ch] = dadd(prefix[ch], dmul(c[ch], wgt));
            dsig[ch] = s.delta * (c[ch] * T_next + prefix[ch]);
          }
          prefix_d = dadd(prefix_d, dmul(s.t, wgt));
          dsig[3] = s.delta * (s.t * T_next + prefix_d);
          const bool sgate = sraw > 0.0;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const double gs = sgate ? s.delta * Gs[a] : 0.0;
            Bo[a] += gs;
            Bd[a] = fma(s.t, gs, Bd[a]);
          }
#pragma unroll
          for (int r = 0; r < 4; ++r) {
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              double gv = sgate ? dsig[r] * Gs[a] : 0.0;
              if (r < 3 && !clamped[r]) gv += wgt * Gc[r][a];
              Jo[r][a] += gv;
              Jd[r][a] = fma(s.t, gv, Jd[r][a]);
            }
          }
          T = T_next;
          if (T < p.eps) break;
        }
      }
      if (count > 0) {
        hit = 1;
        samples = count;
        const double4 tg = rgbd[(long long)py * cam.width + px];
        // Ĉ = prefix, D̂ = prefix_d (renderer.cpp:120-126, same accumulation order)
        const double C[4] = {prefix[0], prefix[1], prefix[2], prefix_d};
        const double res[4] = {dsub(C[0], tg.x), dsub(C[1], tg.y), dsub(C[2], tg.z),
                               dsub(C[3], tg.w)};
        // tracking.cpp:117: lambda_p |cres|^2 + lambda_d dres^2
        loss = dadd(dmul(lambda_p, dadd(dadd(dmul(res[0], res[0]), dmul(res[1], res[1])),
                                        dmul(res[2], res[2]))),
                    dmul(dmul(lambda_d, res[3]), res[3]));
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            Jo[r][a] -= C[r] * Bo[a];
            Jd[r][a] -= C[r] * Bd[a];
          }
        // chart (tracking.cpp:125-128): tau <- dL/do, omega <- d x (dL/dd - d (d.dL/dd))
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const double dd = dot3(m.d, Jd[r]);
          double gp[3], om[3];
          for (int a = 0; a < 3; ++a) gp[a] = Jd[r][a] - m.d[a] * dd;
          cross3(m.d, gp, om);
          const double J[6] = {om[0], om[1], om[2], Jo[r][0], Jo[r][1], Jo[r][2]};
          const double lam = r < 3 ? lambda_p : lambda_d;
          int idx = 0;
#pragma unroll
          for (int a = 0; a < 6; ++a) {
#pragma unroll
            for (int b = a; b < 6; ++b) jtj[idx++] += lam * J[a] * J[b];
            jtr[a] += lam * J[a] * res[r];
          }
        }
      }
    }
  }
  // CTA reduction in a fixed order (warp butterflies, then warps in order)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double vals[28];
#pragma unroll
  for (int k = 0; k < 21; ++k) vals[k] = jtj[k];
#pragma unroll
  for (int k = 0; k < 6; ++k) vals[21 + k] = jtr[k];
  vals[27] = loss;
#pragma unroll
  for (int k = 0; k < 28; ++k) {
    double v = warp_sum(vals[k]);
    if (lane == 0) s_d[wid][k] = v;
  }
  long long sw = warp_sum(samples);
  int hw = warp_sum(hit);
  if (lane == 0) {
    s_l[wid] = sw;
    s_i[wid] = hw;
  }
  __syncthreads();
  if (threadIdx.x < 28) {
    double acc = 0.0;
    for (int w = 0; w < kT / 32; ++w) acc += s_d[w][threadIdx.x];
    PosePartial* out = partials + blockIdx.x;
    if (threadIdx.x < 21)
      out->jtj[threadIdx.x] = acc;
    else if (threadIdx.x < 27)
      out->jtr[threadIdx.x - 21] = acc;
    else
      out->loss = acc;
  }
  if (threadIdx.x == 32) {
    long long sl = 0;
    int sm = 0;
    for (int w = 0; w < kT / 32; ++w) {
      sl += s_l[w];
      sm += s_i[w];
    }
    partials[blockIdx.x].samples = sl;
    partials[blockIdx.x].m = sm;
    partials[blockIdx.x].bad = 0;
  }
}

// ------------------------------------------------------------------ sample-parallel
// One warp per ray; lane l owns schedule segment k0 + l of each 32-segment chunk,
// so a ray's samples are shaded in parallel and the front-to-back recurrences
// become warp scans: T = carry * prefix product of exp(-sigma delta),
// prefix[ch] = carry + prefix sum of c w (gradients.cpp:69-97). Termination is
// the first lane whose update drives T below eps (renderer.cpp:127-131).
__device__ __forceinline__ double scan_prod(double v, int lane) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double o = __shfl_up_sync(0xffffffffu, v, off);
    if (lane >= off) v *= o;
  }
  return v;
}
// Exclusive prefix product (lane 0 -> 1).
__device__ __forceinline__ double excl_prod(double v, int lane) {
  const double incl = scan_prod(v, lane);
  const double e = __shfl_up_sync(0xffffffffu, incl, 1);
  return lane == 0 ? 1.0 : e;
}
__device__ __forceinline__ double scan_sum(double v, int lane) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double o = __shfl_up_sync(0xffffffffu, v, off);
    if (lane >= off) v += o;
  }
  return v;
}

struct LaneSample {
  bool valid;
  Sample s;
  double w[8];
  Shade sh;
  double decay, alpha;
};

// Locates + shades this lane's segment of the chunk; returns the chunk's next
// start (empty-block jump taken from the last lane).
template <typename ShT>
__device__ __forceinline__ long long chunk_samples(const DevGrid& g, March& m, long long k0,
                                                   const double basis[9], int lane,
                                                   LaneSample& ls) {
  const long long k = k0 + lane;
  ls.valid = false;
  long long next = k0 + 32;
  if (k < m.nseg) {
    const double s0 = dadd(m.lo, dmul((double)k, m.step));
    const double s0s = dadd(s0, m.step);
    const double s1 = (m.hi < s0s) ? m.hi : s0s;
    const double len = dsub(s1, s0);
    if (len >= 1e-12) {
      const double tm = dmul(0.5, dadd(s0, s1));
      const double p[3] = {dadd(m.o[0], dmul(tm, m.d[0])), dadd(m.o[1], dmul(tm, m.d[1])),
                           dadd(m.o[2], dmul(tm, m.d[2]))};
      if (locate(g, p, ls.s)) {
        if (cell_active(g, ls.s.cell)) {
          ls.valid = true;
          ls.s.t = tm;
          ls.s.delta = len;
        } else if (lane == 31 && !block_active(g, ls.s.cx, ls.s.cy, ls.s.cz)) {
          March mm = m;
          mm.k = k + 1;
          next = skip_empty_block(g, mm, ls.s);
        }
      }
    }
  }
  next = __shfl_sync(0xffffffffu, next, 31);
  if (ls.valid) {
    corner_weights(ls.s, ls.w);
    shade<ShT>(g, ls.s, ls.w, basis, ls.sh);
    const double sigma = (ls.sh.sigma_raw < 0.0) ? 0.0 : ls.sh.sigma_raw;
    ls.decay = exp(dmul(-sigma, ls.s.delta));
    ls.alpha = dsub(1.0, ls.decay);
  } else {
    ls.decay = 1.0;
    ls.alpha = 0.0;
  }
  return next > k0 + 32 ? next : k0 + 32;
}

template <typename ShT>
__global__ void __launch_bounds__(kT) k_pose_warp(
    DevGrid g, DevParams p, DevCam cam, const double4* __restrict__ rgbd_base,
    const int* __restrict__ frame_idx, long long npix, const DevPose* __restrict__ pose_ptr,
    const int* __restrict__ pixels, const uint32_t* __restrict__ order, int n, double lambda_p,
    double lambda_d, PosePartial* __restrict__ partials, int* err) {
  __shared__ double s_d[kT / 32][28];
  __shared__ long long s_l[kT / 32];
  __shared__ int s_i[kT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int warps_total = gridDim.x * (kT / 32);
  const double4* rgbd = rgbd_base + npix * (long long)(*frame_idx);
  const DevPose pose = *pose_ptr;
  double jtj[21], jtr[6], loss = 0.0;  // lane 0 accumulates the warp's rays
#pragma unroll
  for (int k = 0; k < 21; ++k) jtj[k] = 0.0;
#pragma unroll
  for (int k = 0; k < 6; ++k) jtr[k] = 0.0;
  long long samples = 0;
  int hits = 0;
  for (int q = blockIdx.x * (kT / 32) + wid; q < n; q += warps_total) {
    const int i = order ? (int)order[q] : q;
    const int px = pixels[2 * i], py = pixels[2 * i + 1];
    if (px < 0) continue;
    if (px >= cam.width || py < 0 || py >= cam.height) {
      if (lane == 0) atomicOr(err, 2);
      continue;
    }
    March m;
    ray_from_pixel(cam, pose, (double)px, (double)py, m);
    double basis[9];
    if (!sh_basis(m.d, basis)) {
      if (lane == 0) atomicOr(err, 1);
      continue;
    }
    if (!march_begin(g, p, m)) continue;
    // ---- forward: C, D, count
    double Tc = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0, D = 0.0;
    int count = 0;
    for (long long k0 = 0; k0 < m.nseg;) {
      LaneSample ls;
      const long long next = chunk_samples<ShT>(g, m, k0, basis, lane, ls);
      const unsigned vm = __ballot_sync(0xffffffffu, ls.valid);
      if (vm) {
        const double Tb = Tc * excl_prod(ls.decay, lane);
        const double Ta = dmul(Tb, ls.decay);
        const unsigned tm = __ballot_sync(0xffffffffu, ls.valid && Ta < p.eps);
        const unsigned keep = tm ? vm & ((2u << (__ffs(tm) - 1)) - 1u) : vm;
        const bool kept = (keep >> lane) & 1u;
        const double wgt = kept ? dmul(Tb, ls.alpha) : 0.0;
        C0 += warp_sum(kept ? wgt * ls.sh.c[0] : 0.0);
        C1 += warp_sum(kept ? wgt * ls.sh.c[1] : 0.0);
        C2 += warp_sum(kept ? wgt * ls.sh.c[2] : 0.0);
        D += warp_sum(kept ? wgt * ls.s.t : 0.0);
        count += __popc(keep);
        Tc = __shfl_sync(0xffffffffu, Ta, 31 - __clz(keep));
        if (tm) break;
      }
      k0 = next;
    }
    if (count == 0) continue;
    ++hits;
    samples += count;
    const double4 tg = rgbd[(long long)py * cam.width + px];
    const double C[3] = {C0, C1, C2};
    const double res[4] = {dsub(C0, tg.x), dsub(C1, tg.y), dsub(C2, tg.z), dsub(D, tg.w)};
    loss += dadd(dmul(lambda_p, dadd(dadd(dmul(res[0], res[0]), dmul(res[1], res[1])),
                                     dmul(res[2], res[2]))),
                 dmul(dmul(lambda_d, res[3]), res[3]));
    // ---- backward: per-lane Jacobian contributions, recompute march
    double Jo[4][3], Jd[4][3];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int a = 0; a < 3; ++a) Jo[r][a] = Jd[r][a] = 0.0;
    double Tcb = 1.0, pre[4] = {0.0, 0.0, 0.0, 0.0};
    march_begin(g, p, m);
    const double sgn[2] = {-1.0, 1.0};
    for (long long k0 = 0; k0 < m.nseg;) {
      LaneSample ls;
      const long long next = chunk_samples<ShT>(g, m, k0, basis, lane, ls);
      const unsigned vm = __ballot_sync(0xffffffffu, ls.valid);
      if (vm) {
        const double Tb = Tcb * excl_prod(ls.decay, lane);
        const double Ta = dmul(Tb, ls.decay);
        const unsigned tm = __ballot_sync(0xffffffffu, ls.valid && Ta < p.eps);
        const unsigned keep = tm ? vm & ((2u << (__ffs(tm) - 1)) - 1u) : vm;
        const bool kept = (keep >> lane) & 1u;
        const double wgt = kept ? dmul(Tb, ls.alpha) : 0.0;
        double prefix[4];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) prefix[ch] = pre[ch] + scan_sum(kept ? ls.sh.c[ch] * wgt : 0.0, lane);
        prefix[3] = pre[3] + scan_sum(kept ? ls.s.t * wgt : 0.0, lane);
        if (kept) {
          double dsig[4];
#pragma unroll
          for (int ch = 0; ch < 3; ++ch)
            dsig[ch] = ls.s.delta * ((ls.sh.c[ch] * Ta - C[ch]) + prefix[ch]);
          dsig[3] = ls.s.delta * ((ls.s.t * Ta - D) + prefix[3]);
          const double wx[2] = {1.0 - ls.s.fx, ls.s.fx}, wy[2] = {1.0 - ls.s.fy, ls.s.fy},
                       wz[2] = {1.0 - ls.s.fz, ls.s.fz};
          double Gs[3] = {0, 0, 0}, Gc[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll 1
          for (int k = 0; k < 8; ++k) {
            const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
            const double dw[3] = {sgn[dx] * wy[dy] * wz[dz] * g.inv_voxel,
                                  wx[dx] * sgn[dy] * wz[dz] * g.inv_voxel,
                                  wx[dx] * wy[dy] * sgn[dz] * g.inv_voxel};
            const float4* vp4 =
                g.payload + (size_t)corner_index(g, ls.s.base, k) * kVec4PerVertex;
            float v[28];
#pragma unroll
            for (int j = 0; j < kVec4PerVertex; ++j) {
              const float4 a = __ldg(vp4 + j);
              v[4 * j] = a.x;
              v[4 * j + 1] = a.y;
              v[4 * j + 2] = a.z;
              v[4 * j + 3] = a.w;
            }
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
              ShT acc = ShT(0);
#pragma unroll
              for (int mm = 0; mm < 9; ++mm)
                acc = fma((ShT)basis[mm], (ShT)v[1 + ch * 9 + mm], acc);
#pragma unroll
              for (int a = 0; a < 3; ++a) Gc[ch][a] = fma(dw[a], (double)acc, Gc[ch][a]);
            }
#pragma unroll
            for (int a = 0; a < 3; ++a) Gs[a] = fma(dw[a], (double)v[0], Gs[a]);
          }
          const bool sgate = ls.sh.sigma_raw > 0.0;
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              double gv = sgate ? dsig[r] * Gs[a] : 0.0;
              if (r < 3 && !ls.sh.clamped[r]) gv += wgt * Gc[r][a];
              Jo[r][a] += gv;
              Jd[r][a] = fma(ls.s.t, gv, Jd[r][a]);
            }
        }
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) pre[ch] = __shfl_sync(0xffffffffu, prefix[ch], 31);
        Tcb = __shfl_sync(0xffffffffu, Ta, 31 - __clz(keep));
        if (tm) break;
      }
      k0 = next;
    }
    // reduce the lane contributions, chart (tracking.cpp:125-128), accumulate J^T J
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        Jo[r][a] = warp_sum(Jo[r][a]);
        Jd[r][a] = warp_sum(Jd[r][a]);
      }
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const double dd = dot3(m.d, Jd[r]);
        double gp[3], om[3];
        for (int a = 0; a < 3; ++a) gp[a] = Jd[r][a] - m.d[a] * dd;
        cross3(m.d, gp, om);
        const double J[6] = {om[0], om[1], om[2], Jo[r][0], Jo[r][1], Jo[r][2]};
        const double lam = r < 3 ? lambda_p : lambda_d;
        int idx = 0;
#pragma unroll
        for (int a = 0; a < 6; ++a) {
#pragma unroll
          for (int b = a; b < 6; ++b) jtj[idx++] += lam * J[a] * J[b];
          jtr[a] += lam * J[a] * res[r];
        }
      }
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 21; ++k) s_d[wid][k] = jtj[k];
#pragma unroll
    for (int k = 0; k < 6; ++k) s_d[wid][21 + k] = jtr[k];
    s_d[wid][27] = loss;
    s_l[wid] = samples;
    s_i[wid] = hits;
  }
  __syncthreads();
  if (threadIdx.x < 28) {
    double acc = 0.0;
    for (int w = 0; w < kT / 32; ++w) acc += s_d[w][threadIdx.x];
    PosePartial* out = partials + blockIdx.x;
    if (threadIdx.x < 21)
      out->jtj[threadIdx.x] = acc;
    else if (threadIdx.x < 27)
      out->jtr[threadIdx.x - 21] = acc;
    else
      out->loss = acc;
  }
  if (threadIdx.x == 32) {
    long long sl = 0;
    int sm = 0;
    for (int w = 0; w < kT / 32; ++w) {
      sl += s_l[w];
      sm += s_i[w];
    }
    partials[blockIdx.x].samples = sl;
    partials[blockIdx.x].m = sm;
    partials[blockIdx.x].bad = 0;
  }
}

__global__ void __launch_bounds__(64) k_pose_reduce2(const PosePartial* __restrict__ parts,
                                                     int nparts, PosePartial* out) {
  const int v = threadIdx.x;
  if (v < 28) {
    double acc = 0.0;
    for (int k = 0; k < nparts; ++k)
      acc += v < 21 ? parts[k].jtj[v] : (v < 27 ? parts[k].jtr[v - 21] : parts[k].loss);
    if (v < 21)
      out->jtj[v] = acc;
    else if (v < 27)
      out->jtr[v - 21] = acc;
    else
      out->loss = acc;
  } else if (v == 32) {
    long long s = 0;
    int m = 0;
    for (int k = 0; k < nparts; ++k) {
      s += parts[k].samples;
      m += parts[k].m;
    }
    out->samples = s;
    out->m = m;
    out->bad = 0;
  }
}

// ---- counter-based RNG (splitmix64 of a packed counter)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t compact_bits(uint32_t x) {  // inverse of spread (even bits)
  x &= 0x55555555;
  x = (x | (x >> 1)) & 0x33333333;
  x = (x | (x >> 2)) & 0x0f0f0f0f;
  x = (x | (x >> 4)) & 0x00ff00ff;
  x = (x | (x >> 8)) & 0x0000ffff;
  return x;
}

// Stratified valid-depth draws: thread t owns tile (Morton decode of t) of a
// tiles_x x tiles_y grid over the image, draws uniformly inside it and redraws
// (max_redraws attempts) until the depth is valid; -1 marks a dropped pixel.
__global__ void k_draw_strat(const double4* __restrict__ rgbd_base,
                             const int* __restrict__ frame_idx, long long npix, int width,
                             int height, int tiles_log2, int max_redraws,
                             const unsigned long long* __restrict__ seed, int iteration,
                             int* __restrict__ pixels, int n) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double4* rgbd = rgbd_base + npix * (long long)(*frame_idx);
  const int tiles = 1 << tiles_log2;
  const int tx = (int)compact_bits((uint32_t)t), ty = (int)compact_bits((uint32_t)t >> 1);
  int px = -1, py = -1;
  if (tx < tiles && ty < tiles) {
    const int x0 = (int)((long long)tx * width / tiles), x1 = (int)((long long)(tx + 1) * width / tiles);
    const int y0 = (int)((long long)ty * height / tiles), y1 = (int)((long long)(ty + 1) * height / tiles);
    const int w = x1 - x0, h = y1 - y0;
    if (w > 0 && h > 0) {
      for (int a = 0; a < max_redraws; ++a) {
        const uint64_t r = mix64(*seed ^ mix64(((uint64_t)iteration << 40) ^ ((uint64_t)t << 8) ^
                                               (uint64_t)a));
        const int cx = x0 + (int)(((r & 0xffffffffULL) * (uint64_t)w) >> 32);
        const int cy = y0 + (int)(((r >> 32) * (uint64_t)h) >> 32);
        if (rgbd[(long long)cy * width + cx].w > 0.0) {
          px = cx;
          py = cy;
          break;
        }
      }
    }
  }
  pixels[2 * t] = px;
  pixels[2 * t + 1] = py;
}

// ---- device pose update (pose.hpp:32-41, tracking.hpp:21-26)
__device__ void d_quat_normalize(double q[4]) {
  const double n2 = (q[1] * q[1] + q[3] * q[3]) + (q[2] * q[2] + q[0] * q[0]);
  if (n2 > 0.0) {
    const double s = sqrt(n2);
    for (int i = 0; i < 4; ++i) q[i] /= s;
  }
}

__global__ void k_gn_step(const PosePartial* __restrict__ ne, DevPose* pose, double damping,
                          double* hist, int iteration) {
  if (threadIdx.x != 0) return;
  const PosePartial r = *ne;
  hist[2 * iteration] = r.m > 0 ? r.loss / r.m : 0.0;
  hist[2 * iteration + 1] = r.m;
  if (r.m == 0) return;
  double A[6][6];
  int idx = 0;
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b) A[a][b] = A[b][a] = r.jtj[idx++];
  for (int a = 0; a < 6; ++a) A[a][a] += damping * A[a][a] + 1e-12;
  double L[6][6] = {};
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = A[i][j];
      for (int k = 0; k < j; ++k) s -= L[i][k] * L[j][k];
      if (i == j) {
        if (!(s > 0.0)) return;
        L[i][i] = sqrt(s);
      } else {
        L[i][j] = s / L[j][j];
      }
    }
  double y[6], x[6];
  for (int i = 0; i < 6; ++i) {
    double s = -r.jtr[i];
    for (int k = 0; k < i; ++k) s -= L[i][k] * y[k];
    y[i] = s / L[i][i];
  }
  for (int i = 5; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < 6; ++k) s -= L[k][i] * x[k];
    x[i] = s / L[i][i];
  }
  // exp_so3(omega) * q, renormalised; t += tau
  double e[4];
  const double angle = sqrt((x[0] * x[0] + x[1] * x[1]) + x[2] * x[2]);
  if (angle < 1e-8) {
    e[0] = 1.0;
    e[1] = 0.5 * x[0];
    e[2] = 0.5 * x[1];
    e[3] = 0.5 * x[2];
    d_quat_normalize(e);
  } else {
    const double ha = 0.5 * angle, sh = sin(ha) / angle;
    e[0] = cos(ha);
    e[1] = sh * x[0];
    e[2] = sh * x[1];
    e[3] = sh * x[2];
  }
  DevPose P = *pose;
  const double* b = P.q;
  double q[4] = {e[0] * b[0] - e[1] * b[1] - e[2] * b[2] - e[3] * b[3],
                 e[0] * b[1] + e[1] * b[0] + e[2] * b[3] - e[3] * b[2],
                 e[0] * b[2] + e[2] * b[0] + e[3] * b[1] - e[1] * b[3],
                 e[0] * b[3] + e[3] * b[0] + e[1] * b[2] - e[2] * b[1]};
  d_quat_normalize(q);
  for (int i = 0; i < 4; ++i) P.q[i] = q[i];
  for (int a = 0; a < 3; ++a) P.t[a] += x[3 + a];
  *pose = P;
}

}  // namespace

// Thread-per-ray by default (r01: 13.4 ms vs 16.0 ms per 1200x680 GN frame);
// VRF_POSE_KERNEL=warp selects the sample-parallel warp-per-ray kernel (A/B).
static bool pose_warp() {
  static const bool w = [] {
    const char* e = getenv("VRF_POSE_KERNEL");
    return e && std::string(e) == "warp";
  }();
  return w;
}

int pose_fused_blocks(int n) {
  if (pose_warp()) return std::max(1, std::min((n + kT / 32 - 1) / (kT / 32), 148 * 32));
  return (n + kT - 1) / kT;
}

void launch_pose_fused(bool fp64_sh, const DevGrid& g, const DevParams& p, const DevCam& cam,
                       const double4* rgbd_base, const int* frame_idx, long long npix,
                       const DevPose* pose, const int* pixels, const uint32_t* order, int n,
                       double lambda_p, double lambda_d, PosePartial* partials, int* err,
                       cudaStream_t s) {
  if (n <= 0) return;
  if (pose_warp()) {
    if (fp64_sh)
      k_pose_warp<double><<<pose_fused_blocks(n), kT, 0, s>>>(
          g, p, cam, rgbd_base, frame_idx, npix, pose, pixels, order, n, lambda_p, lambda_d,
          partials, err);
    else
      k_pose_warp<float><<<pose_fused_blocks(n), kT, 0, s>>>(
          g, p, cam, rgbd_base, frame_idx, npix, pose, pixels, order, n, lambda_p, lambda_d,
          partials, err);
    return;
  }
  if (fp64_sh)
    k_pose_fused<double><<<pose_fused_blocks(n), kT, 0, s>>>(
        g, p, cam, rgbd_base, frame_idx, npix, pose, pixels, order, n, lambda_p, lambda_d,
        partials, err);
  else
    k_pose_fused<float><<<pose_fused_blocks(n), kT, 0, s>>>(
        g, p, cam, rgbd_base, frame_idx, npix, pose, pixels, order, n, lambda_p, lambda_d,
        partials, err);
}

void launch_pose_reduce2(const PosePartial* partials, int nparts, PosePartial* out,
                         cudaStream_t s) {
  k_pose_reduce2<<<1, 64, 0, s>>>(partials, nparts, out);
}

void launch_draw_strat(const double4* rgbd_base, const int* frame_idx, long long npix, int width,
                       int height, int tiles_log2, int max_redraws,
                       const unsigned long long* seed, int iteration, int* pixels, int n,
                       cudaStream_t s) {
  k_draw_strat<<<(n + 255) / 256, 256, 0, s>>>(rgbd_base, frame_idx, npix, width, height,
                                               tiles_log2, max_redraws, seed, iteration, pixels,
                                               n);
}

void launch_gn_step(const PosePartial* ne, DevPose* pose, double damping, double* hist,
                    int iteration, cudaStream_t s) {
  k_gn_step<<<1, 32, 0, s>>>(ne, pose, damping, hist, iteration);
}

}  // namespace vrf
