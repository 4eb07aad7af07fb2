// Tracking kernels.
//
//   k_pose_group   one march per ray, 8 lanes per ray (one trilinear corner
//                  each): composites Ĉ, D̂ and builds the ray's 4x6 Jacobian of
//                  [C; D] w.r.t. the pose chart [omega; tau] (gradients.cpp:116-143
//                  with unit upstreams, chart as tracking.cpp:125-128) -> per-CTA
//                  partial J^T J (21) + J^T r (6) + loss + hit count. The
//                  reference's 1/m normalisation (tracking.cpp:118-120) is a
//                  host-side scale, so no global sync is needed inside the pass.
//                  <double>: FP64 SH and Jacobian partials — the reference-parity
//                  path (pose_gradient, track_frame). <float>: the checker of the
//                  GN kernel below (same arithmetic, group-independent control).
//   k_pose_group_u the Gauss-Newton path's pose kernel: the same per-ray
//                  arithmetic as k_pose_group<float>, warp-synchronous control.
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
#include <type_traits>

#include "vrf_internal.h"

namespace vrf {

namespace {

#ifndef VRF_POSE_KT
#define VRF_POSE_KT 128  // threads per CTA of the pose kernels (A/B knob)
#endif
constexpr int kT = VRF_POSE_KT;
static_assert(kT >= 64 && kT % 32 == 0, "the CTA reduction uses threads 0-32");

// ------------------------------------------------------------------ corner-parallel
// LPR lanes per ray (LPR = 8: one trilinear corner per lane). The tracking batch
// is small (16,384 rays = 111 threads per SM at one thread per ray), so the
// thread-per-ray kernel is latency bound; splitting each sample's 8 corner
// gathers and SH contractions across LPR lanes gives LPR x the warps in flight.
// Every lane of a group carries the same ray state (march, T, prefix), so the
// loop is group-uniform and group-masked shuffles are safe:
//   * sigma_raw: the 8 products w_k v_k[0] are gathered to every lane and
//     summed in corner order k = 0..7 — the reference's exact FP64 order, so
//     T and termination stay bit-identical (renderer.cpp:113-131);
//   * colour: the per-lane basis-contracted partials are gathered and summed in
//     lane order (identical on every lane);
//   * the Jacobian terms are linear in each corner's spatial gradients, so every
//     lane accumulates its own partial Jo / Jd / B and the group reduces once
//     per ray.
// MINB = 3 CTAs/SM (168 registers). r01: capping registers for more warps lost
// (4 CTAs, 128 regs + spills: 494 frames/s; 5: 460; 7: 458; 3: 525). r01 also
// measured 4 lanes per ray, a thread-per-ray kernel and a segment-by-segment
// march here; all were slower and were removed in r02.
template <typename ShT, int MINB = 3>
__global__ void __launch_bounds__(kT, MINB) k_pose_group(
    DevGrid g, DevParams p, DevCam cam, const double4* __restrict__ rgbd_base,
    const int* __restrict__ frame_idx, long long npix, const DevPose* __restrict__ pose_ptr,
    const int* __restrict__ pixels, const uint32_t* __restrict__ order, int n, double lambda_p,
    double lambda_d, PosePartial* __restrict__ partials, int* err) {
  constexpr int LPR = 8, CPL = 1;  // lanes per ray, corners per lane
  __shared__ double s_d[kT / 32][32];
  __shared__ long long s_l[kT / 32];
  __shared__ int s_i[kT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int sub = lane & (LPR - 1), gbase = lane & ~(LPR - 1);
  const unsigned gmask = 0xffu << gbase;
  const int t = blockIdx.x * (kT / LPR) + threadIdx.x / LPR;
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
      if (sub == 0) atomicOr(err, 2);
    } else {
      const DevPose pose = *pose_ptr;
      March m;
      ray_from_pixel(cam, pose, (double)px, (double)py, m);
      double basis[9];
      // Jacobian partials: fp32 on the fast (GN) path, fp64 on the parity path
      using JT = typename std::conditional<sizeof(ShT) == 4, float, double>::type;
      JT Jo[4][3], Jd[4][3], Bo[3] = {0, 0, 0}, Bd[3] = {0, 0, 0};
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int a = 0; a < 3; ++a) Jo[r][a] = Jd[r][a] = JT(0);
      double T = 1.0, prefix[3] = {0, 0, 0}, prefix_d = 0.0;
      int count = 0;
      if (!sh_basis(m.d, basis)) {
        if (sub == 0) atomicOr(err, 1);
      } else if (march_begin(g, p, m)) {
        const double sgn[2] = {-1.0, 1.0};
        ShT bs[9];
#pragma unroll
        for (int mm = 0; mm < 9; ++mm) bs[mm] = ShT(basis[mm]);
        Sample s;
        GroupMarch<LPR> gm;
        while (gm.next(g, m, s, sub, gbase, gmask)) {
          const double wx[2] = {dsub(1.0, s.fx), s.fx}, wy[2] = {dsub(1.0, s.fy), s.fy},
                       wz[2] = {dsub(1.0, s.fz), s.fz};
          double pk[CPL];
          ShT cp[3] = {ShT(0), ShT(0), ShT(0)};
          JT Gs[3] = {0, 0, 0}, Gc[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
          const JT wxj[2] = {JT(wx[0]), JT(wx[1])}, wyj[2] = {JT(wy[0]), JT(wy[1])},
                   wzj[2] = {JT(wz[0]), JT(wz[1])};
          const JT iv = JT(g.inv_voxel);
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            const int k = sub + LPR * c;
            const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
            const double wk = dmul(dmul(wx[dx], wy[dy]), wz[dz]);
            const JT dw[3] = {JT(sgn[dx]) * wyj[dy] * wzj[dz] * iv,
                              wxj[dx] * JT(sgn[dy]) * wzj[dz] * iv,
                              wxj[dx] * wyj[dy] * JT(sgn[dz]) * iv};
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
            pk[c] = dmul(wk, (double)v[0]);
            JT shd[3];
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
              ShT acc = ShT(0);
#pragma unroll
              for (int mm = 0; mm < 9; ++mm) acc = fma(bs[mm], (ShT)v[1 + ch * 9 + mm], acc);
              shd[ch] = JT(acc);
              cp[ch] = fma(ShT(wk), acc, cp[ch]);
            }
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              Gs[a] = fma(dw[a], JT(v[0]), Gs[a]);
#pragma unroll
              for (int ch = 0; ch < 3; ++ch) Gc[ch][a] = fma(dw[a], shd[ch], Gc[ch][a]);
            }
          }
          // sigma_raw in corner order k = c * LPR + j (the reference's order)
          double sraw = 0.0;
#pragma unroll
          for (int c = 0; c < CPL; ++c)
#pragma unroll
            for (int j = 0; j < LPR; ++j) sraw = dadd(sraw, __shfl_sync(gmask, pk[c], gbase + j));
          ShT csum[3] = {ShT(0), ShT(0), ShT(0)};
#pragma unroll
          for (int j = 0; j < LPR; ++j)
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) csum[ch] += __shfl_sync(gmask, cp[ch], gbase + j);
          double c[3];
          bool clamped[3];
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const double v = 0.5 + (double)csum[ch];
            clamped[ch] = (v <= 0.0 || v >= 1.0);
            c[ch] = (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v);
          }
          const double sigma = (sraw < 0.0) ? 0.0 : sraw;
          const double decay = exp(dmul(-sigma, s.delta));
          const double wgt = dmul(T, dsub(1.0, decay));
          const double T_next = dmul(T, decay);
          ++count;
          JT dsig[4];
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            prefix[ch] = dadd(prefix[ch], dmul(c[ch], wgt));
            dsig[ch] = JT(s.delta * (c[ch] * T_next + prefix[ch]));
          }
          prefix_d = dadd(prefix_d, dmul(s.t, wgt));
          dsig[3] = JT(s.delta * (s.t * T_next + prefix_d));
          const bool sgate = sraw > 0.0;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const JT gs = sgate ? JT(s.delta) * Gs[a] : JT(0);
            Bo[a] += gs;
            Bd[a] = fma(JT(s.t), gs, Bd[a]);
          }
#pragma unroll
          for (int r = 0; r < 4; ++r) {
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              JT gv = sgate ? dsig[r] * Gs[a] : JT(0);
              if (r < 3 && !clamped[r]) gv += JT(wgt) * Gc[r][a];
              Jo[r][a] += gv;
              Jd[r][a] = fma(JT(s.t), gv, Jd[r][a]);
            }
          }
          T = T_next;
          if (T < p.eps) break;
        }
      }
      // group reduction of the lane partials (fixed butterfly order)
#pragma unroll
      for (int off = LPR / 2; off > 0; off >>= 1) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          Bo[a] += __shfl_xor_sync(gmask, Bo[a], off);
          Bd[a] += __shfl_xor_sync(gmask, Bd[a], off);
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            Jo[r][a] += __shfl_xor_sync(gmask, Jo[r][a], off);
            Jd[r][a] += __shfl_xor_sync(gmask, Jd[r][a], off);
          }
        }
      }
      if (count > 0 && sub == 0) {
        hit = 1;
        samples = count;
        const double4 tg = rgbd[(long long)py * cam.width + px];
        const double C[4] = {prefix[0], prefix[1], prefix[2], prefix_d};
        const double res[4] = {dsub(C[0], tg.x), dsub(C[1], tg.y), dsub(C[2], tg.z),
                               dsub(C[3], tg.w)};
        loss = dadd(dmul(lambda_p, dadd(dadd(dmul(res[0], res[0]), dmul(res[1], res[1])),
                                        dmul(res[2], res[2]))),
                    dmul(dmul(lambda_d, res[3]), res[3]));
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          double jo[3], jd[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            jo[a] = (double)Jo[r][a] - C[r] * (double)Bo[a];
            jd[a] = (double)Jd[r][a] - C[r] * (double)Bd[a];
          }
          // chart (tracking.cpp:125-128): tau <- dL/do, omega <- d x (dL/dd - d (d.dL/dd))
          const double dd = dot3(m.d, jd);
          double gp[3], om[3];
          for (int a = 0; a < 3; ++a) gp[a] = jd[a] - m.d[a] * dd;
          cross3(m.d, gp, om);
          const double J[6] = {om[0], om[1], om[2], jo[0], jo[1], jo[2]};
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

// Warp-synchronous k_pose_group for the GN path (fp32 SH, 8 lanes per ray).
// In k_pose_group the four ray groups of a warp march independently, so the
// group-masked ballots of GroupMarch run while the groups are diverged and the
// compiler emulates them (WARPSYNC.COLLECTIVE; ~17% of the kernel's stall
// samples, r01). Here the groups advance in lockstep rounds: in each round a
// group without a pending sample evaluates its next 8 segments, then every
// group with a pending sample shades one. All ballots and shuffles run with
// the full warp mask. The arithmetic (sample order, sigma in corner order,
// colour in lane order, Jacobian partials) is the same as k_pose_group<float>,
// and tests/test_gpu_pose.py holds the two bit-identical.
//
// fp32 only (the FP64 parity path is k_pose_group<double>). r01's FP64-SH
// instance and r02's 4-CTA/SM build composited one sample per ray: ptxas
// (CUDA 12.9) spilled the ray origin to stack slots it never stored
// (profiles/r02_pose_spill_bug.md). The march therefore reads the origin from
// the pose (the 8-lane build has no spills; the default 4-lane build at 4 CTAs/SM
// spills 76 B, all stored before use); every build
// rejects never-stored stack loads (_build.unwritten_local_loads).
#ifndef VRF_POSE_U_MINB
#define VRF_POSE_U_MINB 4  // CTAs per SM of k_pose_group_u (128 registers)
#endif
#ifndef VRF_POSE_U_LPR
#define VRF_POSE_U_LPR 4  // lanes per ray of k_pose_group_u (r02: 4 -> ~753 frames/s
                          // at 4 CTAs/SM, 8 -> ~638; tools/ab/pose_lpr.sh)
#endif
template <int MINB = VRF_POSE_U_MINB, int LPR = VRF_POSE_U_LPR>
__global__ void __launch_bounds__(kT, MINB) k_pose_group_u(
    DevGrid g, DevParams p, DevCam cam, const double4* __restrict__ rgbd_base,
    const int* __restrict__ frame_idx, long long npix, const DevPose* __restrict__ pose_ptr,
    const int* __restrict__ pixels, const uint32_t* __restrict__ order, int n, double lambda_p,
    double lambda_d, PosePartial* __restrict__ partials, int* err) {
  // LPR lanes per ray, CPL = 8 / LPR trilinear corners per lane (corners sub,
  // sub + LPR, ...). LPR = 4 (default): 8 rays per warp, so the per-ray scalar
  // work (FP64 compositing, exp, sample hand-out) is shared by 4 lanes, not 8.
  // sigma and colour still sum in corner order (bit-identical to the 8-lane
  // checker); the lane Jacobian partials sum two corners per lane first.
  constexpr int CPL = 8 / LPR;
  static_assert(LPR == 8 || LPR == 4 || LPR == 2, "lanes per ray");
  constexpr unsigned GMASK = (1u << LPR) - 1u;
  constexpr unsigned FULL = 0xffffffffu;
  using ShT = float;
  using JT = float;
  __shared__ double s_d[kT / 32][32];
  __shared__ long long s_l[kT / 32];
  __shared__ int s_i[kT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int sub = lane & (LPR - 1), gbase = lane & ~(LPR - 1);
  const int t = blockIdx.x * (kT / LPR) + threadIdx.x / LPR;
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
  bool alive = false;
  March m;
  ShT bs[9];
  if (t < n && px >= 0) {
    if (px >= cam.width || py < 0 || py >= cam.height) {
      if (sub == 0) atomicOr(err, 2);
    } else {
      const DevPose pose = *pose_ptr;
      ray_from_pixel(cam, pose, (double)px, (double)py, m);
      double basis[9];
      if (!sh_basis(m.d, basis)) {
        if (sub == 0) atomicOr(err, 1);
      } else if (march_begin(g, p, m)) {
        alive = true;
#pragma unroll
        for (int mm = 0; mm < 9; ++mm) bs[mm] = ShT(basis[mm]);
      }
    }
  }
  JT Jo[4][3], Jd[4][3], Bo[3] = {0, 0, 0}, Bd[3] = {0, 0, 0};
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int a = 0; a < 3; ++a) Jo[r][a] = Jd[r][a] = JT(0);
  double T = 1.0, prefix[3] = {0, 0, 0}, prefix_d = 0.0;
  int count = 0;
  Sample mine{};  // value-initialised: lanes read it only after a located segment
  unsigned act = 0;
  while (__any_sync(FULL, alive)) {
    // ---- round A: groups without a pending sample locate their next 8 segments
    const bool need = alive && act == 0;
    bool a = false, eb = false;
    if (need) {
      const long long kk = m.k + sub;
      if (kk < m.nseg) {
        const double s0 = dadd(m.lo, dmul((double)kk, m.step));
        const double s0s = dadd(s0, m.step);
        const double s1 = (m.hi < s0s) ? m.hi : s0s;
        const double len = dsub(s1, s0);
        if (len >= 1e-12) {
          const double tm = dmul(0.5, dadd(s0, s1));
          // the origin is the pose translation, shared by every ray: read it
          // (uniform address, L1 broadcast) instead of keeping m.o live
          const double* po = pose_ptr->t;
          const double pp[3] = {dadd(__ldg(po), dmul(tm, m.d[0])),
                                dadd(__ldg(po + 1), dmul(tm, m.d[1])),
                                dadd(__ldg(po + 2), dmul(tm, m.d[2]))};
          if (locate(g, pp, mine)) {
            if (cell_active(g, mine.cell)) {
              a = true;
              mine.t = tm;
              mine.delta = len;
            } else {
              eb = !block_active(g, mine.cx, mine.cy, mine.cz);
            }
          }
        }
      }
    }
    const unsigned ba = __ballot_sync(FULL, a), be = __ballot_sync(FULL, eb);
    int jskip = -1;
    if (need) {
      act = (ba >> gbase) & GMASK;
      const unsigned ebm = (be >> gbase) & GMASK;
      m.k += LPR;
      if (act == 0 && ebm) jskip = 31 - __clz(ebm);
    }
    long long kn = 0;
    if (jskip >= 0 && sub == jskip)
      kn = skip_empty_box<true>(g, m, mine,
                                super_active(g, mine.cx, mine.cy, mine.cz) ? kBlockLog2 : kSuperLog2,
                                pose_ptr->t);
    kn = __shfl_sync(FULL, kn, gbase + (jskip >= 0 ? jskip : 0));
    if (jskip >= 0 && kn > m.k) m.k = kn;
    if (need && act == 0 && m.k >= m.nseg) alive = false;  // ray exhausted
    // ---- round B: groups with a pending sample shade the first one
    const bool has = alive && act != 0;
    if (!__any_sync(FULL, has)) continue;
    const int src = gbase + (has ? (__ffs(act) - 1) : 0);
    if (has) act &= act - 1;
    Sample s{};
    s.t = __shfl_sync(FULL, mine.t, src);
    s.delta = __shfl_sync(FULL, mine.delta, src);
    s.fx = __shfl_sync(FULL, mine.fx, src);
    s.fy = __shfl_sync(FULL, mine.fy, src);
    s.fz = __shfl_sync(FULL, mine.fz, src);
    s.base = __shfl_sync(FULL, mine.base, src);
    double pk[CPL];
    ShT cp[CPL][3];
    JT Gs[3] = {0, 0, 0}, Gc[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int cc = 0; cc < CPL; ++cc) {
      pk[cc] = 0.0;
      cp[cc][0] = cp[cc][1] = cp[cc][2] = ShT(0);
    }
#pragma unroll
    for (int cc = 0; cc < CPL; ++cc) {
    // this lane's corner kc and its signs (sgn[d] of k_pose_group: -1 for d = 0)
    const int kc = sub + cc * LPR, dx = kc & 1, dy = (kc >> 1) & 1, dz = (kc >> 2) & 1;
    const JT sx = dx ? JT(1) : JT(-1), sy = dy ? JT(1) : JT(-1), sz = dz ? JT(1) : JT(-1);
    if (has) {
      // the lane's own corner weights, selected rather than indexed (the [2]
      // arrays of k_pose_group live in local memory here): the same values, so
      // the same arithmetic bit for bit
      const double wxl = dx ? s.fx : dsub(1.0, s.fx), wyl = dy ? s.fy : dsub(1.0, s.fy),
                   wzl = dz ? s.fz : dsub(1.0, s.fz);
      const JT wxj = JT(wxl), wyj = JT(wyl), wzj = JT(wzl);
      const JT iv = JT(g.inv_voxel);
      const double wk = dmul(dmul(wxl, wyl), wzl);
      const JT dw[3] = {sx * wyj * wzj * iv, wxj * sy * wzj * iv, wxj * wyj * sz * iv};
      const float4* vp4 = g.payload + (size_t)corner_index(g, s.base, kc) * kVec4PerVertex;
      float v[28];
#pragma unroll
      for (int j = 0; j < kVec4PerVertex; ++j) {
        const float4 q = __ldg(vp4 + j);
        v[4 * j] = q.x;
        v[4 * j + 1] = q.y;
        v[4 * j + 2] = q.z;
        v[4 * j + 3] = q.w;
      }
      pk[cc] = dmul(wk, (double)v[0]);
      JT shd[3];
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        ShT acc = ShT(0);
#pragma unroll
        for (int mm = 0; mm < 9; ++mm) acc = fma(bs[mm], (ShT)v[1 + ch * 9 + mm], acc);
        shd[ch] = JT(acc);
        cp[cc][ch] = fma(ShT(wk), acc, cp[cc][ch]);
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        Gs[q] = fma(dw[q], JT(v[0]), Gs[q]);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) Gc[ch][q] = fma(dw[q], shd[ch], Gc[ch][q]);
      }
    }
    }
    // sigma_raw in corner order (the reference's), colour in corner order too
    // (corner cc * LPR + j is lane j's cc-th)
    double sraw = 0.0;
    ShT csum[3] = {ShT(0), ShT(0), ShT(0)};
#pragma unroll
    for (int cc = 0; cc < CPL; ++cc)
#pragma unroll
      for (int j = 0; j < LPR; ++j) sraw = dadd(sraw, __shfl_sync(FULL, pk[cc], gbase + j));
#pragma unroll
    for (int cc = 0; cc < CPL; ++cc)
#pragma unroll
      for (int j = 0; j < LPR; ++j)
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) csum[ch] += __shfl_sync(FULL, cp[cc][ch], gbase + j);
    if (has) {
      double c[3];
      bool clamped[3];
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const double cv = 0.5 + (double)csum[ch];
        clamped[ch] = (cv <= 0.0 || cv >= 1.0);
        c[ch] = (cv < 0.0) ? 0.0 : ((1.0 < cv) ? 1.0 : cv);
      }
      const double sigma = (sraw < 0.0) ? 0.0 : sraw;
      const double decay = exp(dmul(-sigma, s.delta));
      const double wgt = dmul(T, dsub(1.0, decay));
      const double T_next = dmul(T, decay);
      ++count;
      JT dsig[4];
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        prefix[ch] = dadd(prefix[ch], dmul(c[ch], wgt));
        dsig[ch] = JT(s.delta * (c[ch] * T_next + prefix[ch]));
      }
      prefix_d = dadd(prefix_d, dmul(s.t, wgt));
      dsig[3] = JT(s.delta * (s.t * T_next + prefix_d));
      const bool sgate = sraw > 0.0;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const JT gs = sgate ? JT(s.delta) * Gs[q] : JT(0);
        Bo[q] += gs;
        Bd[q] = fma(JT(s.t), gs, Bd[q]);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          JT gv = sgate ? dsig[r] * Gs[q] : JT(0);
          if (r < 3 && !clamped[r]) gv += JT(wgt) * Gc[r][q];
          Jo[r][q] += gv;
          Jd[r][q] = fma(JT(s.t), gv, Jd[r][q]);
        }
      }
#if VRF_POSE_DEBUG
      if (blockIdx.x == 0 && threadIdx.x < 16)
        printf("dbg t%d cnt%d sraw %.6g delta %.6g st %.6g decay %.6g T %.6g->%.6g act %x k %lld nseg %lld\n",
               threadIdx.x, count, sraw, s.delta, s.t, decay, T, T_next, act, m.k, m.nseg);
#endif
      T = T_next;
      if (T < p.eps) alive = false;
    }
  }
  // group reduction of the lane partials (fixed butterfly order, full-warp shuffles)
#pragma unroll
  for (int off = LPR / 2; off > 0; off >>= 1) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      Bo[q] += __shfl_xor_sync(FULL, Bo[q], off);
      Bd[q] += __shfl_xor_sync(FULL, Bd[q], off);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        Jo[r][q] += __shfl_xor_sync(FULL, Jo[r][q], off);
        Jd[r][q] += __shfl_xor_sync(FULL, Jd[r][q], off);
      }
    }
  }
  if (count > 0 && sub == 0) {
    hit = 1;
    samples = count;
    const double4 tg = rgbd[(long long)py * cam.width + px];
    const double C[4] = {prefix[0], prefix[1], prefix[2], prefix_d};
    const double res[4] = {dsub(C[0], tg.x), dsub(C[1], tg.y), dsub(C[2], tg.z),
                           dsub(C[3], tg.w)};
    loss = dadd(dmul(lambda_p, dadd(dadd(dmul(res[0], res[0]), dmul(res[1], res[1])),
                                    dmul(res[2], res[2]))),
                dmul(dmul(lambda_d, res[3]), res[3]));
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double jo[3], jd[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        jo[q] = (double)Jo[r][q] - C[r] * (double)Bo[q];
        jd[q] = (double)Jd[r][q] - C[r] * (double)Bd[q];
      }
      const double dd = dot3(m.d, jd);
      double gp[3], om[3];
      for (int q = 0; q < 3; ++q) gp[q] = jd[q] - m.d[q] * dd;
      cross3(m.d, gp, om);
      const double J[6] = {om[0], om[1], om[2], jo[0], jo[1], jo[2]};
      const double lam = r < 3 ? lambda_p : lambda_d;
      int idx = 0;
#pragma unroll
      for (int a2 = 0; a2 < 6; ++a2) {
#pragma unroll
        for (int b2 = a2; b2 < 6; ++b2) jtj[idx++] += lam * J[a2] * J[b2];
        jtr[a2] += lam * J[a2] * res[r];
      }
    }
  }
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

// Fixed-order reduction of the CTA partials: thread t folds partials t, t+256,
// ... (strided, fixed), then the block folds the 256 thread sums in a fixed
// tree — deterministic, and parallel (one thread per field walking all
// partials serially was 0.46 ms for 1,024 partials).
constexpr int kRedT = 256;
__global__ void __launch_bounds__(kRedT) k_pose_reduce2(const PosePartial* __restrict__ parts,
                                                        int nparts, PosePartial* out) {
  __shared__ double s_v[kRedT / 32][29];
  __shared__ long long s_s[kRedT / 32];
  __shared__ int s_m[kRedT / 32];
  double v[28];
#pragma unroll
  for (int k = 0; k < 28; ++k) v[k] = 0.0;
  long long smp = 0;
  int m = 0;
  for (int k = threadIdx.x; k < nparts; k += kRedT) {
    const PosePartial q = parts[k];
#pragma unroll
    for (int j = 0; j < 21; ++j) v[j] += q.jtj[j];
#pragma unroll
    for (int j = 0; j < 6; ++j) v[21 + j] += q.jtr[j];
    v[27] += q.loss;
    smp += q.samples;
    m += q.m;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < 28; ++j) {
    const double w = warp_sum(v[j]);
    if (lane == 0) s_v[wid][j] = w;
  }
  const long long ws = warp_sum(smp);
  const int wm = warp_sum(m);
  if (lane == 0) {
    s_s[wid] = ws;
    s_m[wid] = wm;
  }
  __syncthreads();
  if (threadIdx.x < 28) {
    double acc = 0.0;
    for (int w = 0; w < kRedT / 32; ++w) acc += s_v[w][threadIdx.x];
    if (threadIdx.x < 21)
      out->jtj[threadIdx.x] = acc;
    else if (threadIdx.x < 27)
      out->jtr[threadIdx.x - 21] = acc;
    else
      out->loss = acc;
  } else if (threadIdx.x == 32) {
    long long sl = 0;
    int sm = 0;
    for (int w = 0; w < kRedT / 32; ++w) {
      sl += s_s[w];
      sm += s_m[w];
    }
    out->samples = sl;
    out->m = sm;
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

// Stratified valid-depth draws over a 2^L x 2^L tile grid (4^L <= n < 4^(L+1)):
// thread t owns tile (Morton decode of t mod 4^L), so the first 4^L draws cover
// every tile once and the rest start a second pass in Morton order (warps stay
// coherent). Each draws uniformly inside its tile and redraws (max_redraws
// attempts) until the depth is valid; -1 marks a dropped pixel. The counter
// (iteration, t, attempt) keys the RNG, so every one of the n draws is distinct.
__global__ void k_draw_strat(const double4* __restrict__ rgbd_base,
                             const int* __restrict__ frame_idx, long long npix, int width,
                             int height, int tiles_log2, int max_redraws,
                             const unsigned long long* __restrict__ seed, int iteration,
                             int* __restrict__ pixels, int n) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double4* rgbd = rgbd_base + npix * (long long)(*frame_idx);
  const int tiles = 1 << tiles_log2;
  const uint32_t tile = (uint32_t)t & ((1u << (2 * tiles_log2)) - 1u);
  const int tx = (int)compact_bits(tile), ty = (int)compact_bits(tile >> 1);
  int px = -1, py = -1;
  if (tx < tiles && ty < tiles) {
    const int x0 = (int)((long long)tx * width / tiles);
    int x1 = (int)((long long)(tx + 1) * width / tiles);
    const int y0 = (int)((long long)ty * height / tiles);
    int y1 = (int)((long long)(ty + 1) * height / tiles);
    // more tiles than pixel rows / columns: a tile keeps at least its first pixel
    if (x1 <= x0) x1 = x0 + 1;
    if (y1 <= y0) y1 = y0 + 1;
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
  hist[3 * iteration] = r.m > 0 ? r.loss / r.m : 0.0;
  hist[3 * iteration + 1] = r.m;
  hist[3 * iteration + 2] = (double)r.samples;
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

int pose_fused_blocks(int n, PoseKernel which) {
  const int rays_per_cta = kT / (which == PoseKernel::kGnUniform ? VRF_POSE_U_LPR : 8);
  return (n + rays_per_cta - 1) / rays_per_cta;
}

void launch_pose_fused(PoseKernel which, const DevGrid& g, const DevParams& p, const DevCam& cam,
                       const double4* rgbd_base, const int* frame_idx, long long npix,
                       const DevPose* pose, const int* pixels, const uint32_t* order, int n,
                       double lambda_p, double lambda_d, PosePartial* partials, int* err,
                       cudaStream_t s) {
  if (n <= 0) return;
  const int nb = pose_fused_blocks(n, which);
#define VRF_POSE_ARGS \
  g, p, cam, rgbd_base, frame_idx, npix, pose, pixels, order, n, lambda_p, lambda_d, partials, err
  switch (which) {
    case PoseKernel::kParityFp64:
      k_pose_group<double><<<nb, kT, 0, s>>>(VRF_POSE_ARGS);
      break;
    case PoseKernel::kGroupFp32:
      k_pose_group<float><<<nb, kT, 0, s>>>(VRF_POSE_ARGS);
      break;
    case PoseKernel::kGnUniform:
      k_pose_group_u<><<<nb, kT, 0, s>>>(VRF_POSE_ARGS);
      break;
  }
#undef VRF_POSE_ARGS
}

void launch_pose_reduce2(const PosePartial* partials, int nparts, PosePartial* out,
                         cudaStream_t s) {
  k_pose_reduce2<<<1, kRedT, 0, s>>>(partials, nparts, out);
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
