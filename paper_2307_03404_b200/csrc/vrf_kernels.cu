// sm_100a kernels of the per-ray hot path.
//
//   K1 k_render_image      render_image          renderer.cpp:149-174 (+51-140)
//   K0+fwd k_map_forward_rec  mapping_step forward (hit counts M_c/M_d, loss
//                          partials) + 24 B per-sample records  mapping.cpp:130-200
//   K2 k_map_backward_rec  reverse walk over the records: suffix-form dL/dsigma,
//                          dL/dc + aggregated trilinear adjoint scatter
//                          (red.global.add.v4.f32)   gradients.cpp:69-114, mapping.cpp:172-195
//      k_map_backward      recompute-march variant (rays longer than the record cap)
//      k_map_forward       forward without records (deterministic mode, >cap budgets)
//   K3 k_map_records +     deterministic mode: per-sample fp64 records, stable
//      k_segmented_reduce  radix sort by vertex, in-order fp64 segment sums
//                                                gradients.cpp:28-57 (sorted merge)
//   K4 k_rmsprop           sparse RMSProp (skip g == 0), clears g   mapping.cpp:218-231
//   K5 (vrf_track.cu)      fused pose forward + Jacobian -> J^T J, J^T r
//   utilities              prune, upsample, block occupancy, pack / convert
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <cstdlib>
#include <climits>

#include "vrf_internal.h"

namespace vrf {

namespace {

constexpr int kThreads = 128;

// ------------------------------------------------------------------ K1
template <typename ShT>
__global__ void __launch_bounds__(kThreads) k_render_image(DevGrid g, DevParams p, DevCam cam,
                                                           DevPose pose, int stride, int out_w,
                                                           int out_h, double* __restrict__ color,
                                                           double* __restrict__ depth,
                                                           int* err) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)out_w * out_h) return;
  const int px = (int)(idx % out_w), py = (int)(idx / out_w);
  March m;
  ray_from_pixel(cam, pose, (double)px * stride, (double)py * stride, m);
  Composite st;
  double basis[9];
  if (!render_forward<ShT>(g, p, m, st, basis)) {
    atomicOr(err, 1);
    return;
  }
  color[idx * 3 + 0] = st.C[0];
  color[idx * 3 + 1] = st.C[1];
  color[idx * 3 + 2] = st.C[2];
  depth[idx] = st.count > 0 ? st.D : 0.0;
}

// ------------------------------------------------------------------ inspection
__global__ void __launch_bounds__(kThreads) k_debug_rays(DevGrid g, DevParams p,
                                                         const double* __restrict__ rays, int n,
                                                         int cap, int* counts, double* t,
                                                         double* delta, uint32_t* cells,
                                                         double* out, int* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  March m;
  for (int a = 0; a < 3; ++a) {
    m.o[a] = rays[6 * i + a];
    m.d[a] = rays[6 * i + 3 + a];
  }
  if (counts) {  // sample_ray: the full schedule (no termination)
    int c = 0;
    if (march_begin(g, p, m)) {
      Sample s;
      while (march_next(g, m, s)) {
        if (c < cap) {
          t[(long long)i * cap + c] = s.t;
          delta[(long long)i * cap + c] = s.delta;
          cells[(long long)i * cap + c] = s.cell;
        }
        ++c;
      }
    }
    counts[i] = c;
  }
  if (out) {  // render_ray
    Composite st;
    double basis[9];
    if (!render_forward<double>(g, p, m, st, basis)) {
      atomicOr(err, 1);
      return;
    }
    double* o = out + 8 * (long long)i;
    o[0] = st.C[0];
    o[1] = st.C[1];
    o[2] = st.C[2];
    o[3] = st.D;
    o[4] = st.T;
    o[5] = st.count;
    o[6] = st.count > 0;
    o[7] = st.terminated;
  }
}

// ------------------------------------------------------------------ block reductions
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  T r = T(0);
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += smem[w];  // fixed order
  return r;  // valid in thread 0
}

__device__ __forceinline__ int block_min(int v, int* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, off));
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  int r = INT_MAX;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = min(r, smem[w]);
  return r;
}

// ------------------------------------------------------------------ K0 + mapping forward
template <typename ShT>
__global__ void __launch_bounds__(kThreads) k_map_forward(
    DevGrid g, DevParams p, DevCam cam, const double4* __restrict__ rgbd,
    const DevPose* __restrict__ poses, int n_frames, const int* __restrict__ batch, int n,
    double4* __restrict__ ray_cd, uint8_t* __restrict__ flags, MapPartial* partials,
    int* __restrict__ ray_count, int* err, const uint32_t* __restrict__ order) {
  __shared__ double s_d[32];
  __shared__ long long s_l[32];
  __shared__ int s_i[32];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = (order && t < n) ? (int)order[t] : t;  // coherent ray order when given
  double lp = 0.0, lg = 0.0;
  long long samples = 0;
  int mc = 0, md = 0, bad = INT_MAX;
  if (t < n) {
    const int f = batch[3 * i], px = batch[3 * i + 1], py = batch[3 * i + 2];
    uint8_t fl = 0;
    if (f < 0 || f >= n_frames || px < 0 || px >= cam.width || py < 0 || py >= cam.height) {
      atomicOr(err, 2);  // generate_ray: pixel outside image
    } else {
      March m;
      ray_from_pixel(cam, poses[f], (double)px, (double)py, m);
      Composite st;
      double basis[9];
      if (!render_forward<ShT>(g, p, m, st, basis)) atomicOr(err, 1);
      const double4 tg = rgbd[(long long)f * cam.width * cam.height + (long long)py * cam.width + px];
      if (st.count > 0) {
        fl |= kHit;
        mc = 1;
        samples = st.count;
        const double r0 = dsub(st.C[0], tg.x), r1 = dsub(st.C[1], tg.y), r2 = dsub(st.C[2], tg.z);
        const double sq = dadd(dadd(dmul(r0, r0), dmul(r1, r1)), dmul(r2, r2));
        if (!isfinite(sq) || !isfinite(st.D)) {
          bad = i;
        } else {
          lp = sq;
          if (tg.w > 0.0) {
            fl |= kDepthValid;
            md = 1;
            const double dr = dsub(st.D, tg.w);
            lg = dmul(dr, dr);
          }
        }
      }
      ray_cd[i] = make_double4(st.C[0], st.C[1], st.C[2], st.D);
    }
    flags[i] = fl;
    if (ray_count) ray_count[i] = (fl & kHit) ? (int)samples : 0;
  }
  const double blp = block_sum(lp, s_d);
  const double blg = block_sum(lg, s_d);
  const long long bs = block_sum(samples, s_l);
  const int bmc = block_sum(mc, s_i);
  const int bmd = block_sum(md, s_i);
  const int bbad = block_min(bad, s_i);
  const int bmax = -block_min(-(int)samples, s_i);
  if (threadIdx.x == 0) {
    MapPartial q;
    q.lp = blp;
    q.lg = blg;
    q.samples = bs;
    q.m_c = bmc;
    q.m_d = bmd;
    q.bad = bbad;
    q.max_count = bmax;
    partials[blockIdx.x] = q;
  }
}

// Record slot of sample c of the ray in slot t: warp-tiled sample-major
// ("AoSoA"): the 32 rays of a warp own one contiguous K x 32-record region of
// each plane, and within it sample c of all 32 lanes is contiguous. The rays of
// a warp are coherent (Morton tiles), so its lanes mostly composite (and walk
// back) their c-th samples together: those stores and loads coalesce. (A
// ray-major layout measured 10.7 / 13.9 ms for K0 / K2 against 8.7 / 11.8, r02.)
__device__ __forceinline__ size_t rec_index(int t, int c, int K) {
  return ((size_t)(t >> 5) * (size_t)K + (size_t)c) * 32 + (size_t)(t & 31);
}

// VRF_REC_HINT: the records stream through L2 at evict-first priority (written
// once by K0, read once by K2) to keep the payload and gradient lines resident.
// Bit 0: K0's record stores; bit 1: K2's record loads (also no L1 allocation).
#ifndef VRF_REC_HINT
#define VRF_REC_HINT 1
#endif
#if VRF_REC_HINT
__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
#endif
// Stores one sample record (vrf_internal.h: RecBuf): a 16 B and an 8 B store.
// A clamped channel's colour is stored negated (its sign bit is the clamp
// flag; the clamped value is 0 or 1, and -0.f keeps the bit).
__device__ __forceinline__ void store_record(RecBuf rec, size_t idx, double wgt, const Shade& sh,
                                             int cx, int cy, int cz, double tm) {
  float c[3];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) c[ch] = sh.clamped[ch] ? -(float)sh.c[ch] : (float)sh.c[ch];
#if VRF_REC_HINT & 1
  const unsigned long long pol = evict_first_policy();
  const uint32_t cw = pack_cell(cx, cy, cz) | (sh.sigma_raw > 0.0 ? kRecSigmaPos : 0u);
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;"
               :: "l"(rec.a + idx), "f"((float)wgt), "f"(c[0]), "f"(c[1]), "f"(c[2]), "l"(pol)
               : "memory");
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;"
               :: "l"(rec.b + idx), "r"(cw), "r"(__float_as_uint((float)tm)), "l"(pol)
               : "memory");
#else
  rec.a[idx] = make_float4((float)wgt, c[0], c[1], c[2]);
  rec.b[idx] = make_uint2(pack_cell(cx, cy, cz) | (sh.sigma_raw > 0.0 ? kRecSigmaPos : 0u),
                          __float_as_uint((float)tm));
#endif
}

// Fast forward (fp32 SH) that records every composited sample for the
// backward: identical march, sigma_raw replay, compositing and termination as
// k_map_forward<float>; per sample it stores w_i, T_{i+1}, the clamped colour,
// clamp / sigma gates, cell and midpoint — 24 B — so the backward never
// gathers the 896 B of corner payload again. Records are warp-tiled
// sample-major (rec_index): the lanes of a warp composite their c-th samples in
// the same loop iteration, so each record store is coalesced.
// 4 CTAs/SM (128 registers): r01 measured 3 / 4 / 5 CTAs at 8.83 / 8.21 / 8.75 ms.
#ifndef VRF_K0_MINB
#define VRF_K0_MINB 4
#endif
#ifndef VRF_K0_CARVEOUT
#define VRF_K0_CARVEOUT -1  // driver default
#endif
#ifndef VRF_K0_COOP
#define VRF_K0_COOP 0  // A/B: warp-cooperative corner staging in shared memory
#endif
__global__ void __launch_bounds__(kThreads, VRF_K0_MINB) k_map_forward_rec(
    DevGrid g, DevParams p, DevCam cam, const double4* __restrict__ rgbd,
    const DevPose* __restrict__ poses, int n_frames, const int* __restrict__ batch, int n,
    double4* __restrict__ ray_cd, uint8_t* __restrict__ flags, MapPartial* partials, int* err,
    const uint32_t* __restrict__ order, RecBuf rec, int K,
    int2* __restrict__ rec_count) {
  __shared__ double s_d[32];
  __shared__ long long s_l[32];
  __shared__ int s_i[32];
#if VRF_K0_CACHE
  static_assert(kThreads == kCacheStride, "corner cache layout");
  __shared__ float4 s_cache[8 * kThreads];
#endif
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = (order && t < n) ? (int)order[t] : t;
  double lp = 0.0, lg = 0.0;
  long long samples = 0;
  int mc = 0, md = 0, bad = INT_MAX;
  if (t < n) {
    const int f = batch[3 * i], px = batch[3 * i + 1], py = batch[3 * i + 2];
    uint8_t fl = 0;
    int stored = 0;
    float tfin = 1.f;  // T after the ray's last composited sample
    if (f < 0 || f >= n_frames || px < 0 || px >= cam.width || py < 0 || py >= cam.height) {
      atomicOr(err, 2);  // generate_ray: pixel outside image
    } else {
      March m;
      ray_from_pixel(cam, poses[f], (double)px, (double)py, m);
      Composite st;
      st.T = 1.0;
      st.C[0] = st.C[1] = st.C[2] = 0.0;
      st.D = 0.0;
      st.count = 0;
      st.terminated = false;
      float bf[9];
      bool basis_ok;
      {
        double basis[9];
        basis_ok = sh_basis(m.d, basis);
#pragma unroll
        for (int mm = 0; mm < 9; ++mm) bf[mm] = (float)basis[mm];
      }
      if (!basis_ok) {
        atomicOr(err, 1);
      } else if (march_begin(g, p, m)) {
        Sample s;
#if VRF_K0_CACHE
        CornerCache cc{s_cache + threadIdx.x, 0u, 0xffffffffu};
#endif
        while (march_next(g, m, s)) {
          Shade sh;
          {
            double w[8];
            corner_weights(s, w);
#if VRF_K0_CACHE
            shade_cached(g, s, w, bf, cc, sh);
#else
            shade_fast(g, s, w, bf, sh);
#endif
          }
          double decay;
          const double wgt = composite_step(st, sh, s.t, s.delta, p.eps, decay);
          if (st.count <= K) {
            store_record(rec, rec_index(t, st.count - 1, K), wgt, sh, s.cx, s.cy, s.cz, s.t);
          }
          if (st.terminated) break;
        }
      }
      if (st.count == 0) {
        st.C[0] = st.C[1] = st.C[2] = 0.0;
        st.D = 0.0;
      }
      const double4 tg = rgbd[(long long)f * cam.width * cam.height + (long long)py * cam.width + px];
      if (st.count > 0) {
        fl |= kHit;
        if (st.count > K) fl |= kOverflow;
        stored = st.count > K ? 0 : st.count;
        tfin = (float)st.T;
        mc = 1;
        samples = st.count;
        const double r0 = dsub(st.C[0], tg.x), r1 = dsub(st.C[1], tg.y), r2 = dsub(st.C[2], tg.z);
        const double sq = dadd(dadd(dmul(r0, r0), dmul(r1, r1)), dmul(r2, r2));
        if (!isfinite(sq) || !isfinite(st.D)) {
          bad = i;
        } else {
          lp = sq;
          if (tg.w > 0.0) {
            fl |= kDepthValid;
            md = 1;
            const double dr = dsub(st.D, tg.w);
            lg = dmul(dr, dr);
          }
        }
      }
      ray_cd[i] = make_double4(st.C[0], st.C[1], st.C[2], st.D);
    }
    flags[i] = fl;
    rec_count[t] = make_int2(stored, __float_as_int(tfin));
  }
  const double blp = block_sum(lp, s_d);
  const double blg = block_sum(lg, s_d);
  const long long bs = block_sum(samples, s_l);
  const int bmc = block_sum(mc, s_i);
  const int bmd = block_sum(md, s_i);
  const int bbad = block_min(bad, s_i);
  const int bmax = -block_min(-(int)samples, s_i);
  if (threadIdx.x == 0) {
    MapPartial q;
    q.lp = blp;
    q.lg = blg;
    q.samples = bs;
    q.m_c = bmc;
    q.m_d = bmd;
    q.bad = bbad;
    q.max_count = bmax;
    partials[blockIdx.x] = q;
  }
}

#if VRF_K0_COOP
// K0 with warp-cooperative corner staging (A/B, -DVRF_K0_COOP=1). The 32 rays of
// a warp are coherent, so at one march step they sit in a handful of distinct
// cells; the thread-per-ray gather reads every corner through L1 once per lane
// (56 LDG.128 per sample, ~5.6 L1 wavefronts each: K0 is bound by the L1 data
// pipe). Here each step groups the lanes by cell (__match_any_sync), the warp
// loads each distinct cell's 8 corners once with coalesced 112-B runs into shared
// memory, and every lane shades from there. Same values, same FP64 arithmetic:
// bit-identical to k_map_forward_rec.
constexpr int kCoopSlots = 8;    // distinct cells staged per round
constexpr int kCoopStride = 57;  // float4 per staged cell: 8 corners x 7 + 1 (bank spread)

__device__ __forceinline__ void shade_staged(const float4* cell, const double w[8],
                                             const float bf[9], Shade& out) {
  double sraw = 0.0;
  float cr = 0.f, cg = 0.f, cb = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float v[28];
#pragma unroll
    for (int j = 0; j < kVec4PerVertex; ++j) {
      const float4 a = cell[k * kVec4PerVertex + j];
      v[4 * j] = a.x;
      v[4 * j + 1] = a.y;
      v[4 * j + 2] = a.z;
      v[4 * j + 3] = a.w;
    }
    sraw = dadd(sraw, dmul(w[k], (double)v[0]));
    float dr = 0.f, dg = 0.f, db = 0.f;
#pragma unroll
    for (int m = 0; m < 9; ++m) {
      dr = fmaf(bf[m], v[1 + m], dr);
      dg = fmaf(bf[m], v[10 + m], dg);
      db = fmaf(bf[m], v[19 + m], db);
    }
    const float wk = (float)w[k];
    cr = fmaf(wk, dr, cr);
    cg = fmaf(wk, dg, cg);
    cb = fmaf(wk, db, cb);
  }
  out.sigma_raw = sraw;
  const float cc[3] = {cr, cg, cb};
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    const double v = 0.5 + (double)cc[ch];
    out.clamped[ch] = (v <= 0.0 || v >= 1.0);
    out.c[ch] = (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v);
  }
}

__global__ void __launch_bounds__(kThreads, VRF_K0_MINB) k_map_forward_coop(
    DevGrid g, DevParams p, DevCam cam, const double4* __restrict__ rgbd,
    const DevPose* __restrict__ poses, int n_frames, const int* __restrict__ batch, int n,
    double4* __restrict__ ray_cd, uint8_t* __restrict__ flags, MapPartial* partials, int* err,
    const uint32_t* __restrict__ order, RecBuf rec, int K,
    int2* __restrict__ rec_count) {
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ double s_d[32];
  __shared__ long long s_l[32];
  __shared__ int s_i[32];
  __shared__ __align__(16) float4 s_cells[kThreads / 32][kCoopSlots * kCoopStride];
  __shared__ uint32_t s_base[kThreads / 32][kCoopSlots];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = (order && t < n) ? (int)order[t] : t;
  double lp = 0.0, lg = 0.0;
  long long samples = 0;
  int mc = 0, md = 0, bad = INT_MAX;
  int f = 0, px = 0, py = 0;
  bool valid = false, alive = false;
  March m;
  Composite st;
  st.T = 1.0;
  st.C[0] = st.C[1] = st.C[2] = 0.0;
  st.D = 0.0;
  st.count = 0;
  st.terminated = false;
  float bf[9];
  for (int mm = 0; mm < 9; ++mm) bf[mm] = 0.f;
  if (t < n) {
    f = batch[3 * i];
    px = batch[3 * i + 1];
    py = batch[3 * i + 2];
    if (f < 0 || f >= n_frames || px < 0 || px >= cam.width || py < 0 || py >= cam.height) {
      atomicOr(err, 2);  // generate_ray: pixel outside image
    } else {
      valid = true;
      ray_from_pixel(cam, poses[f], (double)px, (double)py, m);
      double basis[9];
      const bool basis_ok = sh_basis(m.d, basis);
#pragma unroll
      for (int mm = 0; mm < 9; ++mm) bf[mm] = (float)basis[mm];
      if (!basis_ok)
        atomicOr(err, 1);
      else
        alive = march_begin(g, p, m);
    }
  }
  float4* cells = s_cells[wid];
  uint32_t* bases = s_base[wid];
  while (__any_sync(FULL, alive)) {
    Sample s;
    bool has = false;
    if (alive) {
      has = march_next(g, m, s);
      if (!has) alive = false;
    }
    const unsigned grp = __match_any_sync(FULL, has ? s.base : 0xffffffffu);
    const int leader = __ffs(grp) - 1;
    const unsigned lm = __ballot_sync(FULL, has && lane == leader);  // one bit per distinct cell
    const int D = __popc(lm);
    const int slot = __popc(lm & ((1u << leader) - 1u));
    for (int r0 = 0; r0 < D; r0 += kCoopSlots) {
      const int nd = min(kCoopSlots, D - r0);
      if (has && lane == leader && slot >= r0 && slot < r0 + kCoopSlots) bases[slot - r0] = s.base;
      __syncwarp();
      // the staged cells' 8 corners, 7 float4 each, as contiguous 112-B runs
      for (int it = lane; it < nd * 8 * kVec4PerVertex; it += 32) {
        const int vs = it / kVec4PerVertex, j = it - vs * kVec4PerVertex;
        const int c = vs >> 3, k = vs & 7;
        const float4* src = g.payload + (size_t)corner_index(g, bases[c], k) * kVec4PerVertex;
        cells[c * kCoopStride + k * kVec4PerVertex + j] = __ldg(src + j);
      }
      __syncwarp();
      if (has && slot >= r0 && slot < r0 + kCoopSlots) {
        Shade sh;
        {
          double w[8];
          corner_weights(s, w);
          shade_staged(cells + (slot - r0) * kCoopStride, w, bf, sh);
        }
        double decay;
        const double wgt = composite_step(st, sh, s.t, s.delta, p.eps, decay);
        if (st.count <= K) {
          store_record(rec, rec_index(t, st.count - 1, K), wgt, sh, s.cx, s.cy, s.cz, s.t);
        }
        if (st.terminated) alive = false;
      }
      __syncwarp();
    }
  }
  if (t < n) {
    uint8_t fl = 0;
    int stored = 0;
    float tfin = 1.f;  // T after the ray's last composited sample
    if (valid) {
      if (st.count == 0) {
        st.C[0] = st.C[1] = st.C[2] = 0.0;
        st.D = 0.0;
      }
      const double4 tg =
          rgbd[(long long)f * cam.width * cam.height + (long long)py * cam.width + px];
      if (st.count > 0) {
        fl |= kHit;
        if (st.count > K) fl |= kOverflow;
        stored = st.count > K ? 0 : st.count;
        tfin = (float)st.T;
        mc = 1;
        samples = st.count;
        const double r0 = dsub(st.C[0], tg.x), r1 = dsub(st.C[1], tg.y), r2 = dsub(st.C[2], tg.z);
        const double sq = dadd(dadd(dmul(r0, r0), dmul(r1, r1)), dmul(r2, r2));
        if (!isfinite(sq) || !isfinite(st.D)) {
          bad = i;
        } else {
          lp = sq;
          if (tg.w > 0.0) {
            fl |= kDepthValid;
            md = 1;
            const double dr = dsub(st.D, tg.w);
            lg = dmul(dr, dr);
          }
        }
      }
      ray_cd[i] = make_double4(st.C[0], st.C[1], st.C[2], st.D);
    }
    flags[i] = fl;
    rec_count[t] = make_int2(stored, __float_as_int(tfin));
  }
  const double blp = block_sum(lp, s_d);
  const double blg = block_sum(lg, s_d);
  const long long bs = block_sum(samples, s_l);
  const int bmc = block_sum(mc, s_i);
  const int bmd = block_sum(md, s_i);
  const int bbad = block_min(bad, s_i);
  const int bmax = -block_min(-(int)samples, s_i);
  if (threadIdx.x == 0) {
    MapPartial q;
    q.lp = blp;
    q.lg = blg;
    q.samples = bs;
    q.m_c = bmc;
    q.m_d = bmd;
    q.bad = bbad;
    q.max_count = bmax;
    partials[blockIdx.x] = q;
  }
}
#endif

// Fixed-order reduction of the per-block partials (deterministic).
__global__ void __launch_bounds__(1024) k_map_reduce(const MapPartial* __restrict__ parts,
                                                     int nparts, MapStats* out) {
  __shared__ double s_d[32];
  __shared__ long long s_l[32];
  __shared__ int s_i[32];
  double lp = 0.0, lg = 0.0;
  long long samples = 0;
  int mc = 0, md = 0, bad = INT_MAX, mx = 0;
  for (int k = threadIdx.x; k < nparts; k += blockDim.x) {
    const MapPartial q = parts[k];
    lp += q.lp;
    lg += q.lg;
    samples += q.samples;
    mc += q.m_c;
    md += q.m_d;
    bad = min(bad, q.bad);
    mx = max(mx, q.max_count);
  }
  const double blp = block_sum(lp, s_d);
  const double blg = block_sum(lg, s_d);
  const long long bs = block_sum(samples, s_l);
  const int bmc = block_sum(mc, s_i);
  const int bmd = block_sum(md, s_i);
  const int bbad = block_min(bad, s_i);
  const int bmx = -block_min(-mx, s_i);
  if (threadIdx.x == 0) {
    MapStats r;
    r.lp = blp;
    r.lg = blg;
    r.samples = bs;
    r.m_c = bmc;
    r.m_d = bmd;
    r.bad = bbad;
    r.max_count = bmx;
    *out = r;
  }
}

// ------------------------------------------------------------------ K2 mapping backward
// Per-sample upstream of the map-parameter gradient (gradients.cpp:69-114):
// prefix-form dL/dsigma_i and dL/dc_i, gated by sigma_raw > 0 and the clamp flags.
struct MapUp {
  double upc[3];
  double upd;
  bool use_depth;
  double C[3], D;
};

__device__ __forceinline__ bool map_upstream(const MapStats& st, const int* global_counts,
                                             const double4 cd, const double4 tg, uint8_t fl,
                                             double lambda_d, MapUp& u) {
  const int mc = global_counts ? global_counts[0] : st.m_c;
  const int md = global_counts ? global_counts[1] : st.m_d;
  if (mc == 0) return false;
  u.C[0] = cd.x;
  u.C[1] = cd.y;
  u.C[2] = cd.z;
  u.D = cd.w;
  const double tgc[3] = {tg.x, tg.y, tg.z};
  for (int ch = 0; ch < 3; ++ch) u.upc[ch] = ddiv(dmul(2.0, dsub(u.C[ch], tgc[ch])), (double)mc);
  const bool depth_ok = (fl & kDepthValid) && md > 0;
  u.upd = depth_ok ? ddiv(dmul(dmul(lambda_d, 2.0), dsub(u.D, tg.w)), (double)md) : 0.0;
  u.use_depth = depth_ok && u.upd != 0.0;
  return true;
}

// Walks the samples of one ray again and hands each sample's 28-slot upstream
// and corner weights to `emit`.
template <typename ShT, bool SKIP = true, typename Emit>
__device__ __forceinline__ void map_backward_ray(const DevGrid& g, const DevParams& p, March& m,
                                                 const MapUp& u, Emit&& emit) {
  double basis[9];
  if (!sh_basis(m.d, basis)) return;
  if (!march_begin(g, p, m)) return;
  double T = 1.0, prefix[3] = {0.0, 0.0, 0.0}, prefix_d = 0.0;
  Sample s;
  int idx = 0;
  while (march_next<SKIP>(g, m, s)) {
    double w[8];
    corner_weights(s, w);
    Shade sh;
    shade<ShT>(g, s, w, basis, sh);
    const double sigma = (sh.sigma_raw < 0.0) ? 0.0 : sh.sigma_raw;
    const double decay = exp(dmul(-sigma, s.delta));
    const double wgt = dmul(T, dsub(1.0, decay));
    const double T_next = dmul(T, decay);
    double ds = 0.0, dcol[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      prefix[ch] = dadd(prefix[ch], dmul(sh.c[ch], wgt));
      dcol[ch] = dmul(u.upc[ch], wgt);
      ds = dadd(ds, dmul(dmul(u.upc[ch], s.delta),
                         dadd(dsub(dmul(sh.c[ch], T_next), u.C[ch]), prefix[ch])));
    }
    if (u.use_depth) {
      prefix_d = dadd(prefix_d, dmul(s.t, wgt));
      ds = dadd(ds, dmul(dmul(u.upd, s.delta), dadd(dsub(dmul(s.t, T_next), u.D), prefix_d)));
    }
    const double up0 = sh.sigma_raw > 0.0 ? ds : 0.0;
    emit(idx, s, w, up0, dcol, sh.clamped, basis);
    ++idx;
    T = T_next;
    if (T < p.eps) break;
  }
}

// K0g: K0 for small batches, 8 lanes per ray. Below ~1e5 rays the thread-per-
// ray K0 leaves one warp per SM sub-partition and each sample is a serial chain
// of 56 gathers and the FP64 march (16K rays: ~10 us per sample). Here the ray
// group locates 8 segments at once (GroupMarch) and each lane gathers one
// trilinear corner. sigma_raw is summed from the lanes' w_k * sigma_k products
// in corner order and the colour from their (w_k, basis-contracted corner
// colour) pairs, again in corner order, so samples, T, records and outputs are
// bit-identical to K0 (k_map_forward_rec). Lane 0 of the group writes.
constexpr int kFwdLanes = 8;
__global__ void __launch_bounds__(kThreads) k_map_forward_rec_g(
    DevGrid g, DevParams p, DevCam cam, const double4* __restrict__ rgbd,
    const DevPose* __restrict__ poses, int n_frames, const int* __restrict__ batch, int n,
    double4* __restrict__ ray_cd, uint8_t* __restrict__ flags, MapPartial* partials, int* err,
    const uint32_t* __restrict__ order, RecBuf rec, int K,
    int2* __restrict__ rec_count) {
  constexpr int LPR = kFwdLanes;
  __shared__ double s_d[32];
  __shared__ long long s_l[32];
  __shared__ int s_i[32];
  const int lane = threadIdx.x & 31, sub = lane & (LPR - 1), gbase = lane & ~(LPR - 1);
  const unsigned gmask = ((1u << LPR) - 1u) << gbase;
  const bool lead = sub == 0;
  const int t = blockIdx.x * (kThreads / LPR) + threadIdx.x / LPR;
  const int i = (order && t < n) ? (int)order[t] : t;
  double lp = 0.0, lg = 0.0;
  long long samples = 0;
  int mc = 0, md = 0, bad = INT_MAX;
  if (t < n) {
    const int f = batch[3 * i], px = batch[3 * i + 1], py = batch[3 * i + 2];
    uint8_t fl = 0;
    int stored = 0;
    float tfin = 1.f;  // T after the ray's last composited sample
    if (f < 0 || f >= n_frames || px < 0 || px >= cam.width || py < 0 || py >= cam.height) {
      if (lead) atomicOr(err, 2);  // generate_ray: pixel outside image
    } else {
      March m;
      ray_from_pixel(cam, poses[f], (double)px, (double)py, m);
      Composite st;
      st.T = 1.0;
      st.C[0] = st.C[1] = st.C[2] = 0.0;
      st.D = 0.0;
      st.count = 0;
      st.terminated = false;
      float bf[9];
      bool basis_ok;
      {
        double basis[9];
        basis_ok = sh_basis(m.d, basis);
#pragma unroll
        for (int mm = 0; mm < 9; ++mm) bf[mm] = (float)basis[mm];
      }
      if (!basis_ok) {
        if (lead) atomicOr(err, 1);
      } else if (march_begin(g, p, m)) {
        Sample s;
        GroupMarch<LPR> gm;
        const int k = sub, dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
        while (gm.next(g, m, s, sub, gbase, gmask)) {
          // this lane's corner: weight (corner_weights order), payload, contraction
          const double wxk = dx ? s.fx : dsub(1.0, s.fx);
          const double wyk = dy ? s.fy : dsub(1.0, s.fy);
          const double wzk = dz ? s.fz : dsub(1.0, s.fz);
          const double wk = dmul(dmul(wxk, wyk), wzk);
          const float4* vp = g.payload + (size_t)corner_index(g, s.base, k) * kVec4PerVertex;
          float v[28];
#pragma unroll
          for (int j = 0; j < kVec4PerVertex; ++j) {
            const float4 a = __ldg(vp + j);
            v[4 * j] = a.x;
            v[4 * j + 1] = a.y;
            v[4 * j + 2] = a.z;
            v[4 * j + 3] = a.w;
          }
          const double pk = dmul(wk, (double)v[0]);
          float dr = 0.f, dg = 0.f, db = 0.f;
#pragma unroll
          for (int mm = 0; mm < 9; ++mm) {
            dr = fmaf(bf[mm], v[1 + mm], dr);
            dg = fmaf(bf[mm], v[10 + mm], dg);
            db = fmaf(bf[mm], v[19 + mm], db);
          }
          const float wkf = (float)wk;
          Shade sh;
          double sraw = 0.0;
          float cr = 0.f, cg = 0.f, cb = 0.f;
#pragma unroll
          for (int j = 0; j < LPR; ++j) {  // corner order, identical on every lane
            sraw = dadd(sraw, __shfl_sync(gmask, pk, gbase + j));
            const float wj = __shfl_sync(gmask, wkf, gbase + j);
            cr = fmaf(wj, __shfl_sync(gmask, dr, gbase + j), cr);
            cg = fmaf(wj, __shfl_sync(gmask, dg, gbase + j), cg);
            cb = fmaf(wj, __shfl_sync(gmask, db, gbase + j), cb);
          }
          sh.sigma_raw = sraw;
          const float col[3] = {cr, cg, cb};
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const double cv = 0.5 + (double)col[ch];
            sh.clamped[ch] = (cv <= 0.0 || cv >= 1.0);
            sh.c[ch] = (cv < 0.0) ? 0.0 : ((1.0 < cv) ? 1.0 : cv);
          }
          double decay;
          const double wgt = composite_step(st, sh, s.t, s.delta, p.eps, decay);
          if (lead && st.count <= K) {
            store_record(rec, rec_index(t, st.count - 1, K), wgt, sh, s.cx, s.cy, s.cz, s.t);
          }
          if (st.terminated) break;
        }
      }
      if (st.count == 0) {
        st.C[0] = st.C[1] = st.C[2] = 0.0;
        st.D = 0.0;
      }
      const double4 tg = rgbd[(long long)f * cam.width * cam.height + (long long)py * cam.width + px];
      if (st.count > 0) {
        fl |= kHit;
        if (st.count > K) fl |= kOverflow;
        stored = st.count > K ? 0 : st.count;
        tfin = (float)st.T;
        mc = 1;
        samples = st.count;
        const double r0 = dsub(st.C[0], tg.x), r1 = dsub(st.C[1], tg.y), r2 = dsub(st.C[2], tg.z);
        const double sq = dadd(dadd(dmul(r0, r0), dmul(r1, r1)), dmul(r2, r2));
        if (!isfinite(sq) || !isfinite(st.D)) {
          bad = i;
        } else {
          lp = sq;
          if (tg.w > 0.0) {
            fl |= kDepthValid;
            md = 1;
            const double dr = dsub(st.D, tg.w);
            lg = dmul(dr, dr);
          }
        }
      }
      if (lead) ray_cd[i] = make_double4(st.C[0], st.C[1], st.C[2], st.D);
    }
    if (lead) {
      flags[i] = fl;
      rec_count[t] = make_int2(stored, __float_as_int(tfin));
    }
  }
  if (!lead) {  // one contribution per ray
    lp = lg = 0.0;
    samples = 0;
    mc = md = 0;
    bad = INT_MAX;
  }
  const double blp = block_sum(lp, s_d);
  const double blg = block_sum(lg, s_d);
  const long long bs = block_sum(samples, s_l);
  const int bmc = block_sum(mc, s_i);
  const int bmd = block_sum(md, s_i);
  const int bbad = block_min(bad, s_i);
  const int bmax = -block_min(-(int)samples, s_i);
  if (threadIdx.x == 0) {
    MapPartial q;
    q.lp = blp;
    q.lg = blg;
    q.samples = bs;
    q.m_c = bmc;
    q.m_d = bmd;
    q.bad = bbad;
    q.max_count = bmax;
    partials[blockIdx.x] = q;
  }
}

// ---- per-ray corner aggregation (all K2 variants)
// The 28-slot upstream of a sample is [dL/dsigma, dcol_ch * basis_m], and the SH
// basis is constant along a ray, so the contribution to corner k over any run of
// samples factorises into a[0][k] = sum w_k up_sigma and a[1+ch][k] = sum w_k
// dcol_ch (clamp-gated): 32 registers instead of 224. A corner is flushed
// (expanded to 28 slots and reduced into the gradient) only when the ray leaves
// it. The corners a move to a neighbouring cell (face, edge or vertex adjacent)
// keeps are carried, and carried by RELABELLING rather than by moving registers:
// logical corner k of the current cell lives in register slot k ^ X. A shared
// vertex's corner labels in the two cells differ exactly in the bits of the
// moved axes, so a move along the axis mask M flushes the departing slots and
// sets X ^= M; the trilinear weights follow by swapping each axis' (1 - f, f)
// pair where X has the bit. Every move direction runs the same straight-line
// code. (r01 moved the registers with one shift routine per direction; a warp
// ran those variants one after another: ~35 warp instructions per sample at 15
// active lanes, ncu v23.)
struct CornerAgg {
  float a[4][8];  // slot s: logical corner s ^ X of the current cell
  uint32_t nz;    // slots that may hold a nonzero sum (free-space samples add zeros)
  uint32_t X;
  uint32_t base;  // vertex_index of the current cell; kNoCell before the first
  int cx, cy, cz;
};
constexpr uint32_t kNoCell = 0xffffffffu;

__device__ __forceinline__ void agg_init(CornerAgg& A) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int k = 0; k < 8; ++k) A.a[c][k] = 0.f;
  A.nz = 0;
  A.X = 0;
  A.base = kNoCell;
  A.cx = A.cy = A.cz = 0;
}

// Vertex offset of logical corner k from the cell's base vertex (corner_index).
__device__ __forceinline__ uint32_t corner_off(const DevGrid& g, uint32_t k) {
  return (k & 1u) + ((k >> 1) & 1u) * (uint32_t)g.rx + (k >> 2) * g.rxy;
}

// Flushes the slots in `slots` (bit s = slot s) to the sink and zeroes them.
template <typename Sink>
__device__ __forceinline__ void agg_flush(CornerAgg& A, Sink& sink, const DevGrid& g,
                                          uint32_t slots) {
  // all-zero corners add nothing and are not flushed: a slot is nonzero only if a
  // sample with a nonzero upstream reached it since it was last flushed (free-
  // space samples with sigma_raw <= 0 carry w = 0 and a gated dL/dsigma)
  const uint32_t live = slots & A.nz;
  A.nz &= ~slots;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    if (live & (1u << s)) {
      sink(A.base + corner_off(g, (uint32_t)s ^ A.X), A.a[0][s], A.a[1][s], A.a[2][s],
           A.a[3][s]);
      A.a[0][s] = A.a[1][s] = A.a[2][s] = A.a[3][s] = 0.f;
    }
  }
}

// The ray's next sample is in cell s: flush what it leaves, relabel what it keeps.
// Returns true when the cell changed.
template <typename Sink>
__device__ __forceinline__ bool agg_enter(CornerAgg& A, Sink& sink, const DevGrid& g,
                                          const Sample& s) {
  if (s.base == A.base) return false;
  if (A.base != kNoCell) {
    const int dx = s.cx - A.cx, dy = s.cy - A.cy, dz = s.cz - A.cz;
    uint32_t dep = 0xffu, M = 0;
    if (dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 && dz <= 1) {
      // departing logical corners: bit = 0 on an axis moved up, 1 on one moved
      // down; in slot terms the per-axis half-masks swap where X has the bit
      dep = 0;
      if (dx != 0) dep |= ((A.X & 1u) ^ (uint32_t)(dx < 0)) ? 0xAAu : 0x55u;
      if (dy != 0) dep |= (((A.X >> 1) & 1u) ^ (uint32_t)(dy < 0)) ? 0xCCu : 0x33u;
      if (dz != 0) dep |= (((A.X >> 2) & 1u) ^ (uint32_t)(dz < 0)) ? 0xF0u : 0x0Fu;
      M = (uint32_t)(dx != 0) | ((uint32_t)(dy != 0) << 1) | ((uint32_t)(dz != 0) << 2);
    }
    agg_flush(A, sink, g, dep);
    A.X ^= M;
  }
  A.base = s.base;
  A.cx = s.cx;
  A.cy = s.cy;
  A.cz = s.cz;
  return true;
}

// Adds a sample's (u_sigma, u_r, u_g, u_b) with trilinear weights (fx, fy, fz).
__device__ __forceinline__ void agg_add(CornerAgg& A, float fx, float fy, float fz, float u0,
                                        float u1, float u2, float u3) {
  if (u0 != 0.f || u1 != 0.f || u2 != 0.f || u3 != 0.f) A.nz = 0xffu;
  const bool sx = A.X & 1u, sy = (A.X >> 1) & 1u, sz = (A.X >> 2) & 1u;
  const float gx = 1.f - fx, gy = 1.f - fy, gz = 1.f - fz;
  const float wx[2] = {sx ? fx : gx, sx ? gx : fx};
  const float wy[2] = {sy ? fy : gy, sy ? gy : fy};
  const float wz[2] = {sz ? fz : gz, sz ? gz : fz};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float wk = wx[k & 1] * wy[(k >> 1) & 1] * wz[(k >> 2) & 1];
    A.a[0][k] = fmaf(wk, u0, A.a[0][k]);
    A.a[1][k] = fmaf(wk, u1, A.a[1][k]);
    A.a[2][k] = fmaf(wk, u2, A.a[2][k]);
    A.a[3][k] = fmaf(wk, u3, A.a[3][k]);
  }
}

#ifndef VRF_RED_HINT
#define VRF_RED_HINT 1  // reductions at L2 evict-last priority (r02: K2 10.96 -> 10.80 ms)
#endif
// One vertex's 7 float4 reductions into the gradient. With VRF_RED_HINT they carry
// an L2 evict-last policy: the gradient lines stay resident against the
// streaming sample records.
__device__ __forceinline__ void red_vertex(float4* dst, const float (&x)[28]) {
#if VRF_RED_HINT
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
  for (int j = 0; j < kVec4PerVertex; ++j)
    asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;"
                 :: "l"(dst + j), "f"(x[4 * j]), "f"(x[4 * j + 1]), "f"(x[4 * j + 2]),
                    "f"(x[4 * j + 3]), "l"(pol)
                 : "memory");
#else
#pragma unroll
  for (int j = 0; j < kVec4PerVertex; ++j)
    atomicAdd(dst + j, make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]));
#endif
}

// Direct scatter of a flushed corner: basis expansion + 7 red.global.add.v4.f32.
struct RedSink {
  float4* __restrict__ grad;
  const float* bf;  // the ray's SH basis (9)
  __device__ __forceinline__ void operator()(uint32_t v, float s, float r, float gg, float b) {
    float4* dst = grad + (size_t)v * kVec4PerVertex;
    float x[28];
    x[0] = s;
#pragma unroll
    for (int mm = 0; mm < 9; ++mm) {
      x[1 + mm] = r * bf[mm];
      x[10 + mm] = gg * bf[mm];
      x[19 + mm] = b * bf[mm];
    }
    red_vertex(dst, x);
  }
};

// Fast-path backward of one ray (fp32 SH, fp32 gradient accumulation) by
// re-marching it: the rays the record buffer could not hold (kOverflow) and the
// record-free configuration (vrf_set_record_limits(max_k = 0)). Same schedule,
// sigma_raw replay, T and termination as the forward pass (all FP64, reference
// order), so exactly the forward's samples are visited. The colour / depth terms
// of dL/dsigma_i use the running form
//   sum_ch upc_ch (c_ch T_{i+1} - C_ch + prefix_ch) = uc_i T_{i+1} + Q_i,
//   Q_i = sum_ch upc_ch (prefix_ch,i - C_ch),  uc_i = sum_ch upc_ch c_ch,i
// (gradients.cpp:69-97 regrouped), which keeps 3 FP64 scalars live instead of 11.
template <bool SKIP>
__device__ __forceinline__ void map_backward_fast(const DevGrid& g, const DevParams& p, March& m,
                                                  const MapUp& u, float4* __restrict__ grad) {
  float bf[9];
  {
    double basis[9];
    if (!sh_basis(m.d, basis)) return;
#pragma unroll
    for (int mm = 0; mm < 9; ++mm) bf[mm] = (float)basis[mm];
  }
  if (!march_begin(g, p, m)) return;
  const double upc0 = u.upc[0], upc1 = u.upc[1], upc2 = u.upc[2];
  const bool use_depth = u.use_depth;
  const double upd = use_depth ? u.upd : 0.0;
  double T = 1.0;
  double Q = -(upc0 * u.C[0] + upc1 * u.C[1] + upc2 * u.C[2]);
  double Qd = -upd * u.D;
  CornerAgg A;
  agg_init(A);
  int last_tb = -1;
  RedSink sink{grad, bf};
  Sample s;
  while (march_next<SKIP>(g, m, s)) {
    Shade sh;
    {
      double w[8];
      corner_weights(s, w);
      shade_fast(g, s, w, bf, sh);
    }
    const double sigma = (sh.sigma_raw < 0.0) ? 0.0 : sh.sigma_raw;
    const double decay = exp(dmul(-sigma, s.delta));
    const double wgt = dmul(T, dsub(1.0, decay));
    const double T_next = dmul(T, decay);
    const double uc = upc0 * sh.c[0] + upc1 * sh.c[1] + upc2 * sh.c[2];
    Q += uc * wgt;
    double ds = uc * T_next + Q;
    if (use_depth) {
      Qd += upd * (s.t * wgt);
      ds += upd * (s.t * T_next) + Qd;
    }
    ds *= s.delta;
    if (agg_enter(A, sink, g, s)) mark_touched(g, s.cx, s.cy, s.cz, last_tb);
    const float wf = (float)wgt;
    agg_add(A, (float)s.fx, (float)s.fy, (float)s.fz, sh.sigma_raw > 0.0 ? (float)ds : 0.f,
            sh.clamped[0] ? 0.f : (float)upc0 * wf, sh.clamped[1] ? 0.f : (float)upc1 * wf,
            sh.clamped[2] ? 0.f : (float)upc2 * wf);
    T = T_next;
    if (T < p.eps) break;
  }
  if (A.base != kNoCell) agg_flush(A, sink, g, 0xffu);
}

template <bool SKIP>
__global__ void __launch_bounds__(kThreads, 4) k_map_backward(
    DevGrid g, DevParams p, DevCam cam, const double4* __restrict__ rgbd,
    const DevPose* __restrict__ poses, const int* __restrict__ batch, int n,
    const double4* __restrict__ ray_cd, const uint8_t* __restrict__ flags,
    const MapStats* __restrict__ stats, const int* __restrict__ global_counts,
    float4* __restrict__ grad, double lambda_d, const uint32_t* __restrict__ order,
    bool overflow_only) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int i = order ? (int)order[t] : t;  // coherent (keyframe, Morton tile) ray order
  const MapStats st = *stats;
  if (st.bad != INT_MAX) return;  // non-finite loss: the reference throws before updating
  const uint8_t fl = flags[i];
  if (!(fl & kHit)) return;
  if (overflow_only && !(fl & kOverflow)) return;  // recorded rays: K2q / K2g
  const int f = batch[3 * i], px = batch[3 * i + 1], py = batch[3 * i + 2];
  const double4 tg = rgbd[(long long)f * cam.width * cam.height + (long long)py * cam.width + px];
  MapUp u;
  if (!map_upstream(st, global_counts, ray_cd[i], tg, fl, lambda_d, u)) return;
  March m;
  ray_from_pixel(cam, poses[f], (double)px, (double)py, m);
  map_backward_fast<SKIP>(g, p, m, u, grad);
}

// The ray as the record walk needs it (fp32): origin, direction, segment end
// and step, and the grid origin / inverse voxel for the trilinear weights.
struct WalkRay {
  float o[3], d[3];
  float hi, step;
};
__device__ __forceinline__ WalkRay walk_ray(const March& m) {
  WalkRay w;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    w.o[a] = (float)m.o[a];
    w.d[a] = (float)m.d[a];
  }
  w.hi = (float)m.hi;
  w.step = (float)m.step;
  return w;
}

// One record of the reverse walk, decoded. The cell comes from the record (the
// forward located it in FP64 with the reference's arithmetic), so the scatter
// targets exactly the forward's corners; the trilinear weights are re-derived in
// fp32 from the stored segment midpoint (weight error ~1e-5, far inside the fast
// path's 1e-3 gradient bar), and delta is the step except on the segment
// clipped at t_far, where s1 = hi gives delta = 2 (hi - t_mid).
struct RecSample {
  int cx, cy, cz;
  uint32_t base;
  float fx, fy, fz;
  float tm, delta, w, c0, c1, c2;
  uint32_t kf;
};
__device__ __forceinline__ void decode_record(const DevGrid& g, const WalkRay& m, float4 q0,
                                              uint2 q1, RecSample& r) {
  r.w = q0.x;
  r.c0 = fabsf(q0.y);
  r.c1 = fabsf(q0.z);
  r.c2 = fabsf(q0.w);
  r.kf = (q1.x & kRecSigmaPos) | (__float_as_uint(q0.y) >> 31) |
         ((__float_as_uint(q0.z) >> 31) << 1) | ((__float_as_uint(q0.w) >> 31) << 2);
  const uint32_t cell = q1.x;
  r.tm = __uint_as_float(q1.y);
  r.cx = (int)(cell & 1023u);
  r.cy = (int)((cell >> 10) & 1023u);
  r.cz = (int)((cell >> 20) & 1023u);
  r.base = (uint32_t)r.cx + (uint32_t)g.rx * ((uint32_t)r.cy + (uint32_t)g.ry * (uint32_t)r.cz);
  r.delta = fminf(m.step, 2.f * (m.hi - r.tm));
  const float iv = (float)g.rcp_voxel;
  const float gx = (fmaf(r.tm, m.d[0], m.o[0]) - (float)g.ox) * iv;
  const float gy = (fmaf(r.tm, m.d[1], m.o[1]) - (float)g.oy) * iv;
  const float gz = (fmaf(r.tm, m.d[2], m.o[2]) - (float)g.oz) * iv;
  r.fx = fminf(fmaxf(gx - (float)r.cx, 0.f), 1.f);
  r.fy = fminf(fmaxf(gy - (float)r.cy, 0.f), 1.f);
  r.fz = fminf(fmaxf(gz - (float)r.cz, 0.f), 1.f);
}

__device__ __forceinline__ void load_record(RecBuf rec, int t, int c, int K, float4& q0,
                                            uint2& q1) {
  const size_t i = rec_index(t, c, K);
#if VRF_REC_HINT & 2
  const unsigned long long pol = evict_first_policy();
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
      : "=f"(q0.x), "=f"(q0.y), "=f"(q0.z), "=f"(q0.w) : "l"(rec.a + i), "l"(pol));
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
      : "=r"(q1.x), "=r"(q1.y) : "l"(rec.b + i), "l"(pol));
#else
  q0 = __ldg(rec.a + i);
  q1 = __ldg(rec.b + i);
#endif
}

// The walk's cell as the corner aggregation sees it.
__device__ __forceinline__ Sample rec_cell(const RecSample& r) {
  Sample s{};
  s.base = r.base;
  s.cx = r.cx;
  s.cy = r.cy;
  s.cz = r.cz;
  return s;
}

// Suffix-form sample upstream of the reverse walk (see K2q) and the aggregate
// update; Sc / Sd advance past the sample (fp32: the fast path's precision).
// Tn = T_{i+1} of this sample on entry (the walk starts from the ray's final T)
// and T_i on exit: T_i = T_{i+1} + w_i (renderer.cpp's w_i = T_i alpha_i,
// T_{i+1} = T_i (1 - alpha_i)).
__device__ __forceinline__ void walk_sample(CornerAgg& A, const RecSample& r, float upc0,
                                            float upc1, float upc2, float upd, float& Sc0,
                                            float& Sc1, float& Sc2, float& Sd, float& Tn) {
  float ds = upc0 * (r.c0 * Tn - Sc0) + upc1 * (r.c1 * Tn - Sc1) + upc2 * (r.c2 * Tn - Sc2);
  ds = fmaf(upd, r.tm * Tn - Sd, ds);
  ds *= r.delta;
  Sc0 = fmaf(r.c0, r.w, Sc0);
  Sc1 = fmaf(r.c1, r.w, Sc1);
  Sc2 = fmaf(r.c2, r.w, Sc2);
  Sd = fmaf(r.tm, r.w, Sd);
  Tn += r.w;
  agg_add(A, r.fx, r.fy, r.fz, (r.kf & kRecSigmaPos) ? ds : 0.f,
          (r.kf & 1u) ? 0.f : upc0 * r.w, (r.kf & 2u) ? 0.f : upc1 * r.w,
          (r.kf & 4u) ? 0.f : upc2 * r.w);
}

// K2g: the record walk for small batches, 8 lanes per ray. Below ~40K rays the
// thread-per-ray K2 runs one warp per SM sub-partition or less and each ray's
// ~200 records are a serial chain. Here the ray's records are split into 8
// contiguous chunks. Pass 1: every lane sums its chunk's c_ch w and t w. A
// shuffle suffix-scan gives each lane the sums of the records after its chunk
// (the starting Sc / Sd of the reverse walk). Pass 2: every lane walks its chunk
// backwards exactly as K2q does (suffix-form dL/dsigma, per-lane corner
// aggregation, relabelled carries, red.v4 flushes; chunk ends flush their
// cell). Same gradient up to fp32 summation order.
__global__ void __launch_bounds__(kThreads) k_map_backward_g(
    DevGrid g, DevParams p, DevCam cam, const double4* __restrict__ rgbd,
    const DevPose* __restrict__ poses, const int* __restrict__ batch, int n,
    const double4* __restrict__ ray_cd, const uint8_t* __restrict__ flags,
    const MapStats* __restrict__ stats, const int* __restrict__ global_counts,
    float4* __restrict__ grad, double lambda_d, const uint32_t* __restrict__ order,
    RecBuf rec, int K, const int2* __restrict__ rec_count) {
  constexpr int LPR = 8;
  const int lane = threadIdx.x & 31, sub = lane & (LPR - 1), gbase = lane & ~(LPR - 1);
  const unsigned gmask = ((1u << LPR) - 1u) << gbase;
  const int t = blockIdx.x * (kThreads / LPR) + threadIdx.x / LPR;
  if (t >= n) return;  // group-uniform
  const int i = order ? (int)order[t] : t;
  const MapStats st = *stats;
  if (st.bad != INT_MAX) return;
  const uint8_t fl = flags[i];
  if (!(fl & kHit) || (fl & kOverflow)) return;
  const int f = batch[3 * i], px = batch[3 * i + 1], py = batch[3 * i + 2];
  const double4 tg = rgbd[(long long)f * cam.width * cam.height + (long long)py * cam.width + px];
  MapUp u;
  if (!map_upstream(st, global_counts, ray_cd[i], tg, fl, lambda_d, u)) return;
  March m;
  ray_from_pixel(cam, poses[f], (double)px, (double)py, m);
  float bf[9];
  {
    double basis[9];
    if (!sh_basis(m.d, basis)) return;
#pragma unroll
    for (int mm = 0; mm < 9; ++mm) bf[mm] = (float)basis[mm];
  }
  if (!march_begin(g, p, m)) return;
  const WalkRay wr = walk_ray(m);
  const int2 rc = rec_count[t];
  const int cnt = rc.x;
  const int L = (cnt + LPR - 1) / LPR;
  const int c0 = sub * L, c1 = min(cnt, c0 + L);  // this lane's records [c0, c1)
  // pass 1: chunk sums of c_ch w and t w
  float P0 = 0.f, P1 = 0.f, P2 = 0.f, Pd = 0.f, Pw = 0.f;
  for (int c = c0; c < c1; ++c) {
    float4 q0;
    uint2 q1;
    load_record(rec, t, c, K, q0, q1);
    P0 = fmaf(fabsf(q0.y), q0.x, P0);
    P1 = fmaf(fabsf(q0.z), q0.x, P1);
    P2 = fmaf(fabsf(q0.w), q0.x, P2);
    Pd = fmaf(__uint_as_float(q1.y), q0.x, Pd);
    Pw += q0.x;
  }
  // suffix sums of the later chunks (lanes sub+1 .. 7)
  // (and T_{i+1} of the chunk's last record: the ray's final T plus the
  // weights of the later chunks)
  float Sc0 = 0.f, Sc1 = 0.f, Sc2 = 0.f, Sd = 0.f, Tn = __int_as_float(rc.y);
#pragma unroll
  for (int j = LPR - 1; j > 0; --j) {
    const float a0 = __shfl_sync(gmask, P0, gbase + j), a1 = __shfl_sync(gmask, P1, gbase + j);
    const float a2 = __shfl_sync(gmask, P2, gbase + j), ad = __shfl_sync(gmask, Pd, gbase + j);
    const float aw = __shfl_sync(gmask, Pw, gbase + j);
    if (j > sub) {
      Sc0 += a0;
      Sc1 += a1;
      Sc2 += a2;
      Sd += ad;
      Tn += aw;
    }
  }
  const float upd = u.use_depth ? (float)u.upd : 0.f;
  CornerAgg A;
  agg_init(A);
  int last_tb = -1;
  RedSink sink{grad, bf};
  for (int c = c1 - 1; c >= c0; --c) {
    float4 q0;
    uint2 q1;
    load_record(rec, t, c, K, q0, q1);
    RecSample r;
    decode_record(g, wr, q0, q1, r);
    if (agg_enter(A, sink, g, rec_cell(r))) mark_touched(g, r.cx, r.cy, r.cz, last_tb);
    walk_sample(A, r, (float)u.upc[0], (float)u.upc[1], (float)u.upc[2], upd, Sc0, Sc1, Sc2, Sd,
                Tn);
  }
  if (A.base != kNoCell) agg_flush(A, sink, g, 0xffu);
}

// K2q (default): the reverse record walk with a DEFERRED, convergent scatter.
// Walking each ray's samples last to first turns the prefix form of
// gradients.cpp:69-97 into a suffix form without cancellation,
// -C + prefix_i = -sum_{j>i} c_j w_j:
//   dL/dsigma_i = delta_i [sum_ch upc_ch (c_ch,i T_{i+1} - Sc_ch) + upd (t_i T_{i+1} - Sd)],
// Sc / Sd the running suffix sums; no payload is gathered. The reverse walk also
// staggers the lanes of a warp along their rays, so neighbouring rays do not hit
// the same vertices with atomics at the same time (forward order measured 10%
// slower, r01). A cell the ray leaves is only stored, as one record of its 8
// aggregated corner slots, in the lane's ring in shared memory (the cell-record
// ring below, default since r02; VRF_K2_RING=0 is r01's per-corner entry ring);
// every iteration each lane then pops up to POPS corners and scatters them after
// the warp reconverges, merging same-round duplicates (pop_entry). The
// reductions carry an L2 evict-last policy (red_vertex). The loop runs until
// every lane of the warp has finished its ray AND drained its ring (warp-uniform
// exit; lanes without a ray help drain).
#ifndef VRF_K2_MERGE
#define VRF_K2_MERGE 3  // same-round duplicate merging: 1 leader sums expanded vectors, 3 factor-domain
#endif
#ifndef VRF_K2_POP2
#define VRF_K2_POP2 0  // A/B: load both pops' queue entries up front
#endif
#ifndef VRF_K2_SYNC_ACT
#define VRF_K2_SYNC_ACT 1  // merge synchronised over all popping lanes (r02: 10.80 -> 10.39 ms)
#endif
#ifndef VRF_K2_STAGE2
#define VRF_K2_STAGE2 0  // A/B: double-buffered merge staging, one barrier per round (no gain, r02)
#endif
#ifndef VRF_K2_MERGE_PIPE
#define VRF_K2_MERGE_PIPE 0  // A/B: software-pipelined merge loop (slower, r02)
#endif
#ifndef VRF_K2_POPS
#define VRF_K2_POPS 2  // pop rounds per walk step
#endif
#ifndef VRF_K2_GROUP_MAX
#define VRF_K2_GROUP_MAX 32  // largest merged duplicate group (A/B knob)
#endif
#ifndef VRF_K2_PROBE_NORED
#define VRF_K2_PROBE_NORED 0  // timing probe builds only (tools/ab/k2_probe.sh)
#endif
#ifndef VRF_K2_MERGE_MIN
#define VRF_K2_MERGE_MIN 2  // smallest duplicate group merged before the reduction
#endif
#ifndef VRF_K2_MINB
#define VRF_K2_MINB 4  // CTAs per SM: 128 registers (config 3, r02: 10.39 vs 10.87 ms at 3)
#endif
constexpr int kQ = 16;  // ring entries per thread (power of 2); a step enqueues <= 8
constexpr int kQSmemBytes = kQ * kThreads * (16 + 4);
constexpr int kQMergeSmemBytes = kQSmemBytes + kThreads * kVec4PerVertex * 16;
// Per-warp vertex cache of K2q (VRF_K2_VCACHE=1). The 32 coherent rays of a
// warp span one or two voxels at room depths, so each vertex is flushed by many
// of its lanes over a few iterations, mostly in different pop rounds (where the
// same-round merge cannot see them). The warp keeps kVCache recently flushed
// vertices' 28 sums in shared memory (hashed slots, one owner per slot and
// round) and reduces an entry into the gradient only when its slot is taken
// by another vertex, and at the end of the kernel.
#ifndef VRF_K2_VCACHE
#define VRF_K2_VCACHE 0
#endif
constexpr int kVCache = 28;
// the warp's staging region (float4 units): [0, 32) member factors, then the
// lanes' SH bases (12 floats each, 96 float4); with the cache, its entries
// (kVCache x 7 float4) and tags (kVCache u32) follow
constexpr int kSbfOff = VRF_K2_VCACHE ? 32 : 32 * kVec4PerVertex - 32 * 3;
// (MERGE 4 stages up to 15 holder rows of 7 float4 below kSbfOff = 128)
static_assert(VRF_K2_MERGE != 4 || 16 * kVec4PerVertex <= kSbfOff, "merge-4 rows overlap the bases");
constexpr int kVCacheOff = 128;
constexpr int kWarpStage =
    VRF_K2_VCACHE ? kVCacheOff + kVCache * kVec4PerVertex + kVCache / 4 : 32 * kVec4PerVertex;
static_assert(kVCache % 4 == 0, "tags fill whole float4");
static_assert(!VRF_K2_STAGE2 || (!VRF_K2_VCACHE && VRF_K2_MERGE == 3 && VRF_K2_SYNC_ACT),
              "the second staging buffer uses the factor-merge layout's free rows [32, 64)");
static_assert(!VRF_K2_VCACHE || VRF_K2_MERGE == 3, "the vertex cache sits in the factor-merge layout");
struct QueueSink {
  uint32_t* qv;  // [kQ][kThreads] vertex ids
  float4* qa;    // [kQ][kThreads] (a_sigma, a_r, a_g, a_b)
  int tid;
  uint32_t tail;
  __device__ __forceinline__ void operator()(uint32_t v, float s, float r, float gg, float b) {
    const int slot = (int)(tail & (kQ - 1)) * kThreads + tid;
    qv[slot] = v;
    qa[slot] = make_float4(s, r, gg, b);
    ++tail;
  }
};

#ifndef VRF_K2_GSTATS
#define VRF_K2_GSTATS 0
#endif
#if VRF_K2_GSTATS
__device__ unsigned long long g_k2_gsize[33], g_k2_rmax[33];
#endif
// One pop round: the lane's oldest queued corner. The ~28 lanes popping together
// often hold the same vertex (33% of pops duplicate another lane's vertex in the
// same round, r01 counters): lanes popping the same vertex are grouped
// (__match_any_sync), members stage their expanded 28-vector in the warp's shared
// buffer, and the leader sums the group and issues the only 7 red.v4. This cuts
// the L2 reductions by a third; at config 4, where the 15 GB gradient misses L2,
// it saves DRAM read-modify-writes (K2 29.3 -> 25.7 ms, r01).
// One merged pop of the entry (v, e) the caller loaded (has: the lane popped).
__device__ __forceinline__ void pop_entry(bool has, uint32_t v, float4 e,
                                          float4* __restrict__ grad, const float (&bf)[9],
                                          float4* stage, int buf = 0) {
  if (has) {
    const unsigned act = __activemask();
#if VRF_K2_MERGE_MIN > 2
    // A/B: groups smaller than VRF_K2_MERGE_MIN reduce lane by lane
    unsigned grp = __match_any_sync(act, v);
    if (__popc(grp) < VRF_K2_MERGE_MIN) grp = 1u << (threadIdx.x & 31);
#elif VRF_K2_GROUP_MAX < 32
    // A/B: duplicate groups split into sub-groups of at most VRF_K2_GROUP_MAX
    // lanes (bounds the serial leader loop; each sub-group reduces separately)
    unsigned grp = __match_any_sync(act, v);
    if (__popc(grp) > VRF_K2_GROUP_MAX) {
      const unsigned below = grp & ((1u << (threadIdx.x & 31)) - 1u);
      const unsigned long long key =
          ((unsigned long long)v << 8) | (unsigned)(__popc(below) / VRF_K2_GROUP_MAX);
      grp = __match_any_sync(grp, key);
    }
#else
    const unsigned grp = __match_any_sync(act, v);
#endif
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(grp) - 1;
#if VRF_K2_GSTATS
    // diagnostic build: histogram of duplicate-group sizes (one count per group)
    // and of each pop round's largest group (the merge loop's trip count + 1)
    {
      if (lane == leader) atomicAdd(&g_k2_gsize[__popc(grp)], 1ull);
      const unsigned mx = __reduce_max_sync(act, (unsigned)__popc(grp));
      if (lane == __ffs(act) - 1) atomicAdd(&g_k2_rmax[mx], 1ull);
    }
#endif
    float x[28];
    x[0] = e.x;
#pragma unroll
    for (int mm = 0; mm < 9; ++mm) {
      x[1 + mm] = e.y * bf[mm];
      x[10 + mm] = e.z * bf[mm];
      x[19 + mm] = e.w * bf[mm];
    }
#if VRF_K2_MERGE == 4
    // Pairwise-first merge (A/B). r02 counters (tools/k2_groups.py, config 3):
    // 58 % of pops sit in duplicate groups, a pop round's largest group has
    // 3-4 lanes at the median, and the leader loop below ran 3.2 trips per
    // round on 3 active lanes. Here level 1 runs every pair of a group at once
    // in the factor domain (rank 2j absorbs rank 2j+1), and the leader then sums
    // the surviving even-ranked partial sums as expanded vectors: a group of k
    // costs 1 + ceil(k/2) - 1 serial steps instead of k - 1.
    {
      const unsigned below = grp & ((1u << lane) - 1u);
      const int rank = __popc(below);
      const bool multi = grp != (1u << lane);
      float4* stage_e = stage;  // [32] member factors
      if (multi && (rank & 1)) stage_e[lane] = e;
      __syncwarp(act);
      if (multi && !(rank & 1)) {
        const unsigned above = grp & ~((2u << lane) - 1u);
        if (above) {  // the next lane of the group is this lane's odd partner
          const int o = __ffs(above) - 1;
          const float* sb = reinterpret_cast<const float*>(stage + kSbfOff) + 12 * o;
          const float4 eo = stage_e[o], b0 = reinterpret_cast<const float4*>(sb)[0],
                       b1 = reinterpret_cast<const float4*>(sb)[1];
          const float bb[9] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, sb[8]};
          x[0] += eo.x;
#pragma unroll
          for (int mm = 0; mm < 9; ++mm) {
            x[1 + mm] = fmaf(eo.y, bb[mm], x[1 + mm]);
            x[10 + mm] = fmaf(eo.z, bb[mm], x[10 + mm]);
            x[19 + mm] = fmaf(eo.w, bb[mm], x[19 + mm]);
          }
        }
      }
      // level 2: even ranks >= 2 hold partial sums for their group's leader
      const bool holder = multi && !(rank & 1) && rank >= 2;
      const unsigned hm = __ballot_sync(act, holder);
      const bool any2 = hm != 0u;  // warp-uniform
      if (any2) {
        __syncwarp(act);  // the factor rows are read; their space is reused
        if (holder) {
          float4* row = stage + __popc(hm & ((1u << lane) - 1u)) * kVec4PerVertex;
#pragma unroll
          for (int j = 0; j < kVec4PerVertex; ++j)
            row[j] = make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
        }
        __syncwarp(act);
        if (lane == leader) {
          unsigned rest = grp & hm;
          while (rest) {
            const int o = __ffs(rest) - 1;
            rest &= rest - 1;
            const float4* row = stage + __popc(hm & ((1u << o) - 1u)) * kVec4PerVertex;
#pragma unroll
            for (int j = 0; j < kVec4PerVertex; ++j) {
              const float4 y = row[j];
              x[4 * j] += y.x;
              x[4 * j + 1] += y.y;
              x[4 * j + 2] += y.z;
              x[4 * j + 3] += y.w;
            }
          }
        }
      }
      __syncwarp(act);
    }
    if (false) {
#elif VRF_K2_MERGE == 3 && VRF_K2_SYNC_ACT
    // (the same merge as below, synchronised over all popping lanes: one
    // warp-uniform mask, so WARPSYNC needs no per-group collective emulation)
    {
      const bool multi = grp != (1u << lane);
      // VRF_K2_STAGE2: consecutive pop rounds alternate between two staging
      // buffers, and the loop's full-warp votes separate a buffer's reuse, so
      // the barrier after the leaders' reads is not needed
      float4* stage_e = stage + (VRF_K2_STAGE2 ? 32 * buf : 0);
      if (multi && lane != leader) stage_e[lane] = e;
      __syncwarp(act);
      if (multi && lane == leader) {
        const float4* sbf = stage + kSbfOff;
        unsigned rest = grp & ~(1u << lane);
#if VRF_K2_MERGE_PIPE
        // software-pipelined: the next member's operands load while this one's
        // 27 FMAs run (A/B; needs the registers of a second member)
        int o = __ffs(rest) - 1;
        rest &= rest - 1;
        float4 eo = stage_e[o], b0 = sbf[3 * o], b1 = sbf[3 * o + 1];
        float b8 = sbf[3 * o + 2].x;
        while (true) {
          const bool more = rest != 0;
          const int on = more ? __ffs(rest) - 1 : o;
          rest &= rest - 1;
          const float4 en = stage_e[on], c0 = sbf[3 * on], c1 = sbf[3 * on + 1];
          const float c8 = sbf[3 * on + 2].x;
          const float bb[9] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b8};
          x[0] += eo.x;
#pragma unroll
          for (int mm = 0; mm < 9; ++mm) {
            x[1 + mm] = fmaf(eo.y, bb[mm], x[1 + mm]);
            x[10 + mm] = fmaf(eo.z, bb[mm], x[10 + mm]);
            x[19 + mm] = fmaf(eo.w, bb[mm], x[19 + mm]);
          }
          if (!more) break;
          eo = en;
          b0 = c0;
          b1 = c1;
          b8 = c8;
        }
#else
        while (rest) {
          const int o = __ffs(rest) - 1;
          rest &= rest - 1;
          const float4 eo = stage_e[o], b0 = sbf[3 * o], b1 = sbf[3 * o + 1], b2 = sbf[3 * o + 2];
          const float bb[9] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x};
          x[0] += eo.x;
#pragma unroll
          for (int mm = 0; mm < 9; ++mm) {
            x[1 + mm] = fmaf(eo.y, bb[mm], x[1 + mm]);
            x[10 + mm] = fmaf(eo.z, bb[mm], x[10 + mm]);
            x[19 + mm] = fmaf(eo.w, bb[mm], x[19 + mm]);
          }
        }
#endif
      }
#if !VRF_K2_STAGE2
      __syncwarp(act);
#endif
    }
    if (false) {
#else
    if (grp != (1u << lane)) {
#endif
#if VRF_K2_MERGE == 3
      // factor-domain merge: members stage only their 4 factors; the leader
      // expands each member's factors with that member's SH basis (the warp's
      // s_bf rows) into its own sums
      float4* stage_e = stage;  // [32] of the warp
      if (lane != leader) stage_e[lane] = e;
      __syncwarp(grp);
      if (lane == leader) {
        const float4* sbf = stage + kSbfOff;
        unsigned rest = grp & ~(1u << lane);
        while (rest) {
          const int o = __ffs(rest) - 1;
          rest &= rest - 1;
          const float4 eo = stage_e[o], b0 = sbf[3 * o], b1 = sbf[3 * o + 1], b2 = sbf[3 * o + 2];
          const float bb[9] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x};
          x[0] += eo.x;
#pragma unroll
          for (int mm = 0; mm < 9; ++mm) {
            x[1 + mm] = fmaf(eo.y, bb[mm], x[1 + mm]);
            x[10 + mm] = fmaf(eo.z, bb[mm], x[10 + mm]);
            x[19 + mm] = fmaf(eo.w, bb[mm], x[19 + mm]);
          }
        }
      }
#else
      // leader merge of expanded vectors: members stage their 28-vector, the
      // leader sums the group
      if (lane != leader) {
#pragma unroll
        for (int j = 0; j < kVec4PerVertex; ++j)
          stage[lane * kVec4PerVertex + j] =
              make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
      }
      __syncwarp(grp);
      if (lane == leader) {
        unsigned rest = grp & ~(1u << lane);
        while (rest) {
          const int o = __ffs(rest) - 1;
          rest &= rest - 1;
#pragma unroll
          for (int j = 0; j < kVec4PerVertex; ++j) {
            const float4 y = stage[o * kVec4PerVertex + j];
            x[4 * j] += y.x;
            x[4 * j + 1] += y.y;
            x[4 * j + 2] += y.z;
            x[4 * j + 3] += y.w;
          }
        }
      }
#endif
      __syncwarp(grp);
    }
#if VRF_K2_VCACHE
    // the warp's vertex cache (see kVCache): each leader adds its group's sums
    // into the cached entry for v; a different vertex in that slot is evicted
    // (reduced to the gradient) first. Leaders whose slots collide in this round
    // beyond the first reduce directly.
    const unsigned leaders = __ballot_sync(act, lane == leader);
    if (lane == leader) {
      const uint32_t slot = __umulhi(v * 0x9E3779B1u, (uint32_t)kVCache);
      const unsigned sg = __match_any_sync(leaders, slot);
      float4* ent = stage + kVCacheOff + slot * kVec4PerVertex;
      uint32_t* tag = reinterpret_cast<uint32_t*>(stage + kVCacheOff + kVCache * kVec4PerVertex);
      const bool own = __ffs(sg) - 1 == lane;
      const uint32_t old = own ? tag[slot] : v;
      const bool hit = old == v;
      if (own && !hit) {
        if (old != kNoCell) {
          float4* od = grad + (size_t)old * kVec4PerVertex;
#pragma unroll
          for (int j = 0; j < kVec4PerVertex; ++j) atomicAdd(od + j, ent[j]);
        }
        tag[slot] = v;
      }
      if (own) {
#pragma unroll
        for (int j = 0; j < kVec4PerVertex; ++j) {
          float4 a = make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
          if (hit) {
            const float4 c = ent[j];
            a.x += c.x;
            a.y += c.y;
            a.z += c.z;
            a.w += c.w;
          }
          ent[j] = a;
        }
      } else {
        float4* dst = grad + (size_t)v * kVec4PerVertex;
#pragma unroll
        for (int j = 0; j < kVec4PerVertex; ++j)
          atomicAdd(dst + j, make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]));
      }
    }
#else
    if (lane == leader) {  // (a lone lane is its own leader)
      float4* dst = grad + (size_t)v * kVec4PerVertex;
#if VRF_K2_PROBE_NORED
      // timing probe only (wrong gradient): the reductions replaced by a
      // data-dependent branch that keeps the expansion alive
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < 28; ++j) acc += x[j];
      if (acc == 1234.5f) dst[0] = make_float4(acc, 0.f, 0.f, 0.f);
#else
      red_vertex(dst, x);
#endif
    }
#endif
  }
}

__device__ __forceinline__ void queue_pop_merge(const QueueSink& q, uint32_t& head,
                                                float4* __restrict__ grad, const float (&bf)[9],
                                                float4* stage) {
  const bool has = head != q.tail;
  uint32_t v = 0;
  float4 e = make_float4(0.f, 0.f, 0.f, 0.f);
  if (has) {
    const int slot = (int)(head & (kQ - 1)) * kThreads + q.tid;
    v = q.qv[slot];
    e = q.qa[slot];
    ++head;
  }
  pop_entry(has, v, e, grad, bf, stage);
}

// Two pops with both entries loaded up front: the second entry's shared-memory
// latency hides behind the first pop (ncu r02: short-scoreboard stalls on the
// popped vertex led K2's stall reasons).
__device__ __forceinline__ void queue_pop_merge2(const QueueSink& q, uint32_t& head,
                                                 float4* __restrict__ grad, const float (&bf)[9],
                                                 float4* stage) {
  const uint32_t n = q.tail - head;
  const bool h0 = n > 0, h1 = n > 1;
  uint32_t v0 = 0, v1 = 0;
  float4 e0 = make_float4(0.f, 0.f, 0.f, 0.f), e1 = e0;
  if (h0) {
    const int s0 = (int)(head & (kQ - 1)) * kThreads + q.tid;
    v0 = q.qv[s0];
    e0 = q.qa[s0];
  }
  if (h1) {
    const int s1 = (int)((head + 1) & (kQ - 1)) * kThreads + q.tid;
    v1 = q.qv[s1];
    e1 = q.qa[s1];
  }
  head += (uint32_t)h0 + (uint32_t)h1;
  pop_entry(h0, v0, e0, grad, bf, stage);
  pop_entry(h1, v1, e1, grad, bf, stage);
}

// ---- K2q cell-record ring (VRF_K2_RING=1, the default). A move stores the departing
// cell's whole aggregate (8 slots x 4 factors, unconditionally: 8 STS.128 at
// full warp) plus a header (base vertex, X, live-slot mask) as one record; pops
// pick the live slots of the oldest record in slot order and derive each
// vertex from the header. The entry ring (QueueSink) instead branches per live
// slot at enqueue (corner offset, ring position, two stores), which ran at ~10
// active lanes and took ~20 % of K2's warp instructions (ncu v11 SASS profile).
// Two records per thread: before every step a lane holds at most one pending
// record, as the entry ring held at most 8 pending entries.
#ifndef VRF_K2_RING
#define VRF_K2_RING 1
#endif
constexpr int kRingRecs = 2;
constexpr int kRingSmemBytes =
    kRingRecs * 8 * kThreads * 16 + kRingRecs * kThreads * 8 + (kThreads / 32) * kWarpStage * 16;
#ifndef VRF_K2_HDR_REG
#define VRF_K2_HDR_REG 1  // the head record's base and X in registers
#endif
struct RingQueue {
  float4* rec;   // [kRingRecs][8][kThreads] slot factors
  uint2* hdr;    // [kRingRecs][kThreads] (base vertex, X | live << 8)
  int tid;
  uint32_t st;   // bits 0-7: unpopped live slots of the head record; bit 8: head
                 // record; bits 9-10: records pending; bit 12: pop-round parity;
                 // bits 16-18: the head's X
#if VRF_K2_HDR_REG
  uint32_t hbase;  // the head record's base vertex
#endif
  __device__ __forceinline__ uint32_t pending() const { return (st >> 9) & 3u; }
};

#ifndef VRF_K2_POP_LOGICAL
#define VRF_K2_POP_LOGICAL 1
#endif
// Slot mask -> logical-corner mask (bit k = slot k ^ X).
__device__ __forceinline__ uint32_t slots_to_corners(uint32_t m, uint32_t X) {
  if (X & 1u) m = ((m & 0x55u) << 1) | ((m & 0xAAu) >> 1);
  if (X & 2u) m = ((m & 0x33u) << 2) | ((m & 0xCCu) >> 2);
  if (X & 4u) m = ((m & 0x0Fu) << 4) | ((m & 0xF0u) >> 4);
  return m;
}

// Stores the aggregate's slots `live` (nonzero) as the lane's next record. The
// record's pop mask is kept in logical-corner order (VRF_K2_POP_LOGICAL), so
// neighbouring rays that leave the same cell pop its corners in the same order
// and meet in the same pop round, where the merge catches them.
__device__ __forceinline__ void ring_push(RingQueue& q, const CornerAgg& A, uint32_t live) {
#if VRF_K2_POP_LOGICAL
  live = slots_to_corners(live, A.X);
#endif
  const uint32_t hr = (q.st >> 8) & 1u, np = q.pending();
  const uint32_t r = hr ^ np;  // np <= 1 here
  float4* d = q.rec + (size_t)r * 8 * kThreads + q.tid;
#pragma unroll
  for (int s = 0; s < 8; ++s) d[s * kThreads] = make_float4(A.a[0][s], A.a[1][s], A.a[2][s], A.a[3][s]);
  q.hdr[r * kThreads + q.tid] = make_uint2(A.base, A.X | (live << 8));
#if VRF_K2_HDR_REG
  if (np == 0) {
    q.st = live | (hr << 8) | (1u << 9) | (A.X << 16) | (q.st & (1u << 12));
    q.hbase = A.base;
  } else {
    q.st += 1u << 9;
  }
#else
  q.st = (np == 0 ? (live | (hr << 8)) : (q.st & 0x1ffu)) | ((np + 1) << 9) | (q.st & (1u << 12));
#endif
}

// Zeroes the slots in `dep` (branch-free selects).
__device__ __forceinline__ void agg_zero(CornerAgg& A, uint32_t dep) {
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const bool z = (dep >> s) & 1u;
#pragma unroll
    for (int c = 0; c < 4; ++c) A.a[c][s] = z ? 0.f : A.a[c][s];
  }
  A.nz &= ~dep;
}

// agg_enter for the record ring.
__device__ __forceinline__ bool ring_enter(CornerAgg& A, RingQueue& q, const DevGrid& g,
                                           const Sample& s) {
  if (s.base == A.base) return false;
  if (A.base != kNoCell) {
    const int dx = s.cx - A.cx, dy = s.cy - A.cy, dz = s.cz - A.cz;
    uint32_t dep = 0xffu, M = 0;
    if (dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 && dz <= 1) {
      dep = 0;
      if (dx != 0) dep |= ((A.X & 1u) ^ (uint32_t)(dx < 0)) ? 0xAAu : 0x55u;
      if (dy != 0) dep |= (((A.X >> 1) & 1u) ^ (uint32_t)(dy < 0)) ? 0xCCu : 0x33u;
      if (dz != 0) dep |= (((A.X >> 2) & 1u) ^ (uint32_t)(dz < 0)) ? 0xF0u : 0x0Fu;
      M = (uint32_t)(dx != 0) | ((uint32_t)(dy != 0) << 1) | ((uint32_t)(dz != 0) << 2);
    }
    const uint32_t live = dep & A.nz;
    if (live) {
      ring_push(q, A, live);
      agg_zero(A, dep);
    }
    A.X ^= M;
  }
  A.base = s.base;
  A.cx = s.cx;
  A.cy = s.cy;
  A.cz = s.cz;
  return true;
}

// One merged pop round over the rings.
__device__ __forceinline__ void ring_pop_merge(RingQueue& q, const DevGrid& g,
                                               float4* __restrict__ grad, const float (&bf)[9],
                                               float4* stage) {
  const bool has = q.pending() != 0;
  uint32_t v = 0;
  float4 e = make_float4(0.f, 0.f, 0.f, 0.f);
#if VRF_K2_STAGE2
  q.st ^= 1u << 12;  // round parity (warp-uniform: every lane runs every round)
#endif
  if (has) {
    const uint32_t pm = q.st & 0xffu, hr = (q.st >> 8) & 1u;
#if VRF_K2_HDR_REG
    const uint2 h = make_uint2(q.hbase, (q.st >> 16) & 7u);
#else
    const uint2 h = q.hdr[hr * kThreads + q.tid];
#endif
#if VRF_K2_POP_LOGICAL
    const uint32_t k = (uint32_t)__ffs(pm) - 1u, sl = k ^ (h.y & 7u);
    v = h.x + corner_off(g, k);
#else
    const uint32_t sl = (uint32_t)__ffs(pm) - 1u;
    v = h.x + corner_off(g, sl ^ (h.y & 7u));
#endif
    e = q.rec[(size_t)(hr * 8 + sl) * kThreads + q.tid];
    const uint32_t rest = pm & (pm - 1);
    if (rest) {
      q.st = (q.st & ~0xffu) | rest;
    } else {
      const uint32_t np = q.pending() - 1, nh = hr ^ 1u;
#if VRF_K2_HDR_REG
      uint2 nx = make_uint2(0u, 0u);
      if (np) nx = q.hdr[nh * kThreads + q.tid];
      q.st = (nx.y >> 8) | (nh << 8) | (np << 9) | ((nx.y & 7u) << 16) | (q.st & (1u << 12));
      q.hbase = nx.x;
#else
      const uint32_t npm = np ? (q.hdr[nh * kThreads + q.tid].y >> 8) : 0u;
      q.st = npm | (nh << 8) | (np << 9) | (q.st & (1u << 12));
#endif
    }
  }
  pop_entry(has, v, e, grad, bf, stage, (int)((q.st >> 12) & 1u));
}

template <int MINB, int POPS>
__global__ void __launch_bounds__(kThreads, MINB) k_map_backward_q(
    DevGrid g, DevParams p, DevCam cam, const double4* __restrict__ rgbd,
    const DevPose* __restrict__ poses, const int* __restrict__ batch, int n,
    const double4* __restrict__ ray_cd, const uint8_t* __restrict__ flags,
    const MapStats* __restrict__ stats, const int* __restrict__ global_counts,
    float4* __restrict__ grad, double lambda_d, const uint32_t* __restrict__ order,
    RecBuf rec, int K, const int2* __restrict__ rec_count) {
  // dynamic shared memory (kQMergeSmemBytes): the rings, [kQ][kThreads] float4 +
  // u32, then the per-warp merge staging [32][7] float4
  extern __shared__ __align__(16) float4 s_dyn[];
#if VRF_K2_RING
  // (kRingSmemBytes): the record rings [2][8][kThreads] float4, their headers
  // [2][kThreads] uint2, then the per-warp merge staging
  float4* s_rr = s_dyn;
  uint2* s_rh = reinterpret_cast<uint2*>(s_dyn + kRingRecs * 8 * kThreads);
  float4* stage = s_dyn + kRingRecs * 8 * kThreads + kRingRecs * kThreads / 2 +
                  (threadIdx.x >> 5) * kWarpStage;
#else
  float4* s_qa = s_dyn;
  uint32_t* s_qv = reinterpret_cast<uint32_t*>(s_dyn + kQ * kThreads);
  static_assert(!VRF_K2_VCACHE, "the vertex cache needs the record ring");
  float4* stage = s_dyn + kQ * kThreads + kQ * kThreads / 4 + (threadIdx.x >> 5) * kWarpStage;
#endif
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  // ---- per-ray setup; a lane with nothing to scatter keeps c = -1 but stays in
  // the loop (the loop's exit vote is warp-wide)
  int c = -1;
  WalkRay wr{};
  float upc0 = 0.f, upc1 = 0.f, upc2 = 0.f, upd = 0.f, Tn = 1.f;
  float bf[9];
  for (int mm = 0; mm < 9; ++mm) bf[mm] = 0.f;
  if (t < n) {
    const int i = order ? (int)order[t] : t;
    const MapStats st = *stats;
    const uint8_t fl = flags[i];
    // non-finite loss: the reference throws before updating
    if (st.bad == INT_MAX && (fl & kHit) && !(fl & kOverflow)) {
      const int f = batch[3 * i], px = batch[3 * i + 1], py = batch[3 * i + 2];
      const double4 tg =
          rgbd[(long long)f * cam.width * cam.height + (long long)py * cam.width + px];
      MapUp u;
      if (map_upstream(st, global_counts, ray_cd[i], tg, fl, lambda_d, u)) {
        March m;
        ray_from_pixel(cam, poses[f], (double)px, (double)py, m);
        double basis[9];
        if (sh_basis(m.d, basis)) {
#pragma unroll
          for (int mm = 0; mm < 9; ++mm) bf[mm] = (float)basis[mm];
          if (march_begin(g, p, m)) {
            const int2 rc = rec_count[t];
            c = rc.x - 1;
            Tn = __int_as_float(rc.y);
            wr = walk_ray(m);
            upc0 = (float)u.upc[0];
            upc1 = (float)u.upc[1];
            upc2 = (float)u.upc[2];
            upd = u.use_depth ? (float)u.upd : 0.f;
          }
        }
      }
    }
  }
#if VRF_K2_MERGE >= 3
  {  // the lane's SH basis, read by the group leaders of the factor-domain merge
    float* sbf = reinterpret_cast<float*>(stage + kSbfOff) + 12 * (threadIdx.x & 31);
#pragma unroll
    for (int mm = 0; mm < 9; ++mm) sbf[mm] = bf[mm];
#if VRF_K2_VCACHE
    uint32_t* tag = reinterpret_cast<uint32_t*>(stage + kVCacheOff + kVCache * kVec4PerVertex);
    if ((threadIdx.x & 31) < kVCache) tag[threadIdx.x & 31] = kNoCell;
#endif
    __syncwarp();
  }
#endif
  float Sc0 = 0.f, Sc1 = 0.f, Sc2 = 0.f, Sd = 0.f;
  CornerAgg A;
  agg_init(A);
  int last_tb = -1;
#if VRF_K2_RING
#if VRF_K2_HDR_REG
  RingQueue q{s_rr, s_rh, (int)threadIdx.x, 0u, 0u};
#else
  RingQueue q{s_rr, s_rh, (int)threadIdx.x, 0u};
#endif
#else
  QueueSink q{s_qv, s_qa, (int)threadIdx.x, 0u};
  uint32_t head = 0;
#endif
  bool final_pending = c >= 0;  // the last cell's 8 corners, flushed after the walk
  // records are prefetched one iteration ahead: the dependent load of the next
  // record overlaps this sample's math and scatter
  float4 n0 = make_float4(0.f, 0.f, 0.f, 0.f);
  uint2 n1 = make_uint2(0u, 0u);
  if (c >= 0) load_record(rec, t, c, K, n0, n1);
#if VRF_K2_RING
  while (__any_sync(0xffffffffu, c >= 0 || final_pending || q.pending() != 0)) {
    if (c >= 0) {
      const float4 q0 = n0;
      const uint2 q1 = n1;
      if (c > 0) load_record(rec, t, c - 1, K, n0, n1);
      --c;
      RecSample r;
      decode_record(g, wr, q0, q1, r);
      if (ring_enter(A, q, g, rec_cell(r))) mark_touched(g, r.cx, r.cy, r.cz, last_tb);
      walk_sample(A, r, upc0, upc1, upc2, upd, Sc0, Sc1, Sc2, Sd, Tn);
    } else if (final_pending && q.pending() < (uint32_t)kRingRecs) {
      final_pending = false;
      if (A.nz) ring_push(q, A, A.nz);
    }
#pragma unroll
    for (int r = 0; r < POPS; ++r) ring_pop_merge(q, g, grad, bf, stage);
    while (__any_sync(0xffffffffu, q.pending() >= (uint32_t)kRingRecs))
      ring_pop_merge(q, g, grad, bf, stage);
  }
#if VRF_K2_VCACHE
  // the cached vertices still owed to the gradient, 7 float4 each, by all lanes
  __syncwarp();
  {
    const uint32_t* tag =
        reinterpret_cast<const uint32_t*>(stage + kVCacheOff + kVCache * kVec4PerVertex);
    for (int i = threadIdx.x & 31; i < kVCache * kVec4PerVertex; i += 32) {
      const uint32_t vv = tag[i / kVec4PerVertex];
      if (vv != kNoCell)
        atomicAdd(grad + (size_t)vv * kVec4PerVertex + i % kVec4PerVertex, stage[kVCacheOff + i]);
    }
  }
#endif
#else
  while (__any_sync(0xffffffffu, c >= 0 || final_pending || head != q.tail)) {
    if (c >= 0) {
      const float4 q0 = n0;
      const uint2 q1 = n1;
      if (c > 0) load_record(rec, t, c - 1, K, n0, n1);
      --c;
      RecSample r;
      decode_record(g, wr, q0, q1, r);
      if (agg_enter(A, q, g, rec_cell(r))) mark_touched(g, r.cx, r.cy, r.cz, last_tb);
      walk_sample(A, r, upc0, upc1, upc2, upd, Sc0, Sc1, Sc2, Sd, Tn);
    } else if (final_pending && q.tail - head <= (uint32_t)(kQ - 8)) {
      final_pending = false;
      agg_flush(A, q, g, 0xffu);
    }
    // convergent scatter: every lane with queued corners pops up to POPS, then
    // more until every ring has room for the next step's <= 8 entries
#if VRF_K2_POP2
    static_assert(POPS == 2, "paired pops");
    queue_pop_merge2(q, head, grad, bf, stage);
#else
#pragma unroll
    for (int r = 0; r < POPS; ++r) queue_pop_merge(q, head, grad, bf, stage);
#endif
    while (__any_sync(0xffffffffu, q.tail - head > (uint32_t)(kQ - 8)))
      queue_pop_merge(q, head, grad, bf, stage);
  }
#endif
}

// ------------------------------------------------------------------ K3 deterministic records
// One record per (sample, corner), in the reference's accumulation order
// (ray, sample, corner). values: per sample 8 weights + 28 upstream slots (fp64).
__global__ void __launch_bounds__(kThreads) k_map_records(
    DevGrid g, DevParams p, DevCam cam, const double4* __restrict__ rgbd,
    const DevPose* __restrict__ poses, const int* __restrict__ batch, int n,
    const double4* __restrict__ ray_cd, const uint8_t* __restrict__ flags,
    const MapStats* __restrict__ stats, double lambda_d, const long long* __restrict__ offsets,
    uint32_t* __restrict__ keys, uint32_t* __restrict__ ids, double* __restrict__ values,
    int r0, int r1, long long sid_base) {
  // rays [r0, r1) of the batch; sample ids relative to this chunk's first sample
  const int i = r0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1 || i >= n) return;
  const MapStats st = *stats;
  if (st.bad != INT_MAX) return;
  const uint8_t fl = flags[i];
  if (!(fl & kHit)) return;
  const int f = batch[3 * i], px = batch[3 * i + 1], py = batch[3 * i + 2];
  const double4 tg = rgbd[(long long)f * cam.width * cam.height + (long long)py * cam.width + px];
  MapUp u;
  if (!map_upstream(st, nullptr, ray_cd[i], tg, fl, lambda_d, u)) return;
  March m;
  ray_from_pixel(cam, poses[f], (double)px, (double)py, m);
  const long long base = offsets[i] - sid_base;
  map_backward_ray<double>(
      g, p, m, u,
      [&](int idx, const Sample& s, const double w[8], double up0, const double dcol[3],
          const bool clamped[3], const double basis[9]) {
        const long long sid = base + idx;
        double* v = values + sid * 36;
        for (int k = 0; k < 8; ++k) {
          v[k] = w[k];
          keys[sid * 8 + k] = corner_index(g, s.base, k);
          ids[sid * 8 + k] = (uint32_t)(sid * 8 + k);
        }
        v[8] = up0;
        for (int ch = 0; ch < 3; ++ch)
          for (int mm = 0; mm < 9; ++mm)
            v[9 + ch * 9 + mm] = clamped[ch] ? 0.0 : dmul(dcol[ch], basis[mm]);
      });
}

// In-order fp64 sums over runs of equal vertex keys (GradientBuffer::add order).
// Each segment continues the vertex's running sum from earlier ray chunks, so
// chunking the batch keeps the single sequential (ray, sample, corner) order.
__global__ void __launch_bounds__(kThreads) k_segmented_reduce(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ rec, const double* __restrict__ values,
    long long nrec, double* __restrict__ grad) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  const uint32_t key = keys[r];
  if (r > 0 && keys[r - 1] == key) return;  // not a segment head
  double acc[28];
  const double* run = grad + (size_t)key * 28;
#pragma unroll
  for (int c = 0; c < 28; ++c) acc[c] = run[c];
  for (long long q = r; q < nrec && keys[q] == key; ++q) {
    const uint32_t id = rec[q];
    const double* v = values + (long long)(id >> 3) * 36;
    const double wk = v[id & 7];
#pragma unroll
    for (int c = 0; c < 28; ++c) acc[c] = dadd(acc[c], dmul(wk, v[8 + c]));
  }
  double* dst = grad + (size_t)key * 28;
#pragma unroll
  for (int c = 0; c < 28; ++c) dst[c] = acc[c];
}

// ------------------------------------------------------------------ K4 RMSProp
// Appends an updated float4 group (its index and new theta / v) to the update
// log the drop-in write-back reads (vrf_updates_read); warp-aggregated slot.
__device__ __forceinline__ void log_update(const UpdateLog& log, long long f, float4 th,
                                           float4 v4) {
  const unsigned m = __activemask();
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(log.count, (unsigned long long)__popc(m));
  base = __shfl_sync(m, base, leader);
  const unsigned long long pos = base + __popc(m & ((1u << lane) - 1u));
  if (pos < (unsigned long long)log.cap) {
    log.ids[pos] = (uint32_t)f;
    log.theta[pos] = th;
    log.v[pos] = v4;
  }
}

__global__ void __launch_bounds__(256) k_rmsprop(float4* __restrict__ theta,
                                                 float4* __restrict__ grad,
                                                 float4* __restrict__ vstate, long long f_begin,
                                                 long long f_end, double rho, double lr_sigma,
                                                 double lr_sh, double eps,
                                                 const MapStats* __restrict__ stats,
                                                 unsigned long long* __restrict__ touched,
                                                 UpdateLog log) {
  if (stats) {
    const MapStats st = *stats;
    if (st.bad != INT_MAX || st.m_c == 0) return;
  }
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  unsigned int n_touched = 0;
  for (long long f = f_begin + (long long)blockIdx.x * blockDim.x + threadIdx.x; f < f_end;
       f += (long long)gridDim.x * blockDim.x) {
    const float4 g4 = grad[f];
    if (g4.x == 0.f && g4.y == 0.f && g4.z == 0.f && g4.w == 0.f) continue;
    ++n_touched;
    float4 th = theta[f], v4 = vstate[f];
    const int j = (int)(f % kVec4PerVertex);
    float* thp = &th.x;
    float* vp = &v4.x;
    const float* gp = &g4.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double gg = gp[e];
      if (gg == 0.0) continue;  // mapping.cpp:226
      const double vn = rho * (double)vp[e] + (1.0 - rho) * gg * gg;
      const double lr = (4 * j + e == 0) ? lr_sigma : lr_sh;
      vp[e] = (float)vn;
      thp[e] = (float)((double)thp[e] - lr * gg / sqrt(vn + eps));
    }
    theta[f] = th;
    vstate[f] = v4;
    grad[f] = zero;
    if (log.count) log_update(log, f, th, v4);
  }
  if (touched) {  // float4 groups updated (algorithmic optimizer bytes: 96 B each)
    n_touched = warp_sum(n_touched);
    if ((threadIdx.x & 31) == 0 && n_touched) atomicAdd(touched, (unsigned long long)n_touched);
  }
}

// Block-sparse K4: one CTA per touched 8^3-vertex block (untouched blocks exit
// at once), same per-group update as k_rmsprop. Every nonzero gradient group lies
// in a block the scatter marked (mark_touched), so visiting only those blocks
// updates exactly the reference's touched set (mapping.cpp:218-231).
__global__ void __launch_bounds__(256) k_rmsprop_blocks(
    float4* __restrict__ theta, float4* __restrict__ grad, float4* __restrict__ vstate,
    const uint32_t* __restrict__ tb, int rx, int ry, int rz, int tbx, int tby, double rho,
    double lr_sigma, double lr_sh, double eps, const MapStats* __restrict__ stats,
    unsigned long long* __restrict__ touched, UpdateLog log) {
  const int b = blockIdx.x;
  if (!((tb[b >> 5] >> (b & 31)) & 1u)) return;
  if (stats) {
    const MapStats st = *stats;
    if (st.bad != INT_MAX || st.m_c == 0) return;
  }
  constexpr int E = 1 << kTouchLog2;
  const int bx = b % tbx, by = (b / tbx) % tby, bz = b / (tbx * tby);
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  unsigned int n_touched = 0;
  for (int q = threadIdx.x; q < E * E * E * kVec4PerVertex; q += blockDim.x) {
    const int vl = q / kVec4PerVertex, j = q % kVec4PerVertex;
    const int x = bx * E + (vl % E), y = by * E + ((vl / E) % E), z = bz * E + vl / (E * E);
    if (x >= rx || y >= ry || z >= rz) continue;
    const long long f = ((long long)x + (long long)rx * (y + (long long)ry * z)) * kVec4PerVertex + j;
    const float4 g4 = grad[f];
    if (g4.x == 0.f && g4.y == 0.f && g4.z == 0.f && g4.w == 0.f) continue;
    ++n_touched;
    float4 th = theta[f], v4 = vstate[f];
    float* thp = &th.x;
    float* vp = &v4.x;
    const float* gp = &g4.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double gg = gp[e];
      if (gg == 0.0) continue;  // mapping.cpp:226
      const double vn = rho * (double)vp[e] + (1.0 - rho) * gg * gg;
      const double lr = (4 * j + e == 0) ? lr_sigma : lr_sh;
      vp[e] = (float)vn;
      thp[e] = (float)((double)thp[e] - lr * gg / sqrt(vn + eps));
    }
    theta[f] = th;
    vstate[f] = v4;
    grad[f] = zero;
    if (log.count) log_update(log, f, th, v4);
  }
  if (touched) {
    n_touched = warp_sum(n_touched);
    if ((threadIdx.x & 31) == 0 && n_touched) atomicAdd(touched, (unsigned long long)n_touched);
  }
}

// ------------------------------------------------------------------ block-sparse exchange
// Multi-GPU block-sparse gradient exchange (distributed.py): the touched 8^3-
// vertex blocks are packed into [n][512][28] fp32 (local x-fastest vertex order,
// vertices outside the grid zero), reduced across ranks block-wise, applied by
// the owning rank and the updated payload blocks gathered back. id < 0 = padding.
constexpr int kBlockVerts = 1 << (3 * kTouchLog2);

// Touched vertex blocks from the touched cell blocks: vertex block v (vertices
// [8 v, 8 v + 7] per axis) holds a corner of cell block c (cells [8 c, 8 c + 7],
// vertices [8 c, 8 c + 8]) iff c == v or c == v - 1 on every axis.
__global__ void k_touched_dilate(const uint32_t* __restrict__ tc, int bx, int by, int bz,
                                 uint32_t* __restrict__ tb, int tbx, int tby, int tbz) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= tbx * tby * tbz) return;
  const int vx = v % tbx, vy = (v / tbx) % tby, vz = v / (tbx * tby);
  bool on = false;
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    const int cx = vx - (d & 1), cy = vy - ((d >> 1) & 1), cz = vz - (d >> 2);
    if (cx < 0 || cy < 0 || cz < 0 || cx >= bx || cy >= by || cz >= bz) continue;
    const int c = cx + bx * (cy + by * cz);
    on |= (tc[c >> 5] >> (c & 31)) & 1u;
  }
  const unsigned m = __ballot_sync(__activemask(), on);
  // one word per 32 consecutive vertex blocks: the warp's lane 0 writes it
  if ((threadIdx.x & 31) == 0) atomicOr(tb + (v >> 5), m);
}

__global__ void k_touched_flags(const uint32_t* __restrict__ tb, int nb, uint8_t* __restrict__ f) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nb) f[b] = (tb[b >> 5] >> (b & 31)) & 1u;
}

__device__ __forceinline__ long long block_vertex(int b, int vl, int rx, int ry, int rz, int tbx,
                                                  int tby) {
  constexpr int E = 1 << kTouchLog2;
  const int bx = b % tbx, by = (b / tbx) % tby, bz = b / (tbx * tby);
  const int x = bx * E + (vl % E), y = by * E + ((vl / E) % E), z = bz * E + vl / (E * E);
  if (x >= rx || y >= ry || z >= rz) return -1;
  return (long long)x + (long long)rx * (y + (long long)ry * z);
}

// which: 0 = gradient, 1 = payload.
__global__ void k_blocks_pack(const float4* __restrict__ src, const int* __restrict__ ids, int n,
                              int rx, int ry, int rz, int tbx, int tby, float4* __restrict__ out) {
  const long long total = (long long)n * kBlockVerts * kVec4PerVertex;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(q % kVec4PerVertex);
    const long long r = q / kVec4PerVertex;
    const int vl = (int)(r % kBlockVerts), e = (int)(r / kBlockVerts);
    const int b = ids[e];
    const long long v = b < 0 ? -1 : block_vertex(b, vl, rx, ry, rz, tbx, tby);
    out[q] = v < 0 ? make_float4(0.f, 0.f, 0.f, 0.f) : src[v * kVec4PerVertex + j];
  }
}

__global__ void k_blocks_unpack(float4* __restrict__ dst, const int* __restrict__ ids, int n, int rx,
                                int ry, int rz, int tbx, int tby, const float4* __restrict__ in) {
  const long long total = (long long)n * kBlockVerts * kVec4PerVertex;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(q % kVec4PerVertex);
    const long long r = q / kVec4PerVertex;
    const int vl = (int)(r % kBlockVerts), e = (int)(r / kBlockVerts);
    const int b = ids[e];
    if (b < 0) continue;
    const long long v = block_vertex(b, vl, rx, ry, rz, tbx, tby);
    if (v >= 0) dst[v * kVec4PerVertex + j] = in[q];
  }
}

// RMSProp (mapping.cpp:218-231) on the vertices of the listed blocks with the
// packed, rank-reduced gradient; same per-element rule as k_rmsprop.
__global__ void k_blocks_apply(float4* __restrict__ theta, float4* __restrict__ vstate,
                               const int* __restrict__ ids, int n, int rx, int ry, int rz, int tbx,
                               int tby, const float4* __restrict__ packed, double rho,
                               double lr_sigma, double lr_sh, double eps) {
  const long long total = (long long)n * kBlockVerts * kVec4PerVertex;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(q % kVec4PerVertex);
    const long long r = q / kVec4PerVertex;
    const int vl = (int)(r % kBlockVerts), e = (int)(r / kBlockVerts);
    const int b = ids[e];
    if (b < 0) continue;
    const long long v = block_vertex(b, vl, rx, ry, rz, tbx, tby);
    if (v < 0) continue;
    const float4 g4 = packed[q];
    if (g4.x == 0.f && g4.y == 0.f && g4.z == 0.f && g4.w == 0.f) continue;
    const long long f = v * kVec4PerVertex + j;
    float4 th = theta[f], v4 = vstate[f];
    float* thp = &th.x;
    float* vp = &v4.x;
    const float* gp = &g4.x;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double gg = gp[c];
      if (gg == 0.0) continue;  // mapping.cpp:226
      const double vn = rho * (double)vp[c] + (1.0 - rho) * gg * gg;
      const double lr = (4 * j + c == 0) ? lr_sigma : lr_sh;
      vp[c] = (float)vn;
      thp[c] = (float)((double)thp[c] - lr * gg / sqrt(vn + eps));
    }
    theta[f] = th;
    vstate[f] = v4;
  }
}

// ------------------------------------------------------------------ fused peer exchange
// One kernel for the whole multi-GPU gradient exchange + update:
// the block-sparse path's pack -> reduce-scatter -> RMSProp -> pack ->
// all-gather -> unpack, done over NVLink peer memory. CTA i handles block
// b = rank + world * i (static owner, as the NCCL path). If any rank's
// touched-block bitmap marks b, the CTA reads b's gradient from every rank that
// touched it (P2P loads, summed in rank order: deterministic for a fixed world
// size), applies RMSProp (mapping.cpp:218-231; same per-element rule as
// k_rmsprop) to its own payload / RMSProp state, and stores the updated payload
// group into every rank's payload (P2P stores). Every rank holds the same
// payload before the step, so reading theta locally is exact.
__global__ void __launch_bounds__(256) k_exchange_p2p(PeerTable pt, float4* __restrict__ vstate,
                                                      int nb, int rx, int ry, int rz, int tbx,
                                                      int tby, double rho, double lr_sigma,
                                                      double lr_sh, double eps,
                                                      const MapStats* __restrict__ stats) {
  const int b = pt.rank + pt.world * blockIdx.x;
  if (b >= nb) return;
  if (stats) {
    const MapStats st = *stats;
    if (st.bad != INT_MAX || st.m_c == 0) return;
  }
  __shared__ unsigned s_mask;
  if (threadIdx.x == 0) {
    unsigned m = 0;
    for (int r = 0; r < pt.world; ++r)
      m |= ((__ldcv(pt.tb[r] + (b >> 5)) >> (b & 31)) & 1u) << r;
    s_mask = m;
  }
  __syncthreads();
  const unsigned mask = s_mask;
  if (!mask) return;
  float4* theta = pt.payload[pt.rank];
  for (int q = threadIdx.x; q < kBlockVerts * kVec4PerVertex; q += blockDim.x) {
    const int vl = q / kVec4PerVertex, j = q % kVec4PerVertex;
    const long long v = block_vertex(b, vl, rx, ry, rz, tbx, tby);
    if (v < 0) continue;
    const long long f = v * kVec4PerVertex + j;
    float4 parts[kMaxPeers];
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)  // all loads in flight before the sum
      parts[r] = (r < pt.world && ((mask >> r) & 1u)) ? __ldcv(pt.grad[r] + f)
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 g4 = parts[0];
#pragma unroll
    for (int r = 1; r < kMaxPeers; ++r) {
      g4.x += parts[r].x;
      g4.y += parts[r].y;
      g4.z += parts[r].z;
      g4.w += parts[r].w;
    }
    if (g4.x == 0.f && g4.y == 0.f && g4.z == 0.f && g4.w == 0.f) continue;
    float4 th = theta[f], v4 = vstate[f];
    float* thp = &th.x;
    float* vp = &v4.x;
    const float* gp = &g4.x;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double gg = gp[c];
      if (gg == 0.0) continue;  // mapping.cpp:226
      const double vn = rho * (double)vp[c] + (1.0 - rho) * gg * gg;
      const double lr = (4 * j + c == 0) ? lr_sigma : lr_sh;
      vp[c] = (float)vn;
      thp[c] = (float)((double)thp[c] - lr * gg / sqrt(vn + eps));
    }
    vstate[f] = v4;
    for (int r = 0; r < pt.world; ++r) __stcg(pt.payload[r] + f, th);
  }
  __threadfence_system();  // peer stores visible before the caller's barrier
}

// ------------------------------------------------------------------ utilities
__global__ void k_fill_payload(float* payload, long long nv, float sigma) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nv * kPayload;
       e += (long long)gridDim.x * blockDim.x)
    payload[e] = (e % kPayload == 0) ? sigma : 0.f;
}
__global__ void k_f64_to_f32(const double* in, float* out, long long n) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = (float)in[e];
}
__global__ void k_f32_to_f64(const float* in, double* out, long long n) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = (double)in[e];
}
__global__ void k_pack_occupancy(const uint8_t* occ, uint32_t* bits, long long n_cells) {
  const long long wd = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (wd * 32 >= n_cells) return;
  uint32_t b = 0;
  for (int k = 0; k < 32; ++k) {
    const long long c = wd * 32 + k;
    if (c < n_cells && occ[c]) b |= 1u << k;
  }
  bits[wd] = b;
}
__global__ void k_unpack_occupancy(const uint32_t* bits, uint8_t* occ, long long n_cells) {
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n_cells;
       c += (long long)gridDim.x * blockDim.x)
    occ[c] = (bits[c >> 5] >> (c & 31)) & 1u;
}
__global__ void k_pack_frames(const double* color, const double* depth, double4* rgbd,
                              long long npix) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < npix;
       q += (long long)gridDim.x * blockDim.x)
    rgbd[q] = make_double4(color[3 * q], color[3 * q + 1], color[3 * q + 2], depth[q]);
}
// Sensor-format frame (8-bit RGB, 16-bit depth units), converted exactly as the
// reference's PNG loaders do (image.cpp:53-55 colour / 255.0, :79 depth /
// depth_scale; IEEE double division).
__global__ void k_pack_frames_u8(const uint8_t* __restrict__ rgb, const uint16_t* __restrict__ d,
                                 double depth_scale, double4* rgbd, long long npix) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < npix;
       q += (long long)gridDim.x * blockDim.x)
    rgbd[q] = make_double4(__ddiv_rn((double)rgb[3 * q], 255.0),
                           __ddiv_rn((double)rgb[3 * q + 1], 255.0),
                           __ddiv_rn((double)rgb[3 * q + 2], 255.0),
                           __ddiv_rn((double)d[q], depth_scale));
}
__global__ void k_extract_depth(const double4* __restrict__ rgbd, double* __restrict__ out,
                                long long npix) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < npix;
       q += (long long)gridDim.x * blockDim.x)
    out[q] = rgbd[q].w;
}
// VoxelGrid::prune — voxel_grid.cpp:169-188 (peak of max(sigma,0) over 8 corners < tau).
__global__ void k_prune(DevGrid g, uint32_t* bits, double tau, unsigned long long* count) {
  const long long n_cells = (long long)(g.rx - 1) * (g.ry - 1) * (g.rz - 1);
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n_cells;
       c += (long long)gridDim.x * blockDim.x) {
    if (!((bits[c >> 5] >> (c & 31)) & 1u)) continue;
    const int cx = (int)(c % (g.rx - 1));
    const long long r = c / (g.rx - 1);
    const int cy = (int)(r % (g.ry - 1)), cz = (int)(r / (g.ry - 1));
    const uint32_t base = (uint32_t)(cx + g.rx * (cy + (long long)g.ry * cz));
    double peak = 0.0;
    for (int k = 0; k < 8; ++k) {
      const double s = (double)((const float*)g.payload)[(size_t)corner_index(g, base, k) * kPayload];
      const double sp = (s < 0.0) ? 0.0 : s;
      peak = (peak < sp) ? sp : peak;
    }
    if (peak < tau) {
      atomicAnd(bits + (c >> 5), ~(1u << (c & 31)));
      atomicAdd(count, 1ull);
    }
  }
}

// VoxelGrid::upsampled — voxel_grid.cpp:190-220. Fine vertex (ix,iy,iz) sits at
// coarse coordinates (ix/2, iy/2, iz/2); like the reference it goes through the
// world point p = to_world(g) and locate(p), then trilerps all 28 channels (FP64
// accumulation in the reference corner order, stored fp32).
__global__ void k_upsample(DevGrid c, int frx, int fry, int frz, float* __restrict__ fine) {
  const long long nv = (long long)frx * fry * frz;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nv;
       v += (long long)gridDim.x * blockDim.x) {
    const int ix = (int)(v % frx);
    const long long r = v / frx;
    const int iy = (int)(r % fry), iz = (int)(r / fry);
    const double p[3] = {dadd(c.ox, dmul(ix * 0.5, c.voxel)), dadd(c.oy, dmul(iy * 0.5, c.voxel)),
                         dadd(c.oz, dmul(iz * 0.5, c.voxel))};
    Sample s;
    if (!locate(c, p, s)) {
      // The world round trip put a far-corner vertex an ulp outside the box; the
      // reference throws here (voxel_grid.cpp:107-111). Clamp the grid
      // coordinate into [0, res-1] instead (the boundary vertex's value).
      const double gx = fmin(fmax(div_voxel(c, dsub(p[0], c.ox)), 0.0), (double)c.rx - 1.0);
      const double gy = fmin(fmax(div_voxel(c, dsub(p[1], c.oy)), 0.0), (double)c.ry - 1.0);
      const double gz = fmin(fmax(div_voxel(c, dsub(p[2], c.oz)), 0.0), (double)c.rz - 1.0);
      int cx = (int)ceil(gx) - 1, cy = (int)ceil(gy) - 1, cz = (int)ceil(gz) - 1;
      cx = cx < 0 ? 0 : (cx > c.rx - 2 ? c.rx - 2 : cx);
      cy = cy < 0 ? 0 : (cy > c.ry - 2 ? c.ry - 2 : cy);
      cz = cz < 0 ? 0 : (cz > c.rz - 2 ? c.rz - 2 : cz);
      s.fx = dsub(gx, (double)cx);
      s.fy = dsub(gy, (double)cy);
      s.fz = dsub(gz, (double)cz);
      s.base = (uint32_t)(cx + c.rx * (cy + (long long)c.ry * cz));
    }
    double w[8];
    corner_weights(s, w);
    double acc[28];
#pragma unroll
    for (int q = 0; q < 28; ++q) acc[q] = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float* vp = reinterpret_cast<const float*>(c.payload) +
                        (size_t)corner_index(c, s.base, k) * kPayload;
#pragma unroll
      for (int q = 0; q < 28; ++q) acc[q] = dadd(acc[q], dmul(w[k], (double)__ldg(vp + q)));
    }
    float* dst = fine + (size_t)v * kPayload;
#pragma unroll
    for (int q = 0; q < 28; ++q) dst[q] = (float)acc[q];
  }
}

// Each refined cell inherits its parent's activity (voxel_grid.cpp:214-218).
__global__ void k_upsample_occupancy(const uint32_t* __restrict__ cocc, int crx, int cry,
                                     int frx, int fry, int frz, uint32_t* __restrict__ focc) {
  const long long ncf = (long long)(frx - 1) * (fry - 1) * (frz - 1);
  const long long words = (ncf + 31) / 32;
  for (long long wd = (long long)blockIdx.x * blockDim.x + threadIdx.x; wd < words;
       wd += (long long)gridDim.x * blockDim.x) {
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b) {
      const long long f = wd * 32 + b;
      if (f >= ncf) break;
      const int cx = (int)(f % (frx - 1));
      const long long r = f / (frx - 1);
      const int cy = (int)(r % (fry - 1)), cz = (int)(r / (fry - 1));
      const long long pc = (cx / 2) + (long long)(crx - 1) * ((cy / 2) + (long long)(cry - 1) * (cz / 2));
      if ((cocc[pc >> 5] >> (pc & 31)) & 1u) bits |= 1u << b;
    }
    focc[wd] = bits;
  }
}

// Coarse occupancy: block bit = OR of its (up to) 8^3 cell bits.
__global__ void k_block_occupancy(const uint32_t* __restrict__ occ, int rx, int ry, int rz,
                                  int bx, int by, int bz, uint32_t* __restrict__ bocc,
                                  unsigned int* __restrict__ n_active) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int nb = bx * by * bz;
  if (b >= nb) return;
  const int ix = b % bx, iy = (b / bx) % by, iz = b / (bx * by);
  const int cx0 = ix << kBlockLog2, cy0 = iy << kBlockLog2, cz0 = iz << kBlockLog2;
  const int cx1 = min(cx0 + (1 << kBlockLog2), rx - 1), cy1 = min(cy0 + (1 << kBlockLog2), ry - 1),
            cz1 = min(cz0 + (1 << kBlockLog2), rz - 1);
  bool any = false;
  for (int cz = cz0; cz < cz1 && !any; ++cz)
    for (int cy = cy0; cy < cy1 && !any; ++cy)
      for (int cx = cx0; cx < cx1 && !any; ++cx) {
        const uint32_t c = (uint32_t)(cx + (rx - 1) * (cy + (long long)(ry - 1) * cz));
        any = (occ[c >> 5] >> (c & 31)) & 1u;
      }
  if (any) {
    atomicOr(bocc + (b >> 5), 1u << (b & 31));
    atomicAdd(n_active, 1u);
  }
}

__global__ void k_super_occupancy(const uint32_t* __restrict__ bocc, int bx, int by, int bz,
                                  int sx, int sy, int sz, uint32_t* __restrict__ socc) {
  constexpr int kS = kSuperLog2 - kBlockLog2;
  const int w = blockIdx.x * blockDim.x + threadIdx.x;  // one 32-superblock word
  const int ns = sx * sy * sz;
  if (w * 32 >= ns) return;
  uint32_t bits = 0;
  for (int q = 0; q < 32; ++q) {
    const int sidx = w * 32 + q;
    if (sidx >= ns) break;
    const int ix = sidx % sx, iy = (sidx / sx) % sy, iz = sidx / (sx * sy);
    bool any = false;
    for (int z = iz << kS; z < min((iz + 1) << kS, bz) && !any; ++z)
      for (int y = iy << kS; y < min((iy + 1) << kS, by) && !any; ++y)
        for (int x = ix << kS; x < min((ix + 1) << kS, bx) && !any; ++x) {
          const int b = x + bx * (y + by * z);
          any = (bocc[b >> 5] >> (b & 31)) & 1u;
        }
    if (any) bits |= 1u << q;
  }
  socc[w] = bits;
}

int grid_blocks(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  if (b > 148LL * 32) b = 148LL * 32;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace

// ------------------------------------------------------------------ launchers
void launch_render_image(const DevGrid& g, const DevParams& p, const DevCam& cam,
                         const DevPose& pose, int stride, int out_w, int out_h, double* color,
                         double* depth, int* err, cudaStream_t s) {
  const long long n = (long long)out_w * out_h;
  if (n == 0) return;
  k_render_image<double><<<(unsigned)((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(
      g, p, cam, pose, stride, out_w, out_h, color, depth, err);
}
void launch_debug_rays(const DevGrid& g, const DevParams& p, const double* rays, int n, int cap,
                       int* counts, double* t, double* delta, uint32_t* cells, double* out,
                       int* err, cudaStream_t s) {
  if (n == 0) return;
  k_debug_rays<<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(g, p, rays, n, cap, counts, t,
                                                                   delta, cells, out, err);
}
int map_forward_blocks(int n) { return (n + kThreads - 1) / kThreads; }
void launch_map_forward(const DevGrid& g, const DevParams& p, const DevCam& cam,
                        const double4* rgbd, const DevPose* poses, int n_frames,
                        const int* batch, int n, double4* ray_cd, uint8_t* flags,
                        MapPartial* partials, int* ray_count, int* err, bool fast,
                        const uint32_t* order, cudaStream_t s) {
  const int blocks = map_forward_blocks(n);
  if (fast)
    k_map_forward<float><<<blocks, kThreads, 0, s>>>(g, p, cam, rgbd, poses, n_frames, batch, n,
                                                     ray_cd, flags, partials, ray_count, err,
                                                     order);
  else
    k_map_forward<double><<<blocks, kThreads, 0, s>>>(g, p, cam, rgbd, poses, n_frames, batch, n,
                                                      ray_cd, flags, partials, ray_count, err,
                                                      order);
}
// Rays up to which K0 runs 8 lanes per ray (K0g); VRF_FWD_GROUP_MAX overrides.
// r01 (config-3 scene, forward ms, K0g vs K0): 4K rays 0.67 vs 2.08, 16K 0.99
// vs 1.91, 32K 1.60 vs 1.87, 48K 2.18 vs 1.82 -> crossover ~40K.
int fwd_group_max() {
  static const int v = [] {
    const char* e = std::getenv("VRF_FWD_GROUP_MAX");
    return e ? std::atoi(e) : 40000;
  }();
  return v;
}
int map_forward_rec_blocks(int n) {
  return n <= fwd_group_max() ? (n + kThreads / kFwdLanes - 1) / (kThreads / kFwdLanes)
                              : map_forward_blocks(n);
}
void launch_map_forward_rec(const DevGrid& g, const DevParams& p, const DevCam& cam,
                            const double4* rgbd, const DevPose* poses, int n_frames,
                            const int* batch, int n, double4* ray_cd, uint8_t* flags,
                            MapPartial* partials, int* err, const uint32_t* order, RecBuf rec,
                            int K, int2* rec_count, cudaStream_t s) {
  if (n <= fwd_group_max()) {
    k_map_forward_rec_g<<<map_forward_rec_blocks(n), kThreads, 0, s>>>(
        g, p, cam, rgbd, poses, n_frames, batch, n, ray_cd, flags, partials, err, order, rec, K,
        rec_count);
    return;
  }
#if VRF_K0_COOP
  k_map_forward_coop<<<map_forward_blocks(n), kThreads, 0, s>>>(g, p, cam, rgbd, poses, n_frames,
                                                                batch, n, ray_cd, flags, partials,
                                                                err, order, rec, K, rec_count);
#else
#if VRF_K0_CARVEOUT >= 0
  // A/B: the L1 / shared-memory split of the SMs running K0 (percent shared)
  static const bool carve = cudaFuncSetAttribute(k_map_forward_rec,
                                                 cudaFuncAttributePreferredSharedMemoryCarveout,
                                                 VRF_K0_CARVEOUT) == cudaSuccess;
  (void)carve;
#endif
  k_map_forward_rec<<<map_forward_blocks(n), kThreads, 0, s>>>(g, p, cam, rgbd, poses, n_frames,
                                                               batch, n, ray_cd, flags, partials,
                                                               err, order, rec, K, rec_count);
#endif
}
// Rays up to which K2 runs 8 lanes per ray (K2g); VRF_BWD_GROUP_MAX overrides.
// r01 (config-3 scene, backward ms, K2g vs K2q): 4K rays 0.19 vs 1.07, 16K 0.41
// vs 1.04, 32K 0.67 vs 1.22, 64K 1.19 vs 1.80, 128K 2.17 vs 2.50, 256K 4.23 vs
// 4.13 -> crossover ~200K.
static int bwd_group_max() {
  static const int v = [] {
    const char* e = std::getenv("VRF_BWD_GROUP_MAX");
    return e ? std::atoi(e) : 160000;
  }();
  return v;
}
// Grid size (vertices) from which K2q runs at 3 CTAs/SM; VRF_K2_MINB3_VERTS
// overrides (0: always). r02: config 4 (513^3 sparse) prefers 3 CTAs/SM at 8M rays
// per batch (26.4 against 27.8 ms) and at 1M (5.64 against 5.94 ms, the per-rank
// batch of an 8-GPU run), config 3 (257^3) prefers 4 (10.39 against 10.87 ms):
// the choice follows the grid, not the batch.
static long long k2_minb3_verts() {
  static const long long v = [] {
    const char* e = std::getenv("VRF_K2_MINB3_VERTS");
    return e ? std::atoll(e) : (64LL << 20);
  }();
  return v;
}
template <int MINB, int POPS, int SMEM>
static void launch_k2q(const DevGrid& g, const DevParams& p, const DevCam& cam,
                       const double4* rgbd, const DevPose* poses, const int* batch, int n,
                       const double4* ray_cd, const uint8_t* flags, const MapStats* stats,
                       const int* global_counts, float4* grad, double lambda_d,
                       const uint32_t* order, RecBuf rec, int K, const int2* rec_count,
                       cudaStream_t s) {
  static const bool attr = cudaFuncSetAttribute(k_map_backward_q<MINB, POPS>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                SMEM) == cudaSuccess;
  (void)attr;
  k_map_backward_q<MINB, POPS><<<(n + kThreads - 1) / kThreads, kThreads, SMEM, s>>>(
      g, p, cam, rgbd, poses, batch, n, ray_cd, flags, stats, global_counts, grad, lambda_d,
      order, rec, K, rec_count);
}
void launch_map_backward_rec(const DevGrid& g, const DevParams& p, const DevCam& cam,
                             const double4* rgbd, const DevPose* poses, const int* batch, int n,
                             const double4* ray_cd, const uint8_t* flags, const MapStats* stats,
                             const int* global_counts, float4* grad, double lambda_d,
                             const uint32_t* order, RecBuf rec, int K,
                             const int2* rec_count, cudaStream_t s) {
  if (n <= bwd_group_max()) {  // small batch: 8 lanes per ray (K2g)
    k_map_backward_g<<<(n + kThreads / 8 - 1) / (kThreads / 8), kThreads, 0, s>>>(
        g, p, cam, rgbd, poses, batch, n, ray_cd, flags, stats, global_counts, grad, lambda_d,
        order, rec, K, rec_count);
    return;
  }
  // K2q: 4 CTAs/SM (VRF_K2_MINB), 2 pops per step. r01 (config 3 / config 4, ms): 1, 2 or 3
  // pops 14.54 / 14.63 / 15.02 and 25.82 / 25.71 / 25.78. Grids of >= k2_minb3_verts()
  // vertices run the 3-CTA/SM build (168-register cap).
  constexpr int kPops = VRF_K2_POPS;
  constexpr int kSmem = VRF_K2_RING ? kRingSmemBytes : kQMergeSmemBytes;
  if (VRF_K2_MINB != 3 && (long long)g.rx * g.ry * g.rz >= k2_minb3_verts()) {
    launch_k2q<3, kPops, kSmem>(g, p, cam, rgbd, poses, batch, n, ray_cd, flags, stats,
                                global_counts, grad, lambda_d, order, rec, K, rec_count, s);
    return;
  }
  launch_k2q<VRF_K2_MINB, kPops, kSmem>(g, p, cam, rgbd, poses, batch, n, ray_cd, flags, stats,
                                        global_counts, grad, lambda_d, order, rec, K,
                                        rec_count, s);
}
void launch_map_reduce(const MapPartial* partials, int nparts, MapStats* out, cudaStream_t s) {
  k_map_reduce<<<1, 1024, 0, s>>>(partials, nparts, out);
}
void launch_map_backward(const DevGrid& g, const DevParams& p, const DevCam& cam,
                         const double4* rgbd, const DevPose* poses, const int* batch, int n,
                         const double4* ray_cd, const uint8_t* flags, const MapStats* stats,
                         const int* global_counts, float4* grad, double lambda_d,
                         bool overflow_only, const uint32_t* order, cudaStream_t s) {
  // 4 CTAs x 128 threads per SM (measured best of 2/3/4, r01). The empty-block
  // jump is compiled in only when the grid has empty blocks.
  const int blocks = (n + kThreads - 1) / kThreads;
  if (g.all_blocks_active)
    k_map_backward<false><<<blocks, kThreads, 0, s>>>(g, p, cam, rgbd, poses, batch, n, ray_cd,
                                                      flags, stats, global_counts, grad,
                                                      lambda_d, order, overflow_only);
  else
    k_map_backward<true><<<blocks, kThreads, 0, s>>>(g, p, cam, rgbd, poses, batch, n, ray_cd,
                                                     flags, stats, global_counts, grad, lambda_d,
                                                     order, overflow_only);
}
void launch_map_backward_records(const DevGrid& g, const DevParams& p, const DevCam& cam,
                                 const double4* rgbd, const DevPose* poses, const int* batch,
                                 int n, const double4* ray_cd, const uint8_t* flags,
                                 const MapStats* stats, double lambda_d,
                                 const long long* offsets, uint32_t* keys, uint32_t* ids,
                                 double* values, int r0, int r1, long long sid_base,
                                 cudaStream_t s) {
  if (r1 <= r0) return;
  k_map_records<<<(r1 - r0 + kThreads - 1) / kThreads, kThreads, 0, s>>>(
      g, p, cam, rgbd, poses, batch, n, ray_cd, flags, stats, lambda_d, offsets, keys, ids,
      values, r0, r1, sid_base);
}
void launch_segmented_reduce(const uint32_t* keys, const uint32_t* perm, const double* values,
                             long long nrec, double* grad, cudaStream_t s) {
  if (nrec == 0) return;
  k_segmented_reduce<<<(unsigned)((nrec + kThreads - 1) / kThreads), kThreads, 0, s>>>(
      keys, perm, values, nrec, grad);
}
void launch_rmsprop(float4* theta, float4* grad, float4* v, long long v_begin, long long v_end,
                    double rho, double lr_sigma, double lr_sh, double eps,
                    const MapStats* stats, unsigned long long* touched, cudaStream_t s,
                    const UpdateLog& log) {
  const long long f0 = v_begin * kVec4PerVertex, f1 = v_end * kVec4PerVertex;
  if (f1 <= f0) return;
  k_rmsprop<<<grid_blocks(f1 - f0, 256), 256, 0, s>>>(theta, grad, v, f0, f1, rho, lr_sigma,
                                                      lr_sh, eps, stats, touched, log);
}
void launch_rmsprop_blocks(float4* theta, float4* grad, float4* v, uint32_t* tb, int rx, int ry,
                           int rz, int tbx, int tby, int tbz, double rho, double lr_sigma,
                           double lr_sh, double eps, const MapStats* stats,
                           unsigned long long* touched, cudaStream_t s, const UpdateLog& log) {
  const int nb = tbx * tby * tbz;
  k_rmsprop_blocks<<<nb, 256, 0, s>>>(theta, grad, v, tb, rx, ry, rz, tbx, tby, rho, lr_sigma,
                                      lr_sh, eps, stats, touched, log);
  cudaMemsetAsync(tb, 0, sizeof(uint32_t) * ((nb + 31) / 32 + 1), s);
}
void launch_touched_dilate(uint32_t* tc, int bx, int by, int bz, uint32_t* tb, int tbx, int tby,
                           int tbz, cudaStream_t s) {
  const int nv = tbx * tby * tbz;
  k_touched_dilate<<<(nv + 255) / 256, 256, 0, s>>>(tc, bx, by, bz, tb, tbx, tby, tbz);
  cudaMemsetAsync(tc, 0, sizeof(uint32_t) * (((long long)bx * by * bz + 31) / 32 + 1), s);
}
void launch_touched_flags(const uint32_t* tb, int nb, uint8_t* flags, cudaStream_t s) {
  k_touched_flags<<<(nb + 255) / 256, 256, 0, s>>>(tb, nb, flags);
}
void launch_blocks_pack(const float4* src, const int* ids, int n, int rx, int ry, int rz, int tbx,
                        int tby, float4* out, cudaStream_t s) {
  const long long total = (long long)n * kBlockVerts * kVec4PerVertex;
  if (total > 0)
    k_blocks_pack<<<grid_blocks(total, 256), 256, 0, s>>>(src, ids, n, rx, ry, rz, tbx, tby, out);
}
void launch_blocks_unpack(float4* dst, const int* ids, int n, int rx, int ry, int rz, int tbx,
                          int tby, const float4* in, cudaStream_t s) {
  const long long total = (long long)n * kBlockVerts * kVec4PerVertex;
  if (total > 0)
    k_blocks_unpack<<<grid_blocks(total, 256), 256, 0, s>>>(dst, ids, n, rx, ry, rz, tbx, tby, in);
}
void launch_blocks_apply(float4* theta, float4* v, const int* ids, int n, int rx, int ry, int rz,
                         int tbx, int tby, const float4* packed, double rho, double lr_sigma,
                         double lr_sh, double eps, cudaStream_t s) {
  const long long total = (long long)n * kBlockVerts * kVec4PerVertex;
  if (total > 0)
    k_blocks_apply<<<grid_blocks(total, 256), 256, 0, s>>>(theta, v, ids, n, rx, ry, rz, tbx, tby,
                                                           packed, rho, lr_sigma, lr_sh, eps);
}
void launch_exchange_p2p(const PeerTable& pt, float4* v, int nb, int rx, int ry, int rz, int tbx,
                         int tby, double rho, double lr_sigma, double lr_sh, double eps,
                         const MapStats* stats, cudaStream_t s) {
  const int grid = (nb + pt.world - 1) / pt.world;
  if (grid > 0)
    k_exchange_p2p<<<grid, 256, 0, s>>>(pt, v, nb, rx, ry, rz, tbx, tby, rho, lr_sigma, lr_sh, eps,
                                        stats);
}
#ifdef VRF_GATHER_SOA  // A/B build only (the planar gather layout)
__global__ void k_aos_to_soa(const float4* __restrict__ aos, float4* __restrict__ soa,
                             long long nv) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv * kVec4PerVertex;
       i += (long long)gridDim.x * blockDim.x) {
    const long long v = i / kVec4PerVertex, j = i % kVec4PerVertex;
    soa[j * nv + v] = aos[i];
  }
}
void launch_aos_to_soa(const float4* aos, float4* soa, long long nv, cudaStream_t s) {
  k_aos_to_soa<<<grid_blocks(nv * kVec4PerVertex, 256), 256, 0, s>>>(aos, soa, nv);
}
#endif
// Order-independent 64-bit digest of a word array: sum over i of mix(i, w_i)
// (splitmix64 finaliser of the index-salted word), so any changed word, moved word
// or changed length changes it w.h.p.; per-block sums, one atomic add per block.
__device__ __forceinline__ uint64_t digest_mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__global__ void __launch_bounds__(256) k_digest(const uint32_t* __restrict__ w, long long n,
                                                uint64_t salt, unsigned long long* out) {
  uint64_t acc = 0;
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < n;
       i += (long long)gridDim.x * 256)
    acc += digest_mix(salt ^ ((uint64_t)i << 32) ^ (uint64_t)__ldg(w + i));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  __shared__ uint64_t s[8];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int k = 0; k < 8; ++k) t += s[k];
    atomicAdd(out, (unsigned long long)t);
  }
}
void launch_digest(const uint32_t* words, long long n, uint64_t salt, unsigned long long* out,
                   cudaStream_t s) {
  if (n > 0) k_digest<<<148 * 8, 256, 0, s>>>(words, n, salt, out);
}
void launch_fill_payload(float* payload, long long nv, float sigma, cudaStream_t s) {
  k_fill_payload<<<grid_blocks(nv * kPayload, 256), 256, 0, s>>>(payload, nv, sigma);
}
void launch_f64_to_f32(const double* in, float* out, long long n, cudaStream_t s) {
  if (n) k_f64_to_f32<<<grid_blocks(n, 256), 256, 0, s>>>(in, out, n);
}
void launch_f32_to_f64(const float* in, double* out, long long n, cudaStream_t s) {
  if (n) k_f32_to_f64<<<grid_blocks(n, 256), 256, 0, s>>>(in, out, n);
}
void launch_pack_occupancy(const uint8_t* occ, uint32_t* bits, long long n_cells,
                           cudaStream_t s) {
  const long long words = (n_cells + 31) / 32;
  if (words) k_pack_occupancy<<<(unsigned)((words + 255) / 256), 256, 0, s>>>(occ, bits, n_cells);
}
void launch_unpack_occupancy(const uint32_t* bits, uint8_t* occ, long long n_cells,
                             cudaStream_t s) {
  if (n_cells) k_unpack_occupancy<<<grid_blocks(n_cells, 256), 256, 0, s>>>(bits, occ, n_cells);
}
void launch_pack_frames(const double* color, const double* depth, double4* rgbd, long long npix,
                        cudaStream_t s) {
  if (npix) k_pack_frames<<<grid_blocks(npix, 256), 256, 0, s>>>(color, depth, rgbd, npix);
}
void launch_pack_frames_u8(const uint8_t* rgb, const uint16_t* depth, double depth_scale,
                           double4* rgbd, long long npix, cudaStream_t s) {
  if (npix)
    k_pack_frames_u8<<<grid_blocks(npix, 256), 256, 0, s>>>(rgb, depth, depth_scale, rgbd, npix);
}
void launch_extract_depth(const double4* rgbd, double* out, long long npix, cudaStream_t s) {
  if (npix) k_extract_depth<<<grid_blocks(npix, 256), 256, 0, s>>>(rgbd, out, npix);
}
void launch_upsample(const DevGrid& coarse, int frx, int fry, int frz, float* fine,
                     uint32_t* fine_occ, cudaStream_t s) {
  const long long nv = (long long)frx * fry * frz;
  k_upsample<<<grid_blocks(nv, 128), 128, 0, s>>>(coarse, frx, fry, frz, fine);
  const long long words = ((long long)(frx - 1) * (fry - 1) * (frz - 1) + 31) / 32;
  k_upsample_occupancy<<<grid_blocks(words, 256), 256, 0, s>>>(coarse.occ, coarse.rx, coarse.ry,
                                                               frx, fry, frz, fine_occ);
}
void launch_block_occupancy(const uint32_t* occ, int rx, int ry, int rz, int bx, int by, int bz,
                            uint32_t* bocc, unsigned int* n_active, cudaStream_t s) {
  const int nb = bx * by * bz;
  cudaMemsetAsync(bocc, 0, sizeof(uint32_t) * ((nb + 31) / 32 + 1), s);
  cudaMemsetAsync(n_active, 0, sizeof(unsigned int), s);
  k_block_occupancy<<<(nb + 127) / 128, 128, 0, s>>>(occ, rx, ry, rz, bx, by, bz, bocc,
                                                     n_active);
}
void launch_super_occupancy(const uint32_t* bocc, int bx, int by, int bz, int sx, int sy, int sz,
                            uint32_t* socc, cudaStream_t s) {
  const int words = (sx * sy * sz + 31) / 32;
  k_super_occupancy<<<(words + 63) / 64, 64, 0, s>>>(bocc, bx, by, bz, sx, sy, sz, socc);
}
void launch_prune(const DevGrid& g, uint32_t* bits, double tau, unsigned long long* count,
                  cudaStream_t s) {
  const long long n_cells = (long long)(g.rx - 1) * (g.ry - 1) * (g.rz - 1);
  k_prune<<<grid_blocks(n_cells, 256), 256, 0, s>>>(g, bits, tau, count);
}

}  // namespace vrf

#if VRF_K2_GSTATS
// diagnostic build only: read and clear the K2 duplicate-group histograms
// (out[0..32] group sizes, out[33..65] largest group per pop round)
extern "C" int vrf_debug_k2_hist(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, vrf::g_k2_gsize, sizeof(unsigned long long) * 33);
  cudaMemcpyFromSymbol(out + 33, vrf::g_k2_rmax, sizeof(unsigned long long) * 33);
  static const unsigned long long z[33] = {};
  cudaMemcpyToSymbol(vrf::g_k2_gsize, z, sizeof(z));
  cudaMemcpyToSymbol(vrf::g_k2_rmax, z, sizeof(z));
  return (int)cudaGetLastError();
}
#endif

