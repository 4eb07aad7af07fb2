// Device building blocks of the per-ray hot path (sm_100a).
//
// Numerics contract:
//  * Everything that decides WHICH samples exist and WHERE they land — ray
//    generation, slab clip, the uniform schedule, cell location, occupancy —
//    is FP64 with the reference's exact operation order and no contraction
//    (__dadd_rn/__dmul_rn/__ddiv_rn), so sample counts, cell ids and corner
//    indices are bit-identical to the CPU reference.
//  * sigma_raw (and with it alpha, T and the T < eps termination test) is also
//    an FP64 replay of trilerp (voxel_grid.cpp:113-122) over the fp32 payload,
//    so early termination cannot flip against the oracle.
//  * The 27 SH channels use the ShT accumulator: double (parity/deterministic
//    mode) or float (fast mode; colour error ~1e-7, far inside the 1e-4 bar).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace vrf {

constexpr int kPayload = 28;      // sigma + 27 SH (voxel_grid.hpp:13-16)
constexpr int kVec4PerVertex = 7; // 112 B per vertex

// voxel_grid.cpp:11-17
constexpr double kC0 = 0.28209479177387814;
constexpr double kC1 = 0.4886025119029199;
constexpr double kC2_xy = 1.0925484305920792;
constexpr double kC2_yz = -1.0925484305920792;
constexpr double kC2_zz = 0.31539156525252005;
constexpr double kC2_xz = -1.0925484305920792;
constexpr double kC2_xxyy = 0.5462742152960396;

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

struct DevGrid {
  int rx, ry, rz;
  uint32_t rxy;           // rx * ry (vertex z stride)
  double ox, oy, oz;      // world_min
  double hx, hy, hz;      // world_max (voxel_grid.hpp:44-46)
  double voxel;
  double inv_voxel;       // 1 / voxel (spatial gradient scale, voxel_grid.cpp:136)
  double rcp_voxel;       // RN(1 / voxel), host IEEE division (div_voxel)
  const float4* __restrict__ payload;  // [V][7]
  // A/B only (-DVRF_GATHER_SOA): a channel-group-planar copy [7][soa_stride] of the
  // payload that K0's gathers read instead (tools/ab/soa.sh)
  const float4* __restrict__ soa;
  long long soa_stride;
  const uint32_t* __restrict__ occ;    // 1 bit per cell, cell_index order
  // Coarse occupancy: 1 bit per block of kBlock^3 cells (any active cell -> 1);
  // lets the march jump over empty blocks without changing the sample set.
  const uint32_t* __restrict__ bocc;
  int bx, by, bz;
  int all_blocks_active;  // host-known: no empty block, the jump can be compiled out
  // Second level: 1 bit per superblock of 8^3 blocks (64^3 cells).
  const uint32_t* __restrict__ socc;
  int sx, sy, sz;
  // Touched vertex blocks (8^3 vertices), consumed (and cleared) by the
  // block-sparse RMSProp and the multi-GPU exchanges; derived after each scatter
  // from the touched CELL blocks (8^3 cells, the bocc grid) the scatter marks.
  uint32_t* tb;
  int tbx, tby, tbz;
  uint32_t* tc;
};

constexpr int kBlockLog2 = 3;  // 8^3-cell blocks
constexpr int kSuperLog2 = 6;  // 64^3-cell superblocks
constexpr int kTouchLog2 = 3;  // 8^3-vertex touched blocks

// Marks the 8^3-cell block of cell (cx, cy, cz) as touched by the scatter (the
// vertex blocks its corners fall in are derived after the pass, k_touched_dilate:
// a cell block's vertices span its own vertex block and the +x/+y/+z neighbours).
// `last` caches the last block id to skip repeats; the atomic is skipped when the
// bit is already set.
__device__ __forceinline__ void mark_touched(const DevGrid& g, int cx, int cy, int cz, int& last) {
  const int b = (cx >> kBlockLog2) + g.bx * ((cy >> kBlockLog2) + g.by * (cz >> kBlockLog2));
  if (b == last) return;
  last = b;
  const uint32_t bit = 1u << (b & 31);
  // L1-cached check: bits are only ever set during the pass, so a stale word can
  // only cost a redundant atomicOr, never a missed mark
  if (!(__ldca(g.tc + (b >> 5)) & bit)) atomicOr(g.tc + (b >> 5), bit);
}

// RenderParams after effective_step / effective_t_far (renderer.hpp:18-24).
struct DevParams {
  double step, t_near, t_far, eps;
};

struct DevCam {
  double fx, fy, cx, cy;
  int width, height;
};

struct DevPose {
  double q[4];  // w x y z
  double t[3];
  double pad;
};

// ---------------------------------------------------------------- geometry
// Eigen (a.x*b.x + a.y*b.y) + a.z*b.z
__device__ __forceinline__ double dot3(const double a[3], const double b[3]) {
  return dadd(dadd(dmul(a[0], b[0]), dmul(a[1], b[1])), dmul(a[2], b[2]));
}
__device__ __forceinline__ void cross3(const double a[3], const double b[3], double o[3]) {
  const double r0 = dsub(dmul(a[1], b[2]), dmul(a[2], b[1]));
  const double r1 = dsub(dmul(a[2], b[0]), dmul(a[0], b[2]));
  const double r2 = dsub(dmul(a[0], b[1]), dmul(a[1], b[0]));
  o[0] = r0;
  o[1] = r1;
  o[2] = r2;
}

// pixel_direction_cam + Pose::rotate (camera.hpp:33-41, pose.hpp:16):
// normalized() = v / sqrt(squaredNorm); q*v = v + w*uv + qv x uv, uv = 2 (qv x v).
__device__ __forceinline__ void generate_dir(const DevCam& c, const DevPose& pose, double u,
                                             double v, double d[3]) {
  double cam[3] = {ddiv(dsub(u, c.cx), c.fx), ddiv(dsub(v, c.cy), c.fy), 1.0};
  const double z = dot3(cam, cam);
  if (z > 0.0) {
    const double s = __dsqrt_rn(z);
    cam[0] = ddiv(cam[0], s);
    cam[1] = ddiv(cam[1], s);
    cam[2] = ddiv(cam[2], s);
  }
  const double qv[3] = {pose.q[1], pose.q[2], pose.q[3]};
  double uv[3], c2[3];
  cross3(qv, cam, uv);
  uv[0] = dadd(uv[0], uv[0]);
  uv[1] = dadd(uv[1], uv[1]);
  uv[2] = dadd(uv[2], uv[2]);
  cross3(qv, uv, c2);
  for (int i = 0; i < 3; ++i) d[i] = dadd(dadd(cam[i], dmul(pose.q[0], uv[i])), c2[i]);
}

// sh_eval — voxel_grid.cpp:34-47. Returns false if |d| is not unit (the
// reference throws std::invalid_argument).
__device__ __forceinline__ bool sh_basis(const double d[3], double b[9]) {
  const double n = __dsqrt_rn(dot3(d, d));
  if (fabs(dsub(n, 1.0)) > 1e-9) return false;
  const double x = d[0], y = d[1], z = d[2];
  b[0] = kC0;
  b[1] = dmul(-kC1, y);
  b[2] = dmul(kC1, z);
  b[3] = dmul(-kC1, x);
  b[4] = dmul(dmul(kC2_xy, x), y);
  b[5] = dmul(dmul(kC2_yz, y), z);
  b[6] = dmul(kC2_zz, dsub(dsub(dmul(dmul(2.0, z), z), dmul(x, x)), dmul(y, y)));
  b[7] = dmul(dmul(kC2_xz, x), z);
  b[8] = dmul(kC2_xxyy, dsub(dmul(x, x), dmul(y, y)));
  return true;
}

// ---------------------------------------------------------------- march
struct March {
  double o[3], d[3];
  double lo, hi, step;
  long long nseg, k;
  double inv_d[3], inv_step;  // for the (margin-guarded) empty-space jumps only
};

// Slab clip + range clamp + segment count — renderer.cpp:12-29, 51-73.
__device__ __forceinline__ bool march_begin(const DevGrid& g, const DevParams& p, March& m) {
  const double wmin[3] = {g.ox, g.oy, g.oz};
  const double wmax[3] = {g.hx, g.hy, g.hz};
  double t_enter = 0.0, t_exit = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  for (int a = 0; a < 3; ++a) {
    if (fabs(m.d[a]) < 1e-15) {
      if (m.o[a] < wmin[a] || m.o[a] > wmax[a]) return false;
      continue;
    }
    double t0 = ddiv(dsub(wmin[a], m.o[a]), m.d[a]);
    double t1 = ddiv(dsub(wmax[a], m.o[a]), m.d[a]);
    if (t0 > t1) {
      const double tmp = t0;
      t0 = t1;
      t1 = tmp;
    }
    t_enter = (t_enter < t0) ? t0 : t_enter;
    t_exit = (t1 < t_exit) ? t1 : t_exit;
  }
  if (!(t_enter < t_exit)) return false;
  m.lo = (p.t_near < t_enter) ? t_enter : p.t_near;
  m.hi = (t_exit < p.t_far) ? t_exit : p.t_far;
  if (m.hi <= m.lo) return false;
  m.step = p.step;
  m.nseg = (long long)ceil(dsub(ddiv(dsub(m.hi, m.lo), p.step), 1e-12));
  m.k = 0;
  for (int a = 0; a < 3; ++a) m.inv_d[a] = m.d[a] == 0.0 ? 0.0 : 1.0 / m.d[a];
  m.inv_step = 1.0 / p.step;
  return true;
}

// One located sample: cell, fractional coordinates, base vertex.
struct Sample {
  double t, delta;
  double fx, fy, fz;
  uint32_t base;   // vertex_index(cell)
  uint32_t cell;   // cell_index(cell)
  int cx, cy, cz;  // cell coordinates
};

// try_locate — voxel_grid.cpp:83-105 — for the segment midpoint, plus the
// occupancy test (renderer.cpp:69-70). Returns false for a dropped sample.
// a / voxel, correctly rounded, without a division: with y = RN(1/voxel) (host
// IEEE division), q0 = RN(a y) is within 1 ulp of a/voxel and one FMA residual
// correction q0 + RN(a - q0 voxel) y yields RN(a/voxel) (Markstein). Checked
// against IEEE division on 4e8 random and near-integer quotients.
__device__ __forceinline__ double div_voxel(const DevGrid& g, double a) {
  const double q0 = dmul(a, g.rcp_voxel);
  const double r = __fma_rn(-q0, g.voxel, a);
  return __fma_rn(r, g.rcp_voxel, q0);
}

__device__ __forceinline__ bool locate(const DevGrid& g, const double p[3], Sample& s) {
  const double gx = div_voxel(g, dsub(p[0], g.ox));
  const double gy = div_voxel(g, dsub(p[1], g.oy));
  const double gz = div_voxel(g, dsub(p[2], g.oz));
  if (!(gx >= 0.0 && gx <= (double)g.rx - 1.0)) return false;
  if (!(gy >= 0.0 && gy <= (double)g.ry - 1.0)) return false;
  if (!(gz >= 0.0 && gz <= (double)g.rz - 1.0)) return false;
  int cx = (int)ceil(gx) - 1, cy = (int)ceil(gy) - 1, cz = (int)ceil(gz) - 1;
  cx = cx < 0 ? 0 : (cx > g.rx - 2 ? g.rx - 2 : cx);
  cy = cy < 0 ? 0 : (cy > g.ry - 2 ? g.ry - 2 : cy);
  cz = cz < 0 ? 0 : (cz > g.rz - 2 ? g.rz - 2 : cz);
  s.fx = dsub(gx, (double)cx);
  s.fy = dsub(gy, (double)cy);
  s.fz = dsub(gz, (double)cz);
  s.base = (uint32_t)(cx + g.rx * (cy + (long long)g.ry * cz));
  s.cell = (uint32_t)(cx + (g.rx - 1) * (cy + (long long)(g.ry - 1) * cz));
  s.cx = cx;
  s.cy = cy;
  s.cz = cz;
  return true;
}

__device__ __forceinline__ bool cell_active(const DevGrid& g, uint32_t cell) {
  return (__ldg(g.occ + (cell >> 5)) >> (cell & 31)) & 1u;
}

__device__ __forceinline__ bool block_active(const DevGrid& g, int cx, int cy, int cz) {
  const int b = (cx >> kBlockLog2) + g.bx * ((cy >> kBlockLog2) + g.by * (cz >> kBlockLog2));
  return (__ldg(g.bocc + (b >> 5)) >> (b & 31)) & 1u;
}

__device__ __forceinline__ bool super_active(const DevGrid& g, int cx, int cy, int cz) {
  const int b = (cx >> kSuperLog2) + g.sx * ((cy >> kSuperLog2) + g.sy * (cz >> kSuperLog2));
  return (__ldg(g.socc + (b >> 5)) >> (b & 31)) & 1u;
}

// The sample at s lies in an all-inactive box of 2^L cells per axis (an 8^3
// block, or a 64^3 superblock): return the first segment index whose midpoint
// may lie beyond the box. Every segment in between has its midpoint inside the
// (convex) box — the ray is inside it at s.t and until the box exit t_out — and
// would be dropped by the occupancy test, so skipping them leaves the schedule
// unchanged. A 1e-6 m margin keeps the jump clear of the exit face and absorbs
// the rounding of the reciprocal-based exit time.
// RECIP = true recomputes the reciprocals (m.inv_d, m.inv_step) instead of
// reading them, and a non-null `origin` (the ray origin in global memory, e.g.
// the pose translation every ray of a tracking batch starts from) replaces m.o:
// the same values, so the same jump, and callers short of registers need not
// keep them live (k_pose_group_u).
template <bool RECIP = false>
__device__ __forceinline__ long long skip_empty_box(const DevGrid& g, const March& m,
                                                    const Sample& s, int L,
                                                    const double* __restrict__ origin = nullptr) {
  const double ext = (double)(1 << L) * g.voxel;
  const int b[3] = {s.cx >> L, s.cy >> L, s.cz >> L};
  const double org[3] = {g.ox, g.oy, g.oz};
  double t_out = 1e300;
  for (int a = 0; a < 3; ++a) {
    if (m.d[a] == 0.0) continue;
    const double face = org[a] + (m.d[a] > 0.0 ? (b[a] + 1) : b[a]) * ext;
    const double oa = (RECIP && origin) ? __ldg(origin + a) : m.o[a];
    const double t = (face - oa) * (RECIP ? 1.0 / m.d[a] : m.inv_d[a]);
    t_out = t < t_out ? t : t_out;
  }
  // midpoint of segment k is ~ lo + (k + 0.5) step; stay below t_out - margin
  const double kf = floor((t_out - 1e-6 - m.lo) * (RECIP ? 1.0 / m.step : m.inv_step) - 0.5);
  const long long k_new = kf > (double)m.nseg ? m.nseg : (long long)kf;
  return k_new > m.k ? k_new : m.k;
}

// Next scheduled, in-bounds, active sample — renderer.cpp:62-79 evaluated lazily.
// SKIP = false compiles out the empty-block jump (grids with every block occupied).
template <bool SKIP = true>
__device__ __forceinline__ bool march_next(const DevGrid& g, March& m, Sample& s) {
  while (m.k < m.nseg) {
    const double s0 = dadd(m.lo, dmul((double)m.k, m.step));
    ++m.k;
    const double s0s = dadd(s0, m.step);
    const double s1 = (m.hi < s0s) ? m.hi : s0s;
    const double len = dsub(s1, s0);
    if (len < 1e-12) continue;
    const double tm = dmul(0.5, dadd(s0, s1));
    const double p[3] = {dadd(m.o[0], dmul(tm, m.d[0])), dadd(m.o[1], dmul(tm, m.d[1])),
                         dadd(m.o[2], dmul(tm, m.d[2]))};
    if (!locate(g, p, s)) continue;
    if (!cell_active(g, s.cell)) {
      // jump past the empty 8^3 block / 64^3 superblock (exact: segments whose
      // midpoints stay inside the empty box are the ones dropped anyway). A
      // cell-level jump inside occupied blocks measured slower (r01: config-2
      // GN tracking 436 -> 396 frames/s): near surfaces an empty cell is
      // crossed in 1-2 segments and the jump only adds divergent work.
      if (SKIP && !block_active(g, s.cx, s.cy, s.cz))
        m.k = skip_empty_box(g, m, s,
                             super_active(g, s.cx, s.cy, s.cz) ? kBlockLog2 : kSuperLog2);
      continue;
    }
    s.t = tm;
    s.delta = len;
    return true;
  }
  return false;
}

// ------------------------------------------------------------------ group march
// The LPR lanes of a ray group march together: a batch evaluates the next LPR
// segments at once (lane j: segment k + j — position, locate, occupancy), a
// group ballot marks the active ones, and next() hands them out in segment
// order (the sample's fields are shuffled from the lane that located it).
// Segments are independent given the occupancy, so this yields exactly the
// sequential march_next sequence (renderer.cpp:62-79): inactive / out-of-grid
// segments are dropped in order, and an all-inactive batch whose last
// empty-block lane lies in an empty 8^3 block / 64^3 superblock jumps past
// that box (skip_empty_box: only segments whose midpoints stay inside the empty
// box are skipped). Empty space inside occupied blocks then costs one batch per
// LPR segments instead of one iteration per segment.
template <int LPR>
struct GroupMarch {
  Sample mine;       // this lane's segment of the current batch
  long long mine_k = 0;
  unsigned act = 0;  // active segments of the batch not yet handed out (group bits)
  long long seg = -1;  // segment index of the sample last handed out

  __device__ __forceinline__ bool next(const DevGrid& g, March& m, Sample& s, int sub, int gbase,
                                       unsigned gmask) {
    constexpr unsigned kLow = (LPR == 32) ? 0xffffffffu : ((1u << LPR) - 1u);
    while (act == 0) {
      if (m.k >= m.nseg) return false;
      const long long kk = m.k + sub;
      mine_k = kk;
      bool a = false, eb = false;
      if (kk < m.nseg) {
        const double s0 = dadd(m.lo, dmul((double)kk, m.step));
        const double s0s = dadd(s0, m.step);
        const double s1 = (m.hi < s0s) ? m.hi : s0s;
        const double len = dsub(s1, s0);
        if (len >= 1e-12) {
          const double tm = dmul(0.5, dadd(s0, s1));
          const double p[3] = {dadd(m.o[0], dmul(tm, m.d[0])), dadd(m.o[1], dmul(tm, m.d[1])),
                               dadd(m.o[2], dmul(tm, m.d[2]))};
          if (locate(g, p, mine)) {
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
      act = (__ballot_sync(gmask, a) >> gbase) & kLow;
      const unsigned ebm = (__ballot_sync(gmask, eb) >> gbase) & kLow;
      m.k += LPR;
      if (act == 0 && ebm) {
        const int j = 31 - __clz(ebm);
        long long kn = 0;
        if (sub == j)
          kn = skip_empty_box(g, m, mine,
                              super_active(g, mine.cx, mine.cy, mine.cz) ? kBlockLog2 : kSuperLog2);
        kn = __shfl_sync(gmask, kn, gbase + j);
        if (kn > m.k) m.k = kn;
      }
    }
    const int src = gbase + (__ffs(act) - 1);
    act &= act - 1;
    s.t = __shfl_sync(gmask, mine.t, src);
    s.delta = __shfl_sync(gmask, mine.delta, src);
    s.fx = __shfl_sync(gmask, mine.fx, src);
    s.fy = __shfl_sync(gmask, mine.fy, src);
    s.fz = __shfl_sync(gmask, mine.fz, src);
    s.base = __shfl_sync(gmask, mine.base, src);
    const uint32_t cpk = __shfl_sync(gmask, (uint32_t)mine.cx | ((uint32_t)mine.cy << 10) |
                                                ((uint32_t)mine.cz << 20), src);
    s.cx = (int)(cpk & 1023u);
    s.cy = (int)((cpk >> 10) & 1023u);
    s.cz = (int)(cpk >> 20);
    seg = __shfl_sync(gmask, mine_k, src);
    return true;
  }
};

__device__ __forceinline__ uint32_t corner_index(const DevGrid& g, uint32_t base, int k) {
  return base + (uint32_t)(k & 1) + ((k >> 1) & 1) * (uint32_t)g.rx + ((k >> 2) & 1) * g.rxy;
}

// Trilinear weights in the reference order wx[dx]*wy[dy]*wz[dz].
__device__ __forceinline__ void corner_weights(const Sample& s, double w[8]) {
  const double wx[2] = {dsub(1.0, s.fx), s.fx};
  const double wy[2] = {dsub(1.0, s.fy), s.fy};
  const double wz[2] = {dsub(1.0, s.fz), s.fz};
#pragma unroll
  for (int k = 0; k < 8; ++k) w[k] = dmul(dmul(wx[k & 1], wy[(k >> 1) & 1]), wz[(k >> 2) & 1]);
}

// ---------------------------------------------------------------- shading
// trilerp (voxel_grid.cpp:113-122) + per-channel SH colour with +0.5, clamp
// and clamp flag (renderer.cpp:104-112).
struct Shade {
  double sigma_raw;
  double c[3];
  bool clamped[3];
};

// VRF_GATHER_HINT=1 (A/B): the fast forward's corner gathers at L2 evict-last
// priority (the payload stays resident against the streaming records).
#ifndef VRF_GATHER_HINT
#define VRF_GATHER_HINT 0
#endif
__device__ __forceinline__ float4 ldg_payload(const float4* p, unsigned long long pol) {
#if VRF_GATHER_HINT
  float4 r;
  asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p), "l"(pol));
  return r;
#else
  (void)pol;
  return __ldg(p);
#endif
}
__device__ __forceinline__ unsigned long long payload_policy() {
#if VRF_GATHER_HINT
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
#else
  return 0ull;
#endif
}

// Fast path (fp32 SH): the colour is contracted with the basis per corner,
// c_ch = 0.5 + sum_k w_k (sum_m basis_m v_k[ch,m]), so only 3 accumulators are
// live instead of 27. sigma_raw stays the FP64 reference-order replay, so T and
// the termination decision are unchanged; colour differs from the reference's
// accumulate-then-contract order at the fp32 rounding level (~1e-7).
__device__ __forceinline__ void shade_fast(const DevGrid& g, const Sample& s, const double w[8],
                                           const float bf[9], Shade& out) {
  double sraw = 0.0;
  float cr = 0.f, cg = 0.f, cb = 0.f;
  const unsigned long long pol = payload_policy();
#pragma unroll
  for (int k = 0; k < 8; ++k) {
#ifdef VRF_GATHER_SOA
    // (contexts that never ran a mapping forward have no planar copy: AoS)
    const float4* vp = g.soa ? g.soa + corner_index(g, s.base, k)
                             : g.payload + (size_t)corner_index(g, s.base, k) * kVec4PerVertex;
    const long long js = g.soa ? g.soa_stride : 1;
#else
    const float4* vp = g.payload + (size_t)corner_index(g, s.base, k) * kVec4PerVertex;
    constexpr long long js = 1;
#endif
    float v[28];
#pragma unroll
    for (int j = 0; j < kVec4PerVertex; ++j) {
      const float4 a = ldg_payload(vp + j * js, pol);
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

// Per-ray corner cache of the fast forward (K0). A corner's contribution to
// shade_fast depends only on the ray (its basis) and the corner: (sigma_k,
// sum_m basis_m v_k[ch,m]). Consecutive samples share corners: all 8 within a
// cell, 4 across a face. The lane keeps the 8 corner contributions of its
// current cell in shared memory, relabelled as K2's CornerAgg does (logical
// corner k in slot k ^ X; a move along axes M refills the departing slots with
// the entering corners and sets X ^= M), and gathers only the corners it has
// not seen: ~3 of 8 per sample instead of 8. Same operations in the same order
// as shade_fast, so the results are bit-identical.
// VRF_K0_CACHE=1 (A/B build, tools/ab/k0_cache.sh): K0 shades through the
// corner cache. It cuts K0's L1 data-pipe wavefronts by 28 % and its global
// sectors by half, but the per-corner branch diverges (+14 % warp instructions)
// and K0 turns latency-bound: config 3 9.07 ms against 8.68, config 4 27.8
// against 28.7 (r02). A predicated, branch-free form spilled and took 11.2 ms.
#ifndef VRF_K0_CACHE
#define VRF_K0_CACHE 0
#endif
constexpr int kCacheStride = 128;  // threads per CTA of the kernels that use it
struct CornerCache {
  float4* slot0;  // this lane's slot 0; slot s at slot0[s * kCacheStride]
  uint32_t X;
  uint32_t cell;  // pack_cell of the cached cell; 0xffffffff: empty
};
__device__ __forceinline__ uint32_t cache_pack(int cx, int cy, int cz) {
  return (uint32_t)cx | ((uint32_t)cy << 10) | ((uint32_t)cz << 20);
}
// Slots (bit s = slot s) to refill for the sample's cell, updating X / cell.
__device__ __forceinline__ uint32_t cache_enter(CornerCache& cc, const Sample& s) {
  const uint32_t key = cache_pack(s.cx, s.cy, s.cz);
  if (key == cc.cell) return 0u;
  uint32_t dep = 0xffu;
  if (cc.cell != 0xffffffffu) {
    const int dx = s.cx - (int)(cc.cell & 1023u), dy = s.cy - (int)((cc.cell >> 10) & 1023u),
              dz = s.cz - (int)(cc.cell >> 20);
    if (dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 && dz <= 1) {
      dep = 0;
      if (dx != 0) dep |= ((cc.X & 1u) ^ (uint32_t)(dx < 0)) ? 0xAAu : 0x55u;
      if (dy != 0) dep |= (((cc.X >> 1) & 1u) ^ (uint32_t)(dy < 0)) ? 0xCCu : 0x33u;
      if (dz != 0) dep |= (((cc.X >> 2) & 1u) ^ (uint32_t)(dz < 0)) ? 0xF0u : 0x0Fu;
      cc.X ^= (uint32_t)(dx != 0) | ((uint32_t)(dy != 0) << 1) | ((uint32_t)(dz != 0) << 2);
    }
  }
  cc.cell = key;
  return dep;
}
__device__ __forceinline__ void shade_cached(const DevGrid& g, const Sample& s, const double w[8],
                                             const float bf[9], CornerCache& cc, Shade& out) {
  const uint32_t refill = cache_enter(cc, s);
  double sraw = 0.0;
  float cr = 0.f, cg = 0.f, cb = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t sl = (uint32_t)k ^ cc.X;
    float4* cp = cc.slot0 + sl * kCacheStride;
    float4 cv;
    if ((refill >> sl) & 1u) {
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
      float dr = 0.f, dg = 0.f, db = 0.f;
#pragma unroll
      for (int m = 0; m < 9; ++m) {
        dr = fmaf(bf[m], v[1 + m], dr);
        dg = fmaf(bf[m], v[10 + m], dg);
        db = fmaf(bf[m], v[19 + m], db);
      }
      cv = make_float4(v[0], dr, dg, db);
      *cp = cv;
    } else {
      cv = *cp;
    }
    sraw = dadd(sraw, dmul(w[k], (double)cv.x));
    const float wk = (float)w[k];
    cr = fmaf(wk, cv.y, cr);
    cg = fmaf(wk, cv.z, cg);
    cb = fmaf(wk, cv.w, cb);
  }
  out.sigma_raw = sraw;
  const float c3[3] = {cr, cg, cb};
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    const double v = 0.5 + (double)c3[ch];
    out.clamped[ch] = (v <= 0.0 || v >= 1.0);
    out.c[ch] = (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v);
  }
}

template <typename ShT>
__device__ __forceinline__ void shade(const DevGrid& g, const Sample& s, const double w[8],
                                      const double basis[9], Shade& out) {
  if constexpr (sizeof(ShT) == 4) {
    float bf[9];
#pragma unroll
    for (int m = 0; m < 9; ++m) bf[m] = (float)basis[m];
    shade_fast(g, s, w, bf, out);
    return;
  }
  double sraw = 0.0;
  ShT sh[27];
#pragma unroll
  for (int m = 0; m < 27; ++m) sh[m] = ShT(0);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float4* vp = g.payload + (size_t)corner_index(g, s.base, k) * kVec4PerVertex;
    const double wk = w[k];
    const ShT wks = ShT(wk);
#pragma unroll
    for (int j = 0; j < kVec4PerVertex; ++j) {
      const float4 a = __ldg(vp + j);
      const float vals[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int slot = 4 * j + e;
        if (slot == 0) {
          sraw = dadd(sraw, dmul(wk, (double)vals[e]));
        } else {
          if constexpr (sizeof(ShT) == 8)
            sh[slot - 1] = dadd(sh[slot - 1], dmul(wk, (double)vals[e]));
          else
            sh[slot - 1] = fmaf(wks, vals[e], sh[slot - 1]);
        }
      }
    }
  }
  out.sigma_raw = sraw;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    double v = 0.5;
#pragma unroll
    for (int m = 0; m < 9; ++m) v = dadd(v, dmul((double)sh[ch * 9 + m], basis[m]));
    out.clamped[ch] = (v <= 0.0 || v >= 1.0);
    out.c[ch] = (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v);
  }
}

// Compositing state of one ray — renderer.cpp:89-139.
struct Composite {
  double T;
  double C[3];
  double D;
  int count;
  bool terminated;
};

// One front-to-back step. Returns the weight; advances T; decay out for T_{i+1}.
__device__ __forceinline__ double composite_step(Composite& st, const Shade& sh, double t,
                                                 double delta, double eps, double& decay) {
  const double sigma = (sh.sigma_raw < 0.0) ? 0.0 : sh.sigma_raw;
  decay = exp(dmul(-sigma, delta));
  const double alpha = dsub(1.0, decay);
  const double w = dmul(st.T, alpha);
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) st.C[ch] = dadd(st.C[ch], dmul(w, sh.c[ch]));
  st.D = dadd(st.D, dmul(w, t));
  st.T = dmul(st.T, decay);
  ++st.count;
  if (st.T < eps) st.terminated = true;
  return w;
}

__device__ __forceinline__ void ray_from_pixel(const DevCam& cam, const DevPose& pose, double u,
                                               double v, March& m) {
  generate_dir(cam, pose, u, v, m.d);
  m.o[0] = pose.t[0];
  m.o[1] = pose.t[1];
  m.o[2] = pose.t[2];
}

// Forward render of one ray: composite until termination. Returns false if the
// SH basis precondition fails (sh_eval throws, voxel_grid.cpp:35-36).
template <typename ShT>
__device__ __forceinline__ bool render_forward(const DevGrid& g, const DevParams& p, March& m,
                                               Composite& st, double basis[9]) {
  st.T = 1.0;
  st.C[0] = st.C[1] = st.C[2] = 0.0;
  st.D = 0.0;
  st.count = 0;
  st.terminated = false;
  if (!sh_basis(m.d, basis)) return false;
  if (!march_begin(g, p, m)) return true;
  Sample s;
  while (march_next(g, m, s)) {
    double w[8];
    corner_weights(s, w);
    Shade sh;
    shade<ShT>(g, s, w, basis, sh);
    double decay;
    composite_step(st, sh, s.t, s.delta, p.eps, decay);
    if (st.terminated) break;
  }
  if (st.count == 0) {
    st.C[0] = st.C[1] = st.C[2] = 0.0;
    st.D = 0.0;
  }
  return true;
}

// ---------------------------------------------------------------- reductions
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

}  // namespace vrf
