/* voxrf CPU oracle — TEST INFRASTRUCTURE ONLY (see voxrf_oracle.h).
 *
 * Plain C, FP64, single-threaded. Every function restates the reference
 * function cited beside it with the same operation order, so the results are
 * bit-identical to oracle/_ref (the reference's own sources compiled against
 * the Eigen-subset shim) — tests/test_oracle_pinning.py checks exactly that.
 * Compiled with -ffp-contract=off (the reference's default x86-64 Release
 * build has no FMA contraction). */
#include "voxrf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define SH_N 9
#define PAYLOAD 28

/* voxel_grid.cpp:11-17 */
static const double kC0 = 0.28209479177387814;
static const double kC1 = 0.4886025119029199;
static const double kC2_xy = 1.0925484305920792;
static const double kC2_yz = -1.0925484305920792;
static const double kC2_zz = 0.31539156525252005;
static const double kC2_xz = -1.0925484305920792;
static const double kC2_xxyy = 0.5462742152960396;

/* ---------------------------------------------------------------- Eigen-order vector helpers */
static double dot3(const double a[3], const double b[3]) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}
static double norm3(const double a[3]) { return sqrt(dot3(a, a)); }
static void cross3(const double a[3], const double b[3], double o[3]) {
  double r0 = a[1] * b[2] - a[2] * b[1];
  double r1 = a[2] * b[0] - a[0] * b[2];
  double r2 = a[0] * b[1] - a[1] * b[0];
  o[0] = r0;
  o[1] = r1;
  o[2] = r2;
}
static void normalized3(const double a[3], double o[3]) {
  double z = dot3(a, a);
  if (z > 0.0) {
    double s = sqrt(z);
    o[0] = a[0] / s;
    o[1] = a[1] / s;
    o[2] = a[2] / s;
  } else {
    o[0] = a[0];
    o[1] = a[1];
    o[2] = a[2];
  }
}
/* Eigen QuaternionBase::_transformVector (pose.hpp:16) */
static void quat_rotate(const double q[4], const double v[3], double o[3]) {
  const double qv[3] = {q[1], q[2], q[3]};
  double uv[3], c2[3], t[3];
  cross3(qv, v, uv);
  uv[0] = uv[0] + uv[0];
  uv[1] = uv[1] + uv[1];
  uv[2] = uv[2] + uv[2];
  cross3(qv, uv, c2);
  for (int i = 0; i < 3; ++i) t[i] = v[i] + q[0] * uv[i];
  for (int i = 0; i < 3; ++i) o[i] = t[i] + c2[i];
}
/* quaternion coefficient squaredNorm in Eigen storage order (x,y,z,w), SSE2 packet order */
static void quat_normalize(double q[4]) {
  double x = q[1], y = q[2], z = q[3], w = q[0];
  double n2 = (x * x + z * z) + (y * y + w * w);
  if (n2 > 0.0) {
    double s = sqrt(n2);
    q[0] = w / s;
    q[1] = x / s;
    q[2] = y / s;
    q[3] = z / s;
  }
}
static void quat_mul(const double a[4], const double b[4], double o[4]) {
  double aw = a[0], ax = a[1], ay = a[2], az = a[3];
  double bw = b[0], bx = b[1], by = b[2], bz = b[3];
  double rw = aw * bw - ax * bx - ay * by - az * bz;
  double rx = aw * bx + ax * bw + ay * bz - az * by;
  double ry = aw * by + ay * bw + az * bx - ax * bz;
  double rz = aw * bz + az * bw + ax * by - ay * bx;
  o[0] = rw;
  o[1] = rx;
  o[2] = ry;
  o[3] = rz;
}

/* ---------------------------------------------------------------- rng.hpp:13-81 */
static uint64_t splitmix64(uint64_t* x) {
  *x += 0x9e3779b97f4a7c15ULL;
  uint64_t z = *x;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
void or_rng_seed(uint64_t seed, uint64_t s[4]) {
  uint64_t x = seed;
  for (int i = 0; i < 4; ++i) s[i] = splitmix64(&x);
}
uint64_t or_rng_next(uint64_t s[4]) {
  const uint64_t result = rotl(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}
uint64_t or_rng_uniform_index(uint64_t s[4], uint64_t n) {
  return (uint64_t)(((unsigned __int128)or_rng_next(s) * n) >> 64);
}
double or_rng_uniform(uint64_t s[4]) { return (double)(or_rng_next(s) >> 11) * 0x1.0p-53; }

/* mapping.cpp:121-128 */
void or_draw_batch(uint64_t s[4], int n_frames, int width, int height, int n_rays,
                   int32_t* batch) {
  for (int i = 0; i < n_rays; ++i) {
    batch[3 * i + 0] = (int32_t)or_rng_uniform_index(s, (uint64_t)n_frames);
    batch[3 * i + 1] = (int32_t)or_rng_uniform_index(s, (uint64_t)width);
    batch[3 * i + 2] = (int32_t)or_rng_uniform_index(s, (uint64_t)height);
  }
}

/* ---------------------------------------------------------------- geometry */
/* camera.hpp:33-41 */
int or_generate_ray(const or_intrinsics* in, const or_pose* pose, double u, double v,
                    double o[3], double d[3]) {
  if (u < 0.0 || u >= in->width || v < 0.0 || v >= in->height) return OR_OUT_OF_RANGE;
  double cam[3] = {(u - in->cx) / in->fx, (v - in->cy) / in->fy, 1.0}, n[3];
  normalized3(cam, n);
  quat_rotate(pose->q, n, d);
  o[0] = pose->t[0];
  o[1] = pose->t[1];
  o[2] = pose->t[2];
  return OR_OK;
}

/* voxel_grid.hpp:44-47 */
static void world_max(const or_geometry* g, double hi[3]) {
  for (int a = 0; a < 3; ++a) hi[a] = g->origin[a] + ((double)g->res[a] - 1.0) * g->voxel_size;
}
static double diagonal(const or_geometry* g) {
  double hi[3], e[3];
  world_max(g, hi);
  for (int a = 0; a < 3; ++a) e[a] = hi[a] - g->origin[a];
  return norm3(e);
}
/* voxel_grid.hpp:57-62 */
static uint32_t vertex_index(const or_geometry* g, int ix, int iy, int iz) {
  return (uint32_t)(ix + g->res[0] * (iy + (int64_t)g->res[1] * iz));
}
static uint32_t cell_index(const or_geometry* g, int cx, int cy, int cz) {
  return (uint32_t)(cx + (g->res[0] - 1) * (cy + (int64_t)(g->res[1] - 1) * cz));
}

typedef struct {
  int cell[3];
  double frac[3];
  uint32_t corner[8];
  double weight[8];
} locator;

/* voxel_grid.cpp:83-105 */
static int try_locate(const or_geometry* g, const double p[3], locator* out) {
  double gc[3];
  for (int a = 0; a < 3; ++a) gc[a] = (p[a] - g->origin[a]) / g->voxel_size;
  for (int a = 0; a < 3; ++a)
    if (!(gc[a] >= 0.0 && gc[a] <= g->res[a] - 1.0)) return 0;
  for (int a = 0; a < 3; ++a) {
    int c = (int)ceil(gc[a]) - 1;
    if (c < 0) c = 0;
    if (c > g->res[a] - 2) c = g->res[a] - 2;
    out->cell[a] = c;
    out->frac[a] = gc[a] - c;
  }
  const double wx[2] = {1.0 - out->frac[0], out->frac[0]};
  const double wy[2] = {1.0 - out->frac[1], out->frac[1]};
  const double wz[2] = {1.0 - out->frac[2], out->frac[2]};
  for (int k = 0; k < 8; ++k) {
    const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
    out->corner[k] = vertex_index(g, out->cell[0] + dx, out->cell[1] + dy, out->cell[2] + dz);
    out->weight[k] = wx[dx] * wy[dy] * wz[dz];
  }
  return 1;
}

/* try_locate with the grid coordinate clamped into [0, res-1] instead of
 * rejecting (used only by or_upsample's clamp_outside mode). */
static void locate_clamped(const or_geometry* g, const double p[3], locator* out) {
  double gc[3];
  for (int a = 0; a < 3; ++a) {
    gc[a] = (p[a] - g->origin[a]) / g->voxel_size;
    if (!(gc[a] >= 0.0)) gc[a] = 0.0;
    if (gc[a] > g->res[a] - 1.0) gc[a] = g->res[a] - 1.0;
  }
  for (int a = 0; a < 3; ++a) {
    int c = (int)ceil(gc[a]) - 1;
    if (c < 0) c = 0;
    if (c > g->res[a] - 2) c = g->res[a] - 2;
    out->cell[a] = c;
    out->frac[a] = gc[a] - c;
  }
  const double wx[2] = {1.0 - out->frac[0], out->frac[0]};
  const double wy[2] = {1.0 - out->frac[1], out->frac[1]};
  const double wz[2] = {1.0 - out->frac[2], out->frac[2]};
  for (int k = 0; k < 8; ++k) {
    const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
    out->corner[k] = vertex_index(g, out->cell[0] + dx, out->cell[1] + dy, out->cell[2] + dz);
    out->weight[k] = wx[dx] * wy[dy] * wz[dz];
  }
}

/* voxel_grid.cpp:113-122 */
static void trilerp(const or_grid* g, const locator* loc, double* sigma_raw, double sh[27]) {
  double s = 0.0;
  for (int m = 0; m < 27; ++m) sh[m] = 0.0;
  for (int k = 0; k < 8; ++k) {
    const double w = loc->weight[k];
    const double* v = g->data + (size_t)loc->corner[k] * PAYLOAD;
    s += w * v[0];
    for (int m = 0; m < 27; ++m) sh[m] += w * v[1 + m];
  }
  *sigma_raw = s;
}

/* VoxelGrid::upsampled — voxel_grid.cpp:190-220. `out` holds the refined
 * geometry (2 res - 1, voxel / 2) and (2rx-1)(2ry-1)(2rz-1)*28 doubles;
 * active_out its cell mask. Returns OR_RUNTIME over max_resolution. */
int or_upsample(const or_grid* g, int max_resolution, int clamp_outside, or_geometry* fine,
                double* out, uint8_t* active_out) {
  or_geometry f = g->geom;
  for (int a = 0; a < 3; ++a) f.res[a] = 2 * g->geom.res[a] - 1;
  f.voxel_size = g->geom.voxel_size * 0.5;
  if (f.res[0] > max_resolution || f.res[1] > max_resolution || f.res[2] > max_resolution)
    return OR_RUNTIME;
  *fine = f;
  if (!out) return OR_OK;
  for (int iz = 0; iz < f.res[2]; ++iz)
    for (int iy = 0; iy < f.res[1]; ++iy)
      for (int ix = 0; ix < f.res[0]; ++ix) {
        const double gg[3] = {ix * 0.5, iy * 0.5, iz * 0.5};
        double p[3];
        for (int a = 0; a < 3; ++a) p[a] = g->geom.origin[a] + gg[a] * g->geom.voxel_size;
        locator loc;
        if (!try_locate(&g->geom, p, &loc)) {
          /* The reference throws here (locate, voxel_grid.cpp:107-111) when the
           * world round trip of a far-corner vertex lands an ulp outside the
           * box. clamp_outside != 0 instead clamps the grid coordinate into
           * [0, res-1] (the device behaviour: the boundary vertex's value). */
          if (!clamp_outside) return OR_OUT_OF_RANGE;
          locate_clamped(&g->geom, p, &loc);
        }
        double* v = out + (size_t)vertex_index(&f, ix, iy, iz) * PAYLOAD;
        trilerp(g, &loc, &v[0], &v[1]);
      }
  for (int cz = 0; cz < f.res[2] - 1; ++cz)
    for (int cy = 0; cy < f.res[1] - 1; ++cy)
      for (int cx = 0; cx < f.res[0] - 1; ++cx)
        active_out[cell_index(&f, cx, cy, cz)] =
            g->active[cell_index(&g->geom, cx / 2, cy / 2, cz / 2)];
  return OR_OK;
}

/* voxel_grid.cpp:34-47 */
int or_sh_eval(const double d[3], double b[9]) {
  if (fabs(norm3(d) - 1.0) > 1e-9) return OR_INVALID_ARGUMENT;
  const double x = d[0], y = d[1], z = d[2];
  b[0] = kC0;
  b[1] = -kC1 * y;
  b[2] = kC1 * z;
  b[3] = -kC1 * x;
  b[4] = kC2_xy * x * y;
  b[5] = kC2_yz * y * z;
  b[6] = kC2_zz * (2.0 * z * z - x * x - y * y);
  b[7] = kC2_xz * x * z;
  b[8] = kC2_xxyy * (x * x - y * y);
  return OR_OK;
}

/* renderer.cpp:12-29 */
static int intersect_bounds(const or_geometry* g, const double o[3], const double d[3],
                            double* t_enter, double* t_exit) {
  double hi[3];
  world_max(g, hi);
  *t_enter = 0.0;
  *t_exit = INFINITY;
  for (int a = 0; a < 3; ++a) {
    if (fabs(d[a]) < 1e-15) {
      if (o[a] < g->origin[a] || o[a] > hi[a]) return 0;
      continue;
    }
    double t0 = (g->origin[a] - o[a]) / d[a];
    double t1 = (hi[a] - o[a]) / d[a];
    if (t0 > t1) {
      double tmp = t0;
      t0 = t1;
      t1 = tmp;
    }
    *t_enter = (*t_enter < t0) ? t0 : *t_enter; /* std::max */
    *t_exit = (t1 < *t_exit) ? t1 : *t_exit;    /* std::min */
  }
  return *t_enter < *t_exit;
}

/* renderer.hpp:18-24 */
static double eff_step(const or_render_params* p, const or_geometry* g) {
  return p->step > 0.0 ? p->step : 0.5 * g->voxel_size;
}
static double eff_t_far(const or_render_params* p, const or_geometry* g) {
  return p->t_far > 0.0 ? p->t_far : diagonal(g);
}

typedef struct {
  double* t;
  double* delta;
  uint32_t* cell;
  int n, cap;
} schedule;

static void sched_push(schedule* s, double t, double delta, uint32_t cell) {
  if (s->n == s->cap) {
    s->cap = s->cap ? 2 * s->cap : 256;
    s->t = (double*)realloc(s->t, sizeof(double) * s->cap);
    s->delta = (double*)realloc(s->delta, sizeof(double) * s->cap);
    s->cell = (uint32_t*)realloc(s->cell, sizeof(uint32_t) * s->cap);
  }
  s->t[s->n] = t;
  s->delta[s->n] = delta;
  s->cell[s->n] = cell;
  s->n++;
}
static void sched_free(schedule* s) {
  free(s->t);
  free(s->delta);
  free(s->cell);
}

/* renderer.cpp:51-80 */
static int sample_ray_impl(const or_grid* gr, const double o[3], const double d[3],
                           const or_render_params* p, schedule* out) {
  const or_geometry* g = &gr->geom;
  out->n = 0;
  const double step = eff_step(p, g);
  if (!(step > 0.0)) return OR_INVALID_ARGUMENT;
  if (!(p->t_near >= 0.0) || eff_t_far(p, g) <= p->t_near) return OR_INVALID_ARGUMENT;
  double t_enter = 0.0, t_exit = 0.0;
  if (!intersect_bounds(g, o, d, &t_enter, &t_exit)) return OR_OK;
  const double lo = (p->t_near < t_enter) ? t_enter : p->t_near;
  const double tf = eff_t_far(p, g);
  const double hi = (t_exit < tf) ? t_exit : tf;
  if (hi <= lo) return OR_OK;
  const size_t n_segments = (size_t)ceil((hi - lo) / step - 1e-12);
  locator loc;
  for (size_t k = 0; k < n_segments; ++k) {
    const double s0 = lo + (double)k * step;
    const double s0s = s0 + step;
    const double s1 = (hi < s0s) ? hi : s0s;
    const double len = s1 - s0;
    if (len < 1e-12) continue;
    const double tm = 0.5 * (s0 + s1);
    double pt[3];
    for (int a = 0; a < 3; ++a) pt[a] = o[a] + tm * d[a];
    if (!try_locate(g, pt, &loc)) continue;
    const uint32_t ci = cell_index(g, loc.cell[0], loc.cell[1], loc.cell[2]);
    if (!gr->active[ci]) continue;
    sched_push(out, tm, len, ci);
  }
  return OR_OK;
}

int or_sample_ray(const or_grid* g, const double o[3], const double d[3],
                  const or_render_params* p, int cap, double* t, double* delta,
                  uint32_t* cell) {
  schedule s = {0};
  int rc = sample_ray_impl(g, o, d, p, &s);
  if (rc != OR_OK) {
    sched_free(&s);
    return -rc;
  }
  for (int i = 0; i < s.n && i < cap; ++i) {
    if (t) t[i] = s.t[i];
    if (delta) delta[i] = s.delta[i];
    if (cell) cell[i] = s.cell[i];
  }
  int n = s.n;
  sched_free(&s);
  return n;
}

/* renderer.hpp:42-63 */
typedef struct {
  double o[3], d[3], basis[9];
  int count, hit, terminated_early;
  double T_term, color_out[3], depth_out;
  double *t, *delta, *sigma_raw, *sigma, *T, *w, *pos, *color;
  unsigned char* clamped; /* 3 per sample */
  int cap;
} workspace;

static void ws_reserve(workspace* ws, int n) {
  if (n <= ws->cap) return;
  ws->cap = n;
  ws->t = (double*)realloc(ws->t, sizeof(double) * n);
  ws->delta = (double*)realloc(ws->delta, sizeof(double) * n);
  ws->sigma_raw = (double*)realloc(ws->sigma_raw, sizeof(double) * n);
  ws->sigma = (double*)realloc(ws->sigma, sizeof(double) * n);
  ws->T = (double*)realloc(ws->T, sizeof(double) * n);
  ws->w = (double*)realloc(ws->w, sizeof(double) * n);
  ws->pos = (double*)realloc(ws->pos, sizeof(double) * 3 * n);
  ws->color = (double*)realloc(ws->color, sizeof(double) * 3 * n);
  ws->clamped = (unsigned char*)realloc(ws->clamped, 3 * n);
}
static void ws_free(workspace* ws) {
  free(ws->t);
  free(ws->delta);
  free(ws->sigma_raw);
  free(ws->sigma);
  free(ws->T);
  free(ws->w);
  free(ws->pos);
  free(ws->color);
  free(ws->clamped);
}

/* renderer.cpp:82-140 */
static int render_ray_scheduled(const or_grid* g, const double o[3], const double d[3],
                                const schedule* s, const or_render_params* p, workspace* ws) {
  ws->count = 0;
  ws->hit = 0;
  ws->terminated_early = 0;
  ws->T_term = 1.0;
  ws->color_out[0] = ws->color_out[1] = ws->color_out[2] = 0.0;
  ws->depth_out = 0.0;
  for (int a = 0; a < 3; ++a) {
    ws->o[a] = o[a];
    ws->d[a] = d[a];
  }
  if (or_sh_eval(d, ws->basis) != OR_OK) return OR_INVALID_ARGUMENT;
  ws_reserve(ws, s->n > 0 ? s->n : 1);
  double T = 1.0, sh[27], sraw;
  locator loc;
  int n = 0;
  for (int i = 0; i < s->n; ++i) {
    const double ti = s->t[i], di = s->delta[i];
    double pt[3];
    for (int a = 0; a < 3; ++a) pt[a] = o[a] + ti * d[a];
    if (!try_locate(&g->geom, pt, &loc)) return OR_OUT_OF_RANGE;
    trilerp(g, &loc, &sraw, sh);
    const double sigma = (sraw < 0.0) ? 0.0 : sraw;
    const double decay = exp(-sigma * di);
    const double alpha = 1.0 - decay;
    const double w = T * alpha;
    double c[3];
    unsigned char cl[3];
    for (int ch = 0; ch < 3; ++ch) {
      double v = 0.5;
      const double* coeff = sh + ch * SH_N;
      for (int m = 0; m < SH_N; ++m) v += coeff[m] * ws->basis[m];
      cl[ch] = (v <= 0.0 || v >= 1.0);
      c[ch] = (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v);
    }
    ws->t[n] = ti;
    ws->delta[n] = di;
    ws->sigma_raw[n] = sraw;
    ws->sigma[n] = sigma;
    ws->T[n] = T;
    ws->w[n] = w;
    for (int a = 0; a < 3; ++a) {
      ws->pos[3 * n + a] = pt[a];
      ws->color[3 * n + a] = c[a];
      ws->clamped[3 * n + a] = cl[a];
    }
    ++n;
    for (int ch = 0; ch < 3; ++ch) ws->color_out[ch] += w * c[ch];
    ws->depth_out += w * ti;
    T *= decay;
    if (T < p->termination_eps) {
      ws->terminated_early = 1;
      break;
    }
  }
  ws->count = n;
  ws->T_term = T;
  ws->hit = n > 0;
  if (!ws->hit) {
    ws->color_out[0] = ws->color_out[1] = ws->color_out[2] = 0.0;
    ws->depth_out = 0.0;
  }
  return OR_OK;
}

/* renderer.cpp:142-147 */
static int render_ray_ws(const or_grid* g, const double o[3], const double d[3],
                         const or_render_params* p, workspace* ws, schedule* s) {
  int rc = sample_ray_impl(g, o, d, p, s);
  if (rc != OR_OK) return rc;
  return render_ray_scheduled(g, o, d, s, p, ws);
}

int or_render_ray(const or_grid* g, const double o[3], const double d[3],
                  const or_render_params* p, or_ray_result* out) {
  workspace ws = {0};
  schedule s = {0};
  int rc = render_ray_ws(g, o, d, p, &ws, &s);
  if (rc == OR_OK) {
    for (int a = 0; a < 3; ++a) out->color[a] = ws.color_out[a];
    out->depth = ws.depth_out;
    out->transmittance_terminal = ws.T_term;
    out->count = ws.count;
    out->hit = ws.hit;
    out->terminated_early = ws.terminated_early;
  }
  ws_free(&ws);
  sched_free(&s);
  return rc;
}

/* renderer.cpp:149-174 */
int or_render_image(const or_grid* g, const or_intrinsics* intr, const or_pose* pose,
                    const or_render_params* p, int stride, double* color, double* depth) {
  if (stride < 1) return OR_INVALID_ARGUMENT;
  const int out_w = (intr->width + stride - 1) / stride;
  const int out_h = (intr->height + stride - 1) / stride;
  workspace ws = {0};
  schedule s = {0};
  int rc = OR_OK;
  for (size_t idx = 0; idx < (size_t)out_w * out_h; ++idx) {
    const int px = (int)(idx % out_w), py = (int)(idx / out_w);
    double o[3], d[3];
    rc = or_generate_ray(intr, pose, (double)px * stride, (double)py * stride, o, d);
    if (rc != OR_OK) break;
    rc = render_ray_ws(g, o, d, p, &ws, &s);
    if (rc != OR_OK) break;
    for (int ch = 0; ch < 3; ++ch) color[idx * 3 + ch] = ws.color_out[ch];
    depth[idx] = ws.hit ? ws.depth_out : 0.0;
  }
  ws_free(&ws);
  sched_free(&s);
  return rc;
}

/* ---------------------------------------------------------------- gradients.cpp */
/* gradients.cpp:69-85 — accumulates into d_sigma / d_color */
static void grad_color_wrt_params(const workspace* ws, const double up[3], double* d_sigma,
                                  double* d_color) {
  double prefix[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < ws->count; ++i) {
    const double T_next = (i + 1 < ws->count) ? ws->T[i + 1] : ws->T_term;
    const double w = ws->w[i];
    const double* c = ws->color + 3 * i;
    for (int ch = 0; ch < 3; ++ch) prefix[ch] = prefix[ch] + c[ch] * w;
    double ds = 0.0;
    for (int ch = 0; ch < 3; ++ch) {
      d_color[3 * i + ch] += up[ch] * w;
      ds += up[ch] * ws->delta[i] * (c[ch] * T_next - ws->color_out[ch] + prefix[ch]);
    }
    d_sigma[i] += ds;
  }
}
/* gradients.cpp:87-97 */
static void grad_depth_wrt_sigma(const workspace* ws, double up, double* d_sigma) {
  double prefix = 0.0;
  for (int i = 0; i < ws->count; ++i) {
    const double T_next = (i + 1 < ws->count) ? ws->T[i + 1] : ws->T_term;
    prefix += ws->t[i] * ws->w[i];
    d_sigma[i] += up * ws->delta[i] * (ws->t[i] * T_next - ws->depth_out + prefix);
  }
}
/* gradients.cpp:99-114 + 59-67 + 28-41: scatter into a dense V*28 buffer */
static void backprop_to_vertices(const or_grid* g, const workspace* ws, const double* d_sigma,
                                 const double* d_color, double* buf) {
  double up[PAYLOAD];
  locator loc;
  for (int i = 0; i < ws->count; ++i) {
    for (int c = 0; c < PAYLOAD; ++c) up[c] = 0.0;
    up[0] = ws->sigma_raw[i] > 0.0 ? d_sigma[i] : 0.0;
    for (int ch = 0; ch < 3; ++ch) {
      if (ws->clamped[3 * i + ch]) continue;
      const double gg = d_color[3 * i + ch];
      for (int m = 0; m < SH_N; ++m) up[1 + ch * SH_N + m] = gg * ws->basis[m];
    }
    if (!try_locate(&g->geom, ws->pos + 3 * i, &loc)) continue; /* note_out_of_bounds */
    for (int k = 0; k < 8; ++k) {
      double* dst = buf + (size_t)loc.corner[k] * PAYLOAD;
      const double scale = loc.weight[k];
      for (int c = 0; c < PAYLOAD; ++c) dst[c] += scale * up[c];
    }
  }
}

/* gradients.cpp:116-143 (+ voxel_grid.cpp:130-151) */
static void grad_wrt_ray(const or_grid* g, const workspace* ws, const double up_c[3],
                         double up_d, double d_origin[3], double d_direction[3],
                         double* d_sigma, double* d_color) {
  for (int i = 0; i < ws->count; ++i) {
    d_sigma[i] = 0.0;
    d_color[3 * i] = d_color[3 * i + 1] = d_color[3 * i + 2] = 0.0;
  }
  grad_color_wrt_params(ws, up_c, d_sigma, d_color);
  grad_depth_wrt_sigma(ws, up_d, d_sigma);
  for (int a = 0; a < 3; ++a) d_origin[a] = d_direction[a] = 0.0;
  const double inv_h = 1.0 / g->geom.voxel_size;
  const double sgn[2] = {-1.0, 1.0};
  locator loc;
  for (int i = 0; i < ws->count; ++i) {
    if (!try_locate(&g->geom, ws->pos + 3 * i, &loc)) continue;
    const double fx = loc.frac[0], fy = loc.frac[1], fz = loc.frac[2];
    const double wx[2] = {1.0 - fx, fx}, wy[2] = {1.0 - fy, fy}, wz[2] = {1.0 - fz, fz};
    double ds[3] = {0, 0, 0}, dsh[27][3];
    memset(dsh, 0, sizeof(dsh));
    for (int k = 0; k < 8; ++k) {
      const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
      const double dw[3] = {sgn[dx] * wy[dy] * wz[dz] * inv_h, wx[dx] * sgn[dy] * wz[dz] * inv_h,
                            wx[dx] * wy[dy] * sgn[dz] * inv_h};
      const double* v = g->data + (size_t)loc.corner[k] * PAYLOAD;
      for (int a = 0; a < 3; ++a) ds[a] += dw[a] * v[0];
      for (int m = 0; m < 27; ++m)
        for (int a = 0; a < 3; ++a) dsh[m][a] += dw[a] * v[1 + m];
    }
    double gv[3] = {0, 0, 0};
    if (ws->sigma_raw[i] > 0.0)
      for (int a = 0; a < 3; ++a) gv[a] += d_sigma[i] * ds[a];
    for (int ch = 0; ch < 3; ++ch) {
      if (ws->clamped[3 * i + ch]) continue;
      double gc[3] = {0, 0, 0};
      for (int m = 0; m < SH_N; ++m)
        for (int a = 0; a < 3; ++a) gc[a] += ws->basis[m] * dsh[ch * SH_N + m][a];
      for (int a = 0; a < 3; ++a) gv[a] += d_color[3 * i + ch] * gc[a];
    }
    for (int a = 0; a < 3; ++a) d_origin[a] += gv[a];
    for (int a = 0; a < 3; ++a) d_direction[a] += ws->t[i] * gv[a];
  }
}

/* ---------------------------------------------------------------- mapping.cpp:114-233 */
static int depth_valid(const or_frame* f, const or_intrinsics* in, int x, int y) {
  return f->depth[(size_t)y * in->width + x] > 0.0; /* frame.hpp:18 */
}

static int mapping_step_impl(or_grid* g, const or_frame* frames, int n_frames,
                             const or_intrinsics* intr, const or_mapping_config* cfg,
                             const int32_t* batch, int n_rays, double* rms_v, double* grad_out,
                             int apply, or_map_stats* st, int m_color_global,
                             int m_depth_global);

int or_mapping_step(or_grid* g, const or_frame* frames, int n_frames,
                    const or_intrinsics* intr, const or_mapping_config* cfg,
                    const int32_t* batch, int n_rays, double* rms_v, double* grad_out,
                    int apply, or_map_stats* st) {
  return mapping_step_impl(g, frames, n_frames, intr, cfg, batch, n_rays, rms_v, grad_out,
                           apply, st, 0, 0);
}

/* A rank's share of a ray-sharded step: the gradient of this
 * rank's rays with the upstream normalised by the GLOBAL hit counts. */
int or_mapping_grad_global(or_grid* g, const or_frame* frames, int n_frames,
                           const or_intrinsics* intr, const or_mapping_config* cfg,
                           const int32_t* batch, int n_rays, int m_color, int m_depth,
                           double* grad_out, or_map_stats* st) {
  return mapping_step_impl(g, frames, n_frames, intr, cfg, batch, n_rays, NULL, grad_out, 0, st,
                           m_color, m_depth);
}

static int mapping_step_impl(or_grid* g, const or_frame* frames, int n_frames,
                             const or_intrinsics* intr, const or_mapping_config* cfg,
                             const int32_t* batch, int n_rays, double* rms_v, double* grad_out,
                             int apply, or_map_stats* st, int m_color_global,
                             int m_depth_global) {
  memset(st, 0, sizeof(*st));
  st->bad_ray = -1;
  if (n_frames <= 0) return OR_RUNTIME; /* "mapping_step: no keyframes" */
  const size_t V = (size_t)g->geom.res[0] * g->geom.res[1] * g->geom.res[2];
  schedule* sch = (schedule*)calloc((size_t)n_rays, sizeof(schedule));
  unsigned char* hits = (unsigned char*)calloc((size_t)n_rays, 1);
  int rc = OR_OK;
  /* pass 1 */
  for (int i = 0; i < n_rays && rc == OR_OK; ++i) {
    const int32_t* s = batch + 3 * i;
    double o[3], d[3];
    rc = or_generate_ray(intr, &frames[s[0]].pose, s[1], s[2], o, d);
    if (rc == OR_OK) rc = sample_ray_impl(g, o, d, &cfg->render, &sch[i]);
    hits[i] = sch[i].n > 0;
  }
  int m_color = 0, m_depth = 0;
  for (int i = 0; i < n_rays && rc == OR_OK; ++i) {
    if (!hits[i]) continue;
    ++m_color;
    if (depth_valid(&frames[batch[3 * i]], intr, batch[3 * i + 1], batch[3 * i + 2])) ++m_depth;
  }
  st->rays_color = m_color;
  st->rays_depth = m_depth;
  if (m_color_global > 0) { /* ray-sharded step: normalise by the global counts */
    m_color = m_color_global;
    m_depth = m_depth_global;
  }
  if (rc == OR_OK && m_color == 0) rc = OR_RUNTIME; /* "mapping_step: no ray hit the grid" */

  double* buf = NULL;
  double lp = 0.0, lg = 0.0;
  if (rc == OR_OK) {
    buf = (double*)calloc(V * PAYLOAD, sizeof(double));
    workspace ws = {0};
    double *d_sigma = NULL, *d_color = NULL;
    int dcap = 0;
    for (int i = 0; i < n_rays; ++i) {
      if (!hits[i]) continue;
      const int32_t* s = batch + 3 * i;
      const or_frame* f = &frames[s[0]];
      double o[3], d[3];
      or_generate_ray(intr, &f->pose, s[1], s[2], o, d);
      rc = render_ray_scheduled(g, o, d, &sch[i], &cfg->render, &ws);
      if (rc != OR_OK) break;
      st->samples += ws.count;
      const size_t pix = (size_t)s[2] * intr->width + s[1];
      double res[3];
      for (int ch = 0; ch < 3; ++ch) res[ch] = ws.color_out[ch] - f->color[pix * 3 + ch];
      const double sq = dot3(res, res);
      if (!isfinite(sq) || !isfinite(ws.depth_out)) {
        st->bad_ray = i;
        rc = OR_RUNTIME;
        break;
      }
      lp += sq;
      double upc[3];
      for (int ch = 0; ch < 3; ++ch) upc[ch] = 2.0 * res[ch] / (double)m_color;
      double upd = 0.0;
      const int depth_ok = depth_valid(f, intr, s[1], s[2]) && m_depth > 0;
      if (depth_ok) {
        const double dres = ws.depth_out - f->depth[pix];
        lg += dres * dres;
        upd = cfg->lambda_d * 2.0 * dres / (double)m_depth;
      }
      if (ws.count > dcap) {
        dcap = ws.count;
        d_sigma = (double*)realloc(d_sigma, sizeof(double) * dcap);
        d_color = (double*)realloc(d_color, sizeof(double) * 3 * dcap);
      }
      for (int k = 0; k < ws.count; ++k) {
        d_sigma[k] = 0.0;
        d_color[3 * k] = d_color[3 * k + 1] = d_color[3 * k + 2] = 0.0;
      }
      grad_color_wrt_params(&ws, upc, d_sigma, d_color);
      if (depth_ok && upd != 0.0) grad_depth_wrt_sigma(&ws, upd, d_sigma);
      backprop_to_vertices(g, &ws, d_sigma, d_color, buf);
    }
    free(d_sigma);
    free(d_color);
    ws_free(&ws);
  }
  if (rc == OR_OK) {
    st->loss_photometric = lp / (double)m_color;
    st->loss_geometric = m_depth > 0 ? lg / (double)m_depth : 0.0;
    st->loss_total = st->loss_photometric + cfg->lambda_d * st->loss_geometric;
    /* mapping.cpp:107-110 */
    if (st->loss_photometric <= 0.0)
      st->psnr_estimate = 99.0;
    else {
      double ps = 10.0 * log10(3.0 / st->loss_photometric);
      st->psnr_estimate = ps < 99.0 ? ps : 99.0;
    }
    if (grad_out) memcpy(grad_out, buf, V * PAYLOAD * sizeof(double));
    if (apply) {
      /* mapping.cpp:218-231 (sparse over touched == skip exact zeros) */
      const double rho = cfg->rmsprop_decay;
      for (size_t vtx = 0; vtx < V; ++vtx) {
        const double* gg = buf + vtx * PAYLOAD;
        double* theta = g->data + vtx * PAYLOAD;
        double* v = rms_v + vtx * PAYLOAD;
        for (int c = 0; c < PAYLOAD; ++c) {
          if (gg[c] == 0.0) continue;
          v[c] = rho * v[c] + (1.0 - rho) * gg[c] * gg[c];
          const double lr = (c == 0) ? cfg->lr_sigma : cfg->lr_sh;
          theta[c] -= lr * gg[c] / sqrt(v[c] + cfg->rmsprop_eps);
        }
      }
    }
  }
  free(buf);
  for (int i = 0; i < n_rays; ++i) sched_free(&sch[i]);
  free(sch);
  free(hits);
  return rc;
}

/* ---------------------------------------------------------------- tracking.cpp */
typedef struct {
  double tau[3], omega[3], loss;
  double jtj[21], jtr[6];
  int m;
} pose_accum;

static int pose_common(const or_grid* g, const or_frame* frame, const or_intrinsics* intr,
                       const or_pose* pose, const int32_t* px, int n,
                       const or_tracking_loss* cfg, int normal_eqs, pose_accum* acc) {
  memset(acc, 0, sizeof(*acc));
  if (n == 0) return OR_RUNTIME; /* "pose_gradient: empty pixel set" */
  schedule* sch = (schedule*)calloc((size_t)n, sizeof(schedule));
  int rc = OR_OK, m = 0;
  for (int i = 0; i < n && rc == OR_OK; ++i) {
    double o[3], d[3];
    rc = or_generate_ray(intr, pose, px[2 * i], px[2 * i + 1], o, d);
    if (rc == OR_OK) rc = sample_ray_impl(g, o, d, &cfg->render, &sch[i]);
    m += sch[i].n > 0;
  }
  if (rc == OR_OK && m == 0) rc = OR_RUNTIME; /* "untrackable frame: ..." */
  acc->m = m;
  workspace ws = {0};
  double *d_sigma = NULL, *d_color = NULL;
  int dcap = 0;
  for (int i = 0; i < n && rc == OR_OK; ++i) {
    if (sch[i].n == 0) continue;
    double o[3], d[3];
    or_generate_ray(intr, pose, px[2 * i], px[2 * i + 1], o, d);
    rc = render_ray_scheduled(g, o, d, &sch[i], &cfg->render, &ws);
    if (rc != OR_OK) break;
    const size_t pix = (size_t)px[2 * i + 1] * intr->width + px[2 * i];
    double cres[3];
    for (int ch = 0; ch < 3; ++ch) cres[ch] = ws.color_out[ch] - frame->color[pix * 3 + ch];
    const double dres = ws.depth_out - frame->depth[pix];
    acc->loss += (cfg->lambda_p * dot3(cres, cres) + cfg->lambda_d * dres * dres);
    if (ws.count > dcap) {
      dcap = ws.count;
      d_sigma = (double*)realloc(d_sigma, sizeof(double) * dcap);
      d_color = (double*)realloc(d_color, sizeof(double) * 3 * dcap);
    }
    if (!normal_eqs) {
      double upc[3], dor[3], ddir[3];
      for (int ch = 0; ch < 3; ++ch) upc[ch] = cfg->lambda_p * 2.0 * cres[ch] / (double)m;
      const double upd = cfg->lambda_d * 2.0 * dres / (double)m;
      grad_wrt_ray(g, &ws, upc, upd, dor, ddir, d_sigma, d_color);
      for (int a = 0; a < 3; ++a) acc->tau[a] += dor[a];
      const double dd = dot3(d, ddir);
      double gperp[3], cr[3];
      for (int a = 0; a < 3; ++a) gperp[a] = ddir[a] - d[a] * dd;
      cross3(d, gperp, cr);
      for (int a = 0; a < 3; ++a) acc->omega[a] += cr[a];
    } else {
      /* rows: r, g, b colour residuals (weight sqrt(lambda_p)), depth (sqrt(lambda_d)) */
      for (int row = 0; row < 4; ++row) {
        double upc[3] = {0, 0, 0}, upd = 0.0, dor[3], ddir[3];
        if (row < 3)
          upc[row] = 1.0;
        else
          upd = 1.0;
        grad_wrt_ray(g, &ws, upc, upd, dor, ddir, d_sigma, d_color);
        const double dd = dot3(d, ddir);
        double gperp[3], cr[3], J[6];
        for (int a = 0; a < 3; ++a) gperp[a] = ddir[a] - d[a] * dd;
        cross3(d, gperp, cr);
        const double lam = row < 3 ? cfg->lambda_p : cfg->lambda_d;
        const double r = row < 3 ? cres[row] : dres;
        for (int a = 0; a < 3; ++a) {
          J[a] = cr[a];
          J[3 + a] = dor[a];
        }
        int idx = 0;
        for (int a = 0; a < 6; ++a) {
          for (int b = a; b < 6; ++b) acc->jtj[idx++] += lam * J[a] * J[b];
          acc->jtr[a] += lam * J[a] * r;
        }
      }
    }
  }
  free(d_sigma);
  free(d_color);
  ws_free(&ws);
  for (int i = 0; i < n; ++i) sched_free(&sch[i]);
  free(sch);
  return rc;
}

/* tracking.cpp:76-143 */
int or_pose_gradient(const or_grid* g, const or_frame* frame, const or_intrinsics* intr,
                     const or_pose* pose, const int32_t* pixels, int n,
                     const or_tracking_loss* cfg, or_pose_grad* out) {
  pose_accum acc;
  int rc = pose_common(g, frame, intr, pose, pixels, n, cfg, 0, &acc);
  memset(out, 0, sizeof(*out));
  out->rays_used = acc.m;
  if (rc != OR_OK) return rc;
  for (int a = 0; a < 3; ++a) {
    out->d_tau[a] = 0.0 + acc.tau[a];
    out->d_omega[a] = 0.0 + acc.omega[a];
  }
  out->loss = (0.0 + acc.loss) / (double)acc.m;
  for (int a = 0; a < 3; ++a)
    if (!isfinite(out->d_tau[a]) || !isfinite(out->d_omega[a])) return OR_RUNTIME;
  if (!isfinite(out->loss)) return OR_RUNTIME;
  return OR_OK;
}

int or_pose_normal_eqs(const or_grid* g, const or_frame* frame, const or_intrinsics* intr,
                       const or_pose* pose, const int32_t* pixels, int n,
                       const or_tracking_loss* cfg, or_normal_eqs* out) {
  pose_accum acc;
  int rc = pose_common(g, frame, intr, pose, pixels, n, cfg, 1, &acc);
  memset(out, 0, sizeof(*out));
  out->rays_used = acc.m;
  if (rc != OR_OK) return rc;
  memcpy(out->jtj, acc.jtj, sizeof(acc.jtj));
  memcpy(out->jtr, acc.jtr, sizeof(acc.jtr));
  out->loss = acc.loss;
  return OR_OK;
}

/* tracking.cpp:147-166 */
int or_draw_valid_pixels(const double* depth, int w, int h, int count, int max_redraws,
                         uint64_t s[4], int32_t* out) {
  int n = 0;
  for (int i = 0; i < count; ++i) {
    int px = 0, py = 0, ok = 0;
    for (int attempt = 0; attempt < max_redraws; ++attempt) {
      px = (int)or_rng_uniform_index(s, (uint64_t)w);
      py = (int)or_rng_uniform_index(s, (uint64_t)h);
      if (depth[(size_t)py * w + px] > 0.0) {
        ok = 1;
        break;
      }
    }
    if (ok) {
      out[2 * n] = px;
      out[2 * n + 1] = py;
      ++n;
    }
  }
  return n;
}

/* pose.hpp:32-41 */
static void exp_so3(const double w[3], double q[4]) {
  const double angle = norm3(w);
  if (angle < 1e-8) {
    q[0] = 1.0;
    q[1] = 0.5 * w[0];
    q[2] = 0.5 * w[1];
    q[3] = 0.5 * w[2];
    quat_normalize(q);
    return;
  }
  const double axis[3] = {w[0] / angle, w[1] / angle, w[2] / angle};
  const double ha = 0.5 * angle; /* Eigen AngleAxis -> Quaternion */
  const double sh = sin(ha);
  q[0] = cos(ha);
  q[1] = sh * axis[0];
  q[2] = sh * axis[1];
  q[3] = sh * axis[2];
}

/* tracking.hpp:21-26 */
void or_apply_perturbation(const double omega[3], const double tau[3], const or_pose* in,
                           or_pose* out) {
  double e[4], q[4];
  exp_so3(omega, e);
  quat_mul(e, in->q, q);
  quat_normalize(q);
  or_pose r;
  for (int i = 0; i < 4; ++i) r.q[i] = q[i];
  for (int a = 0; a < 3; ++a) r.t[a] = in->t[a] + tau[a];
  *out = r;
}

/* tracking.cpp:170-252 */
int or_track_frame(const or_grid* g, const or_frame* frame, const or_intrinsics* intr,
                   const or_pose* init, const or_tracking_config* cfg, or_track_result* out,
                   double* loss_trace) {
  memset(out, 0, sizeof(*out));
  out->pose = *init;
  if (cfg->iterations == 0) return OR_OK;
  uint64_t rng[4];
  or_rng_seed(cfg->seed, rng);
  or_pose pose = *init, best_pose = *init;
  double best_loss = INFINITY, initial_loss = 0.0;
  int streak = 0;
  double m_adam[6] = {0}, v_adam[6] = {0};
  or_tracking_loss lc = {cfg->lambda_p, cfg->lambda_d, cfg->render};
  int32_t* px = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)cfg->rays_per_iteration);
  int rc = OR_OK;
  for (int it = 0; it < cfg->iterations; ++it) {
    const int n = or_draw_valid_pixels(frame->depth, intr->width, intr->height,
                                       cfg->rays_per_iteration, cfg->max_redraws, rng, px);
    if (n == 0) {
      rc = OR_RUNTIME; /* "track_frame: no valid-depth pixels to sample" */
      break;
    }
    or_pose_grad pg;
    rc = or_pose_gradient(g, frame, intr, &pose, px, n, &lc, &pg);
    if (rc != OR_OK) break;
    if (loss_trace) loss_trace[it] = pg.loss;
    out->final_loss = pg.loss;
    out->iterations_run++;
    if (it == 0) initial_loss = pg.loss;
    if (pg.loss < best_loss) {
      best_loss = pg.loss;
      best_pose = pose;
    }
    if (pg.loss > cfg->divergence_factor * initial_loss) {
      if (++streak >= cfg->divergence_patience) {
        out->pose = *init;
        out->failed = 1;
        free(px);
        return OR_OK;
      }
    } else {
      streak = 0;
    }
    const double grad[6] = {pg.d_omega[0], pg.d_omega[1], pg.d_omega[2],
                            pg.d_tau[0],   pg.d_tau[1],   pg.d_tau[2]};
    for (int k = 0; k < 6; ++k) {
      m_adam[k] = cfg->beta1 * m_adam[k] + (1.0 - cfg->beta1) * grad[k];
      v_adam[k] = cfg->beta2 * v_adam[k] + (1.0 - cfg->beta2) * (grad[k] * grad[k]);
    }
    const double bc1 = 1.0 - pow(cfg->beta1, it + 1);
    const double bc2 = 1.0 - pow(cfg->beta2, it + 1);
    double om[3], ta[3];
    for (int k = 0; k < 6; ++k) {
      const double mhat = m_adam[k] / bc1;
      const double vhat = v_adam[k] / bc2;
      const double lr = k < 3 ? cfg->lr_omega : cfg->lr_tau;
      const double step = -lr * mhat / (sqrt(vhat) + cfg->adam_eps);
      if (k < 3)
        om[k] = step;
      else
        ta[k - 3] = step;
    }
    or_apply_perturbation(om, ta, &pose, &pose);
    if (cfg->convergence_step > 0.0 && norm3(om) < cfg->convergence_step &&
        norm3(ta) < cfg->convergence_step)
      break;
  }
  if (rc == OR_OK) {
    const int n = or_draw_valid_pixels(frame->depth, intr->width, intr->height,
                                       cfg->rays_per_iteration, cfg->max_redraws, rng, px);
    if (n > 0) {
      or_pose_grad pg;
      rc = or_pose_gradient(g, frame, intr, &pose, px, n, &lc, &pg);
      if (rc == OR_OK && pg.loss < best_loss) {
        best_loss = pg.loss;
        best_pose = pose;
      }
    }
    out->pose = best_pose;
  }
  free(px);
  return rc;
}
