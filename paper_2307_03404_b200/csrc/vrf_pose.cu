// Tracking entry points of the C-ABI: pose_gradient (tracking.cpp:76-143), the
// Gauss-Newton normal equations, track_frame with the reference's Adam loop
// (tracking.cpp:170-252) and a Gauss-Newton/LM tracker.
#include <thread>
#include <vector>

#include "vrf_context.h"

using namespace vrf;
using namespace vrf_host;

namespace {

// ---- rng.hpp:13-81 (xoshiro256** seeded through splitmix64): the reference's
// pixel-draw stream, reproduced on the host so track_frame draws the same pixels.
struct Xoshiro {
  uint64_t s[4];
  static uint64_t splitmix(uint64_t& x) {
    x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  explicit Xoshiro(uint64_t seed) {
    uint64_t x = seed;
    for (auto& w : s) w = splitmix(x);
  }
  static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  uint64_t index(uint64_t n) { return (uint64_t)(((unsigned __int128)next() * n) >> 64); }
};

// Jump-ahead of the xoshiro256** state by k steps. The state transition is
// linear over GF(2)^256, so T^k = product of the cached powers T^(2^j) for the
// set bits of k; each power is kept as its 256 column images (the state bit b
// maps to column b), and applying one is 256 conditional 4-word XORs.
struct XoshiroPowers {
  static constexpr int kMax = 34;  // k < 2^34 draws (3 per ray, n < 2^31)
  uint64_t col[kMax][256][4];
  static void step(uint64_t s[4]) {
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = (s[3] << 45) | (s[3] >> 19);
  }
  static void apply(const uint64_t (&m)[256][4], uint64_t s[4]) {
    uint64_t o[4] = {0, 0, 0, 0};
    for (int b = 0; b < 256; ++b)
      if ((s[b >> 6] >> (b & 63)) & 1u)
        for (int w = 0; w < 4; ++w) o[w] ^= m[b][w];
    for (int w = 0; w < 4; ++w) s[w] = o[w];
  }
  XoshiroPowers() {
    for (int b = 0; b < 256; ++b) {
      uint64_t e[4] = {0, 0, 0, 0};
      e[b >> 6] = 1ull << (b & 63);
      step(e);
      for (int w = 0; w < 4; ++w) col[0][b][w] = e[w];
    }
    for (int j = 1; j < kMax; ++j)
      for (int b = 0; b < 256; ++b) {
        uint64_t e[4];
        for (int w = 0; w < 4; ++w) e[w] = col[j - 1][b][w];
        apply(col[j - 1], e);
        for (int w = 0; w < 4; ++w) col[j][b][w] = e[w];
      }
  }
};
void xoshiro_jump(uint64_t s[4], uint64_t k) {
  if (k == 0) return;
  static const XoshiroPowers* P = new XoshiroPowers();  // built once, 272 KB
  for (int j = 0; k; ++j, k >>= 1)
    if (k & 1u) {
      if (j >= XoshiroPowers::kMax) abort();
      XoshiroPowers::apply(P->col[j], s);
    }
}

// tracking.cpp:147-166
void draw_valid_pixels(const std::vector<double>& depth, int w, int h, int count, int max_redraws,
                       Xoshiro& rng, std::vector<int32_t>& out) {
  out.clear();
  for (int i = 0; i < count; ++i) {
    int px = 0, py = 0;
    bool ok = false;
    for (int a = 0; a < max_redraws; ++a) {
      px = (int)rng.index((uint64_t)w);
      py = (int)rng.index((uint64_t)h);
      if (depth[(size_t)py * w + px] > 0.0) {
        ok = true;
        break;
      }
    }
    if (ok) {
      out.push_back(px);
      out.push_back(py);
    }
  }
}

struct PoseResult {
  double jtj[21], jtr[6], loss;
  int m;
  long long samples;
};

int pose_pass(vrf_context* ctx, int frame, const vrf_intrinsics* intr, const vrf_pose* pose,
              const int32_t* pixels, int n, const vrf_tracking_loss* cfg, PoseResult* res,
              PoseKernel which = PoseKernel::kParityFp64) {
  int rc = need_grid(ctx);
  if (rc) return rc;
  if (frame < 0 || frame >= ctx->n_frames)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "pose_gradient: frame index out of range");
  if ((rc = check_frames(ctx, intr))) return rc;
  if (n <= 0) return set_err(ctx, VRF_ERR_RUNTIME, "pose_gradient: empty pixel set");
  for (int i = 0; i < n; ++i)
    if (pixels[2 * i] < 0 || pixels[2 * i] >= intr->width || pixels[2 * i + 1] < 0 ||
        pixels[2 * i + 1] >= intr->height)
      return set_err(ctx, VRF_ERR_OUT_OF_RANGE, "generate_ray: pixel outside image");
  DevParams p;
  if ((rc = resolve_params(ctx, &cfg->render, &p))) return rc;
  const size_t pix_bytes = sizeof(int32_t) * 2 * (size_t)n;
  if ((rc = ensure(ctx, ctx->s_batch, pix_bytes))) return rc;
  const int nb = pose_fused_blocks(n, which);
  if ((rc = ensure(ctx, ctx->s_partials, sizeof(PosePartial) * nb))) return rc;
  if ((rc = ensure_pinned(ctx, pix_bytes + sizeof(DevPose) + sizeof(int)))) return rc;
  if (!ctx->d_frame) CU(cudaMalloc(&ctx->d_frame, sizeof(int)));
  std::memcpy(ctx->h_pinned, pixels, pix_bytes);
  const DevPose dp = dev_pose(pose);
  std::memcpy((char*)ctx->h_pinned + pix_bytes, &dp, sizeof(DevPose));
  std::memcpy((char*)ctx->h_pinned + pix_bytes + sizeof(DevPose), &frame, sizeof(int));
  CU(cudaMemcpyAsync(ctx->s_batch.ptr, ctx->h_pinned, pix_bytes, cudaMemcpyHostToDevice,
                     ctx->stream));
  CU(cudaMemcpyAsync(ctx->d_pose, (char*)ctx->h_pinned + pix_bytes, sizeof(DevPose),
                     cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(ctx->d_frame, (char*)ctx->h_pinned + pix_bytes + sizeof(DevPose),
                     sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
  const long long npix = (long long)intr->width * intr->height;
  const DevGrid g = dev_grid(ctx);
  const DevCam cam = dev_cam(intr);
  // coherent (Morton 4x4-tile) pixel order for the per-ray kernels
  const size_t tmp = ray_order_tmp_bytes(n);
  if ((rc = ensure(ctx, ctx->s_order, sizeof(uint32_t) * n))) return rc;
  if ((rc = ensure(ctx, ctx->s_okeys, sizeof(uint32_t) * n))) return rc;
  if ((rc = ensure(ctx, ctx->s_okeys2, sizeof(uint32_t) * n))) return rc;
  if ((rc = ensure(ctx, ctx->s_oids, sizeof(uint32_t) * n))) return rc;
  if ((rc = ensure(ctx, ctx->s_otmp, tmp))) return rc;
  const uint32_t* order = (const uint32_t*)ctx->s_order.ptr;
  launch_pixel_order((const int*)ctx->s_batch.ptr, n, (uint32_t*)ctx->s_okeys.ptr,
                     (uint32_t*)ctx->s_oids.ptr, (uint32_t*)ctx->s_okeys2.ptr,
                     (uint32_t*)ctx->s_order.ptr, ctx->s_otmp.ptr, tmp, ctx->stream);
  // K5: forward + Jacobian in one pass per ray (FP64 SH on the reference-parity path)
  cudaEvent_t pb = prof_begin(ctx);
  launch_pose_fused(which, g, p, cam, ctx->rgbd, ctx->d_frame, npix, ctx->d_pose,
                    (const int*)ctx->s_batch.ptr, order, n, cfg->lambda_p, cfg->lambda_d,
                    (PosePartial*)ctx->s_partials.ptr, ctx->d_err, ctx->stream);
  prof_end(ctx, kProfPoseBackward, pb);
  launch_pose_reduce2((const PosePartial*)ctx->s_partials.ptr, nb, ctx->d_pose_out, ctx->stream);
  LAUNCHED(4);
  CU(cudaGetLastError());
  // error flag and result in one round trip (one host sync per pose pass)
  PosePartial out;
  int flag = 0;
  CU(cudaMemcpyAsync(&flag, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(&out, ctx->d_pose_out, sizeof(out), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if ((rc = err_from_flag(ctx, flag))) return rc;
  prof_collect(ctx);
  std::memcpy(res->jtj, out.jtj, sizeof(res->jtj));
  std::memcpy(res->jtr, out.jtr, sizeof(res->jtr));
  res->loss = out.loss;
  res->m = out.m;
  res->samples = out.samples;
  return VRF_OK;
}

int gradient_from(vrf_context* ctx, const PoseResult& r, vrf_pose_gradient_result* out) {
  vrf_pose_gradient_result g{};
  g.rays_used = r.m;
  g.samples = r.samples;
  if (r.m == 0) {
    if (out) *out = g;
    return set_err(ctx, VRF_ERR_RUNTIME, "untrackable frame: all sampled rays miss the grid");
  }
  // pose_gradient == (2/m) J^T r with rows weighted by sqrt(lambda) (tracking.cpp:117-128).
  for (int a = 0; a < 3; ++a) {
    g.d_omega[a] = 2.0 * r.jtr[a] / double(r.m);
    g.d_tau[a] = 2.0 * r.jtr[3 + a] / double(r.m);
  }
  g.loss = r.loss / double(r.m);
  if (out) *out = g;
  bool finite = std::isfinite(g.loss);
  for (int a = 0; a < 3; ++a)
    finite = finite && std::isfinite(g.d_omega[a]) && std::isfinite(g.d_tau[a]);
  if (!finite) return set_err(ctx, VRF_ERR_RUNTIME, "pose_gradient: non-finite result");
  return VRF_OK;
}

// ---- pose.hpp:32-41, tracking.hpp:21-26 (same operation order as the oracle)
void quat_normalize(double q[4]) {
  const double x = q[1], y = q[2], z = q[3], w = q[0];
  const double n2 = (x * x + z * z) + (y * y + w * w);
  if (n2 > 0.0) {
    const double s = std::sqrt(n2);
    q[0] = w / s;
    q[1] = x / s;
    q[2] = y / s;
    q[3] = z / s;
  }
}
void exp_so3(const double w[3], double q[4]) {
  const double angle = std::sqrt((w[0] * w[0] + w[1] * w[1]) + w[2] * w[2]);
  if (angle < 1e-8) {
    q[0] = 1.0;
    q[1] = 0.5 * w[0];
    q[2] = 0.5 * w[1];
    q[3] = 0.5 * w[2];
    quat_normalize(q);
    return;
  }
  const double axis[3] = {w[0] / angle, w[1] / angle, w[2] / angle};
  const double ha = 0.5 * angle, sh = std::sin(ha);
  q[0] = std::cos(ha);
  q[1] = sh * axis[0];
  q[2] = sh * axis[1];
  q[3] = sh * axis[2];
}
void apply_perturbation(const double om[3], const double ta[3], vrf_pose* pose) {
  double e[4];
  exp_so3(om, e);
  const double* b = pose->q;
  double q[4] = {e[0] * b[0] - e[1] * b[1] - e[2] * b[2] - e[3] * b[3],
                 e[0] * b[1] + e[1] * b[0] + e[2] * b[3] - e[3] * b[2],
                 e[0] * b[2] + e[2] * b[0] + e[3] * b[1] - e[1] * b[3],
                 e[0] * b[3] + e[3] * b[0] + e[1] * b[2] - e[2] * b[1]};
  quat_normalize(q);
  for (int i = 0; i < 4; ++i) pose->q[i] = q[i];
  for (int a = 0; a < 3; ++a) pose->t[a] = pose->t[a] + ta[a];
}

}  // namespace

extern "C" {

void vrf_rng_seed(uint64_t seed, uint64_t state[4]) {
  Xoshiro r(seed);
  for (int i = 0; i < 4; ++i) state[i] = r.s[i];
}
uint64_t vrf_rng_next(uint64_t state[4]) {
  Xoshiro r(0);
  for (int i = 0; i < 4; ++i) r.s[i] = state[i];
  const uint64_t v = r.next();
  for (int i = 0; i < 4; ++i) state[i] = r.s[i];
  return v;
}
void vrf_rng_draw_batch(uint64_t state[4], int n_frames, int width, int height, int n,
                        int32_t* batch) {
  // mapping.cpp:121-128: three draws per ray, one raw output each (index(n) =
  // (next * n) >> 64), so ray i starts at stream position 3 i and chunks of a
  // large batch can be drawn in parallel from jumped-ahead states (bit-identical
  // to the sequential stream; the final state is the one after 3 n draws).
  auto draw = [=](Xoshiro r, int i0, int i1) {
    for (int i = i0; i < i1; ++i) {
      batch[3 * i] = (int32_t)r.index((uint64_t)n_frames);
      batch[3 * i + 1] = (int32_t)r.index((uint64_t)width);
      batch[3 * i + 2] = (int32_t)r.index((uint64_t)height);
    }
  };
  Xoshiro r(0);
  for (int i = 0; i < 4; ++i) r.s[i] = state[i];
  const int hw = (int)std::min(16u, std::max(1u, std::thread::hardware_concurrency()));
  const int parts = n >= (1 << 16) ? std::min(hw, n >> 15) : 1;
  if (parts <= 1) {
    for (int i = 0; i < n; ++i) {
      batch[3 * i] = (int32_t)r.index((uint64_t)n_frames);
      batch[3 * i + 1] = (int32_t)r.index((uint64_t)width);
      batch[3 * i + 2] = (int32_t)r.index((uint64_t)height);
    }
    for (int i = 0; i < 4; ++i) state[i] = r.s[i];
    return;
  } else {
    std::vector<std::thread> pool;
    for (int c = 1; c < parts; ++c) {
      const int i0 = (int)((long long)n * c / parts), i1 = (int)((long long)n * (c + 1) / parts);
      Xoshiro rc = r;
      xoshiro_jump(rc.s, 3ull * (uint64_t)i0);
      pool.emplace_back(draw, rc, i0, i1);
    }
    draw(r, 0, (int)((long long)n / parts));
    for (auto& t : pool) t.join();
  }
  xoshiro_jump(r.s, 3ull * (uint64_t)n);
  for (int i = 0; i < 4; ++i) state[i] = r.s[i];
}
int vrf_rng_draw_valid_pixels(uint64_t state[4], const double* depth, int width, int height,
                              int count, int max_redraws, int32_t* pixels) {
  Xoshiro r(0);
  for (int i = 0; i < 4; ++i) r.s[i] = state[i];
  int n = 0;
  for (int i = 0; i < count; ++i) {
    int px = 0, py = 0;
    bool ok = false;
    for (int a = 0; a < max_redraws; ++a) {
      px = (int)r.index((uint64_t)width);
      py = (int)r.index((uint64_t)height);
      if (depth[(size_t)py * width + px] > 0.0) {
        ok = true;
        break;
      }
    }
    if (ok) {
      pixels[2 * n] = px;
      pixels[2 * n + 1] = py;
      ++n;
    }
  }
  for (int i = 0; i < 4; ++i) state[i] = r.s[i];
  return n;
}

int vrf_pose_gradient(vrf_context* ctx, int frame, const vrf_intrinsics* intr,
                      const vrf_pose* pose, const int32_t* pixels, int n,
                      const vrf_tracking_loss* cfg, vrf_pose_gradient_result* out) {
  cudaSetDevice(ctx->device);
  PoseResult r;
  int rc = pose_pass(ctx, frame, intr, pose, pixels, n, cfg, &r);
  if (rc) return rc;
  return gradient_from(ctx, r, out);
}

int vrf_pose_normal_equations(vrf_context* ctx, int frame, const vrf_intrinsics* intr,
                              const vrf_pose* pose, const int32_t* pixels, int n,
                              const vrf_tracking_loss* cfg, vrf_normal_equations* out) {
  return vrf_pose_normal_equations_ex(ctx, frame, intr, pose, pixels, n, cfg,
                                      VRF_POSE_KERNEL_PARITY, out);
}

int vrf_pose_normal_equations_ex(vrf_context* ctx, int frame, const vrf_intrinsics* intr,
                                 const vrf_pose* pose, const int32_t* pixels, int n,
                                 const vrf_tracking_loss* cfg, int kernel,
                                 vrf_normal_equations* out) {
  cudaSetDevice(ctx->device);
  PoseKernel which;
  switch (kernel) {
    case VRF_POSE_KERNEL_PARITY: which = PoseKernel::kParityFp64; break;
    case VRF_POSE_KERNEL_GN: which = PoseKernel::kGnUniform; break;
    case VRF_POSE_KERNEL_GN_CHECK: which = PoseKernel::kGroupFp32; break;
    default: return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "pose_normal_equations: unknown kernel");
  }
  PoseResult r;
  int rc = pose_pass(ctx, frame, intr, pose, pixels, n, cfg, &r, which);
  if (rc) return rc;
  std::memcpy(out->jtj, r.jtj, sizeof(r.jtj));
  std::memcpy(out->jtr, r.jtr, sizeof(r.jtr));
  out->loss = r.loss;
  out->rays_used = r.m;
  out->reserved = 0;
  out->samples = r.samples;
  if (r.m == 0)
    return set_err(ctx, VRF_ERR_RUNTIME, "untrackable frame: all sampled rays miss the grid");
  return VRF_OK;
}

// tracking.cpp:170-252
int vrf_track_frame(vrf_context* ctx, int frame, const vrf_intrinsics* intr, const vrf_pose* init,
                    const vrf_tracking_config* cfg, vrf_track_frame_result* out,
                    double* loss_trace) {
  cudaSetDevice(ctx->device);
  vrf_track_frame_result res{};
  res.pose = *init;
  *out = res;
  if (cfg->iterations == 0) return VRF_OK;
  if (frame < 0 || frame >= ctx->n_frames)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "track_frame: frame index out of range");
  std::vector<double>& depth = ctx->host_depth[frame];
  if (depth.empty()) {  // frame written in sensor format: fetch its depth channel once
    const long long npix = (long long)ctx->fintr.width * ctx->fintr.height;
    int rc2 = ensure(ctx, ctx->s_out, sizeof(double) * (size_t)npix);
    if (rc2) return rc2;
    launch_extract_depth(ctx->rgbd + npix * frame, (double*)ctx->s_out.ptr, npix, ctx->stream);
    LAUNCHED(1);
    depth.resize((size_t)npix);
    CU(cudaMemcpyAsync(depth.data(), ctx->s_out.ptr, sizeof(double) * (size_t)npix,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  Xoshiro rng(cfg->seed);
  vrf_pose pose = *init, best_pose = *init;
  double best_loss = INFINITY, initial_loss = 0.0;
  int streak = 0;
  double m_adam[6] = {0}, v_adam[6] = {0};
  const vrf_tracking_loss lc{cfg->lambda_p, cfg->lambda_d, cfg->render};
  std::vector<int32_t> px;
  int rc;
  for (int it = 0; it < cfg->iterations; ++it) {
    draw_valid_pixels(depth, intr->width, intr->height, cfg->rays_per_iteration, cfg->max_redraws,
                      rng, px);
    if (px.empty())
      return set_err(ctx, VRF_ERR_RUNTIME, "track_frame: no valid-depth pixels to sample");
    PoseResult r;
    vrf_pose_gradient_result g;
    if ((rc = pose_pass(ctx, frame, intr, &pose, px.data(), (int)px.size() / 2, &lc, &r))) return rc;
    if ((rc = gradient_from(ctx, r, &g))) return rc;
    if (loss_trace) loss_trace[it] = g.loss;
    res.final_loss = g.loss;
    ++res.iterations_run;
    if (it == 0) initial_loss = g.loss;
    if (g.loss < best_loss) {
      best_loss = g.loss;
      best_pose = pose;
    }
    if (g.loss > cfg->divergence_factor * initial_loss) {
      if (++streak >= cfg->divergence_patience) {
        res.pose = *init;
        res.failed = 1;
        *out = res;
        return VRF_OK;
      }
    } else {
      streak = 0;
    }
    const double grad[6] = {g.d_omega[0], g.d_omega[1], g.d_omega[2],
                            g.d_tau[0],   g.d_tau[1],   g.d_tau[2]};
    for (int k = 0; k < 6; ++k) {
      m_adam[k] = cfg->beta1 * m_adam[k] + (1.0 - cfg->beta1) * grad[k];
      v_adam[k] = cfg->beta2 * v_adam[k] + (1.0 - cfg->beta2) * (grad[k] * grad[k]);
    }
    const double bc1 = 1.0 - std::pow(cfg->beta1, it + 1);
    const double bc2 = 1.0 - std::pow(cfg->beta2, it + 1);
    double om[3], ta[3];
    for (int k = 0; k < 6; ++k) {
      const double mhat = m_adam[k] / bc1, vhat = v_adam[k] / bc2;
      const double lr = k < 3 ? cfg->lr_omega : cfg->lr_tau;
      const double step = -lr * mhat / (std::sqrt(vhat) + cfg->adam_eps);
      if (k < 3)
        om[k] = step;
      else
        ta[k - 3] = step;
    }
    apply_perturbation(om, ta, &pose);
    const double nom = std::sqrt((om[0] * om[0] + om[1] * om[1]) + om[2] * om[2]);
    const double nta = std::sqrt((ta[0] * ta[0] + ta[1] * ta[1]) + ta[2] * ta[2]);
    if (cfg->convergence_step > 0.0 && nom < cfg->convergence_step && nta < cfg->convergence_step)
      break;
  }
  // Evaluate the final iterate (tracking.cpp:239-249).
  draw_valid_pixels(depth, intr->width, intr->height, cfg->rays_per_iteration, cfg->max_redraws,
                    rng, px);
  if (!px.empty()) {
    PoseResult r;
    vrf_pose_gradient_result g;
    if ((rc = pose_pass(ctx, frame, intr, &pose, px.data(), (int)px.size() / 2, &lc, &r))) return rc;
    if ((rc = gradient_from(ctx, r, &g))) return rc;
    if (g.loss < best_loss) {
      best_loss = g.loss;
      best_pose = pose;
    }
  }
  res.pose = best_pose;
  *out = res;
  return VRF_OK;
}

// Gauss-Newton / LM: per iteration one normal-equation pass and a damped 6x6
// solve; pixel draws from the same valid-depth sampler (seeded stream).
int vrf_track_frame_gn(vrf_context* ctx, int frame, const vrf_intrinsics* intr,
                       const vrf_pose* init, const vrf_gn_config* cfg,
                       vrf_track_frame_result* out) {
  cudaSetDevice(ctx->device);
  vrf_track_frame_result res{};
  res.pose = *init;
  *out = res;
  if (cfg->iterations <= 0) return VRF_OK;
  if (frame < 0 || frame >= ctx->n_frames)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "track_frame: frame index out of range");
  int rc = need_grid(ctx);
  if (rc) return rc;
  if ((rc = check_frames(ctx, intr))) return rc;
  DevParams p;
  if ((rc = resolve_params(ctx, &cfg->render, &p))) return rc;
  // n = rays_per_iteration stratified draws over a 2^L x 2^L tile grid, 4^L <= n
  const int n = cfg->rays_per_iteration;
  if (n <= 0)
    return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "track_frame_gn: rays_per_iteration must be > 0");
  int L = 0;
  while ((4LL << (2 * L)) <= (long long)n) ++L;
  PoseKernel which;
  switch (cfg->kernel) {
    case VRF_POSE_KERNEL_GN: which = PoseKernel::kGnUniform; break;
    case VRF_POSE_KERNEL_GN_CHECK: which = PoseKernel::kGroupFp32; break;
    default: return set_err(ctx, VRF_ERR_INVALID_ARGUMENT, "track_frame_gn: unknown kernel");
  }
  const int iters = cfg->iterations;
  const int nb = pose_fused_blocks(n, which);
  if ((rc = ensure(ctx, ctx->s_batch, sizeof(int32_t) * 2 * (size_t)n))) return rc;
  if ((rc = ensure(ctx, ctx->s_partials, sizeof(PosePartial) * nb))) return rc;
  if (!ctx->d_frame) CU(cudaMalloc(&ctx->d_frame, sizeof(int)));
  if (!ctx->d_gn_pose) CU(cudaMalloc(&ctx->d_gn_pose, sizeof(DevPose)));
  if (!ctx->d_gn_seed) CU(cudaMalloc(&ctx->d_gn_seed, sizeof(unsigned long long)));
  if (ctx->gn_hist_cap < iters) {
    CU(cudaStreamSynchronize(ctx->stream));
    cudaFree(ctx->d_gn_hist);
    CU(cudaMalloc(&ctx->d_gn_hist, sizeof(double) * 3 * iters));
    ctx->gn_hist_cap = iters;
    if (ctx->gn_graph) cudaGraphExecDestroy(ctx->gn_graph);
    ctx->gn_graph = nullptr;
  }
  const DevGrid g = dev_grid(ctx);
  const DevCam cam = dev_cam(intr);
  const long long npix = (long long)intr->width * intr->height;
  // graph key: everything baked into the captured kernel parameters
  std::vector<unsigned char> key;
  auto put = [&key](const void* v, size_t b) {
    key.insert(key.end(), (const unsigned char*)v, (const unsigned char*)v + b);
  };
  put(&g, sizeof(g));
  put(&p, sizeof(p));
  put(&cam, sizeof(cam));
  put(&n, sizeof(n));
  put(&which, sizeof(which));
  put(&iters, sizeof(iters));
  put(&cfg->lambda_p, sizeof(double));
  put(&cfg->lambda_d, sizeof(double));
  put(&cfg->damping, sizeof(double));
  put(&cfg->max_redraws, sizeof(int));
  put(&ctx->rgbd, sizeof(void*));
  put(&ctx->s_batch.ptr, sizeof(void*));
  put(&ctx->s_partials.ptr, sizeof(void*));
  put(&ctx->stream, sizeof(void*));
  put(&ctx->grid_generation, sizeof(long long));
  if (!ctx->gn_graph || key != ctx->gn_key) {
    if (ctx->gn_graph) cudaGraphExecDestroy(ctx->gn_graph);
    ctx->gn_graph = nullptr;
    cudaGraph_t graph;
    // capture on the context's own (non-blocking) stream: the legacy default
    // stream a caller may have selected with vrf_set_stream cannot be captured;
    // the graph is then launched on whichever stream the context runs on
    cudaStream_t cs = ctx->own_stream;
    CU(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    for (int it = 0; it < iters; ++it) {
      launch_draw_strat(ctx->rgbd, ctx->d_frame, npix, intr->width, intr->height, L,
                        cfg->max_redraws, ctx->d_gn_seed, it, (int*)ctx->s_batch.ptr, n, cs);
      launch_pose_fused(which, g, p, cam, ctx->rgbd, ctx->d_frame, npix,
                        ctx->d_gn_pose, (const int*)ctx->s_batch.ptr, nullptr, n, cfg->lambda_p,
                        cfg->lambda_d, (PosePartial*)ctx->s_partials.ptr, ctx->d_err, cs);
      launch_pose_reduce2((const PosePartial*)ctx->s_partials.ptr, nb, ctx->d_pose_out, cs);
      launch_gn_step(ctx->d_pose_out, ctx->d_gn_pose, cfg->damping, ctx->d_gn_hist, it, cs);
    }
    CU(cudaStreamEndCapture(cs, &graph));
    CU(cudaGraphInstantiate(&ctx->gn_graph, graph, 0));
    cudaGraphDestroy(graph);
    ctx->gn_key = key;
  }
  // per-frame inputs: init pose, frame index, seed
  if ((rc = ensure_pinned(ctx, sizeof(DevPose) + 16 + sizeof(double) * 3 * iters))) return rc;
  char* h = (char*)ctx->h_pinned;
  const DevPose dp = dev_pose(init);
  const unsigned long long seed = cfg->seed ^ (0x9e3779b97f4a7c15ULL * (unsigned long long)(frame + 1));
  std::memcpy(h, &dp, sizeof(DevPose));
  std::memcpy(h + sizeof(DevPose), &frame, sizeof(int));
  std::memcpy(h + sizeof(DevPose) + 8, &seed, sizeof(seed));
  CU(cudaMemcpyAsync(ctx->d_gn_pose, h, sizeof(DevPose), cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(ctx->d_frame, h + sizeof(DevPose), sizeof(int), cudaMemcpyHostToDevice,
                     ctx->stream));
  CU(cudaMemcpyAsync(ctx->d_gn_seed, h + sizeof(DevPose) + 8, sizeof(seed),
                     cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
  cudaEvent_t pb = prof_begin(ctx);
  CU(cudaGraphLaunch(ctx->gn_graph, ctx->stream));
  prof_end(ctx, kProfPoseBackward, pb);
  LAUNCHED(4LL * iters);
  DevPose fin;
  double* hist = (double*)(h + sizeof(DevPose) + 16);
  CU(cudaMemcpyAsync(&fin, ctx->d_gn_pose, sizeof(DevPose), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(hist, ctx->d_gn_hist, sizeof(double) * 3 * iters, cudaMemcpyDeviceToHost,
                     ctx->stream));
  if ((rc = check_err_flag(ctx))) return rc;  // syncs the stream
  prof_collect(ctx);
  ctx->gn_last_hist.assign(hist, hist + 3 * iters);
  if (hist[1] == 0.0)
    return set_err(ctx, VRF_ERR_RUNTIME, "untrackable frame: all sampled rays miss the grid");
  for (int a = 0; a < 4; ++a) res.pose.q[a] = fin.q[a];
  for (int a = 0; a < 3; ++a) res.pose.t[a] = fin.t[a];
  res.iterations_run = iters;
  res.final_loss = hist[3 * (iters - 1)];
  if (ctx->profiling)  // composited samples of the frame's iterations (bench roofline)
    for (int it = 0; it < iters; ++it) ctx->prof_track_samples += (long long)hist[3 * it + 2];
  *out = res;
  return VRF_OK;
}

int vrf_track_frame_gn_history(vrf_context* ctx, double* hist, int cap) {
  const int n = (int)ctx->gn_last_hist.size();
  if (hist && cap > 0) std::memcpy(hist, ctx->gn_last_hist.data(), sizeof(double) * std::min(n, cap));
  return n / 3;
}

}  // extern "C"
