// C wrapper over the reference's OWN C++ functions — TEST INFRASTRUCTURE ONLY.
//
// Compiled by oracle/Makefile together with the reference translation units
// (/root/reference/proj/src/{voxel_grid,renderer,gradients,mapping,tracking}.cpp,
// unchanged) into oracle/_ref/libvoxrf_ref.so. Used (a) by the parity tests to
// pin oracle/voxrf_oracle.c against the reference itself and to generate the
// golden fixtures, and (b) by bench.py as the CPU baseline / `--impl reference`
// arm ("kind": "reference"). Never linked into the product library.
#include <chrono>
#include <optional>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "voxrf/eval.hpp"
#include "voxrf/gradients.hpp"
#include "voxrf/mapping.hpp"
#include "voxrf/renderer.hpp"
#include "voxrf/tracking.hpp"
#include "voxrf/trajectory.hpp"

#include "voxrf_oracle.h"  // POD structs shared with the restatement

using namespace voxrf;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define REF_GUARD(...)                                  \
  try {                                                 \
    __VA_ARGS__;                                             \
  } catch (const std::invalid_argument& e) {           \
    return fail(e, OR_INVALID_ARGUMENT);                \
  } catch (const std::out_of_range& e) {               \
    return fail(e, OR_OUT_OF_RANGE);                    \
  } catch (const std::exception& e) {                  \
    return fail(e, OR_RUNTIME);                         \
  }                                                     \
  return OR_OK

GridGeometry to_geom(const or_geometry& g) {
  GridGeometry out;
  out.res = Eigen::Vector3i(g.res[0], g.res[1], g.res[2]);
  out.origin = Eigen::Vector3d(g.origin[0], g.origin[1], g.origin[2]);
  out.voxel_size = g.voxel_size;
  return out;
}
CameraIntrinsics to_intr(const or_intrinsics& i) {
  CameraIntrinsics c;
  c.fx = i.fx;
  c.fy = i.fy;
  c.cx = i.cx;
  c.cy = i.cy;
  c.width = i.width;
  c.height = i.height;
  c.depth_scale = i.depth_scale;
  return c;
}
Pose to_pose(const or_pose& p) {
  Pose out;
  out.q = Eigen::Quaterniond(p.q[0], p.q[1], p.q[2], p.q[3]);
  out.t = Eigen::Vector3d(p.t[0], p.t[1], p.t[2]);
  return out;
}
or_pose from_pose(const Pose& p) {
  or_pose o;
  o.q[0] = p.q.w();
  o.q[1] = p.q.x();
  o.q[2] = p.q.y();
  o.q[3] = p.q.z();
  for (int a = 0; a < 3; ++a) o.t[a] = p.t[a];
  return o;
}
RenderParams to_params(const or_render_params& p) {
  RenderParams r;
  r.step = p.step;
  r.t_near = p.t_near;
  r.t_far = p.t_far;
  r.termination_eps = p.termination_eps;
  return r;
}
Frame to_frame(const or_frame& f, int w, int h) {
  Frame out;
  out.color = ImageF(w, h, 3);
  out.depth = ImageF(w, h, 1);
  std::memcpy(out.color.data.data(), f.color, sizeof(double) * size_t(w) * h * 3);
  std::memcpy(out.depth.data.data(), f.depth, sizeof(double) * size_t(w) * h);
  out.gt_pose = to_pose(f.pose);
  return out;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- grid handle
void* ref_grid_create(const or_geometry* g, const double* data, const uint8_t* active) {
  try {
    auto* grid = new VoxelGrid(to_geom(*g));
    if (data) std::memcpy(grid->data().data(), data, sizeof(double) * grid->data().size());
    if (active) {
      const GridGeometry& gg = grid->geometry();
      for (int cz = 0; cz < gg.res.z() - 1; ++cz)
        for (int cy = 0; cy < gg.res.y() - 1; ++cy)
          for (int cx = 0; cx < gg.res.x() - 1; ++cx)
            grid->set_cell_active(cx, cy, cz, active[gg.cell_index(cx, cy, cz)] != 0);
    }
    return grid;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_grid_destroy(void* grid) { delete static_cast<VoxelGrid*>(grid); }
void ref_grid_read(const void* grid, double* data) {
  const auto* g = static_cast<const VoxelGrid*>(grid);
  std::memcpy(data, g->data().data(), sizeof(double) * g->data().size());
}
int ref_grid_prune(void* grid, double tau) { return int(static_cast<VoxelGrid*>(grid)->prune(tau)); }
void ref_grid_occupancy(const void* grid, uint8_t* active) {
  const auto& occ = static_cast<const VoxelGrid*>(grid)->occupancy();
  std::memcpy(active, occ.data(), occ.size());
}
void* ref_grid_upsampled(const void* grid, int max_resolution) {
  try {
    return new VoxelGrid(static_cast<const VoxelGrid*>(grid)->upsampled(max_resolution));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
int ref_grid_save(const void* grid, const char* path) {
  REF_GUARD(static_cast<const VoxelGrid*>(grid)->save(path));
}
void* ref_grid_load(const char* path) {
  try {
    return new VoxelGrid(VoxelGrid::load(path));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
uint64_t ref_grid_checksum(const void* grid) {
  return static_cast<const VoxelGrid*>(grid)->checksum();
}

// ---- frames handle (a keyframe list for mapping_step / a tracking frame)
struct RefFrames {
  std::vector<Frame> frames;
  std::vector<const Frame*> ptrs;
};
void* ref_frames_create(const or_frame* frames, int n, int width, int height) {
  auto* fs = new RefFrames;
  fs->frames.reserve(n);
  for (int i = 0; i < n; ++i) fs->frames.push_back(to_frame(frames[i], width, height));
  for (const Frame& f : fs->frames) fs->ptrs.push_back(&f);
  return fs;
}
void ref_frames_destroy(void* fs) { delete static_cast<RefFrames*>(fs); }

// fit_grid_geometry (mapping.cpp:235-276) over every frame of the handle.
int ref_fit_grid_geometry(const void* frames, const or_intrinsics* intr, int initial_resolution,
                          double bounds_margin, or_geometry* out) {
  REF_GUARD({
    const auto* fs = static_cast<const RefFrames*>(frames);
    Dataset ds;
    ds.intrinsics = to_intr(*intr);
    MappingConfig cfg;
    cfg.initial_resolution = initial_resolution;
    cfg.bounds_margin = bounds_margin;
    const GridGeometry g = fit_grid_geometry(ds, fs->ptrs, cfg);
    for (int a = 0; a < 3; ++a) {
      out->res[a] = g.res[a];
      out->origin[a] = g.origin[a];
    }
    out->voxel_size = g.voxel_size;
  });
}

// ---- renderer.cpp
int ref_sample_ray(const void* grid, const double o[3], const double d[3],
                   const or_render_params* p, int cap, double* t, double* delta, int* count) {
  REF_GUARD({
    SampleSchedule s;
    sample_ray(*static_cast<const VoxelGrid*>(grid),
               Ray{Eigen::Vector3d(o[0], o[1], o[2]), Eigen::Vector3d(d[0], d[1], d[2])},
               to_params(*p), s);
    *count = int(s.size());
    for (int i = 0; i < int(s.size()) && i < cap; ++i) {
      t[i] = s.t[i];
      delta[i] = s.delta[i];
    }
  });
}
int ref_render_ray(const void* grid, const double o[3], const double d[3],
                   const or_render_params* p, or_ray_result* out) {
  REF_GUARD({
    RayWorkspace ws;
    render_ray(*static_cast<const VoxelGrid*>(grid),
               Ray{Eigen::Vector3d(o[0], o[1], o[2]), Eigen::Vector3d(d[0], d[1], d[2])},
               to_params(*p), ws);
    for (int a = 0; a < 3; ++a) out->color[a] = ws.color_out[a];
    out->depth = ws.depth_out;
    out->transmittance_terminal = ws.transmittance_terminal;
    out->count = ws.count;
    out->hit = ws.hit;
    out->terminated_early = ws.terminated_early;
  });
}
int ref_generate_ray(const or_intrinsics* intr, const or_pose* pose, double u, double v,
                     double o[3], double d[3]) {
  REF_GUARD({
    const Ray r = generate_ray(to_intr(*intr), to_pose(*pose), u, v);
    for (int a = 0; a < 3; ++a) {
      o[a] = r.o[a];
      d[a] = r.d[a];
    }
  });
}
int ref_render_image(const void* grid, const or_intrinsics* intr, const or_pose* pose,
                     const or_render_params* p, int stride, int threads, double* color,
                     double* depth) {
  REF_GUARD({
    const Frame f = render_image(*static_cast<const VoxelGrid*>(grid), to_intr(*intr),
                                 to_pose(*pose), to_params(*p), stride, threads);
    std::memcpy(color, f.color.data.data(), sizeof(double) * f.color.data.size());
    std::memcpy(depth, f.depth.data.data(), sizeof(double) * f.depth.data.size());
  });
}

// ---- mapping.cpp:114-233 (the reference's own function, batch drawn from Rng(seed))
struct RefMapper {
  RmspropState rms;
  Rng rng{1};
};
void* ref_mapper_create(uint64_t seed) {
  auto* m = new RefMapper;
  m->rng = Rng(seed);
  return m;
}
void ref_mapper_destroy(void* m) { delete static_cast<RefMapper*>(m); }
int ref_mapper_rms(const void* m, double* v, size_t n) {
  const auto* mm = static_cast<const RefMapper*>(m);
  if (mm->rms.v.size() != n) return -1;
  std::memcpy(v, mm->rms.v.data(), sizeof(double) * n);
  return 0;
}
int ref_mapping_step(void* grid, const void* frames, const or_intrinsics* intr,
                     const or_mapping_config* cfg, int rays_per_batch, int threads,
                     int deterministic, void* mapper, or_map_stats* stats) {
  REF_GUARD({
    MappingConfig c;
    c.lambda_d = cfg->lambda_d;
    c.lr_sigma = cfg->lr_sigma;
    c.lr_sh = cfg->lr_sh;
    c.rmsprop_decay = cfg->rmsprop_decay;
    c.rmsprop_eps = cfg->rmsprop_eps;
    c.render = to_params(cfg->render);
    c.rays_per_batch = rays_per_batch;
    c.threads = threads;
    c.deterministic = deterministic != 0;
    auto* mm = static_cast<RefMapper*>(mapper);
    const MapStepStats s =
        mapping_step(*static_cast<VoxelGrid*>(grid), static_cast<const RefFrames*>(frames)->ptrs,
                     to_intr(*intr), c, mm->rms, mm->rng);
    std::memset(stats, 0, sizeof(*stats));
    stats->loss_photometric = s.loss_photometric;
    stats->loss_geometric = s.loss_geometric;
    stats->loss_total = s.loss_total;
    stats->rays_color = s.rays_color;
    stats->rays_depth = s.rays_depth;
    stats->psnr_estimate = s.psnr_estimate;
    stats->bad_ray = -1;
  });
}

// Merged gradient of one batch, assembled from the reference's per-ray
// building blocks in mapping_step's exact single-worker order
// (mapping.cpp:134-207): render_ray_scheduled, grad_color_wrt_params,
// grad_depth_wrt_sigma, backprop_to_vertices into one GradientBuffer.
int ref_mapping_grad(const void* grid_h, const void* frames_h, const or_intrinsics* intr_c,
                     const or_mapping_config* cfg, const int32_t* batch, int n_rays,
                     double* grad_out, int64_t* samples) {
  REF_GUARD({
    const auto& grid = *static_cast<const VoxelGrid*>(grid_h);
    const auto& kf = static_cast<const RefFrames*>(frames_h)->ptrs;
    const CameraIntrinsics intr = to_intr(*intr_c);
    const RenderParams params = to_params(cfg->render);
    std::vector<SampleSchedule> sched(n_rays);
    int m_color = 0, m_depth = 0;
    for (int i = 0; i < n_rays; ++i) {
      const int32_t* s = batch + 3 * i;
      sample_ray(grid, generate_ray(intr, *kf[s[0]]->gt_pose, s[1], s[2]), params, sched[i]);
      if (sched[i].empty()) continue;
      ++m_color;
      if (kf[s[0]]->depth_valid(s[1], s[2])) ++m_depth;
    }
    if (m_color == 0) throw std::runtime_error("mapping_step: no ray hit the grid");
    GradientBuffer buf(std::size_t(grid.geometry().num_vertices()));
    RayWorkspace ws;
    MapGradContribution contrib;
    int64_t total = 0;
    for (int i = 0; i < n_rays; ++i) {
      if (sched[i].empty()) continue;
      const int32_t* s = batch + 3 * i;
      const Frame& f = *kf[s[0]];
      const Ray ray = generate_ray(intr, *f.gt_pose, s[1], s[2]);
      render_ray_scheduled(grid, ray, sched[i], params, ws);
      total += ws.count;
      const Eigen::Vector3d target(f.color.at(s[1], s[2], 0), f.color.at(s[1], s[2], 1),
                                   f.color.at(s[1], s[2], 2));
      const Eigen::Vector3d residual = ws.color_out - target;
      const Eigen::Vector3d upstream_c = 2.0 * residual / double(m_color);
      double upstream_d = 0.0;
      const bool depth_ok = f.depth_valid(s[1], s[2]) && m_depth > 0;
      if (depth_ok)
        upstream_d = cfg->lambda_d * 2.0 * (ws.depth_out - double(f.depth.at(s[1], s[2]))) /
                     double(m_depth);
      contrib.resize_zero(ws.count);
      grad_color_wrt_params(ws, upstream_c, contrib);
      if (depth_ok && upstream_d != 0.0) grad_depth_wrt_sigma(ws, upstream_d, contrib);
      backprop_to_vertices(grid, ws, contrib, buf);
    }
    const std::size_t V = std::size_t(grid.geometry().num_vertices());
    std::memset(grad_out, 0, sizeof(double) * V * kPayloadSize);
    for (const std::uint32_t v : buf.sorted_touched())
      std::memcpy(grad_out + std::size_t(v) * kPayloadSize, buf.grad(v),
                  sizeof(double) * kPayloadSize);
    *samples = total;
  });
}

// ---- tracking.cpp
TrackingConfig to_tracking(const or_tracking_config* c, int threads) {
  TrackingConfig t;
  t.rays_per_iteration = c->rays_per_iteration;
  t.iterations = c->iterations;
  t.lr_omega = c->lr_omega;
  t.lr_tau = c->lr_tau;
  t.beta1 = c->beta1;
  t.beta2 = c->beta2;
  t.adam_eps = c->adam_eps;
  t.lambda_p = c->lambda_p;
  t.lambda_d = c->lambda_d;
  t.convergence_step = c->convergence_step;
  t.divergence_factor = c->divergence_factor;
  t.divergence_patience = c->divergence_patience;
  t.max_redraws = c->max_redraws;
  t.seed = c->seed;
  t.threads = threads;
  t.render = to_params(c->render);
  return t;
}

int ref_pose_gradient(const void* grid, const void* frames, const or_intrinsics* intr,
                      const or_pose* pose, const int32_t* pixels, int n,
                      const or_tracking_loss* cfg, int threads, or_pose_grad* out) {
  REF_GUARD({
    TrackingConfig t;
    t.lambda_p = cfg->lambda_p;
    t.lambda_d = cfg->lambda_d;
    t.render = to_params(cfg->render);
    t.threads = threads;
    std::vector<PixelSample> px(n);
    for (int i = 0; i < n; ++i) px[i] = {pixels[2 * i], pixels[2 * i + 1]};
    const PoseGradient g =
        pose_gradient(*static_cast<const VoxelGrid*>(grid),
                      *static_cast<const RefFrames*>(frames)->ptrs[0], to_intr(*intr),
                      to_pose(*pose), px, t);
    for (int a = 0; a < 3; ++a) {
      out->d_omega[a] = g.d_omega[a];
      out->d_tau[a] = g.d_tau[a];
    }
    out->loss = g.loss;
    out->rays_used = g.rays_used;
  });
}

// J^T J / J^T r assembled from the reference's grad_wrt_ray with unit
// upstreams, rows weighted by sqrt(lambda), chart as
// tracking.cpp:125-128.
int ref_pose_normal_eqs(const void* grid_h, const void* frames, const or_intrinsics* intr_c,
                        const or_pose* pose_c, const int32_t* pixels, int n,
                        const or_tracking_loss* cfg, or_normal_eqs* out) {
  REF_GUARD({
    const auto& grid = *static_cast<const VoxelGrid*>(grid_h);
    const Frame& frame = *static_cast<const RefFrames*>(frames)->ptrs[0];
    const CameraIntrinsics intr = to_intr(*intr_c);
    const Pose pose = to_pose(*pose_c);
    const RenderParams params = to_params(cfg->render);
    std::memset(out, 0, sizeof(*out));
    RayWorkspace ws;
    for (int i = 0; i < n; ++i) {
      const Ray ray = generate_ray(intr, pose, pixels[2 * i], pixels[2 * i + 1]);
      render_ray(grid, ray, params, ws);
      if (!ws.hit) continue;
      ++out->rays_used;
      const int px = pixels[2 * i], py = pixels[2 * i + 1];
      const Eigen::Vector3d cres =
          ws.color_out -
          Eigen::Vector3d(frame.color.at(px, py, 0), frame.color.at(px, py, 1),
                          frame.color.at(px, py, 2));
      const double dres = ws.depth_out - frame.depth.at(px, py);
      out->loss += cfg->lambda_p * cres.squaredNorm() + cfg->lambda_d * dres * dres;
      for (int row = 0; row < 4; ++row) {
        Eigen::Vector3d upc = Eigen::Vector3d::Zero();
        double upd = 0.0;
        if (row < 3)
          upc[row] = 1.0;
        else
          upd = 1.0;
        const PoseGradContribution rg = grad_wrt_ray(grid, ws, upc, upd);
        const Eigen::Vector3d g_perp = rg.d_direction - ray.d * ray.d.dot(rg.d_direction);
        const Eigen::Vector3d om = ray.d.cross(g_perp);
        const double J[6] = {om[0], om[1], om[2], rg.d_origin[0], rg.d_origin[1], rg.d_origin[2]};
        const double lam = row < 3 ? cfg->lambda_p : cfg->lambda_d;
        const double r = row < 3 ? cres[row] : dres;
        int idx = 0;
        for (int a = 0; a < 6; ++a) {
          for (int b = a; b < 6; ++b) out->jtj[idx++] += lam * J[a] * J[b];
          out->jtr[a] += lam * J[a] * r;
        }
      }
    }
    if (out->rays_used == 0) throw std::runtime_error("untrackable frame: all sampled rays miss the grid");
  });
}

int ref_track_frame(const void* grid, const void* frames, const or_intrinsics* intr,
                    const or_pose* init, const or_tracking_config* cfg, int threads,
                    or_track_result* out, double* loss_trace) {
  REF_GUARD({
    const TrackFrameResult r =
        track_frame(*static_cast<const VoxelGrid*>(grid),
                    *static_cast<const RefFrames*>(frames)->ptrs[0], to_intr(*intr),
                    to_pose(*init), to_tracking(cfg, threads));
    out->pose = from_pose(r.pose);
    out->failed = r.failed;
    out->iterations_run = r.iterations_run;
    out->final_loss = r.loss_trace.empty() ? 0.0 : r.loss_trace.back();
    if (loss_trace)
      for (std::size_t i = 0; i < r.loss_trace.size(); ++i) loss_trace[i] = r.loss_trace[i];
  });
}

// ---- map_scene (mapping.cpp:278-316) / track_sequence (tracking.cpp:254-295) over
// every frame of a handle (frames carry their gt poses); wall time via steady_clock.
struct or_map_scene_cfg {
  int32_t keyframe_stride, rays_per_batch, iterations_per_stage, initial_resolution;
  int32_t upsample_stages, max_resolution, prune_every, threads, deterministic, pad;
  double lambda_d, lr_sigma, lr_sh, rmsprop_decay, rmsprop_eps, prune_threshold, sigma_init,
      bounds_margin;
  uint64_t seed;
  or_render_params render;
};
void* ref_map_scene(const void* frames, const or_intrinsics* intr, const or_map_scene_cfg* c,
                    const or_geometry* geom, double* final_loss, double* ms) {
  try {
    Dataset ds;
    ds.intrinsics = to_intr(*intr);
    ds.frames = static_cast<const RefFrames*>(frames)->frames;
    MappingConfig m;
    m.keyframe_stride = c->keyframe_stride;
    m.rays_per_batch = c->rays_per_batch;
    m.iterations_per_stage = c->iterations_per_stage;
    m.initial_resolution = c->initial_resolution;
    m.upsample_stages = c->upsample_stages;
    m.max_resolution = c->max_resolution;
    m.prune_every = c->prune_every;
    m.threads = c->threads;
    m.deterministic = c->deterministic != 0;
    m.lambda_d = c->lambda_d;
    m.lr_sigma = c->lr_sigma;
    m.lr_sh = c->lr_sh;
    m.rmsprop_decay = c->rmsprop_decay;
    m.rmsprop_eps = c->rmsprop_eps;
    m.prune_threshold = c->prune_threshold;
    m.sigma_init = c->sigma_init;
    m.bounds_margin = c->bounds_margin;
    m.seed = c->seed;
    m.render = to_params(c->render);
    std::optional<GridGeometry> g;
    if (geom) {
      GridGeometry gg;
      for (int a = 0; a < 3; ++a) {
        gg.res[a] = geom->res[a];
        gg.origin[a] = geom->origin[a];
      }
      gg.voxel_size = geom->voxel_size;
      g = gg;
    }
    const auto t0 = std::chrono::steady_clock::now();
    MapResult r = map_scene(ds, m, g);
    *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    *final_loss = r.log.empty() ? 0.0 : r.log.back().stats.loss_total;
    return new VoxelGrid(std::move(r.grid));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
int ref_track_sequence(const void* grid, const void* frames, const or_intrinsics* intr,
                       const or_tracking_config* cfg, int threads, int constant_velocity,
                       or_pose* poses_out, double* ms) {
  REF_GUARD({
    Dataset ds;
    ds.intrinsics = to_intr(*intr);
    ds.frames = static_cast<const RefFrames*>(frames)->frames;
    TrackingConfig t = to_tracking(cfg, threads);
    t.init_policy = constant_velocity ? TrackingConfig::Init::kConstantVelocity
                                      : TrackingConfig::Init::kPreviousPose;
    const auto t0 = std::chrono::steady_clock::now();
    const TrackSequenceResult r = track_sequence(*static_cast<const VoxelGrid*>(grid), ds, t);
    *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    for (std::size_t i = 0; i < r.trajectory.poses.size(); ++i)
      poses_out[i] = from_pose(r.trajectory.poses[i]);
  });
}

// ---- eval.cpp / trajectory.cpp (metrics and TUM I/O around the hot path)
namespace {
Trajectory to_traj(const double* ts, const or_pose* poses, int n) {
  Trajectory t;
  for (int i = 0; i < n; ++i) t.push(ts[i], to_pose(poses[i]));
  return t;
}
std::vector<ImageF> to_images(const double* data, int n, int w, int h, int c) {
  std::vector<ImageF> out;
  for (int k = 0; k < n; ++k) {
    ImageF im(w, h, c);
    std::memcpy(im.data.data(), data + (size_t)k * w * h * c, sizeof(double) * w * h * c);
    out.push_back(std::move(im));
  }
  return out;
}
std::vector<const ImageF*> ptrs(const std::vector<ImageF>& v) {
  std::vector<const ImageF*> p;
  for (const ImageF& i : v) p.push_back(&i);
  return p;
}
}  // namespace

int ref_ate_rmse(const double* est_ts, const or_pose* est, int n_est, const double* ref_ts,
                 const or_pose* ref, int n_ref, int align, double* out, int* pairs) {
  REF_GUARD({
    *out = ate_rmse(to_traj(est_ts, est, n_est), to_traj(ref_ts, ref, n_ref), align != 0, pairs);
  });
}
int ref_rpe(const double* est_ts, const or_pose* est, int n_est, const double* ref_ts,
            const or_pose* ref, int n_ref, double interval_m, double* rpe_t, double* rpe_r_deg,
            int* pairs) {
  REF_GUARD({
    const RpeResult r = rpe(to_traj(est_ts, est, n_est), to_traj(ref_ts, ref, n_ref), interval_m);
    *rpe_t = r.rpe_t;
    *rpe_r_deg = r.rpe_r_deg;
    *pairs = r.pairs;
  });
}
// n images of w x h: rendered / reference colour n*h*w*3; masks n*h*w or NULL
int ref_psnr(const double* rendered, const double* reference, const double* masks, int n, int w,
             int h, int images, int pixels_per_image, uint64_t seed, double* out, int* samples) {
  REF_GUARD({
    const auto a = to_images(rendered, n, w, h, 3), b = to_images(reference, n, w, h, 3);
    std::vector<ImageF> m;
    if (masks) m = to_images(masks, n, w, h, 1);
    PixelSampleSpec spec;
    spec.images = images;
    spec.pixels_per_image = pixels_per_image;
    spec.seed = seed;
    *out = psnr(ptrs(a), ptrs(b), ptrs(m), spec, samples);
  });
}
int ref_depth_l1(const double* rendered, const double* reference, const double* masks, int n,
                 int w, int h, double* out, int* pixels) {
  REF_GUARD({
    const auto a = to_images(rendered, n, w, h, 1), b = to_images(reference, n, w, h, 1);
    std::vector<ImageF> m;
    if (masks) m = to_images(masks, n, w, h, 1);
    *out = depth_l1(ptrs(a), ptrs(b), ptrs(m), pixels);
  });
}
// evaluate_map_quality over frames[idx] of a frames handle (no exact depth)
int ref_evaluate_map_quality(const void* grid, const void* frames, const or_intrinsics* intr,
                             const int* idx, int n_idx, const or_render_params* p, int images,
                             int pixels_per_image, uint64_t seed, int threads, double* psnr_db,
                             double* depth_l1_m, int* color_samples, int* depth_pixels) {
  REF_GUARD({
    Dataset ds;
    ds.intrinsics = to_intr(*intr);
    ds.frames = static_cast<const RefFrames*>(frames)->frames;
    MapQualityOptions o;
    o.sampling.images = images;
    o.sampling.pixels_per_image = pixels_per_image;
    o.sampling.seed = seed;
    o.render = to_params(*p);
    o.threads = threads;
    const MapQuality q = evaluate_map_quality(*static_cast<const VoxelGrid*>(grid), ds,
                                              std::vector<int>(idx, idx + n_idx), o);
    *psnr_db = q.psnr_db;
    *depth_l1_m = q.depth_l1_m;
    *color_samples = q.color_samples;
    *depth_pixels = q.depth_pixels;
  });
}
int ref_save_tum(const char* path, const double* ts, const or_pose* poses, int n) {
  REF_GUARD({ save_tum(path, to_traj(ts, poses, n)); });
}
// returns the pose count (<= cap written), or -status
int ref_load_tum(const char* path, int cap, double* ts, or_pose* poses) {
  try {
    const Trajectory t = load_tum(path);
    for (int i = 0; i < (int)t.size() && i < cap; ++i) {
      ts[i] = t.timestamps[i];
      poses[i] = from_pose(t.poses[i]);
    }
    return (int)t.size();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -OR_RUNTIME;
  }
}

}  // extern "C"
