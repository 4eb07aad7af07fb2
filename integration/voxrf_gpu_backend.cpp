// The reference-side C++ binding of libvoxrf_b200: drop-in definitions of the
// voxrf batch entry points with the reference's exact signatures, exception
// types and messages, implemented on the C-ABI in include/voxrf_b200.h.
//
//   render_image   renderer.hpp:83-84   (renderer.cpp:149-174)
//   mapping_step   mapping.hpp:80-82    (mapping.cpp:114-233)
//   map_scene      mapping.hpp:98-99    (mapping.cpp:278-316)
//   pose_gradient  tracking.hpp:70-73   (tracking.cpp:76-143)
//   track_frame    tracking.hpp:82-84   (tracking.cpp:170-252)
//   track_sequence tracking.hpp:102-103 (tracking.cpp:254-295)
//
// A maintainer compiles this TU against the reference headers
// (proj/include/voxrf) and links it in place of those six definitions
// (INTEGRATION.md); everything else (VoxelGrid, per-ray CPU functions used by
// tests and gradcheck, dataset/eval/CLI) is unchanged.
//
// Device residency: the caller's grid, RMSProp state and keyframes stay in HBM
// between calls. Each host buffer the device mirrors is write-tracked
// (host_mirror.hpp), so a repeat call uploads only what the caller changed, and
// mapping_step writes back only the float4 groups its RMSProp pass updated (the
// reference's touched set, mapping.cpp:218-231) — untouched vertices keep their
// host fp64 values, as in the reference's in-place update.
#include <immintrin.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "voxrf/mapping.hpp"
#include "voxrf/renderer.hpp"
#include "voxrf/tracking.hpp"
#include "host_mirror.hpp"
#include "voxrf_b200.h"

namespace voxrf {
namespace {

using voxrf_b200::HostMirror;

vrf_context* ctx() {
  static vrf_context* c = [] {
    vrf_context* h = nullptr;
    const char* dev = std::getenv("VOXRF_DEVICE");
    const int rc = vrf_context_create(dev ? std::atoi(dev) : 0, &h);
    if (rc != VRF_OK)
      throw std::runtime_error("voxrf_b200: no usable CUDA device (status " +
                               std::to_string(rc) + "); there is no CPU fallback");
    vrf_track_updates(h, 1);  // mapping_step's sparse write-back
    return h;
  }();
  return c;
}

void check(int rc) {
  if (rc == VRF_OK) return;
  const std::string msg = vrf_last_error(ctx());
  if (rc == VRF_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == VRF_ERR_OUT_OF_RANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

vrf_grid_geometry to_c(const GridGeometry& g) {
  vrf_grid_geometry o{};
  for (int a = 0; a < 3; ++a) {
    o.res[a] = g.res[a];
    o.origin[a] = g.origin[a];
  }
  o.voxel_size = g.voxel_size;
  return o;
}
vrf_intrinsics to_c(const CameraIntrinsics& i) {
  return vrf_intrinsics{i.fx, i.fy, i.cx, i.cy, i.width, i.height, i.depth_scale};
}
vrf_pose to_c(const Pose& p) {
  return vrf_pose{{p.q.w(), p.q.x(), p.q.y(), p.q.z()}, {p.t.x(), p.t.y(), p.t.z()}};
}
Pose from_c(const vrf_pose& p) {
  Pose o;
  o.q = Eigen::Quaterniond(p.q[0], p.q[1], p.q[2], p.q[3]);
  o.t = Eigen::Vector3d(p.t[0], p.t[1], p.t[2]);
  return o;
}
vrf_render_params to_c(const RenderParams& r) {
  return vrf_render_params{r.step, r.t_near, r.t_far, r.termination_eps};
}

// ---- device residency
struct Residency {
  // drop-in mapping_step wall time by phase (ms, cumulative): batch draw,
  // residency sync, device step, write-back (voxrf_b200_dropin_phase_ms)
  double phase_ms[4] = {0.0, 0.0, 0.0, 0.0};
  double wb_ms[2] = {0.0, 0.0};  // write-back: blocked in the D2H reads, the rest (host work not overlapped)
  bool grid_valid = false;
  const double* data = nullptr;
  std::size_t data_n = 0;
  const std::uint8_t* occ = nullptr;
  std::size_t occ_n = 0;
  GridGeometry geom;
  const double* rms = nullptr;  // host RMSProp buffer the device state matches
  std::size_t rms_n = 0;
  struct Slot {
    const double* c = nullptr;
    const double* d = nullptr;
    std::size_t cn = 0, dn = 0;
    vrf_pose pose{};
  };
  std::vector<Slot> slots;
  vrf_intrinsics intr{};
  // statistics for tests / the bench: bytes uploaded and written back
  std::uint64_t up_bytes = 0, back_bytes = 0;
  std::int64_t last_samples = 0;  // composited samples of the last mapping_step
};
Residency g_res;

bool same_geom(const GridGeometry& a, const GridGeometry& b) {
  return a.res == b.res && a.origin == b.origin && a.voxel_size == b.voxel_size;
}

constexpr std::size_t kVertexBytes = sizeof(double) * kPayloadSize;

// Vertex ranges covering dirty byte ranges of a [V][28] fp64 buffer.
template <typename F>
void for_dirty_vertices(const double* buf, F&& f) {
  for (const auto& r : HostMirror::dirty(buf)) {
    const std::size_t v0 = r.first / kVertexBytes;
    const std::size_t v1 = (r.second + kVertexBytes - 1) / kVertexBytes;
    f(v0, v1 - v0);
  }
}

void sync_grid(const VoxelGrid& grid) {
  HostMirror::refresh();
  const double* d = grid.data().data();
  const std::size_t n = grid.data().size();
  const std::uint8_t* o = grid.occupancy().data();
  const std::size_t on = grid.occupancy().size();
  const bool same = g_res.grid_valid && d == g_res.data && n == g_res.data_n &&
                    o == g_res.occ && on == g_res.occ_n &&
                    same_geom(grid.geometry(), g_res.geom) &&
                    HostMirror::tracked(d, n * sizeof(double)) && HostMirror::tracked(o, on);
  if (!same) {
    const vrf_grid_geometry g = to_c(grid.geometry());
    check(vrf_grid_upload(ctx(), &g, d, o));  // (re-allocates: RMSProp state restarts)
    g_res.up_bytes += n * sizeof(double) + on;
    HostMirror::track(d, n * sizeof(double));
    HostMirror::track(o, on);
    g_res.grid_valid = true;
    g_res.data = d;
    g_res.data_n = n;
    g_res.occ = o;
    g_res.occ_n = on;
    g_res.geom = grid.geometry();
    g_res.rms = nullptr;
    return;
  }
  if (!HostMirror::dirty(o).empty()) {  // set_cell_active / prune since the last call
    check(vrf_grid_set_occupancy(ctx(), o));
    g_res.up_bytes += on;
    HostMirror::clean(o);
  }
  for_dirty_vertices(d, [&](std::size_t v0, std::size_t nv) {
    check(vrf_grid_write_vertices(ctx(), std::int64_t(v0), std::int64_t(nv), d + v0 * kPayloadSize));
    g_res.up_bytes += nv * kVertexBytes;
  });
  HostMirror::clean(d);
}

// mapping.cpp:219: a state of the wrong size restarts at zero.
void sync_rmsprop(RmspropState& st, std::size_t n) {
  if (st.v.size() != n) st.reset(n);
  double* v = st.v.data();
  if (v == g_res.rms && n == g_res.rms_n && HostMirror::tracked(v, n * sizeof(double))) {
    for_dirty_vertices(v, [&](std::size_t v0, std::size_t nv) {
      check(vrf_rmsprop_write_vertices(ctx(), std::int64_t(v0), std::int64_t(nv),
                                       v + v0 * kPayloadSize));
      g_res.up_bytes += nv * kVertexBytes;
    });
  } else {
    check(vrf_rmsprop_upload(ctx(), v));
    g_res.up_bytes += n * sizeof(double);
    HostMirror::track(v, n * sizeof(double));
    g_res.rms = v;
    g_res.rms_n = n;
  }
  HostMirror::clean(v);
}

// The frames of the call in slots 0..n-1; a slot is rewritten only when its
// buffers changed (new buffers, or writes since they were uploaded).
void sync_frames(const CameraIntrinsics& intr, const std::vector<const Frame*>& frames) {
  const vrf_intrinsics ic = to_c(intr);
  const bool same_intr = std::memcmp(&ic, &g_res.intr, sizeof(ic)) == 0;
  if (!same_intr || g_res.slots.size() < frames.size()) {
    const std::size_t cap = std::max(frames.size(), same_intr ? 2 * g_res.slots.size() : 0);
    check(vrf_frames_reserve(ctx(), &ic, int(cap)));
    g_res.slots.assign(cap, {});
    g_res.intr = ic;
  }
  for (std::size_t i = 0; i < frames.size(); ++i) {
    const Frame& f = *frames[i];
    Residency::Slot want{f.color.data.data(), f.depth.data.data(), f.color.data.size(),
                         f.depth.data.size(), to_c(f.gt_pose ? *f.gt_pose : Pose{})};
    Residency::Slot& have = g_res.slots[i];
    const bool same_buffers = have.c == want.c && have.d == want.d && have.cn == want.cn &&
                              have.dn == want.dn &&
                              HostMirror::tracked(want.c, want.cn * sizeof(double)) &&
                              HostMirror::tracked(want.d, want.dn * sizeof(double)) &&
                              HostMirror::dirty(want.c).empty() &&
                              HostMirror::dirty(want.d).empty();
    if (!same_buffers) {
      check(vrf_frame_set(ctx(), int(i), want.c, want.d, &want.pose));
      g_res.up_bytes += (want.cn + want.dn) * sizeof(double);
      HostMirror::track(want.c, want.cn * sizeof(double));
      HostMirror::track(want.d, want.dn * sizeof(double));
      have = want;
    } else if (std::memcmp(&have.pose, &want.pose, sizeof(vrf_pose)) != 0) {
      check(vrf_frame_set_pose(ctx(), int(i), &want.pose));
      have.pose = want.pose;
    }
  }
}

// Writes mapping_step's result back into the caller's grid and RMSProp state:
// the updated float4 groups only, or everything when most groups changed.
// Host worker pool for the write-back: splits [0, n) over up to `threads` threads.
template <typename F>
void parallel_for(std::int64_t n, int threads, F&& f) {
  const int nt = n < (1 << 15) ? 1 : threads;
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(f, n * t / nt, n * (t + 1) / nt);
  f(0, n / nt);
  for (auto& th : pool) th.join();
}

// dst[i] = double(src[i]) for a contiguous run. The dense write-back widens
// 2 x 1.9 GB of fp32 into 2 x 3.8 GB of the caller's fp64 buffers; with
// non-temporal stores the host does not read the destination lines first.
__attribute__((target("avx2"))) void widen_stream_avx2(double* dst, const float* src,
                                                       std::int64_t n) {
  std::int64_t i = 0;
  for (; i < n && (reinterpret_cast<std::uintptr_t>(dst + i) & 31); ++i) dst[i] = double(src[i]);
  for (; i + 4 <= n; i += 4)
    _mm256_stream_pd(dst + i, _mm256_cvtps_pd(_mm_loadu_ps(src + i)));
  for (; i < n; ++i) dst[i] = double(src[i]);
  _mm_sfence();
}
void widen(double* dst, const float* src, std::int64_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) return widen_stream_avx2(dst, src, n);
  for (std::int64_t i = 0; i < n; ++i) dst[i] = double(src[i]);
}

int writeback_threads() {
  static const int n = int(std::min<unsigned>(32, std::max(1u, std::thread::hardware_concurrency())));
  return n;
}

// In-place contract of mapping_step (mapping.hpp:80): the device's updated theta
// and RMSProp v reach the caller's fp64 buffers. Chunked through two page-locked
// staging buffers, so the D2H of chunk i+1 runs while host threads convert /
// scatter chunk i.
//  * sparse (the RMSProp update log, sorted by group id on the device, so the
//    scatter walks the caller's arrays forward): 36 B per updated float4 group;
//  * dense (when over a third of the groups changed): both fp32 arrays, widened
//    on the host.
void write_back(VoxelGrid& grid, RmspropState& st) {
  double* d = grid.data().data();
  double* v = st.v.data();
  const std::size_t groups = grid.data().size() / 4;
  std::int64_t n = 0;
  check(vrf_updates_count(ctx(), &n));
  HostMirror::unprotect(d);
  HostMirror::unprotect(v);
  constexpr std::int64_t kChunk = std::int64_t(1) << 21;  // entries (sparse) / 4-float groups (dense)
  static void* stage[2] = {nullptr, nullptr};
  constexpr std::size_t kStageBytes = std::size_t(kChunk) * (sizeof(std::uint32_t) + 8 * sizeof(float));
  for (void*& b : stage)
    if (!b && !(b = vrf_host_alloc(kStageBytes)))
      throw std::runtime_error("voxrf_b200: page-locked staging allocation failed");
  const int nt = writeback_threads();
  const auto w0 = std::chrono::steady_clock::now();
  double d2h_ms = 0.0;
  std::thread worker;  // host work on the previous chunk
  auto timed_read = [&](auto&& read) {
    const auto a = std::chrono::steady_clock::now();
    read();
    d2h_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
  };
  if (std::size_t(n) * 3 > groups) {  // dense: cheaper than the indexed form
    const std::int64_t total = std::int64_t(grid.data().size());  // floats per array
    const std::int64_t step = 4 * kChunk;
    int k = 0;
    for (int which = 0; which < 2; ++which) {
      double* dst = which == 0 ? d : v;
      for (std::int64_t off = 0; off < total; off += step, k ^= 1) {
        const std::int64_t cnt = std::min(step, total - off);
        float* buf = static_cast<float*>(stage[k]);
        timed_read([&] { check(vrf_state_read_f32(ctx(), which, off, cnt, buf)); });
        if (worker.joinable()) worker.join();
        worker = std::thread([=] {
          parallel_for(cnt, nt, [=](std::int64_t i0, std::int64_t i1) {
            widen(dst + off + i0, buf + i0, i1 - i0);
          });
        });
      }
    }
    if (worker.joinable()) worker.join();
    g_res.back_bytes += 2 * groups * 4 * sizeof(float);
  } else if (n > 0) {
    int k = 0;
    for (std::int64_t off = 0; off < n; off += kChunk, k ^= 1) {
      const std::int64_t cnt = std::min(kChunk, n - off);
      float* th = static_cast<float*>(stage[k]);
      float* vv = th + 4 * kChunk;
      std::uint32_t* ids = reinterpret_cast<std::uint32_t*>(vv + 4 * kChunk);
      timed_read([&] { check(vrf_updates_read_range(ctx(), off, cnt, 1, ids, th, vv)); });
      if (worker.joinable()) worker.join();
      // the logged groups are distinct, so the threads never write the same element
      worker = std::thread([=] {
        parallel_for(cnt, nt, [=](std::int64_t i0, std::int64_t i1) {
          for (std::int64_t i = i0; i < i1; ++i) {
            const std::size_t o = 4 * std::size_t(ids[std::size_t(i)]);  // == vertex * 28 + 4 group
            for (int e = 0; e < 4; ++e) {
              d[o + e] = th[4 * std::size_t(i) + e];
              v[o + e] = vv[4 * std::size_t(i) + e];
            }
          }
        });
      });
    }
    if (worker.joinable()) worker.join();
    g_res.back_bytes += std::size_t(n) * (4 + 32);
  }
  const double total_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
  g_res.wb_ms[0] += d2h_ms;
  g_res.wb_ms[1] += total_ms - d2h_ms;
  HostMirror::clean(d);
  HostMirror::clean(v);
}

void upload_frames(const CameraIntrinsics& intr, const std::vector<const Frame*>& frames) {
  std::vector<const double*> colors, depths;
  std::vector<vrf_pose> poses;
  for (const Frame* f : frames) {
    colors.push_back(f->color.data.data());
    depths.push_back(f->depth.data.data());
    poses.push_back(to_c(f->gt_pose ? *f->gt_pose : Pose{}));
  }
  const vrf_intrinsics ic = to_c(intr);
  check(vrf_frames_upload(ctx(), &ic, int(frames.size()), colors.data(), depths.data(),
                          poses.data()));
  g_res.slots.clear();  // the slot store was replaced
  g_res.intr = vrf_intrinsics{};
}

vrf_mapping_config to_c(const MappingConfig& c) {
  vrf_mapping_config o{};
  o.lambda_d = c.lambda_d;
  o.lr_sigma = c.lr_sigma;
  o.lr_sh = c.lr_sh;
  o.rmsprop_decay = c.rmsprop_decay;
  o.rmsprop_eps = c.rmsprop_eps;
  o.deterministic = c.deterministic ? 1 : 0;
  o.render = to_c(c.render);
  return o;
}

// mapping.cpp:121-128: the batch is drawn from the caller's Rng. The library's
// vrf_rng_draw_batch produces the same stream (one raw draw per index, so large
// batches are drawn in parallel from jumped-ahead states) and leaves the Rng
// where the reference's loop would. Rng is xoshiro256**'s four words and nothing
// else (rng.hpp:13-81), so its state is copied bytewise.
static_assert(std::is_trivially_copyable_v<Rng> && sizeof(Rng) == 4 * sizeof(std::uint64_t),
              "voxrf::Rng is expected to hold exactly the xoshiro256** state");
std::vector<int32_t> draw_batch(Rng& rng, int n_frames, const CameraIntrinsics& intr, int n) {
  std::vector<int32_t> b(3 * std::size_t(n));
  std::uint64_t st[4];
  std::memcpy(st, &rng, sizeof(st));
  vrf_rng_draw_batch(st, n_frames, intr.width, intr.height, n, b.data());
  std::memcpy(static_cast<void*>(&rng), st, sizeof(st));
  return b;
}

MapStepStats to_stats(const vrf_map_step_stats& s) {
  MapStepStats o;
  o.loss_photometric = s.loss_photometric;
  o.loss_geometric = s.loss_geometric;
  o.loss_total = s.loss_total;
  o.rays_color = s.rays_color;
  o.rays_depth = s.rays_depth;
  o.psnr_estimate = s.psnr_estimate;
  return o;
}

vrf_tracking_config to_c(const TrackingConfig& c) {
  vrf_tracking_config o{};
  o.rays_per_iteration = c.rays_per_iteration;
  o.iterations = c.iterations;
  o.lr_omega = c.lr_omega;
  o.lr_tau = c.lr_tau;
  o.beta1 = c.beta1;
  o.beta2 = c.beta2;
  o.adam_eps = c.adam_eps;
  o.lambda_p = c.lambda_p;
  o.lambda_d = c.lambda_d;
  o.convergence_step = c.convergence_step;
  o.divergence_factor = c.divergence_factor;
  o.divergence_patience = c.divergence_patience;
  o.max_redraws = c.max_redraws;
  o.seed = c.seed;
  o.render = to_c(c.render);
  return o;
}

TrackFrameResult track_uploaded(int frame, const CameraIntrinsics& intr, const Pose& init,
                                const TrackingConfig& config) {
  const vrf_intrinsics ic = to_c(intr);
  const vrf_pose pc = to_c(init);
  const vrf_tracking_config tc = to_c(config);
  vrf_track_frame_result r{};
  std::vector<double> trace(std::size_t(std::max(config.iterations, 1)));
  check(vrf_track_frame(ctx(), frame, &ic, &pc, &tc, &r, trace.data()));
  TrackFrameResult out;
  out.pose = from_c(r.pose);
  out.failed = r.failed != 0;
  out.iterations_run = r.iterations_run;
  out.loss_trace.assign(trace.begin(), trace.begin() + r.iterations_run);
  return out;
}

}  // namespace

Frame render_image(const VoxelGrid& grid, const CameraIntrinsics& intr, const Pose& pose,
                   const RenderParams& params, int stride, int /*threads*/) {
  if (stride < 1) throw std::invalid_argument("render_image: stride must be >= 1");
  const int out_w = (intr.width + stride - 1) / stride;
  const int out_h = (intr.height + stride - 1) / stride;
  Frame frame;
  frame.color = ImageF(out_w, out_h, 3);
  frame.depth = ImageF(out_w, out_h, 1);
  frame.gt_pose = pose;
  sync_grid(grid);
  const vrf_intrinsics ic = to_c(intr);
  const vrf_pose pc = to_c(pose);
  const vrf_render_params rp = to_c(params);
  check(vrf_render_image(ctx(), &ic, &pc, &rp, stride, frame.color.data.data(),
                         frame.depth.data.data()));
  return frame;
}

MapStepStats mapping_step(VoxelGrid& grid, const std::vector<const Frame*>& keyframes,
                          const CameraIntrinsics& intrinsics, const MappingConfig& config,
                          RmspropState& rmsprop, Rng& rng) {
  if (keyframes.empty()) throw std::runtime_error("mapping_step: no keyframes");
  using clock = std::chrono::steady_clock;
  const auto t0 = clock::now();
  const std::vector<int32_t> batch =
      draw_batch(rng, int(keyframes.size()), intrinsics, config.rays_per_batch);
  const auto t1 = clock::now();
  sync_grid(grid);
  sync_rmsprop(rmsprop, grid.data().size());
  sync_frames(intrinsics, keyframes);
  const auto t2 = clock::now();
  const vrf_mapping_config cc = to_c(config);
  vrf_map_step_stats st{};
  const int rc = vrf_mapping_step(ctx(), &cc, batch.data(), config.rays_per_batch, &st);
  if (rc != VRF_OK) {
    g_res.grid_valid = false;  // (no update happened; re-sync next call)
    check(rc);
  }
  g_res.last_samples = st.samples;
  const auto t3 = clock::now();
  // In-place contract (mapping.hpp:80): grid and RMSProp state are updated.
  write_back(grid, rmsprop);
  const auto t4 = clock::now();
  const auto ms = [](clock::time_point a, clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  g_res.phase_ms[0] += ms(t0, t1);
  g_res.phase_ms[1] += ms(t1, t2);
  g_res.phase_ms[2] += ms(t2, t3);
  g_res.phase_ms[3] += ms(t3, t4);
  return to_stats(st);
}

MapResult map_scene(const Dataset& dataset, const MappingConfig& config,
                    const std::optional<GridGeometry>& geometry) {
  if (dataset.frames.empty()) throw std::runtime_error("map_scene: empty dataset");
  std::vector<const Frame*> keyframes;
  for (std::size_t i = 0; i < dataset.frames.size(); i += config.keyframe_stride) {
    if (!dataset.frames[i].gt_pose)
      throw std::runtime_error("map_scene: keyframe " + std::to_string(i) + " has no pose");
    keyframes.push_back(&dataset.frames[i]);
  }
  const GridGeometry geom = geometry ? *geometry : fit_grid_geometry(dataset, keyframes, config);
  MapResult result{VoxelGrid(geom, config.sigma_init), {}};
  upload_frames(dataset.intrinsics, keyframes);
  g_res.grid_valid = false;  // the device grid becomes map_scene's own
  const vrf_mapping_config cc = to_c(config);
  const auto t0 = std::chrono::steady_clock::now();
  int iteration = 0;
  // The grid, its RMSProp state and the keyframes stay in HBM for the whole
  // schedule: stages refine on the device (vrf_grid_upsample ==
  // VoxelGrid::upsampled + RMSProp reset, mapping.cpp:297-300) and the host
  // grid is written back once at the end.
  {
    const vrf_grid_geometry g0 = to_c(result.grid.geometry());
    check(vrf_grid_upload(ctx(), &g0, result.grid.data().data(), result.grid.occupancy().data()));
  }
  check(vrf_rmsprop_reset(ctx()));
  uint64_t rs[4];
  vrf_rng_seed(config.seed, rs);  // == Rng(config.seed), mapping.cpp:292
  const int kf = int(keyframes.size());
  for (int stage = 0; stage <= config.upsample_stages; ++stage) {
    if (stage > 0) check(vrf_grid_upsample(ctx(), config.max_resolution));
    int left = config.iterations_per_stage;
    while (left > 0) {
      // one pipelined vrf_mapping_steps call up to the next prune point
      int n = left;
      if (config.prune_every > 0)
        n = std::min(n, config.prune_every - iteration % config.prune_every);
      std::vector<vrf_map_step_stats> st(n);
      check(vrf_mapping_steps(ctx(), &cc, rs, kf, config.rays_per_batch, n, st.data()));
      const double ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      for (int k = 0; k < n; ++k, ++iteration) {
        MapLogRow row;
        row.iteration = iteration;
        row.stats = to_stats(st[k]);
        row.elapsed_ms = ms;
        result.log.push_back(row);
      }
      left -= n;
      if (config.prune_every > 0 && iteration % config.prune_every == 0) {
        int64_t off = 0;
        check(vrf_grid_prune(ctx(), config.prune_threshold, &off));
      }
    }
  }
  vrf_grid_geometry fg{};
  check(vrf_grid_get_geometry(ctx(), &fg));
  GridGeometry g;
  for (int a = 0; a < 3; ++a) {
    g.res[a] = fg.res[a];
    g.origin[a] = fg.origin[a];
  }
  g.voxel_size = fg.voxel_size;
  result.grid = VoxelGrid(g);
  std::vector<std::uint8_t> occ(result.grid.occupancy().size());
  check(vrf_grid_download(ctx(), result.grid.data().data(), occ.data()));
  for (int cz = 0; cz < g.res.z() - 1; ++cz)
    for (int cy = 0; cy < g.res.y() - 1; ++cy)
      for (int cx = 0; cx < g.res.x() - 1; ++cx)
        result.grid.set_cell_active(cx, cy, cz, occ[g.cell_index(cx, cy, cz)] != 0);
  return result;
}

PoseGradient pose_gradient(const VoxelGrid& grid, const Frame& frame,
                           const CameraIntrinsics& intrinsics, const Pose& pose,
                           const std::vector<PixelSample>& pixels, const TrackingConfig& config) {
  if (pixels.empty()) throw std::runtime_error("pose_gradient: empty pixel set");
  sync_grid(grid);
  sync_frames(intrinsics, {&frame});
  std::vector<int32_t> px(2 * pixels.size());
  for (std::size_t i = 0; i < pixels.size(); ++i) {
    px[2 * i] = pixels[i].px;
    px[2 * i + 1] = pixels[i].py;
  }
  const vrf_intrinsics ic = to_c(intrinsics);
  const vrf_pose pc = to_c(pose);
  const vrf_tracking_loss lc{config.lambda_p, config.lambda_d, to_c(config.render)};
  vrf_pose_gradient_result r{};
  check(vrf_pose_gradient(ctx(), 0, &ic, &pc, px.data(), int(pixels.size()), &lc, &r));
  PoseGradient out;
  out.d_omega = Eigen::Vector3d(r.d_omega[0], r.d_omega[1], r.d_omega[2]);
  out.d_tau = Eigen::Vector3d(r.d_tau[0], r.d_tau[1], r.d_tau[2]);
  out.loss = r.loss;
  out.rays_used = r.rays_used;
  return out;
}

TrackFrameResult track_frame(const VoxelGrid& grid, const Frame& frame,
                             const CameraIntrinsics& intrinsics, const Pose& init,
                             const TrackingConfig& config) {
  if (config.iterations == 0) {
    TrackFrameResult r;
    r.pose = init;
    return r;
  }
  sync_grid(grid);
  sync_frames(intrinsics, {&frame});
  return track_uploaded(0, intrinsics, init, config);
}

TrackSequenceResult track_sequence(const VoxelGrid& grid, const Dataset& dataset,
                                   const TrackingConfig& config) {
  if (dataset.frames.empty()) throw std::runtime_error("track_sequence: empty dataset");
  if (!dataset.frames.front().gt_pose)
    throw std::runtime_error("track_sequence: first frame needs a pose");
  sync_grid(grid);
  std::vector<const Frame*> all;
  for (const Frame& f : dataset.frames) all.push_back(&f);
  sync_frames(dataset.intrinsics, all);

  TrackSequenceResult result;
  const Pose first = *dataset.frames.front().gt_pose;
  result.trajectory.push(dataset.frames.front().timestamp, first);
  result.status.push_back({0, 0, 0.0, 0.0, false});
  Pose prev = first, prev_prev = first;
  bool have_two = false;
  for (std::size_t i = 1; i < dataset.frames.size(); ++i) {
    Pose init = prev;
    if (config.init_policy == TrackingConfig::Init::kConstantVelocity && have_two)
      init = prev * (prev_prev.inverse() * prev);
    TrackingConfig fc = config;
    fc.seed = config.seed + 0x9e3779b9u * std::uint64_t(i);
    const auto t0 = std::chrono::steady_clock::now();
    const TrackFrameResult tf =
        fc.iterations == 0 ? TrackFrameResult{init, {}, false, 0}
                           : track_uploaded(int(i), dataset.intrinsics, init, fc);
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    result.trajectory.push(dataset.frames[i].timestamp, tf.pose);
    result.status.push_back({int(i), tf.iterations_run,
                             tf.loss_trace.empty() ? 0.0 : tf.loss_trace.back(), ms, tf.failed});
    if (!tf.failed) {
      prev_prev = prev;
      prev = tf.pose;
      have_two = true;
    }
  }
  return result;
}

}  // namespace voxrf

// Residency counters of the drop-in (tests, bench): bytes uploaded to the device
// and written back to the caller's buffers since the process started.
// Cumulative drop-in mapping_step wall time by phase (ms): [0] batch draw, [1]
// residency sync, [2] device step, [3] write-back, [4] of which the update-log
// D2H, [5] of which the host scatter.
extern "C" void voxrf_b200_dropin_phase_ms(double* out) {
  for (int i = 0; i < 4; ++i) out[i] = voxrf::g_res.phase_ms[i];
  out[4] = voxrf::g_res.wb_ms[0];
  out[5] = voxrf::g_res.wb_ms[1];
}
extern "C" void voxrf_b200_dropin_traffic(std::uint64_t* uploaded, std::uint64_t* written_back) {
  *uploaded = voxrf::g_res.up_bytes;
  *written_back = voxrf::g_res.back_bytes;
}
// Composited samples of the last drop-in mapping_step (MapStepStats has no such
// field; the bench's samples/s needs it).
extern "C" std::int64_t voxrf_b200_dropin_last_samples() { return voxrf::g_res.last_samples; }
