// e2e leg of bench.py through the reference's own C++ signature: voxrf::mapping_step
// (mapping.hpp:80-82) as linked from integration/voxrf_gpu_backend.cpp, called in
// a loop the way map_scene calls it (one Rng, one RmspropState, the grid mutated
// in place). Every call: host Rng batch draw, residency check of grid / RMSProp /
// keyframes (nothing re-sent once resident), the device step, and the in-place
// write-back of the updated float4 groups into the caller's fp64 grid and state.
//
// Workload = bench.py's config 3: 257^3-vertex grid at sigma_init 0.1 over the
// config-2 room bounds, 10 keyframes of 1200x680 (rendered here by the drop-in
// render_image from a procedural map; their content does not change the sample
// count, which depends on the map being trained), batches of --rays rays.
// usage: voxrf_dropin_bench RAYS STEPS WARMUP -> one JSON line on stdout
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "voxrf/mapping.hpp"
#include "voxrf/renderer.hpp"

extern "C" void voxrf_b200_dropin_traffic(std::uint64_t* uploaded, std::uint64_t* written_back);
extern "C" void voxrf_b200_dropin_phase_ms(double* out);
extern "C" std::int64_t voxrf_b200_dropin_last_samples();

using namespace voxrf;

int main(int argc, char** argv) {
  const int rays = argc > 1 ? std::atoi(argv[1]) : 4096;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 5;
  const int warmup = argc > 3 ? std::atoi(argv[3]) : 2;
  // the config-2 room bounds: [0,7] x [0,6] x [0,3] m, 257^3 vertices, 7.7/256 m voxels
  GridGeometry geom{Eigen::Vector3i(257, 257, 257), {-0.35, -0.85, -2.35}, 7.7 / 256.0};
  // a procedural target map: walls of the box + a ball, SH DC from position
  VoxelGrid target(geom, 0.0);
  const Eigen::Vector3d lo(0, 0, 0), hi(7, 6, 3), ball(4.5, 3.5, 1.2);
  for (int iz = 0; iz < 257; ++iz)
    for (int iy = 0; iy < 257; ++iy)
      for (int ix = 0; ix < 257; ++ix) {
        const Eigen::Vector3d p = geom.to_world(Eigen::Vector3d(ix, iy, iz));
        double d = 1e9;
        for (int a = 0; a < 3; ++a) d = std::min({d, std::abs(p[a] - lo[a]), std::abs(p[a] - hi[a])});
        d = std::min(d, std::abs((p - ball).norm() - 0.6));
        double* v = target.vertex(geom.vertex_index(ix, iy, iz));
        v[0] = float(200.0 * std::max(0.0, 1.0 - d / (1.5 * geom.voxel_size)));
        for (int ch = 0; ch < 3; ++ch) v[1 + 9 * ch] = float(0.5 * std::sin(1.3 * p[ch] + ch));
      }
  CameraIntrinsics intr{600.0, 600.0, 599.5, 339.5, 1200, 680, 6553.5};
  std::vector<Frame> frames;
  for (int k = 0; k < 10; ++k) {
    const double a = 0.6 * k;
    const Pose pose = look_at({3.5 + 1.2 * std::cos(a), 3.0 + 1.0 * std::sin(a), 1.5},
                              {3.5 + 2.5 * std::cos(a + 1.0), 3.0 + 2.0 * std::sin(a + 1.0), 1.2});
    Frame f = render_image(target, intr, pose, RenderParams{}, 1);
    f.gt_pose = pose;
    frames.push_back(std::move(f));
  }
  std::vector<const Frame*> kf;
  for (const Frame& f : frames) kf.push_back(&f);
  VoxelGrid grid(geom, 0.1);  // the map being trained (map_scene's sigma_init)
  RmspropState rms;
  MappingConfig cfg;
  cfg.rays_per_batch = rays;
  Rng rng(1);
  for (int i = 0; i < warmup; ++i) mapping_step(grid, kf, intr, cfg, rms, rng);
  std::uint64_t up0, back0, up1, back1;
  voxrf_b200_dropin_traffic(&up0, &back0);
  double ph0[6], ph1[6];
  voxrf_b200_dropin_phase_ms(ph0);
  long long samples = 0;
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < steps; ++i) {
    mapping_step(grid, kf, intr, cfg, rms, rng);
    samples += voxrf_b200_dropin_last_samples();
  }
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  voxrf_b200_dropin_traffic(&up1, &back1);
  voxrf_b200_dropin_phase_ms(ph1);
  std::printf("{\"api\": \"voxrf::mapping_step (reference C++ signature, drop-in)\", "
              "\"rays_per_step\": %d, \"steps\": %d, \"samples_per_s\": %.6e, "
              "\"rays_per_s\": %.6e, \"ms_per_step\": %.4f, \"upload_bytes_per_step\": %.0f, "
              "\"writeback_bytes_per_step\": %.0f, \"grid_bytes_fp64\": %zu, "
              "\"phase_ms_per_step\": {\"draw\": %.3f, \"sync\": %.3f, \"device_step\": %.3f, "
              "\"write_back\": %.3f, \"write_back_d2h\": %.3f, \"write_back_scatter\": %.3f}}\n",
              rays, steps, samples / s, double(rays) * steps / s, 1e3 * s / steps,
              double(up1 - up0) / steps, double(back1 - back0) / steps,
              grid.data().size() * sizeof(double), (ph1[0] - ph0[0]) / steps,
              (ph1[1] - ph0[1]) / steps, (ph1[2] - ph0[2]) / steps, (ph1[3] - ph0[3]) / steps,
              (ph1[4] - ph0[4]) / steps, (ph1[5] - ph0[5]) / steps);
  return 0;
}
