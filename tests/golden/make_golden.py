"""Generates tests/golden/voxrf_golden.npz from the REFERENCE itself
(oracle/_ref/libvoxrf_ref.so: the reference sources compiled unchanged).

Run here (needs /root/reference): python tests/golden/make_golden.py
The fixture is committed; tests/test_golden.py checks the C oracle (and the GPU
path, on the box) against it without needing /root/reference."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import oracle as orc  # noqa: E402
from paper_2307_03404_b200.api import (CameraIntrinsics, Frame, GridGeometry, MappingConfig,  # noqa: E402
                                       RenderParams, TrackingConfig, VoxelGrid)
from paper_2307_03404_b200 import synth  # noqa: E402


def inputs():
    rng = np.random.default_rng(2024)
    n = 7
    geom = GridGeometry((n, n, n), (-0.1, 0.05, -0.2), 0.2)
    grid = VoxelGrid(geom)
    grid.data[:, 0] = rng.uniform(-0.5, 6.0, geom.num_vertices)
    grid.data[:, 1:] = rng.uniform(-0.6, 0.6, (geom.num_vertices, 27))
    grid.data[:] = grid.data.astype(np.float32).astype(np.float64)
    grid.active[rng.uniform(size=geom.num_cells) < 0.15] = 0
    intr = CameraIntrinsics(20.0, 20.0, 8.0, 6.0, 16, 12, 1000.0)
    c = geom.world_min() + 0.5 * (geom.world_max() - geom.world_min())
    poses = [synth.look_at(c + np.array([1.5 * np.cos(a), 1.5 * np.sin(a), 0.3]), c)
             for a in (0.0, 0.4, 0.8)]
    return grid, intr, poses


def main():
    ref = orc.RefLib()
    grid, intr, poses = inputs()
    gh = ref.grid(grid)
    out = {"grid_data": grid.data, "grid_active": grid.active,
           "geom": np.array([*grid.geom.res, *grid.geom.origin, grid.geom.voxel_size]),
           "intr": np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height,
                             intr.depth_scale]),
           "poses": np.array([[*p.q, *p.t] for p in poses])}
    frames = []
    for k, p in enumerate(poses):
        c, d = ref.render_image(gh, intr, p, RenderParams(), 1, 1)
        out[f"render_color_{k}"], out[f"render_depth_{k}"] = c, d
        c, d = synth.quantize_frame(np.clip(c + 0.05 * (k - 1), 0, 1), d * (1 + 0.02 * k),
                                    intr.depth_scale)
        frames.append(Frame(c, d, 0.0, p))
        out[f"frame_color_{k}"], out[f"frame_depth_{k}"] = c, d
    c, d = ref.render_image(gh, intr, poses[1], RenderParams(), 3, 1)
    out["render_color_stride3"], out["render_depth_stride3"] = c, d
    # schedules
    rng = np.random.default_rng(7)
    rays = np.concatenate([rng.uniform(-0.2, 1.4, (24, 3)),
                           rng.normal(size=(24, 3))], axis=1)
    rays[:, 3:] /= np.linalg.norm(rays[:, 3:], axis=1, keepdims=True)
    out["rays"] = rays
    counts, ts, ds = [], [], []
    for r in rays:
        t, dl = ref.sample_ray(gh, r[:3], r[3:], RenderParams())
        counts.append(len(t))
        ts.append(np.pad(t, (0, 64 - len(t))))
        ds.append(np.pad(dl, (0, 64 - len(t))))
    out["sched_count"], out["sched_t"], out["sched_delta"] = np.array(counts), np.array(ts), np.array(ds)
    # mapping gradient + one mapping_step (the reference draws batch from Rng(17))
    fh = ref.frames(frames, intr)
    cfg = MappingConfig()
    batch = orc.Oracle().draw_batch(17, len(frames), intr.width, intr.height, 96)
    out["map_batch"] = batch
    grad, samples = ref.mapping_grad(gh, fh, intr, cfg, batch, grid.geom.num_vertices)
    out["map_grad"], out["map_samples"] = grad, np.array([samples])
    mapper = ref.lib.ref_mapper_create(17)
    st = ref.mapping_step(gh, fh, intr, cfg, 96, 1, True, mapper)
    out["map_step_data"] = ref.read_grid(gh, grid.geom.num_vertices)
    v = np.zeros(grid.data.size)
    ref.lib.ref_mapper_rms(mapper, orc._ptr(v), v.size)
    out["map_step_v"] = v
    out["map_step_stats"] = np.array([st.loss_photometric, st.loss_geometric, st.loss_total,
                                      st.rays_color, st.rays_depth, st.psnr_estimate])
    ref.lib.ref_mapper_destroy(mapper)
    ref.lib.ref_grid_destroy(gh)
    ref.lib.ref_frames_destroy(fh)
    # tracking on the original grid
    gh = ref.grid(grid)
    fh = ref.frames([frames[1]], intr)
    px = np.stack([rng.integers(0, intr.width, 80), rng.integers(0, intr.height, 80)], 1)
    out["pose_pixels"] = px
    pose = synth.Pose(poses[1].q, tuple(np.asarray(poses[1].t) + [0.02, -0.01, 0.015]))
    out["pose_eval"] = np.array([*pose.q, *pose.t])
    g = ref.pose_gradient(gh, fh, intr, pose, px, 1.0, 1.0, RenderParams())
    out["pose_grad"] = np.array([*g.d_omega, *g.d_tau, g.loss, g.rays_used])
    ne = ref.normal_eqs(gh, fh, intr, pose, px, 1.0, 0.5, RenderParams())
    out["normal_jtj"], out["normal_jtr"] = np.array(ne.jtj), np.array(ne.jtr)
    out["normal_misc"] = np.array([ne.loss, ne.rays_used])
    tc = TrackingConfig(rays_per_iteration=48, iterations=5)
    tr, trace = ref.track_frame(gh, fh, intr, pose, tc)
    out["track_pose"] = np.array([*tr.pose.q, *tr.pose.t, tr.failed, tr.iterations_run])
    out["track_trace"] = trace
    ref.lib.ref_grid_destroy(gh)
    ref.lib.ref_frames_destroy(fh)
    np.savez_compressed(Path(__file__).with_name("voxrf_golden.npz"), **out)
    print("wrote", Path(__file__).with_name("voxrf_golden.npz"))


if __name__ == "__main__":
    main()
