"""Golden vectors generated from the reference itself (tests/golden/make_golden.py,
oracle/_ref = the reference sources compiled unchanged). The C oracle must
reproduce them bit for bit (CPU, runs anywhere); the GPU path within the parity
tolerances (gpu marker)."""
from pathlib import Path

import numpy as np
import pytest

from paper_2307_03404_b200.api import (CameraIntrinsics, Frame, GridGeometry, MappingConfig, Pose,
                                       RenderParams, TrackingConfig, VoxelGrid)

G = np.load(Path(__file__).with_name("golden") / "voxrf_golden.npz")


def scene():
    gm = G["geom"]
    geom = GridGeometry(tuple(int(x) for x in gm[:3]), tuple(gm[3:6]), float(gm[6]))
    grid = VoxelGrid.__new__(VoxelGrid)
    grid.geom, grid.data, grid.active = geom, G["grid_data"].copy(), G["grid_active"].copy()
    i = G["intr"]
    intr = CameraIntrinsics(i[0], i[1], i[2], i[3], int(i[4]), int(i[5]), i[6])
    poses = [Pose(tuple(p[:4]), tuple(p[4:])) for p in G["poses"]]
    frames = [Frame(G[f"frame_color_{k}"], G[f"frame_depth_{k}"], 0.0, poses[k])
              for k in range(len(poses))]
    return grid, intr, poses, frames


def test_oracle_render_matches_golden(oracle):
    grid, intr, poses, _ = scene()
    for k, p in enumerate(poses):
        c, d = oracle.render_image(grid, intr, p, RenderParams())
        assert np.array_equal(c, G[f"render_color_{k}"]) and np.array_equal(d, G[f"render_depth_{k}"])
    c, d = oracle.render_image(grid, intr, poses[1], RenderParams(), 3)
    assert np.array_equal(c, G["render_color_stride3"]) and np.array_equal(d, G["render_depth_stride3"])


def test_oracle_schedules_match_golden(oracle):
    grid, *_ = scene()
    for r, n, t, dl in zip(G["rays"], G["sched_count"], G["sched_t"], G["sched_delta"]):
        tt, dd, _ = oracle.sample_ray(grid, r[:3], r[3:], RenderParams())
        assert len(tt) == n and np.array_equal(tt, t[:n]) and np.array_equal(dd, dl[:n])


def test_oracle_mapping_matches_golden(oracle):
    grid, intr, _, frames = scene()
    cfg = MappingConfig()
    _, _, grad, st = oracle.mapping_step(grid, frames, intr, cfg, G["map_batch"], apply=False,
                                         want_grad=True)
    assert st.samples == G["map_samples"][0]
    assert np.array_equal(grad, G["map_grad"])
    data, v, _, st = oracle.mapping_step(grid, frames, intr, cfg, G["map_batch"])
    assert np.array_equal(data, G["map_step_data"])
    assert np.array_equal(v.reshape(-1), G["map_step_v"])
    s = G["map_step_stats"]
    assert [st.loss_photometric, st.loss_geometric, st.loss_total, st.rays_color, st.rays_depth,
            st.psnr_estimate] == list(s)


def test_oracle_tracking_matches_golden(oracle):
    grid, intr, _, frames = scene()
    pe = G["pose_eval"]
    pose = Pose(tuple(pe[:4]), tuple(pe[4:]))
    g = oracle.pose_gradient(grid, frames[1], intr, pose, G["pose_pixels"], 1.0, 1.0,
                             RenderParams())
    assert [*g.d_omega, *g.d_tau, g.loss, g.rays_used] == list(G["pose_grad"])
    ne = oracle.normal_eqs(grid, frames[1], intr, pose, G["pose_pixels"], 1.0, 0.5, RenderParams())
    np.testing.assert_allclose(ne.jtj, G["normal_jtj"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(ne.jtr, G["normal_jtr"], rtol=1e-12, atol=1e-15)
    tr, trace = oracle.track_frame(grid, frames[1], intr, pose,
                                   TrackingConfig(rays_per_iteration=48, iterations=5))
    assert [*tr.pose.q, *tr.pose.t, tr.failed, tr.iterations_run] == list(G["track_pose"])
    assert np.array_equal(trace, G["track_trace"])


@pytest.mark.gpu
def test_gpu_matches_golden(ctx):
    grid, intr, poses, frames = scene()
    ctx.load_grid(grid)
    for k, p in enumerate(poses):
        img = ctx.render_image(intr, p)
        np.testing.assert_allclose(img.color, G[f"render_color_{k}"], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(img.depth, G[f"render_depth_{k}"], rtol=1e-10, atol=1e-12)
    counts, t, delta, _ = ctx.sample_rays(G["rays"], cap=64)
    assert np.array_equal(counts, G["sched_count"])
    for i, n in enumerate(counts):
        assert np.array_equal(t[i, :n], G["sched_t"][i, :n])
    ctx.load_frames(intr, frames)
    grad, st = ctx.mapping_gradient(MappingConfig(deterministic=True), G["map_batch"])
    assert st.samples == G["map_samples"][0]
    scale = np.abs(G["map_grad"]).max()
    np.testing.assert_allclose(grad, G["map_grad"], rtol=1e-9, atol=1e-12 * scale)
    ctx.rmsprop_reset()
    ctx.mapping_step(MappingConfig(deterministic=True), G["map_batch"])
    d = ctx.download_grid().data
    ref = G["map_step_data"]
    np.testing.assert_allclose(d, ref, rtol=2e-6, atol=2e-6 * np.abs(ref).max())
    ctx.load_grid(grid)
    pe = G["pose_eval"]
    g = ctx.pose_gradient(1, intr, Pose(tuple(pe[:4]), tuple(pe[4:])), G["pose_pixels"],
                          TrackingConfig())
    ref = G["pose_grad"]
    got = np.array([*g.d_omega, *g.d_tau])
    np.testing.assert_allclose(got, ref[:6], rtol=1e-7, atol=1e-10 * np.abs(ref[:6]).max())
    assert g.rays_used == ref[7]
