"""The interleaved SLAM driver (slam.py) on a small room: frame slots, keyframe
mapping and GN tracking composed on one context."""
import numpy as np
import pytest

from paper_2307_03404_b200 import Context, GNConfig, MappingConfig, synth
from paper_2307_03404_b200.api import Frame, GridGeometry
from paper_2307_03404_b200 import metrics
from paper_2307_03404_b200.slam import SlamConfig, SlamSystem

pytestmark = pytest.mark.gpu


def _scene(n_frames):
    room = synth.Room()
    gt = synth.scene_grid(65, room, seed=2, prune_tau=1e-3)
    intr = synth.small_intrinsics()
    poses, ts = synth.ellipse_trajectory(400, room)
    sensor = Context(0)
    sensor.load_grid(gt)
    frames = []
    for i in range(n_frames):
        img = sensor.render_image(intr, poses[i])
        c, d = synth.quantize_frame(img.color, img.depth, intr.depth_scale)
        frames.append(Frame(c, d, ts[i], poses[i]))
    return gt, intr, frames, poses[:n_frames], ts[:n_frames]


def test_slam_on_the_ground_truth_map_holds_the_trajectory():
    gt, intr, frames, poses, ts = _scene(12)
    cfg = SlamConfig(keyframe_stride=5, map_steps=0, bootstrap_steps=0, max_keyframes=8,
                     tracking=GNConfig(rays_per_iteration=4096, iterations=8))
    ctx = Context(0)
    slam = SlamSystem(ctx, intr, GridGeometry(gt.geom.res, gt.geom.origin, gt.geom.voxel_size),
                      cfg)
    ctx.load_grid(gt)  # plumbing check: track against the map the frames came from
    for f in frames:
        slam.process(f)
    ate, _ = metrics.ate_rmse(slam.poses, ts, poses, ts, align=False)
    assert ate < 1e-3
    assert slam.n_keyframes == 3 and ctx.n_frames == cfg.max_keyframes + 1


def test_slam_maps_and_tracks_online():
    gt, intr, frames, poses, ts = _scene(8)
    cfg = SlamConfig(keyframe_stride=4, map_steps=20, bootstrap_steps=300, max_keyframes=4,
                     tracking=GNConfig(rays_per_iteration=4096, iterations=6, lambda_d=0.1),
                     mapping=MappingConfig(rays_per_batch=4096))
    ctx = Context(0)
    slam = SlamSystem(ctx, intr, GridGeometry(gt.geom.res, gt.geom.origin, gt.geom.voxel_size),
                      cfg)
    for f in frames:
        slam.process(f)
    assert len(slam.poses) == 8 and slam.n_keyframes == 2
    assert all(np.all(np.isfinite(p.t)) for p in slam.poses)
    # the bootstrap map renders the first view far better than the sigma_init fog
    q = metrics.evaluate_map_quality(ctx, intr, frames, [0], images=1, pixels_per_image=2000)
    assert q.psnr_db > 14.0
