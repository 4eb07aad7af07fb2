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


def _slam_worker(rank, world, port, out_dir):
    import os
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(__file__))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gt, intr, frames, poses, ts = _scene(8)
        cfg = SlamConfig(keyframe_stride=4, map_steps=10, bootstrap_steps=100, max_keyframes=4,
                         coarse_levels=1,  # also exercises the mapper rebuild after upsample
                         tracking=GNConfig(rays_per_iteration=4096, iterations=6, lambda_d=0.1),
                         mapping=MappingConfig(rays_per_batch=4096))
        ctx = Context(0, shard_multiple=world)
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        slam = SlamSystem(ctx, intr,
                          GridGeometry(gt.geom.res, gt.geom.origin, gt.geom.voxel_size), cfg,
                          distributed=True)
        for f in frames:
            slam.process(f)
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, f"poses{rank}.npy"),
                np.array([list(p.q) + list(p.t) for p in slam.poses]))
        np.save(os.path.join(out_dir, f"grid{rank}.npy"), ctx.download_grid().data)
    finally:
        dist.destroy_process_group()


def test_slam_distributed_replicas_agree(tmp_path):
    """Multi-GPU SLAM (slam.SlamSystem(distributed=True)): two ranks on one
    device (gloo host collectives, CUDA IPC peer table for the fused exchange).
    Keyframe mapping is ray-sharded, tracking runs as replicas: both ranks must
    hold the same map and the same trajectory."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(_slam_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    p0, p1 = (np.load(tmp_path / f"poses{r}.npy") for r in range(2))
    g0, g1 = (np.load(tmp_path / f"grid{r}.npy") for r in range(2))
    assert np.array_equal(g0, g1)
    assert np.array_equal(p0, p1)
    assert p0.shape == (8, 7) and np.all(np.isfinite(p0))
