#!/usr/bin/env python
"""Config 5: interleaved SLAM on a closed-loop ellipse through the config-2 room.

Frames are rendered on demand from the ground-truth 257^3 room map in a second
context (the "sensor"; excluded from the timing), quantised like image.cpp, and
fed to the SLAM system one at a time. Prints one JSON line: frames/s, tracking
and mapping ms per frame, ATE (aligned / unaligned), RPE at 1 m, and map PSNR /
depth L1 on held-out views rendered from the SLAM map.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2307_03404_b200 import Context, GNConfig, MappingConfig, synth  # noqa: E402
from paper_2307_03404_b200.api import Frame, GridGeometry  # noqa: E402
from paper_2307_03404_b200 import metrics  # noqa: E402
from paper_2307_03404_b200.slam import SlamConfig, SlamSystem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=2000, help="frames processed")
    ap.add_argument("--loop", type=int, default=2000, help="frames in the closed loop")
    ap.add_argument("--res", type=int, default=257)
    ap.add_argument("--width", type=int, default=1200)
    ap.add_argument("--height", type=int, default=680)
    ap.add_argument("--stride", type=int, default=10)
    ap.add_argument("--map-steps", type=int, default=25)
    ap.add_argument("--map-rays", type=int, default=65536)
    ap.add_argument("--bootstrap", type=int, default=3000)
    ap.add_argument("--track-rays", type=int, default=16384)
    ap.add_argument("--track-iters", type=int, default=10)
    ap.add_argument("--sigma-init", type=float, default=0.1)
    ap.add_argument("--window", type=int, default=0, help="map over the last N keyframes")
    ap.add_argument("--coarse", type=int, default=0,
                    help="bootstrap coarse-to-fine: start at (res-1)/2^L+1, upsample L times")
    ap.add_argument("--recent", type=float, default=0.0,
                    help="share of each mapping batch drawn from the newest keyframe")
    ap.add_argument("--track-lambda-d", type=float, default=0.1,
                    help="tracking depth weight (r01 sweep: 1.0 drifts, 0.1 holds 2 cm ATE)")
    ap.add_argument("--trace", action="store_true", help="print per-frame position error")
    ap.add_argument("--gt-map", action="store_true",
                    help="plumbing check: track against the ground-truth map, no mapping")
    ap.add_argument("--out", default="")
    ap.add_argument("--distributed", action="store_true",
                    help="one process per GPU under torchrun: ray-sharded keyframe mapping "
                         "(fused peer-memory exchange), tracking replicas")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    distributed = args.distributed or world > 1
    if distributed:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")

    room = synth.Room().scaled(7.0 / 4.0, 6.0 / 4.0, 1.0)
    gt = synth.scene_grid(args.res, room, seed=2, prune_tau=1e-3)
    s = args.width / 1200.0
    intr = synth.CameraIntrinsics(600.0 * s, 600.0 * s, args.width / 2 - 0.5,
                                  args.height / 2 - 0.5, args.width, args.height, 6553.5)
    poses, ts = synth.ellipse_trajectory(args.loop, room)
    poses, ts = poses[:args.frames], ts[:args.frames]
    sensor = Context(local)
    sensor.load_grid(gt)

    def frame(i):
        img = sensor.render_image(intr, poses[i])
        return synth.sensor_frame(img.color, img.depth, intr.depth_scale, ts[i], poses[i])

    geom = GridGeometry(gt.geom.res, gt.geom.origin, gt.geom.voxel_size)
    cfg = SlamConfig(keyframe_stride=args.stride, map_steps=args.map_steps, window=args.window,
                     recent_fraction=args.recent, coarse_levels=args.coarse,
                     bootstrap_steps=args.bootstrap,
                     max_keyframes=(args.frames + args.stride - 1) // args.stride + 1,
                     tracking=GNConfig(rays_per_iteration=args.track_rays,
                                       iterations=args.track_iters,
                                       lambda_d=args.track_lambda_d),
                     mapping=MappingConfig(rays_per_batch=args.map_rays,
                                           sigma_init=args.sigma_init))
    if distributed:
        ctx = Context(local, shard_multiple=world)
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    else:
        ctx = Context(local)
    slam = SlamSystem(ctx, intr, geom, cfg, distributed=distributed)
    if args.gt_map:
        ctx.load_grid(gt)
        cfg.bootstrap_steps = cfg.map_steps = 0
    slam_s = 0.0
    gen_s = 0.0
    for i in range(args.frames):
        t0 = time.perf_counter()
        f = frame(i)
        t1 = time.perf_counter()
        slam.process(f)
        t2 = time.perf_counter()
        gen_s += t1 - t0
        if i > 0:
            slam_s += t2 - t1
        if args.trace and (i % 10 == 0 or i < 10):
            e = np.linalg.norm(np.asarray(slam.poses[-1].t) - np.asarray(poses[i].t))
            print(f"frame {i}: pos err {e:.4f} m, loss {slam.log[-1].final_loss:.4g}",
                  file=sys.stderr)
    est = slam.poses
    ate, pairs = metrics.ate_rmse(est, ts, poses, ts, align=True)
    ate_u, _ = metrics.ate_rmse(est, ts, poses, ts, align=False)
    try:
        r = metrics.rpe(est, ts, poses, ts, 1.0)
        rpe = {"rpe_t_m": r.rpe_t, "rpe_r_deg": r.rpe_r_deg, "pairs": r.pairs}
    except RuntimeError as e:
        rpe = {"error": str(e)}
    # map quality on views half-way between keyframes
    held = list(range(args.stride // 2, args.frames, max(1, args.frames // 10)))[:10]
    views = {i: frame(i) for i in held}
    q = metrics.evaluate_map_quality(ctx, intr, views, held, images=10, pixels_per_image=2000)
    logs = slam.log[1:]
    n = len(logs)
    out = {
        "config": f"config5: SLAM, {args.width}x{args.height}, {args.res}^3 grid, "
                  f"closed-loop ellipse of {args.loop} frames",
        "frames": args.frames, "keyframes": slam.n_keyframes,
        "mapping": ("ray-sharded over %d GPUs, %s exchange; tracking replicas" % (world, cfg.exchange))
        if distributed else "1 GPU",
        "frames_per_s": n / slam_s if slam_s > 0 else None,
        "track_ms_per_frame": float(np.mean([l.track_ms for l in logs])) if n else None,
        "map_ms_per_keyframe": float(np.mean([l.map_ms for l in logs if l.keyframe]))
        if any(l.keyframe for l in logs) else None,
        "bootstrap_ms": slam.log[0].map_ms,
        "ate_rmse_m": ate, "ate_unaligned_m": ate_u, "pose_pairs": pairs, **rpe,
        "psnr_db": q.psnr_db, "depth_l1_m": q.depth_l1_m,
        "settings": {"stride": args.stride, "map_steps": args.map_steps, "window": args.window,
                     "recent_fraction": args.recent, "coarse_levels": args.coarse,
                     "track_lambda_d": args.track_lambda_d,
                     "map_rays": args.map_rays, "bootstrap_steps": args.bootstrap,
                     "track": f"GN {args.track_rays} rays x {args.track_iters} it"},
        "sensor_render_s": gen_s,
    }
    out["n_gpus"] = world
    if distributed:
        dist.destroy_process_group()
    if rank != 0:
        return
    line = json.dumps(out)
    print(line)
    if args.out:
        Path(args.out).write_text(line + "\n")


if __name__ == "__main__":
    main()
