#!/usr/bin/env python
"""BASELINE.json configs 1 and 2, GPU beside the reference CPU build (oracle/_ref).

Config 1 (64^3 cells, 160x120, 10 frames, mapping + tracking — the config the
CPU reference runs in full): map_scene with keyframe_stride 1, 4096 rays x 500
iterations, no upsampling, explicit 65^3 geometry; then
track_sequence (Adam defaults: 2048 rays x 40 iterations, previous-pose init)
on the mapped grid. GPU and CPU each run the reference-named API; both tracking
runs use the same (GPU-mapped) grid so the trajectories are comparable.

Config 2 (257^3 map, 1200x680, tracking only): the reference's track_sequence
on a short prefix (all host cores) beside the GPU Adam path (same algorithm,
same pixel stream) and the GPU Gauss-Newton tracker.

Prints one JSON line per config. Needs oracle/_ref (built here, travels to the
GPU box as a prebuilt .so).
"""
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import oracle as orc  # noqa: E402
from paper_2307_03404_b200 import Context, GNConfig, MappingConfig, TrackingConfig, synth  # noqa: E402
from paper_2307_03404_b200 import api  # noqa: E402
from paper_2307_03404_b200.api import Frame, GridGeometry, Pose  # noqa: E402
from paper_2307_03404_b200.metrics import ate_rmse, rotation_angle_rad  # noqa: E402


def render_frames(ctx, intr, poses, fps=30.0):
    out = []
    for i, p in enumerate(poses):
        img = ctx.render_image(intr, p)
        c, d = synth.quantize_frame(img.color, img.depth, intr.depth_scale)
        out.append(Frame(c, d, i / fps, p))
    return out


def traj_diff(a, b):
    dt = max(float(np.linalg.norm(np.asarray(x.t) - np.asarray(y.t))) for x, y in zip(a, b))
    dr = max(math.degrees(rotation_angle_rad(api.pose_compose(api.pose_inverse(x), y).q))
             for x, y in zip(a, b))
    return dt, dr


def config1(ref, cores):
    room = synth.Room()
    gt = synth.scene_grid(65, room, seed=2, prune_tau=1e-3)
    intr = synth.small_intrinsics()
    poses = synth.circle_trajectory(10, (2.0, 2.0, 0.0), 0.8, 1.5, (2.0, 3.5, 1.5), arc_deg=9.0)
    sensor = Context(0)
    sensor.load_grid(gt)
    frames = render_frames(sensor, intr, poses)
    ts = [f.timestamp for f in frames]
    geom = GridGeometry((65, 65, 65), (-0.2, -0.2, -0.7), 4.4 / 64)
    mcfg = MappingConfig(keyframe_stride=1, rays_per_batch=4096, iterations_per_stage=500,
                         upsample_stages=0, sigma_init=0.1, seed=1)
    ctx = Context(0)
    api.map_scene(frames, intr, MappingConfig(**{**mcfg.__dict__, "iterations_per_stage": 5}),
                  geom, ctx=ctx)  # warm-up (allocations)
    t0 = time.perf_counter()
    grid_gpu, log = api.map_scene(frames, intr, mcfg, geom, ctx=ctx)
    gpu_map_s = time.perf_counter() - t0
    fh = ref.frames(frames, intr)
    h, cpu_loss, cpu_map_ms = ref.map_scene(fh, intr, mcfg, geom, threads=cores)
    ref.lib.ref_grid_destroy(h)
    # tracking on the GPU-mapped grid, both sides
    tcfg = TrackingConfig()
    api._DEFAULT = ctx
    t0 = time.perf_counter()
    gpu_poses, _ = api.track_sequence(grid_gpu, frames, intr, tcfg)
    gpu_track_s = time.perf_counter() - t0
    gh = ref.grid(grid_gpu)
    cpu_p, cpu_track_ms = ref.track_sequence(gh, fh, intr, tcfg, len(frames), threads=cores)
    ref.lib.ref_grid_destroy(gh)
    ref.lib.ref_frames_destroy(fh)
    cpu_poses = [Pose(q, t) for q, t in cpu_p]
    dt, dr = traj_diff(gpu_poses, cpu_poses)
    gt_poses = [f.gt_pose for f in frames]
    return {
        "config": "config1: 65^3-vertex grid, 160x120, 10 frames, map_scene 500 x 4096 rays "
                  "(keyframe_stride 1) + track_sequence (Adam 2048 x 40)",
        "mapping": {"gpu_s": gpu_map_s, "cpu_s": cpu_map_ms / 1e3, "cpu_cores": cores,
                    "speedup": cpu_map_ms / 1e3 / gpu_map_s,
                    "final_loss_gpu": log[-1][1].loss_total, "final_loss_cpu": cpu_loss,
                    "gpu_steps_per_s": len(log) / gpu_map_s},
        "tracking": {"gpu_frames_per_s": (len(frames) - 1) / gpu_track_s,
                     "cpu_frames_per_s": (len(frames) - 1) / (cpu_track_ms / 1e3),
                     "cpu_cores": cores,
                     "gpu_vs_cpu_max_dt_m": dt, "gpu_vs_cpu_max_drot_deg": dr,
                     "ate_gpu_m": ate_rmse(gpu_poses, ts, gt_poses, ts)[0],
                     "ate_cpu_m": ate_rmse(cpu_poses, ts, gt_poses, ts)[0]},
    }


def config2(ref, cores, n_frames=4):
    room = synth.Room().scaled(7.0 / 4.0, 6.0 / 4.0, 1.0)
    gt = synth.scene_grid(257, room, seed=2, prune_tau=1e-3)
    intr = synth.replica_intrinsics()
    poses = synth.room_path(n_frames, room, seed=4)
    ctx = Context(0)
    ctx.load_grid(gt)
    frames = render_frames(ctx, intr, poses)
    ts = [f.timestamp for f in frames]
    tcfg = TrackingConfig()
    # grid and frames resident first (the reference's track_sequence also starts
    # from an in-memory grid); the timed loop is track_sequence's own
    # (tracking.cpp:268-292: previous-pose init, per-frame seed)
    ctx.load_frames(intr, frames)
    ctx.track_frame(1, intr, poses[0], tcfg)  # warm-up
    t0 = time.perf_counter()
    gpu_poses = [poses[0]]
    for i in range(1, n_frames):
        fc = TrackingConfig(**{**tcfg.__dict__})
        fc.seed = (tcfg.seed + 0x9E3779B9 * i) & (2**64 - 1)
        r = ctx.track_frame(i, intr, gpu_poses[-1], fc)
        gpu_poses.append(r.pose if not r.failed else gpu_poses[-1])
    gpu_s = time.perf_counter() - t0
    gn = GNConfig(rays_per_iteration=16384, iterations=10)
    ctx.track_frame_gn(1, intr, poses[0], gn)
    t0 = time.perf_counter()
    prev = poses[0]
    gn_poses = [poses[0]]
    for i in range(1, n_frames):
        prev = ctx.track_frame_gn(i, intr, prev, gn).pose
        gn_poses.append(prev)
    gn_s = time.perf_counter() - t0
    fh = ref.frames(frames, intr)
    gh = ref.grid(gt)
    # render_image (A20) at 1200x680 on the same map: GPU vs the reference's own
    ctx.render_image(intr, poses[0])
    t0 = time.perf_counter()
    for pz in poses:
        gimg = ctx.render_image(intr, pz)
    gpu_render_s = (time.perf_counter() - t0) / len(poses)
    t0 = time.perf_counter()
    rc, rd = ref.render_image(gh, intr, poses[-1], api.RenderParams(), 1, cores)
    cpu_render_s = time.perf_counter() - t0
    render_diff = float(np.max(np.abs(gimg.depth - rd)))
    cpu_p, cpu_ms = ref.track_sequence(gh, fh, intr, tcfg, n_frames, threads=cores)
    ref.lib.ref_grid_destroy(gh)
    ref.lib.ref_frames_destroy(fh)
    cpu_poses = [Pose(q, t) for q, t in cpu_p]
    dt, dr = traj_diff(gpu_poses, cpu_poses)
    return {
        "config": f"config2: 257^3 room map, 1200x680, tracking only, {n_frames - 1} tracked frames",
        "adam_2048x40": {"gpu_frames_per_s": (n_frames - 1) / gpu_s,
                         "cpu_frames_per_s": (n_frames - 1) / (cpu_ms / 1e3), "cpu_cores": cores,
                         "gpu_vs_cpu_max_dt_m": dt, "gpu_vs_cpu_max_drot_deg": dr},
        "gn_16384x10": {"gpu_frames_per_s": (n_frames - 1) / gn_s,
                        "ate_vs_gt_m": ate_rmse(gn_poses, ts, poses, ts, align=False)[0]},
        "render_image_1200x680": {"gpu_ms": 1e3 * gpu_render_s, "cpu_ms": 1e3 * cpu_render_s,
                                  "cpu_cores": cores, "max_depth_diff_m": render_diff},
    }


def main():
    cores = os.cpu_count() or 1
    ref = orc.RefLib()
    which = sys.argv[1:] or ["1", "2"]
    if "1" in which:
        print(json.dumps(config1(ref, cores)), flush=True)
    if "2" in which:
        print(json.dumps(config2(ref, cores)), flush=True)


if __name__ == "__main__":
    main()
