#!/usr/bin/env python
"""Tracking-only timing (config 2: 1200x680 frames of the fixed 257^3 room map,
Gauss-Newton 16384 rays x 10 iterations). Used for ncu captures of k_pose_fused."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2307_03404_b200 import Context, GNConfig, synth  # noqa: E402
from paper_2307_03404_b200.api import Frame  # noqa: E402


def main(frames=6, rays=16384, iters=10):
    room = synth.Room().scaled(7.0 / 4.0, 6.0 / 4.0, 1.0)
    gt = synth.scene_grid(257, room, seed=2, prune_tau=1e-3)
    intr = synth.replica_intrinsics()
    path = synth.room_path(frames + 1, room, seed=4)
    ctx = Context(0)
    ctx.load_grid(gt)
    fr = []
    for p in path:
        img = ctx.render_image(intr, p)
        c, d = synth.quantize_frame(img.color, img.depth, intr.depth_scale)
        fr.append(Frame(c, d, 0.0, p))
    ctx.load_frames(intr, fr)
    cfg = GNConfig(rays_per_iteration=rays, iterations=iters)
    ctx.track_frame_gn(1, intr, path[0], cfg)
    t0 = time.perf_counter()
    prev = path[0]
    err = []
    for i in range(1, len(fr)):
        r = ctx.track_frame_gn(i, intr, prev, cfg)
        prev = r.pose
        err.append(np.linalg.norm(np.asarray(r.pose.t) - np.asarray(path[i].t)))
    dt = (time.perf_counter() - t0) / (len(fr) - 1)
    print(f"GN tracking: {1e3 * dt:.2f} ms/frame ({1 / dt:.1f} fps), max err {max(err):.2e} m")


if __name__ == "__main__":
    main()
