#!/usr/bin/env python
"""Diagnose SLAM bootstrap: map one frame, then score the map and track frame 1."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2307_03404_b200 import Context, GNConfig, MappingConfig, Rng, synth  # noqa: E402
from paper_2307_03404_b200.api import Frame  # noqa: E402


def main(steps=1000, rays=65536, sigma_init=0.1, lr_sigma=30.0):
    room = synth.Room().scaled(7.0 / 4.0, 6.0 / 4.0, 1.0)
    gt = synth.scene_grid(257, room, seed=2, prune_tau=1e-3)
    intr = synth.replica_intrinsics()
    poses, ts = synth.ellipse_trajectory(2000, room)
    sensor = Context(0)
    sensor.load_grid(gt)
    fr = []
    for i in range(3):
        img = sensor.render_image(intr, poses[i])
        c, d = synth.quantize_frame(img.color, img.depth, intr.depth_scale)
        fr.append(Frame(c, d, ts[i], poses[i]))
    print("valid depth frac", float((fr[0].depth > 0).mean()), "depth range",
          float(fr[0].depth[fr[0].depth > 0].min()), float(fr[0].depth.max()))
    ctx = Context(0)
    ctx.init_grid(gt.geom, sigma_init)
    ctx.load_frames(intr, fr[:1])
    cfg = MappingConfig(rays_per_batch=rays, sigma_init=sigma_init, lr_sigma=lr_sigma)
    rng = Rng(1)
    for k in range(0, steps, 100):
        st = ctx.mapping_steps(cfg, rng, 1, 100)
        print(f"step {k + 100}: Lp {st[-1].loss_photometric:.4g} Lg {st[-1].loss_geometric:.4g} "
              f"samples/ray {st[-1].samples / max(1, st[-1].rays_color):.1f}")
    for i in range(3):
        r = ctx.render_image(intr, poses[i])
        ok = fr[i].depth > 0
        print(f"view {i}: color mse {np.mean((r.color - fr[i].color) ** 2):.4g} "
              f"depth L1 {np.mean(np.abs(r.depth[ok] - fr[i].depth[ok])):.4g}")
    ctx.load_frames(intr, fr)
    for init_name, init in (("gt", poses[1]), ("prev", poses[0])):
        res = ctx.track_frame_gn(1, intr, init, GNConfig())
        e = np.linalg.norm(np.asarray(res.pose.t) - np.asarray(poses[1].t))
        print(f"track frame 1 from {init_name}: err {e:.4f} m, loss {res.loss_trace[-1]:.4g}")
    # the same on the ground-truth map
    sensor.load_frames(intr, fr)
    res = sensor.track_frame_gn(1, intr, poses[0], GNConfig())
    print("gt map: err", np.linalg.norm(np.asarray(res.pose.t) - np.asarray(poses[1].t)))


def slam_check(steps=1000):
    from paper_2307_03404_b200.slam import SlamConfig, SlamSystem
    room = synth.Room().scaled(7.0 / 4.0, 6.0 / 4.0, 1.0)
    gt = synth.scene_grid(257, room, seed=2, prune_tau=1e-3)
    intr = synth.replica_intrinsics()
    poses, ts = synth.ellipse_trajectory(2000, room)
    sensor = Context(0)
    sensor.load_grid(gt)
    fr = []
    for i in range(3):
        img = sensor.render_image(intr, poses[i])
        c, d = synth.quantize_frame(img.color, img.depth, intr.depth_scale)
        fr.append(Frame(c, d, ts[i], poses[i]))
    ctx = Context(0)
    s = SlamSystem(ctx, intr, gt.geom, SlamConfig(bootstrap_steps=steps, max_keyframes=8))
    s.process(fr[0])
    r = ctx.render_image(intr, poses[0])
    ok = fr[0].depth > 0
    print(f"slam view 0: color mse {np.mean((r.color - fr[0].color) ** 2):.4g} "
          f"depth L1 {np.mean(np.abs(r.depth[ok] - fr[0].depth[ok])):.4g}")
    p = s.process(fr[1])
    print("slam frame 1 err", np.linalg.norm(np.asarray(p.t) - np.asarray(poses[1].t)))


if __name__ == "__main__":
    if sys.argv[1:2] == ["slam"]:
        slam_check(int(sys.argv[2]) if len(sys.argv) > 2 else 1000)
        sys.exit(0)
    kw = {}
    for a in sys.argv[1:]:
        k, v = a.split("=")
        kw[k] = type({"steps": 1, "rays": 1, "sigma_init": 1.0, "lr_sigma": 1.0}[k])(v)
    main(**kw)
