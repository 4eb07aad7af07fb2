#!/usr/bin/env python
"""Diagnostic (r02): lane balance of the thread-per-ray kernels K0 / K2 at config 3.

A warp of K0/K2 runs as long as its longest ray; lanes whose ray has ended idle.
This takes the bench's map after its warm-up steps, draws the next 1M-ray
batch, renders those rays (vrf_debug_render_rays: the composited-sample count
of each ray), orders them as k_ray_keys does (keyframe, Morton order of 4x4
tiles; stable), and reports sum(count) / sum(32 * max(count) per warp), the
fraction of lane-steps that do work, for warps of 32 consecutive rays.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2307_03404_b200 import Context, Rng  # noqa: E402
from paper_2307_03404_b200.api import MappingConfig, RenderParams  # noqa: E402


def spread(x):
    x = x.astype(np.uint32) & 0x3FF
    x = (x | (x << 16)) & 0x030000FF
    x = (x | (x << 8)) & 0x0300F00F
    x = (x | (x << 4)) & 0x030C30C3
    x = (x | (x << 2)) & 0x09249249
    return x


def main():
    sys.argv = [sys.argv[0]]
    args = bench.parse()
    room, gt, intr, path = bench.make_scene(args)
    keyposes = path[::10][:10]
    g = Context(0)
    g.load_grid(gt)
    frames = bench.render_frames(g, intr, keyposes)
    del g
    ctx = Context(0)
    ctx.init_grid(gt.geom, 0.1)
    ctx.load_frames(intr, frames)
    ctx.rmsprop_reset()
    cfg = MappingConfig()
    rng = Rng(1)
    for _ in range(3):
        ctx.mapping_step(cfg, rng.draw_batch(len(frames), intr.width, intr.height, args.rays))
    b = rng.draw_batch(len(frames), intr.width, intr.height, args.rays).astype(np.int64)
    f, px, py = b[:, 0], b[:, 1], b[:, 2]
    cam = np.stack([(px - intr.cx) / intr.fx, (py - intr.cy) / intr.fy, np.ones(len(b))], 1)
    cam /= np.linalg.norm(cam, axis=1, keepdims=True)
    d = np.empty_like(cam)
    o = np.empty_like(cam)
    for k, p in enumerate(keyposes):
        sel = f == k
        d[sel] = cam[sel] @ p.rotation().T
        o[sel] = np.asarray(p.t)
    out = ctx.render_rays(np.concatenate([o, d], 1), RenderParams())
    cnt = out[:, 5]
    key = (f.astype(np.uint64) << 20) | spread(px >> 2).astype(np.uint64) | \
        (spread(py >> 2).astype(np.uint64) << 1)
    order = np.argsort(key, kind="stable")
    c = cnt[order]
    n = len(c) // 32 * 32
    w = c[:n].reshape(-1, 32)
    eff = w.sum() / (32 * w.max(1)).sum()
    ww = c[: len(c) // 128 * 128].reshape(-1, 128)
    print(f"samples/ray mean {cnt.mean():.1f} p10 {np.percentile(cnt, 10):.0f} "
          f"p90 {np.percentile(cnt, 90):.0f} max {cnt.max():.0f}")
    print(f"warp lane efficiency (32 consecutive rays): {eff:.3f}")
    print(f"CTA efficiency (128 rays, longest ray): {ww.sum() / (128 * ww.max(1)).sum():.3f}")
    # if each warp took its rays from a 4-warp pool (lanes refill as rays end)
    pool = c[: len(c) // 128 * 128].reshape(-1, 128)
    print(f"pooled-refill bound (128-ray pools, 32 lanes): "
          f"{pool.sum() / (32 * np.maximum(pool.sum(1) / 32, pool.max(1))).sum():.3f}")
    uw = 1.0 - eff
    print(f"idle lane-steps in the walk: {uw:.3f}")


if __name__ == "__main__":
    main()
