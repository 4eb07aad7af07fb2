#!/usr/bin/env python
"""Per-ray composited-sample distribution of the tracking workload (config 2) on
the GPU (render_rays inspection entry point). Diagnostic only."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2307_03404_b200 import Context, synth  # noqa: E402
from paper_2307_03404_b200.api import RenderParams  # noqa: E402


def main():
    room = synth.Room().scaled(7.0 / 4.0, 6.0 / 4.0, 1.0)
    gt = synth.scene_grid(257, room, seed=2, prune_tau=1e-3)
    intr = synth.replica_intrinsics()
    pose = synth.room_path(100, room, seed=4)[1]
    ctx = Context(0)
    ctx.load_grid(gt)
    rng = np.random.default_rng(0)
    n = 16384
    px = rng.uniform(0, intr.width, n)
    py = rng.uniform(0, intr.height, n)
    cam = np.stack([(px - intr.cx) / intr.fx, (py - intr.cy) / intr.fy, np.ones(n)], 1)
    cam /= np.linalg.norm(cam, axis=1, keepdims=True)
    d = cam @ pose.rotation().T
    o = np.broadcast_to(np.asarray(pose.t), d.shape)
    out = ctx.render_rays(np.concatenate([o, d], 1), RenderParams())
    cnt = out[:, 5]
    counts, _, _, _ = ctx.sample_rays(np.concatenate([o, d], 1)[:2048], RenderParams(), cap=1)
    print("composited samples/ray: mean %.1f p50 %d p90 %d p99 %d max %d" %
          (cnt.mean(), np.percentile(cnt, 50), np.percentile(cnt, 90), np.percentile(cnt, 99),
           cnt.max()))
    print("active schedule segments/ray (no termination): mean %.1f max %d" %
          (counts.mean(), counts.max()))
    print("hit fraction %.3f, terminated %.3f" % (out[:, 6].mean(), out[:, 7].mean()))


if __name__ == "__main__":
    main()
