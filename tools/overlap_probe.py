#!/usr/bin/env python
"""Probe (r02): would K0 of one batch overlap usefully with K2 of another?

Two contexts on one GPU, each on its own torch stream, hold the config-3 map
after a few mapping steps. Times, with CUDA events / wall clock around a
device synchronize:
  seq : ctx A's backward (K2) then ctx B's forward (K0), one after the other;
  conc: the same two calls issued from two host threads at once.
If conc is well below seq, a pipelined step (K2 of chunk j beside K0 of chunk
j+1, hit counts from a pre-pass) would pay; if not, K0 and K2 compete for the
same SM resources (L1 / shared-memory data pipe).
usage: python tools/overlap_probe.py [--rays N]
"""
import argparse
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_03404_b200 import Context, Rng  # noqa: E402
from paper_2307_03404_b200.api import MappingConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rays", type=int, default=1 << 20)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    sys.argv = [sys.argv[0]]
    args = bench.parse()
    room, gt, intr, path = bench.make_scene(args)
    keyposes = path[::10][:10]
    gt_ctx = Context(0)
    gt_ctx.load_grid(gt)
    frames = bench.render_frames(gt_ctx, intr, keyposes)
    del gt_ctx
    cfg = MappingConfig()
    rng = Rng(1)
    batches = [torch.from_numpy(rng.draw_batch(len(frames), intr.width, intr.height, a.rays))
               .cuda() for _ in range(4)]
    ctxs, streams = [], []
    for k in range(2):
        s = torch.cuda.Stream()
        c = Context(0)
        c.set_stream(s.cuda_stream)
        c.init_grid(gt.geom, 0.1)
        c.load_frames(intr, frames)
        c.rmsprop_reset()
        for i in range(3):
            c.mapping_step_device(cfg, batches[i].data_ptr(), a.rays)
        ctxs.append(c)
        streams.append(s)
    torch.cuda.synchronize()
    A, B = ctxs
    bt = batches[3]

    def fwd(c):
        return c.map_forward(cfg, bt.data_ptr(), a.rays)

    pa = fwd(A)
    rc, rd = pa.rays_color, pa.rays_depth

    def bwd():
        A.map_backward(cfg, rc, rd)

    def f_b():
        fwd(B)

    def timed(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return 1e3 * (time.perf_counter() - t0)

    res = {"bwd": [], "fwd": [], "seq": [], "conc": []}
    for _ in range(a.reps):
        fwd(A)  # fresh records for A
        res["bwd"].append(timed(bwd))
        res["fwd"].append(timed(f_b))
        fwd(A)
        res["seq"].append(timed(lambda: (bwd(), f_b())))
        fwd(A)

        def both():
            th = threading.Thread(target=bwd)
            th.start()
            f_b()
            th.join()
        res["conc"].append(timed(both))
    for k, v in res.items():
        v = sorted(v)
        print(f"{k}: median {v[len(v) // 2]:.3f} ms  min {v[0]:.3f}")


if __name__ == "__main__":
    main()
