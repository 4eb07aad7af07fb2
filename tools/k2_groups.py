#!/usr/bin/env python
"""Diagnostic (r02): K2's same-round duplicate groups at config 3.

Needs the VRF_K2_GSTATS build:
  python tools/ab/build_variants.py gstats=VRF_K2_GSTATS=1
  VRF_LIB=tools/ab/_lib_gstats/libvoxrf_b200.so python tools/k2_groups.py
Runs the bench's map through 3 warm-up steps, then one 1M-ray step, and prints
the histogram of duplicate-group sizes (lanes popping the same vertex in one pop
round) and of each round's largest group, whose size - 1 is the merge loop's
trip count in that round.
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2307_03404_b200 import Context, Rng, _capi  # noqa: E402
from paper_2307_03404_b200.api import MappingConfig  # noqa: E402


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
    cfg = MappingConfig(rays_per_batch=args.rays)
    lib = _capi.load()
    rd = lib.vrf_debug_k2_hist
    rd.argtypes = [C.POINTER(C.c_uint64)]
    h = (C.c_uint64 * 66)()
    rng = Rng(1)
    ctx.mapping_steps(cfg, rng, len(frames), 3)
    rd(h)  # clear
    ctx.mapping_steps(cfg, rng, len(frames), 1)
    rd(h)
    gs = np.array(h[:33], dtype=np.float64)
    rm = np.array(h[33:], dtype=np.float64)
    k = np.arange(33)
    pops = (gs * k).sum()
    print(f"pops {pops:.4g}, groups {gs.sum():.4g} (reductions), rounds {rm.sum():.4g}")
    print("group size: share of pops  " +
          " ".join(f"{i}:{gs[i] * i / pops:.3f}" for i in range(1, 33) if gs[i]))
    print("largest group per round: share of rounds  " +
          " ".join(f"{i}:{rm[i] / rm.sum():.3f}" for i in range(1, 33) if rm[i]))
    trips = (rm[1:] * (k[1:] - 1)).sum()
    members = (gs[2:] * (k[2:] - 1)).sum()
    print(f"merge-loop trips {trips:.4g} (sum over rounds of max size - 1); "
          f"members merged {members:.4g}; lanes per trip {members / max(trips, 1):.2f}")
    print(f"rounds with a multi-lane group: {rm[2:].sum() / rm.sum():.3f}")


if __name__ == "__main__":
    main()
