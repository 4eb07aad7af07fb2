"""Deterministic small scenes shared by the parity tests (inputs only).

Target frames are rendered by the CPU oracle so the non-GPU tests can use the
same scenes as the GPU parity tests."""
from __future__ import annotations

import functools

import numpy as np

from paper_2307_03404_b200.api import (CameraIntrinsics, Frame, GridGeometry, MappingConfig,
                                       RenderParams, TrackingConfig, VoxelGrid)
from paper_2307_03404_b200 import synth


@functools.lru_cache(maxsize=None)
def room_scene(res: int = 17, width: int = 32, height: int = 24, n_frames: int = 3):
    """Voxelised primitive room + oracle-rendered, quantised RGB-D keyframes."""
    import oracle as orc

    grid = synth.scene_grid(res, seed=2, prune_tau=1e-3)
    f = 0.86 * width
    intr = CameraIntrinsics(f, f, width / 2.0, height / 2.0, width, height, 1000.0)
    room = synth.Room()
    poses = synth.circle_trajectory(n_frames, (2.0, 2.0, 0.0), 0.8, 1.5, (2.0, 3.5, 1.5),
                                    arc_deg=9.0)
    o = orc.Oracle()
    frames = []
    for p in poses:
        c, d = o.render_image(grid, intr, p, RenderParams())
        c, d = synth.quantize_frame(c, d, intr.depth_scale)
        frames.append(Frame(c, d, 0.0, p))
    return grid, intr, frames


def fresh_grid(grid: VoxelGrid, sigma_init=0.1, seed=3, sh_noise=0.05) -> VoxelGrid:
    """A grid to optimise: same geometry/occupancy, sigma_init + small SH noise (fp32-exact)."""
    rng = np.random.default_rng(seed)
    g = VoxelGrid(grid.geom, sigma_init)
    g.active[:] = grid.active
    g.data[:, 1:] = rng.uniform(-sh_noise, sh_noise, g.data[:, 1:].shape)
    g.data[:] = g.data.astype(np.float32).astype(np.float64)
    return g


def random_rays(grid: VoxelGrid, n: int, seed: int = 5, spread: float = 0.6):
    """Rays from around the grid centre in random unit directions."""
    rng = np.random.default_rng(seed)
    lo, hi = grid.geom.world_min(), grid.geom.world_max()
    c = 0.5 * (lo + hi)
    o = c + rng.uniform(-spread, spread, (n, 3)) * (hi - lo) * 0.5
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.concatenate([o, d], axis=1)
