"""Interleaved SLAM driver (config 5).

The reference is offline only: map_scene with GT poses, then track_sequence
against the finished map. This driver composes the same two
hot paths online, the way the paper runs them: every frame is tracked against
the map being built (device Gauss-Newton, Context.track_frame_gn), and every
``keyframe_stride``-th frame joins the keyframe set at its *estimated* pose and
triggers ``map_steps`` mapping_step calls over all keyframes so far.

Device residency: the grid, its RMSProp state, the keyframes and the tracking
frame live in one Context (frame slots: 0..max_keyframes-1 keyframes, slot
max_keyframes the frame being tracked). Per frame the host uploads only that
frame (its RGB-D image, as a sensor would deliver it) and reads back a pose.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .api import (CameraIntrinsics, Context, Frame, GNConfig, GridGeometry, MappingConfig, Pose,
                  Rng, pose_compose, pose_inverse)


@dataclass
class SlamConfig:
    keyframe_stride: int = 10
    map_steps: int = 10                 # mapping_step calls per new keyframe
    bootstrap_steps: int = 200          # mapping_step calls on frame 0 before tracking
    max_keyframes: int = 256
    window: int = 0                     # map over the last `window` keyframes (0 = all)
    recent_fraction: float = 0.0        # share of each mapping batch drawn from the newest keyframe
    exchange: str = "p2p"               # multi-GPU mapping exchange (distributed=True)
    coarse_levels: int = 0              # bootstrap coarse-to-fine: start at (res-1)/2^L+1 and
                                        # upsample L times (voxel_grid.cpp:190-220) during it
    constant_velocity: bool = True      # track_sequence init policy (tracking.cpp:271-272)
    tracking: GNConfig = field(default_factory=GNConfig)
    mapping: MappingConfig = field(default_factory=lambda: MappingConfig(rays_per_batch=65536))


@dataclass
class SlamFrameLog:
    frame: int
    keyframe: bool
    track_ms: float
    map_ms: float
    final_loss: float


class SlamSystem:
    """Online tracking + keyframe mapping on one device context."""

    def __init__(self, ctx: Context, intrinsics: CameraIntrinsics, geometry: GridGeometry,
                 config: SlamConfig, distributed: bool = False):
        """distributed: one process per GPU (torch.distributed initialised, the
        context created with shard_multiple=world and running on torch's current
        stream). Every rank holds the whole grid and every keyframe and tracks
        every frame as a replica (the GN frame graph is deterministic and the maps
        are identical after each exchange, so the replicas agree without
        communication); each keyframe's mapping steps are ray-sharded: a rank draws
        rays_per_batch / world rays from its own stream and the gradients are
        combined by the mapper's exchange (default: the fused peer-memory kernel)."""
        self.ctx = ctx
        self.intr = intrinsics
        self.cfg = config
        self.distributed = distributed
        L = config.coarse_levels
        if L > 0:
            if any((int(r) - 1) % (1 << L) for r in geometry.res):
                raise ValueError("slam: coarse_levels needs (res - 1) divisible by 2^L")
            geometry = GridGeometry(tuple(((int(r) - 1) >> L) + 1 for r in geometry.res),
                                    geometry.origin, geometry.voxel_size * (1 << L))
        ctx.init_grid(geometry, config.mapping.sigma_init)
        ctx.reserve_frames(intrinsics, config.max_keyframes + 1)
        self.track_slot = config.max_keyframes
        self.n_keyframes = 0
        self.mapper = None
        rank = 0
        if distributed:
            import torch.distributed as dist
            from .distributed import DistributedMapper, GpuEngine
            ctx.rmsprop_reset()
            self.mapper = DistributedMapper(GpuEngine(ctx, config.mapping))
            rank = dist.get_rank()
        self.rng = Rng(config.mapping.seed + 7919 * rank)
        self.poses: List[Pose] = []
        self.log: List[SlamFrameLog] = []

    def _draw(self, n: int) -> np.ndarray:
        """One mapping batch of n rays under the keyframe policy (recent share,
        window, or uniform over all keyframes)."""
        w, h = self.intr.width, self.intr.height
        f = self.cfg.recent_fraction
        if f > 0.0 and self.n_keyframes > 1:
            n_new = int(round(f * n))
            a = self.rng.draw_batch(1, w, h, n_new)
            a[:, 0] = self.n_keyframes - 1
            b = self.rng.draw_batch(self.n_keyframes, w, h, n - n_new)
            return np.concatenate([a, b])
        if self.cfg.window <= 0 or self.cfg.window >= self.n_keyframes:
            return self.rng.draw_batch(self.n_keyframes, w, h, n)
        first = self.n_keyframes - self.cfg.window
        b = self.rng.draw_batch(self.cfg.window, w, h, n)
        b[:, 0] += first
        return b

    def _map(self, steps: int):
        m = self.cfg.mapping
        if self.mapper is not None:
            import torch
            world = self.mapper.world
            n = m.rays_per_batch // world + (1 if self.mapper.rank < m.rays_per_batch % world else 0)
            for _ in range(steps):
                b = torch.from_numpy(self._draw(n)).to(self.mapper.e.grad.device)
                self.mapper.step(b, m.lambda_d, exchange=self.cfg.exchange)
            return
        f = self.cfg.recent_fraction
        if f > 0.0 and self.n_keyframes > 1:
            # newest keyframe over-sampled: the region the camera just entered is
            # the least constrained part of the map
            n_new = int(round(f * m.rays_per_batch))
            w = self.intr.width
            h = self.intr.height
            for _ in range(steps):
                a = self.rng.draw_batch(1, w, h, n_new)
                a[:, 0] = self.n_keyframes - 1
                b = self.rng.draw_batch(self.n_keyframes, w, h, m.rays_per_batch - n_new)
                self.ctx.mapping_step(m, np.concatenate([a, b]))
            return
        if self.cfg.window <= 0 or self.cfg.window >= self.n_keyframes:
            # all keyframes: map_scene's pipelined inner loop (host draws overlap steps)
            self.ctx.mapping_steps(m, self.rng, self.n_keyframes, steps)
            return
        w = self.cfg.window
        first = self.n_keyframes - w
        for _ in range(steps):
            batch = self.rng.draw_batch(w, self.intr.width, self.intr.height, m.rays_per_batch)
            batch[:, 0] += first  # keyframe slots [first, n_keyframes)
            self.ctx.mapping_step(m, batch)

    def _put(self, slot: int, frame: Frame, pose: Pose):
        if frame.color_u8 is not None and frame.depth_u16 is not None:
            self.ctx.set_frame_u8u16(slot, frame.color_u8, frame.depth_u16, pose)  # 5 B/px
        else:
            self.ctx.set_frame(slot, frame, pose)

    def _add_keyframe(self, frame: Frame, pose: Pose):
        if self.n_keyframes >= self.cfg.max_keyframes:
            raise RuntimeError("slam: keyframe capacity exhausted")
        self._put(self.n_keyframes, frame, pose)
        self.n_keyframes += 1

    def process(self, frame: Frame, init_pose: Optional[Pose] = None) -> Pose:
        """Track (or, for the first frame, anchor at init_pose) and map."""
        i = len(self.poses)
        t0 = time.perf_counter()
        if i == 0:
            pose = init_pose or frame.gt_pose
            if pose is None:
                raise RuntimeError("slam: the first frame needs a pose")
            loss = 0.0
            t1 = time.perf_counter()
            self._add_keyframe(frame, pose)
            L = self.cfg.coarse_levels
            per = self.cfg.bootstrap_steps // (L + 1)
            for lv in range(L + 1):
                self._map(per if lv < L else self.cfg.bootstrap_steps - per * L)
                if lv < L:
                    self.ctx.upsample()  # resets the RMSProp state, as the reference
                    if self.mapper is not None:  # new grid buffers: new engine and peers
                        from .distributed import DistributedMapper, GpuEngine
                        self.mapper = DistributedMapper(GpuEngine(self.ctx, self.cfg.mapping))
            self.poses.append(pose)
            self.log.append(SlamFrameLog(0, True, 0.0, (time.perf_counter() - t1) * 1e3, loss))
            return pose
        prev = self.poses[-1]
        init = prev
        if self.cfg.constant_velocity and i >= 2:
            init = pose_compose(prev, pose_compose(pose_inverse(self.poses[-2]), prev))
        self._put(self.track_slot, frame, init)
        r = self.ctx.track_frame_gn(self.track_slot, self.intr, init, self.cfg.tracking)
        pose = r.pose
        t1 = time.perf_counter()
        key = i % self.cfg.keyframe_stride == 0
        if key:
            self._add_keyframe(frame, pose)
            self._map(self.cfg.map_steps)
        t2 = time.perf_counter()
        self.poses.append(pose)
        self.log.append(SlamFrameLog(i, key, (t1 - t0) * 1e3, (t2 - t1) * 1e3,
                                     r.loss_trace[-1] if r.loss_trace else 0.0))
        return pose


def run_slam(ctx: Context, intrinsics: CameraIntrinsics, geometry: GridGeometry, frames,
             config: SlamConfig = None):
    """Runs the loop over an iterable of Frames (gt_pose used for frame 0 only).
    Returns (estimated poses, per-frame log)."""
    s = SlamSystem(ctx, intrinsics, geometry, config or SlamConfig())
    for f in frames:
        s.process(f)
    return s.poses, s.log
