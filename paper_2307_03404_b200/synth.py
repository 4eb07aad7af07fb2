"""Synthetic inputs of the named benchmark shapes, numpy only.

This is input generation, not part of the hot path: a voxelised primitive
room (walls + sphere + box, checker-textured, after dataset.cpp:187-195) turned
into a sigma/SH grid, camera trajectories from look_at (pose.hpp:44-61), and
the test helper grids of proj/tests/test_helpers.hpp. Grid values are rounded
to fp32 so the FP64 oracle and the fp32 device payload see identical numbers.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .api import CameraIntrinsics, Frame, GridGeometry, Pose, VoxelGrid

C0 = 0.28209479177387814


def look_at(eye, target, up=(0.0, 0.0, 1.0)) -> Pose:
    """look_at — pose.hpp:44-61 (x right, y down, z forward)."""
    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    fwd = fwd / math.sqrt(float(fwd @ fwd))
    right = np.cross(fwd, np.asarray(up, np.float64))
    if right @ right < 1e-12:
        right = np.cross(fwd, np.array([1.0, 0, 0]))
        if right @ right < 1e-12:
            right = np.cross(fwd, np.array([0, 1.0, 0]))
    right = right / math.sqrt(float(right @ right))
    down = np.cross(fwd, right)
    m = np.stack([right, down, fwd], axis=1)
    # Eigen quaternionbase_assign_impl (matrix -> quaternion)
    t = m[0, 0] + m[1, 1] + m[2, 2]
    q = np.zeros(4)  # x y z w
    if t > 0:
        t = math.sqrt(t + 1.0)
        q[3] = 0.5 * t
        t = 0.5 / t
        q[0] = (m[2, 1] - m[1, 2]) * t
        q[1] = (m[0, 2] - m[2, 0]) * t
        q[2] = (m[1, 0] - m[0, 1]) * t
    else:
        i = 0
        if m[1, 1] > m[0, 0]:
            i = 1
        if m[2, 2] > m[i, i]:
            i = 2
        j = (i + 1) % 3
        k = (j + 1) % 3
        t = math.sqrt(m[i, i] - m[j, j] - m[k, k] + 1.0)
        q[i] = 0.5 * t
        t = 0.5 / t
        q[3] = (m[k, j] - m[j, k]) * t
        q[j] = (m[j, i] + m[i, j]) * t
        q[k] = (m[k, i] + m[i, k]) * t
    q = q / math.sqrt(float(q @ q))
    return Pose((q[3], q[0], q[1], q[2]), tuple(eye))


def random_grid(rng: np.random.Generator, n=4, voxel=0.25, origin=(0, 0, 0), sigma_lo=0.0,
                sigma_hi=2.0) -> VoxelGrid:
    """testing::random_grid — proj/tests/test_helpers.hpp:10-24 (numpy stream)."""
    g = VoxelGrid(GridGeometry((n, n, n), tuple(map(float, origin)), voxel))
    g.data[:, 0] = rng.uniform(sigma_lo, sigma_hi, g.geom.num_vertices)
    g.data[:, 1:] = rng.uniform(-0.5, 0.5, (g.geom.num_vertices, 27))
    g.data[:] = g.data.astype(np.float32).astype(np.float64)
    return g


@dataclass
class Room:
    room_min: tuple = (0.0, 0.0, 0.0)
    room_max: tuple = (4.0, 4.0, 3.0)
    wall_albedo: float = 0.65
    checker_period: float = 0.25
    checker_albedo2: float = 0.1
    sphere_c: tuple = (2.0, 3.3, 1.1)
    sphere_r: float = 0.35
    sphere_albedo: tuple = (0.8, 0.3, 0.2)
    box_min: tuple = (2.6, 2.4, 0.0)
    box_max: tuple = (3.2, 3.0, 0.8)
    box_albedo: tuple = (0.2, 0.5, 0.8)

    def scaled(self, sx, sy, sz) -> "Room":
        s = np.array([sx, sy, sz])
        return Room(tuple(np.array(self.room_min) * s), tuple(np.array(self.room_max) * s),
                    self.wall_albedo, self.checker_period, self.checker_albedo2,
                    tuple(np.array(self.sphere_c) * s), self.sphere_r * min(sx, sy, sz),
                    self.sphere_albedo, tuple(np.array(self.box_min) * s),
                    tuple(np.array(self.box_max) * s), self.box_albedo)

    def sdf_albedo(self, p: np.ndarray):
        """Unsigned distance to the nearest surface and its albedo, p: (N,3)."""
        lo, hi = np.array(self.room_min), np.array(self.room_max)
        d_wall = np.minimum(p - lo, hi - p).min(axis=1)
        d_wall = np.abs(d_wall)
        d_sph = np.abs(np.linalg.norm(p - np.array(self.sphere_c), axis=1) - self.sphere_r)
        bc = 0.5 * (np.array(self.box_min) + np.array(self.box_max))
        bh = 0.5 * (np.array(self.box_max) - np.array(self.box_min))
        q = np.abs(p - bc) - bh
        d_box = np.abs(np.linalg.norm(np.maximum(q, 0.0), axis=1) + np.minimum(q.max(axis=1), 0.0))
        d = np.stack([d_wall, d_sph, d_box], axis=1)
        which = d.argmin(axis=1)
        par = np.floor(p / self.checker_period).astype(np.int64).sum(axis=1) & 1
        wall = np.where(par[:, None] == 1, self.checker_albedo2, self.wall_albedo) * np.ones((1, 3))
        alb = np.where((which == 0)[:, None], wall,
                       np.where((which == 1)[:, None], np.array(self.sphere_albedo),
                                np.array(self.box_albedo)))
        return d.min(axis=1), alb


def scene_grid(res: int, room: Room = None, seed: int = 2, sigma_peak: float = 200.0,
               band: float = 1.5, prune_tau: float = 1e-3, margin: float = 0.2,
               chunk: int = 1 << 21) -> VoxelGrid:
    """Config-2 map: sigma = peak * clamp(1 - |sdf| / (band * voxel), 0, 1), SH DC =
    (albedo - 0.5) / C0, higher SH U(-0.05, 0.05); occupancy pruned at tau
    (voxel_grid.cpp:169-188). res counts vertices per axis (e.g. 257)."""
    room = room or Room()
    lo = np.array(room.room_min) - margin
    hi = np.array(room.room_max) + margin
    voxel = float((hi - lo).max() / (res - 1))
    geom = GridGeometry((res, res, res), tuple(lo), voxel)
    grid = VoxelGrid.__new__(VoxelGrid)
    grid.geom = geom
    V = geom.num_vertices
    data = np.empty((V, 28), np.float32)
    rng = np.random.default_rng(seed)
    idx = np.arange(V, dtype=np.int64)
    for s in range(0, V, chunk):
        e = min(V, s + chunk)
        i = idx[s:e]
        ix = i % res
        iy = (i // res) % res
        iz = i // (res * res)
        p = lo + np.stack([ix, iy, iz], axis=1) * voxel
        d, alb = room.sdf_albedo(p)
        data[s:e, 0] = sigma_peak * np.clip(1.0 - d / (band * voxel), 0.0, 1.0)
        sh = rng.uniform(-0.05, 0.05, (e - s, 27)).astype(np.float32)
        sh[:, 0] = (alb[:, 0] - 0.5) / C0
        sh[:, 9] = (alb[:, 1] - 0.5) / C0
        sh[:, 18] = (alb[:, 2] - 0.5) / C0
        data[s:e, 1:] = sh
    grid.data = data.astype(np.float64)
    grid.active = np.ones(geom.num_cells, np.uint8)
    if prune_tau > 0:
        prune(grid, prune_tau)
    return grid


def prune(grid: VoxelGrid, tau: float) -> int:
    """VoxelGrid::prune — voxel_grid.cpp:169-188 (vectorised)."""
    rx, ry, rz = grid.geom.res
    s = np.maximum(grid.data[:, 0], 0.0).reshape(rz, ry, rx)
    peak = s[:-1, :-1, :-1]
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                peak = np.maximum(peak, s[dz:rz - 1 + dz, dy:ry - 1 + dy, dx:rx - 1 + dx])
    off = (peak.reshape(-1) < tau) & (grid.active != 0)
    grid.active[off] = 0
    return int(off.sum())


def circle_trajectory(n, center, radius, height, look_target, arc_deg=9.0, start_deg=0.0):
    """TrajectorySpec kCircle (dataset.cpp:156-185) with an explicit arc."""
    poses = []
    for i in range(n):
        a = math.radians(start_deg + arc_deg * (i / max(n - 1, 1)))
        eye = (center[0] + radius * math.cos(a), center[1] + radius * math.sin(a), height)
        poses.append(look_at(eye, look_target))
    return poses


def room_path(n, room: Room, seed=4, step_m=0.01, step_deg=0.5, height=1.5):
    """Smooth waypoint path inside the room (<= step_m, <= step_deg per frame)."""
    rng = np.random.default_rng(seed)
    lo, hi = np.array(room.room_min), np.array(room.room_max)
    c = 0.5 * (lo + hi)
    r = 0.25 * min(hi[0] - lo[0], hi[1] - lo[1])
    poses = []
    yaw0 = rng.uniform(0, 2 * math.pi)
    for i in range(n):
        a = yaw0 + math.radians(step_deg) * i
        eye = np.array([c[0] + r * math.cos(a * 0.5), c[1] + r * math.sin(a * 0.5), height])
        target = eye + np.array([math.cos(a + math.pi / 2), math.sin(a + math.pi / 2), -0.15])
        poses.append(look_at(eye, target))
    return poses


def ellipse_trajectory(n, room: Room, height=1.5, fps=30.0, a_frac=0.3, b_frac=0.25,
                       look_out=0.6, pitch=-0.15):
    """Closed-loop ellipse (config 5): the camera circles the room
    centre once over n frames, heading along the tangent turned outward by
    ``look_out`` rad toward the walls. Returns (poses, timestamps)."""
    lo, hi = np.array(room.room_min), np.array(room.room_max)
    c = 0.5 * (lo + hi)
    a = a_frac * (hi[0] - lo[0])
    b = b_frac * (hi[1] - lo[1])
    poses, ts = [], []
    for i in range(n):
        th = 2.0 * math.pi * i / n
        eye = np.array([c[0] + a * math.cos(th), c[1] + b * math.sin(th), height])
        tangent = np.array([-a * math.sin(th), b * math.cos(th), 0.0])
        tangent /= np.linalg.norm(tangent)
        outward = np.array([tangent[1], -tangent[0], 0.0])
        fwd = math.cos(look_out) * tangent + math.sin(look_out) * outward
        target = eye + np.array([fwd[0], fwd[1], pitch])
        poses.append(look_at(eye, target))
        ts.append(i / fps)
    return poses, ts


def quantize_frame(color: np.ndarray, depth: np.ndarray, depth_scale: float):
    """quantize_color / quantize_depth — image.cpp:15-30."""
    c8 = np.clip(np.floor(color * 255.0 + 0.5), 0, 255) / 255.0
    du = np.where(depth > 0, np.clip(np.floor(depth * depth_scale + 0.5), 0, 65535), 0)
    return c8, du / depth_scale


def sensor_frame(color: np.ndarray, depth: np.ndarray, depth_scale: float, timestamp=0.0,
                 pose=None) -> Frame:
    """A Frame as an RGB-D sensor / the reference's PNG dataset delivers it: 8-bit
    colour and 16-bit depth units (image.cpp:13-30), plus the decoded doubles."""
    c8 = np.clip(np.floor(color * 255.0 + 0.5), 0, 255).astype(np.uint8)
    du = np.where(depth > 0, np.clip(np.floor(depth * depth_scale + 0.5), 0, 65535),
                  0).astype(np.uint16)
    return Frame(c8 / 255.0, du / depth_scale, timestamp, pose, c8, du)


def replica_intrinsics() -> CameraIntrinsics:
    return CameraIntrinsics(600.0, 600.0, 599.5, 339.5, 1200, 680, 6553.5)


def small_intrinsics() -> CameraIntrinsics:
    return CameraIntrinsics(138.5, 138.5, 80.0, 60.0, 160, 120, 1000.0)


def frames_from_renders(renders, poses, depth_scale):
    out = []
    for (color, depth), pose in zip(renders, poses):
        c, d = quantize_frame(color, depth, depth_scale)
        out.append(Frame(c, d, 0.0, pose))
    return out


def synth_from_grid(ctx, grid, poses, timestamps, intrinsics, params=None):
    """synth_from_grid — dataset.cpp:443-462, on the device: render every pose of
    the trajectory from `grid` (K1, one full-resolution render_image per frame),
    then quantise colour and depth like the reference's PNG path (quantize_color /
    quantize_depth, image.cpp:26-30). grid=None renders the grid already loaded in
    ctx. Returns the Frames (gt_pose and timestamp set)."""
    if grid is not None:
        ctx.load_grid(grid)
    out = []
    for pose, ts in zip(poses, timestamps):
        img = ctx.render_image(intrinsics, pose, params) if params is not None else \
            ctx.render_image(intrinsics, pose)
        c, d = quantize_frame(img.color, img.depth, intrinsics.depth_scale)
        out.append(Frame(c, d, float(ts), pose))
    return out
