"""Evaluation metrics around the hot path (eval.cpp) and TUM trajectory I/O
(trajectory.cpp).

The trajectory metrics (ATE, RPE) are O(frames) host arithmetic, as in the
reference. Map quality renders the evaluation views on the GPU and scores them
in HBM (vrf_evaluate_views) with the reference's PSNR sampling stream, so the
figure is comparable with the reference's own evaluate_map_quality on the same
frames. psnr / depth_l1 below are the host restatements over given images.
All of it is pinned to the reference's eval.cpp / trajectory.cpp by
tests/test_eval_reference.py and tests/test_gpu_eval.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .api import Pose, RenderParams, Rng, pose_compose, pose_inverse


def associate_trajectories(est_ts: Sequence[float], ref_ts: Sequence[float],
                           max_dt: float = 0.02):
    """associate_trajectories — eval.cpp:124-138 (nearest reference timestamp,
    monotone scan)."""
    pairs = []
    j = 0
    for i, ts in enumerate(est_ts):
        while j + 1 < len(ref_ts) and abs(ref_ts[j + 1] - ts) <= abs(ref_ts[j] - ts):
            j += 1
        if len(ref_ts) and abs(ref_ts[j] - ts) <= max_dt:
            pairs.append((i, j))
    return pairs


def ate_rmse(est: Sequence[Pose], est_ts, ref: Sequence[Pose], ref_ts, align: bool = True):
    """ate_rmse — eval.cpp:140-172: rigid (no scale) SVD alignment of the
    positions, then the RMS position error. Returns (rmse, pairs)."""
    pairs = associate_trajectories(est_ts, ref_ts)
    if len(pairs) < 2:
        raise RuntimeError("ate_rmse: fewer than 2 matched poses")
    pe = np.array([est[i].t for i, _ in pairs], np.float64)
    pr = np.array([ref[j].t for _, j in pairs], np.float64)
    rot = np.eye(3)
    trans = np.zeros(3)
    if align:
        ce, cr = pe.mean(0), pr.mean(0)
        cov = (pr - cr).T @ (pe - ce)
        u, _, vt = np.linalg.svd(cov)
        flip = np.eye(3)
        if np.linalg.det(u @ vt) < 0:
            flip[2, 2] = -1.0
        rot = u @ flip @ vt
        trans = cr - rot @ ce
    err = (pe @ rot.T + trans) - pr
    return math.sqrt(float(np.sum(err * err)) / len(pairs)), len(pairs)


def save_tum(path, poses: Sequence[Pose], timestamps) -> None:
    """save_tum — trajectory.cpp:10-23: "# timestamp tx ty tz qx qy qz qw" header,
    then one line per pose, every value printed with %.17g (doubles round-trip)."""
    with open(path, "w") as f:
        f.write("# timestamp tx ty tz qx qy qz qw\n")
        for ts, p in zip(timestamps, poses):
            w, x, y, z = (float(v) for v in p.q)
            tx, ty, tz = (float(v) for v in p.t)
            f.write("%.17g %.17g %.17g %.17g %.17g %.17g %.17g %.17g\n"
                    % (float(ts), tx, ty, tz, x, y, z, w))


def load_tum(path):
    """load_tum — trajectory.cpp:25-46: skips blank and '#' lines; a line without
    eight numbers raises. Returns (poses, timestamps)."""
    poses, stamps = [], []
    with open(path) as f:
        for lineno, line in enumerate(f, 1):
            s = line.strip(" \t\r\n")
            if not s or s[0] == "#":
                continue
            try:
                v = [float(x) for x in s.split()[:8]]
                if len(v) < 8:
                    raise ValueError
            except ValueError:
                raise RuntimeError(f"load_tum: malformed line {lineno} in {path}") from None
            ts, tx, ty, tz, qx, qy, qz, qw = v
            stamps.append(ts)
            poses.append(Pose((qw, qx, qy, qz), (tx, ty, tz)))
    return poses, stamps


def rotation_angle_rad(q) -> float:
    """rotation_angle_rad — pose.hpp:51-54."""
    q = np.asarray(q, np.float64)
    w = min(1.0, abs(q[0] / np.linalg.norm(q)))
    return 2.0 * math.acos(w)


@dataclass
class RpeResult:
    rpe_t: float
    rpe_r_deg: float
    pairs: int


def rpe(est: Sequence[Pose], est_ts, ref: Sequence[Pose], ref_ts, interval_m: float = 1.0):
    """rpe — eval.cpp:174-208: relative pose error over path-length intervals
    measured along the reference."""
    pairs = associate_trajectories(est_ts, ref_ts)
    if len(pairs) < 2:
        raise RuntimeError("rpe: fewer than 2 matched poses")
    n = len(pairs)
    cum = np.zeros(n)
    for k in range(1, n):
        cum[k] = cum[k - 1] + np.linalg.norm(np.asarray(ref[pairs[k][1]].t) -
                                             np.asarray(ref[pairs[k - 1][1]].t))
    sum_t = sum_r = 0.0
    count = 0
    j = 0
    for i in range(n):
        while j < n and cum[j] - cum[i] < interval_m:
            j += 1
        if j >= n:
            break
        pi, pj = est[pairs[i][0]], est[pairs[j][0]]
        qi, qj = ref[pairs[i][1]], ref[pairs[j][1]]
        e = pose_compose(pose_inverse(pose_compose(pose_inverse(qi), qj)),
                         pose_compose(pose_inverse(pi), pj))
        sum_t += float(np.dot(e.t, e.t))
        a = rotation_angle_rad(e.q)
        sum_r += a * a
        count += 1
    if count == 0:
        raise RuntimeError("rpe: reference path shorter than the interval")
    return RpeResult(math.sqrt(sum_t / count), math.degrees(math.sqrt(sum_r / count)), count)


def psnr(rendered, reference, masks=None, images: int = 10, pixels_per_image: int = 10000,
         seed: int = 0):
    """psnr — eval.cpp:64-97: pixels drawn from the reference Rng stream; peak 1.0,
    capped at 99 dB. Returns (psnr_db, samples)."""
    if not rendered or len(rendered) != len(reference):
        raise RuntimeError("psnr: empty or mismatched image sets")
    rng = Rng(seed)
    sum_sq = 0.0
    samples = 0
    for _ in range(images):
        img = rng.uniform_index(len(rendered))
        a, b = rendered[img], reference[img]
        if a.shape != b.shape:
            raise RuntimeError("psnr: image dimensions differ")
        h, w = a.shape[:2]
        m = None if masks is None else masks[img]
        for _ in range(pixels_per_image):
            x = rng.uniform_index(w)
            y = rng.uniform_index(h)
            if m is not None and not m[y, x] > 0.0:
                continue
            d = a[y, x, :3].astype(np.float64) - b[y, x, :3]
            sum_sq += float(d @ d)
            samples += 1
    if samples == 0:
        raise RuntimeError("psnr: no valid pixels sampled")
    mse = sum_sq / (samples * 3)
    if mse <= 0.0:
        return 99.0, samples
    return min(99.0, 10.0 * math.log10(1.0 / mse)), samples


def depth_l1(rendered, reference, masks=None):
    """depth_l1 — eval.cpp:99-122: mean |D - D*| over valid reference depth (and
    the rendered hit mask). Returns (l1_m, pixels)."""
    if not rendered or len(rendered) != len(reference):
        raise RuntimeError("depth_l1: empty or mismatched image sets")
    s = 0.0
    count = 0
    for k, (a, b) in enumerate(zip(rendered, reference)):
        if a.shape != b.shape:
            raise RuntimeError("depth_l1: image dimensions differ")
        ok = b > 0.0
        if masks is not None:
            ok &= masks[k] > 0.0
        s += float(np.abs(a[ok].astype(np.float64) - b[ok]).sum())
        count += int(ok.sum())
    if count == 0:
        raise RuntimeError("depth_l1: empty valid mask")
    return s / count, count


@dataclass
class MapQuality:
    psnr_db: float
    depth_l1_m: float
    color_samples: int
    depth_pixels: int


def evaluate_map_quality(ctx, intrinsics, frames, frame_indices, render: Optional[RenderParams] = None,
                         images: int = 10, pixels_per_image: int = 10000, seed: int = 0,
                         exact_depth=None) -> MapQuality:
    """evaluate_map_quality — eval.cpp:210-240 on the device: the evaluation views
    are rendered on the grid resident in ``ctx`` and scored in HBM
    (Context.evaluate_views / vrf_evaluate_views); only the sums come back. The
    PSNR pixels are the reference's Rng draws (eval.cpp:72-83), the depth
    reference is exact_depth[idx] when given (prefer_exact_depth), else the
    frame's depth."""
    if not frame_indices:
        raise RuntimeError("evaluate_map_quality: no frames")
    poses, colors, depths = [], [], []
    for idx in frame_indices:
        f = frames[idx]
        if f.gt_pose is None:
            raise RuntimeError("evaluate_map_quality: frame without pose")
        poses.append(f.gt_pose)
        colors.append(f.color)
        use_exact = exact_depth is not None and idx < len(exact_depth) and exact_depth[idx] is not None
        depths.append(exact_depth[idx] if use_exact else f.depth)
    samples = Rng(seed).draw_eval_samples(len(poses), intrinsics.width, intrinsics.height, images,
                                          pixels_per_image)
    sq, ns, l1s, npx = ctx.evaluate_views(intrinsics, poses, colors, depths, samples, render)
    if ns == 0:
        raise RuntimeError("psnr: no valid pixels sampled")
    if npx == 0:
        raise RuntimeError("depth_l1: empty valid mask")
    mse = sq / (ns * 3)
    p = 99.0 if mse <= 0.0 else min(99.0, 10.0 * math.log10(1.0 / mse))
    return MapQuality(p, l1s / npx, int(ns), int(npx))
