"""Host-side evaluation metrics (metrics.py, eval.cpp:64-208) on closed-form cases."""
import math

import numpy as np
import pytest

from paper_2307_03404_b200.api import Pose, pose_compose
from paper_2307_03404_b200 import metrics, synth


def _traj(n=50):
    poses, ts = synth.ellipse_trajectory(n, synth.Room())
    return poses, ts


def test_ate_is_zero_for_identical_and_rigidly_moved_trajectories():
    poses, ts = _traj()
    assert metrics.ate_rmse(poses, ts, poses, ts)[0] < 1e-12
    # a rigid transform of the estimate is removed by the alignment (eval.cpp:154-165)
    a = 0.3
    T = Pose((math.cos(a / 2), 0.0, 0.0, math.sin(a / 2)), (1.0, -2.0, 0.5))
    moved = [pose_compose(T, p) for p in poses]
    assert metrics.ate_rmse(moved, ts, poses, ts, align=True)[0] < 1e-9
    un = metrics.ate_rmse(moved, ts, poses, ts, align=False)[0]
    assert un > 0.5


def test_ate_unaligned_equals_a_constant_offset():
    poses, ts = _traj()
    off = np.array([0.03, -0.04, 0.0])
    est = [Pose(p.q, tuple(np.asarray(p.t) + off)) for p in poses]
    assert metrics.ate_rmse(est, ts, poses, ts, align=False)[0] == pytest.approx(0.05, rel=1e-9)


def test_association_is_nearest_timestamp_within_max_dt():
    pairs = metrics.associate_trajectories([0.0, 0.1, 0.2, 5.0], [0.0, 0.11, 0.19, 0.3])
    assert pairs == [(0, 0), (1, 1), (2, 2)]


def test_rpe_is_zero_for_identical_trajectories_and_sees_a_scale_error():
    poses, ts = _traj(200)
    r = metrics.rpe(poses, ts, poses, ts, 1.0)
    assert r.rpe_t < 1e-12 and r.rpe_r_deg < 1e-6 and r.pairs > 0
    scaled = [Pose(p.q, tuple(1.1 * np.asarray(p.t))) for p in poses]
    assert metrics.rpe(scaled, ts, poses, ts, 1.0).rpe_t > 0.05
    with pytest.raises(RuntimeError, match="shorter than the interval"):
        metrics.rpe(poses[:3], ts[:3], poses[:3], ts[:3], 100.0)


def test_psnr_and_depth_l1():
    rng = np.random.default_rng(0)
    a = rng.uniform(size=(12, 16, 3))
    assert metrics.psnr([a], [a], images=2, pixels_per_image=50)[0] == 99.0
    b = a + 0.1
    p, n = metrics.psnr([b], [a], images=2, pixels_per_image=50)
    assert p == pytest.approx(20.0, abs=1e-9) and n == 100
    d = rng.uniform(1, 2, size=(12, 16))
    l1, cnt = metrics.depth_l1([d + 0.25], [d])
    assert l1 == pytest.approx(0.25) and cnt == d.size
