"""metrics.py (the evaluation layer around the hot path) against the reference's
own eval.cpp / trajectory.cpp, compiled unchanged into oracle/_ref.

* ate_rmse (eval.cpp:140-172, aligned and unaligned), rpe (eval.cpp:174-208),
  associate_trajectories (eval.cpp:124-138), psnr (eval.cpp:64-97: the
  reference's Rng pixel stream) and depth_l1 (eval.cpp:99-122): equal to the
  reference within 1e-12 relative (summation-order noise of the SVD and sums).
* save_tum / load_tum (trajectory.cpp:10-46): the file we write is byte-identical
  to the reference's, and each side reads the other's.
"""
import math

import numpy as np
import pytest

from paper_2307_03404_b200 import metrics, synth
from paper_2307_03404_b200.api import Pose, pose_compose

pytestmark = pytest.mark.ref


def _noisy(poses, sigma_t, sigma_r, seed):
    rng = np.random.default_rng(seed)
    out = []
    for p in poses:
        ax = rng.normal(size=3)
        ax /= np.linalg.norm(ax)
        a = rng.normal(0.0, sigma_r)
        dq = (math.cos(a / 2), *(math.sin(a / 2) * ax))
        out.append(pose_compose(Pose(dq, tuple(rng.normal(0.0, sigma_t, 3))), p))
    return out


def _cases():
    poses, ts = synth.ellipse_trajectory(240, synth.Room())
    ts = list(ts)
    yield "noise", _noisy(poses, 0.02, 0.01, 1), ts, poses, ts
    # a rigidly moved estimate with noise: alignment removes the rigid part
    a = 0.4
    T = Pose((math.cos(a / 2), 0.0, math.sin(a / 2), 0.0), (0.5, -1.0, 0.25))
    yield "rigid", [pose_compose(T, p) for p in _noisy(poses, 0.01, 0.0, 2)], ts, poses, ts
    # estimate timestamps jittered and subsampled: association drops / pairs frames
    rng = np.random.default_rng(3)
    est_ts = [t + rng.uniform(-0.015, 0.015) for t in ts[::2]]
    yield "assoc", _noisy(poses[::2], 0.03, 0.02, 4), est_ts, poses, ts


@pytest.mark.parametrize("case", ["noise", "rigid", "assoc"])
def test_ate_and_rpe_match_reference(ref, case):
    name, est, est_ts, gt, gt_ts = next(c for c in _cases() if c[0] == case)
    for align in (True, False):
        ours, n = metrics.ate_rmse(est, est_ts, gt, gt_ts, align=align)
        theirs, n_ref = ref.ate_rmse(est, est_ts, gt, gt_ts, align=align)
        assert n == n_ref
        assert ours == pytest.approx(theirs, rel=1e-12, abs=1e-15)
    for interval in (0.5, 1.0, 2.0):
        r = metrics.rpe(est, est_ts, gt, gt_ts, interval)
        t, deg, pairs = ref.rpe(est, est_ts, gt, gt_ts, interval)
        assert r.pairs == pairs
        assert r.rpe_t == pytest.approx(t, rel=1e-12, abs=1e-15)
        assert r.rpe_r_deg == pytest.approx(deg, rel=1e-9, abs=1e-12)


def test_metric_errors_match_reference(ref):
    poses, ts = synth.ellipse_trajectory(10, synth.Room())
    for fn in (lambda m: m.ate_rmse(poses[:1], ts[:1], poses[:1], ts[:1]),
               lambda m: m.rpe(poses[:3], ts[:3], poses[:3], ts[:3], 100.0)):
        with pytest.raises(RuntimeError):
            fn(metrics)
        with pytest.raises(RuntimeError):
            fn(ref)


@pytest.mark.parametrize("seed", [0, 7])
def test_psnr_and_depth_l1_match_reference(ref, seed):
    rng = np.random.default_rng(seed)
    n, h, w = 3, 24, 40
    a = [rng.uniform(size=(h, w, 3)) for _ in range(n)]
    b = [np.clip(x + rng.normal(0, 0.05, x.shape), 0, 1) for x in a]
    da = [rng.uniform(0.5, 3.0, (h, w)) * (rng.uniform(size=(h, w)) > 0.2) for _ in range(n)]
    db = [np.where(rng.uniform(size=(h, w)) > 0.1, d + rng.normal(0, 0.01, d.shape), 0.0)
          for d in da]
    for masks in (None, da):
        p, ns = metrics.psnr(a, b, masks, images=7, pixels_per_image=300, seed=seed)
        pr, nr = ref.psnr(a, b, masks, images=7, pixels_per_image=300, seed=seed)
        assert ns == nr
        assert p == pytest.approx(pr, rel=1e-12)
        l1, npx = metrics.depth_l1(da, db, masks)
        l1r, npr = ref.depth_l1(da, db, masks)
        assert npx == npr
        assert l1 == pytest.approx(l1r, rel=1e-12)
    # identical images cap at 99 dB on both sides
    assert metrics.psnr(a, a, images=2, pixels_per_image=10)[0] == ref.psnr(
        a, a, images=2, pixels_per_image=10)[0] == 99.0


def test_tum_files_are_byte_identical_and_cross_readable(ref, tmp_path):
    poses, ts = synth.ellipse_trajectory(50, synth.Room())
    poses = _noisy(poses, 0.01, 0.01, 5)
    ours, theirs = tmp_path / "ours.txt", tmp_path / "theirs.txt"
    metrics.save_tum(ours, poses, ts)
    ref.save_tum(theirs, poses, ts)
    assert ours.read_bytes() == theirs.read_bytes()
    p2, t2 = metrics.load_tum(theirs)
    r2, rt2 = ref.load_tum(ours)
    assert np.array_equal(np.asarray(t2), np.asarray(ts)) and np.array_equal(rt2, np.asarray(ts))
    for a, b, (q, t) in zip(poses, p2, r2):
        assert tuple(a.q) == tuple(b.q) == tuple(q)  # %.17g round-trips every double
        assert tuple(a.t) == tuple(b.t) == tuple(t)


def test_tum_reader_rejects_malformed_lines_like_the_reference(ref, tmp_path):
    f = tmp_path / "bad.txt"
    f.write_text("# header\n\n1.0 0 0 0 0 0 0 1\n2.0 0 0 0 0 0\n")
    with pytest.raises(RuntimeError, match="malformed line 4"):
        metrics.load_tum(f)
    with pytest.raises(RuntimeError, match="malformed line 4"):
        ref.load_tum(f)
