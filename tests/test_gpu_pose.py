"""The Gauss-Newton tracker's pose kernel (k_pose_group_u, K5 on the GN path)
against the CPU oracle and against its checker kernel.

The GN kernel keeps the reference's FP64 march, sigma replay, transmittance and
compositing, and contracts SH and accumulates the per-lane Jacobian partials in
fp32. So:
  * the hit count m and the composited-sample count are exact;
  * the loss is within 1e-4 relative (fp32 colour, ~1e-7 per channel, against
    residuals as small as the 8-bit quantisation at the true pose);
  * J^T r within 1e-4 and J^T J within 1e-3, relative to the largest entry
    (fp32 partials summed over a ray's samples; tolerance as VERDICT r01 asks).
The oracle is or_pose_normal_eqs (oracle/voxrf_oracle.c), pinned to the
reference's grad_wrt_ray (gradients.cpp:116-143) and the chart of
tracking.cpp:104-130 by tests/test_oracle_pinning.py.

k_pose_group<float> (VRF_POSE_KERNEL_GN_CHECK) is an independent control-flow
implementation of the same arithmetic (group-masked march instead of
warp-lockstep rounds): the two must agree bit for bit, per pass and over whole
track_frame_gn frames.
"""
import numpy as np
import pytest

from paper_2307_03404_b200 import _capi as capi
from paper_2307_03404_b200.api import GNConfig, Pose, RenderParams, TrackingConfig, unpack_sym6

from scenes import room_scene

pytestmark = pytest.mark.gpu

RTOL_LOSS = 1e-4
RTOL_JTR = 1e-4
RTOL_JTJ = 1e-3


def _pixels(intr, n, seed):
    rng = np.random.default_rng(seed)
    return np.stack([rng.integers(0, intr.width, n), rng.integers(0, intr.height, n)],
                    1).astype(np.int32)


def _oracle_samples(oracle, grid, intr, pose, px):
    """sum over hit rays of the reference's RayWorkspace::count (renderer.cpp:133)."""
    total = 0
    for x, y in px:
        o, d = oracle.generate_ray(intr, pose, float(x), float(y))
        r = oracle.render_ray(grid, o, d, RenderParams())
        total += r.count
    return total


def _perturbed(pose, dt):
    return Pose(pose.q, tuple(np.asarray(pose.t) + np.asarray(dt)))


SCENES = [(17, 32, 24, 400), (33, 64, 48, 1500)]


@pytest.mark.parametrize("res,w,h,n", SCENES)
@pytest.mark.parametrize("lambda_d", [1.0, 0.1])
def test_gn_kernel_normal_equations_match_oracle(ctx, oracle, res, w, h, n, lambda_d):
    grid, intr, frames = room_scene(res=res, width=w, height=h)
    frame = frames[1]
    ctx.load_grid(grid)
    ctx.load_frames(intr, frames)
    px = _pixels(intr, n, seed=res)
    for dt in ([0.0, 0.0, 0.0], [0.02, -0.015, 0.01]):
        pose = _perturbed(frame.gt_pose, dt)
        tc = TrackingConfig(lambda_d=lambda_d)
        ne = ctx.pose_normal_equations(1, intr, pose, px, tc, kernel=capi.POSE_KERNEL_GN)
        no = oracle.normal_eqs(grid, frame, intr, pose, px, 1.0, lambda_d, RenderParams())
        assert ne.rays_used == no.rays_used
        assert ne.samples == _oracle_samples(oracle, grid, intr, pose, px)
        assert ne.samples > ne.rays_used  # every hit ray composites several samples here
        assert abs(ne.loss - no.loss) <= RTOL_LOSS * abs(no.loss)
        jtr = np.array(no.jtr)
        jtj = unpack_sym6(no.jtj)
        assert np.max(np.abs(ne.jtr - jtr)) <= RTOL_JTR * np.abs(jtr).max()
        assert np.max(np.abs(ne.jtj - jtj)) <= RTOL_JTJ * np.abs(jtj).max()
        # and the FP64 parity kernel on the same pixels is far tighter
        nf = ctx.pose_normal_equations(1, intr, pose, px, tc, kernel=capi.POSE_KERNEL_PARITY)
        assert nf.samples == ne.samples and nf.rays_used == ne.rays_used
        assert np.max(np.abs(nf.jtj - jtj)) <= 1e-9 * np.abs(jtj).max()
        assert np.max(np.abs(nf.jtr - jtr)) <= 1e-9 * np.abs(jtr).max()


def test_gn_kernel_gauss_newton_step_matches_oracle_step(ctx, oracle):
    """The LM step solved from the GN kernel's normal equations equals the step
    from the oracle's within 1e-3 relative (what the tracker actually applies)."""
    grid, intr, frames = room_scene(res=33, width=64, height=48)
    frame = frames[2]
    ctx.load_grid(grid)
    ctx.load_frames(intr, frames)
    px = _pixels(intr, 2000, seed=9)
    pose = _perturbed(frame.gt_pose, [0.015, 0.01, -0.02])
    ne = ctx.pose_normal_equations(2, intr, pose, px, TrackingConfig(),
                                   kernel=capi.POSE_KERNEL_GN)
    no = oracle.normal_eqs(grid, frame, intr, pose, px, 1.0, 1.0, RenderParams())
    A_o = unpack_sym6(no.jtj)

    def step(A, b, lam=1e-4):
        A = A + lam * np.diag(np.diag(A)) + 1e-12 * np.eye(6)
        return np.linalg.solve(A, -np.asarray(b))

    x_gpu, x_o = step(ne.jtj, ne.jtr), step(A_o, no.jtr)
    assert np.linalg.norm(x_gpu - x_o) <= 1e-3 * np.linalg.norm(x_o)


@pytest.mark.parametrize("res,w,h,n", SCENES + [(33, 64, 48, 37)])
def test_gn_kernel_matches_checker(ctx, res, w, h, n):
    """The production GN kernel (4 lanes per ray, two corners per lane) against
    the independent 8-lane checker: the same samples and rays (sigma and colour
    sum in corner order in both), the loss to FP64 block-sum order, and JᵀJ / Jᵀr
    to the fp32 lane-partial order (two corners summed per lane first)."""
    grid, intr, frames = room_scene(res=res, width=w, height=h)
    ctx.load_grid(grid)
    ctx.load_frames(intr, frames)
    px = _pixels(intr, n, seed=res + n)
    for f in range(len(frames)):
        pose = _perturbed(frames[f].gt_pose, [0.01 * f, -0.01, 0.005])
        a = ctx.pose_normal_equations(f, intr, pose, px, TrackingConfig(),
                                      kernel=capi.POSE_KERNEL_GN)
        b = ctx.pose_normal_equations(f, intr, pose, px, TrackingConfig(),
                                      kernel=capi.POSE_KERNEL_GN_CHECK)
        assert a.samples == b.samples and a.rays_used == b.rays_used
        assert abs(a.loss - b.loss) <= 1e-12 * abs(b.loss)
        assert np.max(np.abs(a.jtj - b.jtj)) <= 1e-5 * np.max(np.abs(b.jtj))
        assert np.max(np.abs(a.jtr - b.jtr)) <= 1e-5 * np.max(np.abs(b.jtr))


@pytest.mark.parametrize("rays", [4096, 2048, 3000])
def test_track_frame_gn_kernels_agree_per_iteration(ctx, rays):
    """Whole GN frames (device draws, pose kernel, reduce, LM step; one CUDA
    graph) through the production kernel and the checker: the same draws and
    hits per iteration, losses and sample counts that agree to the fp32
    Jacobian-order noise, and poses within 1e-6. Non-power-of-4 ray counts draw
    exactly rays_per_iteration pixels."""
    grid, intr, frames = room_scene(res=33, width=64, height=48)
    frame = frames[1]
    ctx.load_grid(grid)
    ctx.load_frames(intr, frames)
    init = _perturbed(frame.gt_pose, [0.03, -0.02, 0.01])
    out = {}
    for k in (capi.POSE_KERNEL_GN, capi.POSE_KERNEL_GN_CHECK):
        r = ctx.track_frame_gn(1, intr, init, GNConfig(rays_per_iteration=rays, iterations=6,
                                                        kernel=k))
        out[k] = (r, ctx.track_frame_gn_history())
    (ra, ha), (rb, hb) = out[capi.POSE_KERNEL_GN], out[capi.POSE_KERNEL_GN_CHECK]
    assert ha.shape == (6, 3)
    assert np.array_equal(ha[:, 1], hb[:, 1])
    assert ha[0, 2] == hb[0, 2] and ha[0, 0] == pytest.approx(hb[0, 0], rel=1e-12)
    np.testing.assert_allclose(ha[:, 0], hb[:, 0], rtol=1e-4)
    np.testing.assert_allclose(ha[:, 2], hb[:, 2], rtol=1e-3)
    np.testing.assert_allclose(ra.pose.t, rb.pose.t, atol=1e-6)
    np.testing.assert_allclose(ra.pose.q, rb.pose.q, atol=1e-6)
    # every pixel of this frame has valid depth and the room encloses the camera:
    # all rays_per_iteration draws hit, and each composites more than one sample
    assert np.all(ha[:, 1] == rays)
    assert np.all(ha[:, 2] > 2 * ha[:, 1])
    gt = np.asarray(frame.gt_pose.t)
    assert np.linalg.norm(np.asarray(ra.pose.t) - gt) < 0.5 * np.linalg.norm(
        np.asarray(init.t) - gt)


def test_track_frame_gn_rejects_bad_arguments(ctx):
    grid, intr, frames = room_scene()
    ctx.load_grid(grid)
    ctx.load_frames(intr, frames)
    with pytest.raises(ValueError):
        ctx.track_frame_gn(1, intr, frames[1].gt_pose, GNConfig(rays_per_iteration=0))
    with pytest.raises(ValueError):
        ctx.track_frame_gn(1, intr, frames[1].gt_pose, GNConfig(kernel=capi.POSE_KERNEL_PARITY))
