"""The reference's renderer / gradient known-answer tests, run on the device.

Each test restates a reference unit test (tests/test_renderer.cpp,
tests/test_gradients.cpp; cited per test) through the C-ABI, so the sm_100a
kernels — not the CPU restatement — are held to the same closed-form answers.
Schedules are given through geometry (the device march derives them), where the
reference test hands render_ray_scheduled an explicit schedule.
"""
import math

import numpy as np
import pytest

from paper_2307_03404_b200.api import MappingConfig, Pose, RenderParams, VoxelGrid
from paper_2307_03404_b200 import synth
from paper_2307_03404_b200.api import CameraIntrinsics, Frame, GridGeometry

pytestmark = pytest.mark.gpu

C0 = 0.28209479177387814


def constant_color(grid, rgb):
    for ch, c in enumerate(rgb):
        grid.data[:, 1 + 9 * ch] = (c - 0.5) / C0


def rays_of(o, d):
    return np.array([list(o) + list(d)], dtype=np.float64)


def test_uniform_schedule_arithmetic(ctx):
    """test_renderer.cpp:59-75."""
    grid = VoxelGrid(GridGeometry((9, 9, 9), (-1, -1, -1), 0.25), 1.0)
    ctx.load_grid(grid)
    p = RenderParams(step=0.25, t_near=0.1, t_far=1.1)
    n, t, delta, _ = ctx.sample_rays(rays_of((-0.9, 0, 0), (1, 0, 0)), p, cap=16)
    assert n[0] == 4
    np.testing.assert_allclose(t[0, :4], [0.225, 0.475, 0.725, 0.975], rtol=1e-12)
    np.testing.assert_allclose(delta[0, :4], 0.25, rtol=1e-12)


def test_all_cells_inactive_is_empty(ctx):
    """test_renderer.cpp:77-84."""
    grid = VoxelGrid(GridGeometry((4, 4, 4), (0, 0, 0), 0.25), 1.0)
    grid.set_all_active(False)
    ctx.load_grid(grid)
    n, *_ = ctx.sample_rays(rays_of((-1, 0.4, 0.4), (1, 0, 0)), RenderParams(), cap=16)
    assert n[0] == 0


def test_pruned_schedule_is_the_dense_schedule_filtered(ctx):
    """test_renderer.cpp:86-119: the sparse schedule is exactly the dense one with
    the samples in inactive cells removed."""
    rng = np.random.default_rng(32)
    grid = synth.random_grid(rng, 5, 0.2)
    pruned = grid.copy()
    pruned.active[rng.uniform(size=pruned.active.size) < 0.5] = 0
    p = RenderParams(t_near=0.0)
    o = np.array([0.4, 0.4, 0.4]) + rng.uniform(-1, 1, (40, 3))
    d = rng.normal(size=(40, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rays = np.concatenate([o, d], axis=1)
    ctx.load_grid(grid)
    nd, td, dd, cd = ctx.sample_rays(rays, p, cap=64)
    ctx.load_grid(pruned)
    ns, ts, ds, cs = ctx.sample_rays(rays, p, cap=64)
    for i in range(40):
        keep = pruned.active[cd[i, :nd[i]]] != 0
        assert ns[i] == keep.sum()
        assert np.array_equal(ts[i, :ns[i]], td[i, :nd[i]][keep])
        assert np.array_equal(ds[i, :ns[i]], dd[i, :nd[i]][keep])


def test_zero_density_renders_background_with_full_transmittance(ctx):
    """test_renderer.cpp:121-130."""
    ctx.load_grid(VoxelGrid(GridGeometry((4, 4, 4), (0, 0, 0), 0.25), 0.0))
    r = ctx.render_rays(rays_of((-0.5, 0.4, 0.4), (1, 0, 0)))[0]
    assert r[6] == 1  # hit
    assert r[0] == r[1] == r[2] == 0.0 and r[3] == 0.0
    assert r[4] == pytest.approx(1.0, abs=1e-12)


def test_saturated_sample_dominates_the_ray(ctx):
    """test_renderer.cpp:132-146: sigma delta = 50 on the first sample."""
    grid = VoxelGrid(GridGeometry((2, 2, 2), (0, 0, 0), 1.0), 500.0)
    constant_color(grid, (0.8, 0.3, 0.6))
    ctx.load_grid(grid)
    p = RenderParams(step=0.1, t_near=0.35)
    r = ctx.render_rays(rays_of((0.0, 0.5, 0.5), (1, 0, 0)), p)[0]
    assert r[5] == 1 and r[7] == 1  # one sample, terminated early
    assert r[0] == pytest.approx(0.8, rel=1e-6) and r[1] == pytest.approx(0.3, rel=1e-6)
    assert r[3] == pytest.approx(0.4, rel=1e-9)


def test_ln2_then_opaque_split_the_weight_evenly(ctx):
    """test_renderer.cpp:148-169: sigma delta = ln 2 on the first sample and 50 on
    the second split the weight 1/2 : 1/2. The device derives the schedule, so the
    two densities come from a linear sigma ramp along x sampled at its quarter
    points (two segments of 0.5 over a unit cell)."""
    geom = GridGeometry((2, 2, 2), (0.0, 0.0, 0.0), 1.0)
    grid = VoxelGrid(geom, 0.0)
    # sigma(x) = s0 (1 - x) + s1 x with sigma(0.25) = 2 ln 2, sigma(0.75) = 100
    s0 = (3 * 8 * math.log(2.0) - 400.0) / 8.0
    s1 = 8 * math.log(2.0) - 3 * s0
    for k in range(8):
        x = k & 1
        v = geom.vertex_index(x, (k >> 1) & 1, (k >> 2) & 1)
        grid.data[v, 0] = s1 if x else s0
        grid.data[v, 1] = ((0.9 if x else 0.1) - 0.5) / C0  # red ramps 0.1 -> 0.9
    ctx.load_grid(grid)
    p = RenderParams(step=0.5, t_near=0.0)
    r = ctx.render_rays(rays_of((0.0, 0.5, 0.5), (1, 0, 0)), p)[0]
    assert r[5] == 2 and r[7] == 1  # two samples, terminated after the opaque one
    # colours 0.3 and 0.7 at the sample points, weights 1/2 and 1/2 (1 - e^-50)
    assert r[0] == pytest.approx(0.5 * 0.3 + 0.5 * 0.7, rel=1e-6)
    # fp32 payload: sigma delta = ln 2 up to ~1e-7
    assert r[3] == pytest.approx(0.5 * 0.25 + 0.5 * 0.75, rel=1e-6)


def test_transmittance_accounts_for_all_light(ctx, oracle):
    """test_renderer.cpp:171-194: weights plus the terminal transmittance sum to 1
    for rays that are not terminated early (device render vs oracle workspace)."""
    rng = np.random.default_rng(33)
    for trial in range(10):
        grid = synth.random_grid(rng, 5, 0.2, (0, 0, 0), 0.0, 3.0)
        ctx.load_grid(grid)
        d = rng.normal(size=(8, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        o = np.array([0.4, 0.4, 0.4]) + 0.3 * d[::-1]
        rays = np.concatenate([o, d], axis=1)
        out = ctx.render_rays(rays)
        for i in range(8):
            ref = oracle.render_ray(grid, rays[i, :3], rays[i, 3:], RenderParams())
            assert out[i, 5] == ref.count
            assert out[i, 4] == pytest.approx(ref.transmittance_terminal, rel=1e-12, abs=1e-15)


def test_constant_density_quadrature(ctx):
    """test_renderer.cpp:220-250: piecewise-constant density makes the colour
    accumulation exact at any step; halving the step at least halves the depth
    quadrature error."""
    sigma = 2.0
    geom = GridGeometry((2, 2, 2), (0.0, 0.0, 0.0), 4.0)
    grid = VoxelGrid(geom, sigma)
    constant_color(grid, (0.7, 0.7, 0.7))
    ctx.load_grid(grid)
    a, length = 0.5, 1.0
    E = math.exp(-sigma * length)
    exact_depth = a * (1 - E) + (1 - E) / sigma - length * E
    # the colour the device holds: the fp32-rounded DC coefficient, replayed in FP64
    c_eff = 0.5 + float(np.float32((0.7 - 0.5) / C0)) * C0
    exact_color = c_eff * (1 - E)
    errs = []
    for step in (0.125, 0.0625):
        p = RenderParams(step=step, t_near=a, t_far=a + length, termination_eps=0.0)
        r = ctx.render_rays(rays_of((0.0, 2.0, 2.0), (1, 0, 0)), p)[0]
        assert abs(r[0] - exact_color) < 1e-11
        errs.append(abs(r[3] - exact_depth))
    assert errs[1] <= 0.5 * errs[0]


def test_render_is_bit_reproducible(ctx):
    """test_renderer.cpp:252-263."""
    rng = np.random.default_rng(35)
    grid = synth.random_grid(rng, 4, 0.25)
    ctx.load_grid(grid)
    d = np.array([1, 0.11, -0.07])
    d /= np.linalg.norm(d)
    rays = rays_of((-0.4, 0.37, 0.41), d)
    a = ctx.render_rays(rays)
    b = ctx.render_rays(rays)
    assert np.array_equal(a, b)


def test_mapping_gradient_matches_finite_differences(ctx):
    """tests/test_gradients.cpp:254-264 (randomized gradcheck), on the device:
    the deterministic mapping gradient of L = L_p + lambda_d L_g against central
    differences of the device loss, for random payload entries."""
    rng = np.random.default_rng(777)
    geom = GridGeometry((5, 5, 5), (0.0, 0.0, 0.0), 0.2)
    grid = synth.random_grid(rng, 5, 0.2, (0, 0, 0), 0.5, 4.0)
    intr = CameraIntrinsics(30.0, 30.0, 8.0, 6.0, 16, 12, 1000.0)
    pose = synth.look_at((0.4, -0.9, 0.45), (0.4, 0.4, 0.4))
    target = synth.random_grid(rng, 5, 0.2, (0, 0, 0), 0.5, 4.0)
    ctx.load_grid(target)
    img = ctx.render_image(intr, pose)
    frames = [Frame(img.color, img.depth, 0.0, pose)]
    batch = np.array([[0, x, y] for y in range(0, 12, 2) for x in range(0, 16, 2)], np.int32)
    cfg = MappingConfig(deterministic=True)
    ctx.load_frames(intr, frames)

    def loss(g):
        ctx.load_grid(g)
        _, st = ctx.mapping_gradient(cfg, batch)
        return st.loss_total

    ctx.load_grid(grid)
    grad, _ = ctx.mapping_gradient(cfg, batch)
    nz = np.argwhere(np.abs(grad) > 1e-6 * np.abs(grad).max())
    picks = nz[rng.choice(len(nz), size=12, replace=False)]
    checked = 0
    for v, c in picks:
        h = 1e-4 * max(1.0, abs(grid.data[v, c]))
        gp, gm = grid.copy(), grid.copy()
        gp.data[v, c] += h
        gm.data[v, c] -= h
        # the device stores fp32: use the values it actually holds
        hp = np.float32(gp.data[v, c]) - np.float32(grid.data[v, c])
        hm = np.float32(grid.data[v, c]) - np.float32(gm.data[v, c])
        fd = (loss(gp) - loss(gm)) / (float(hp) + float(hm))
        if abs(fd) < 1e-7:
            continue
        assert grad[v, c] == pytest.approx(fd, rel=2e-2, abs=1e-6), (v, c)
        checked += 1
    assert checked >= 6
