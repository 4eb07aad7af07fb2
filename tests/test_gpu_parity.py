"""GPU parity: libvoxrf_b200 (sm_100a) against the CPU oracle on identical inputs.

Bars (BASELINE.json north_star): bit-exact sample schedules / cell ids /
occupancy decisions; colour and depth within 1e-4 relative; gradients within
1e-3 relative in deterministic mode; pose within 1 mm / 0.05 deg."""
import os
from pathlib import Path

import numpy as np
import pytest

from paper_2307_03404_b200.api import (GNConfig, MappingConfig, Pose, RenderParams,
                                       TrackingConfig, VoxelGrid)
from paper_2307_03404_b200 import synth

from scenes import fresh_grid, random_rays, room_scene

pytestmark = pytest.mark.gpu

RTOL_RENDER = 1e-4
RTOL_GRAD = 1e-3


def rel_err(a, b, floor):
    return np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor))


def test_sample_schedule_and_cell_ids_bit_exact(ctx, oracle):
    grid, intr, frames = room_scene()
    ctx.load_grid(grid)
    rays = random_rays(grid, 300)
    counts, t, delta, cells = ctx.sample_rays(rays, RenderParams(), cap=512)
    for i, row in enumerate(rays):
        t0, d0, c0 = oracle.sample_ray(grid, row[:3], row[3:], RenderParams())
        assert counts[i] == len(t0)
        assert np.array_equal(t[i, :counts[i]], t0)
        assert np.array_equal(delta[i, :counts[i]], d0)
        assert np.array_equal(cells[i, :counts[i]], c0)


def test_cell_location_on_lattice_faces_bit_exact(ctx, oracle):
    """Axis-aligned rays whose segment midpoints land on cell faces (g within an
    ulp of an integer, voxel 0.1 not representable): exact faces resolve to the
    lower cell (voxel_grid.cpp:88-90); the device's division-free locate must
    agree with the reference's IEEE division bit for bit."""
    rng = np.random.default_rng(11)
    geom = synth.GridGeometry((33, 33, 33), (0.0, 0.0, 0.0), 0.1)
    grid = VoxelGrid(geom, 1.0)
    grid.active[rng.uniform(size=geom.num_cells) < 0.3] = 0
    ctx.load_grid(grid)
    rays = []
    for axis in range(3):
        for sgn in (1.0, -1.0):
            for _ in range(40):
                o = rng.integers(1, 32, 3) * 0.1 + rng.choice([0.0, 0.05], 3)
                o[axis] = -0.1 if sgn > 0 else 3.3
                d = np.zeros(3)
                d[axis] = sgn
                rays.append(np.concatenate([o, d]))
    rays = np.array(rays)
    params = RenderParams(step=0.2, t_near=0.0)
    counts, t, delta, cells = ctx.sample_rays(rays, params, cap=64)
    for i, row in enumerate(rays):
        t0, d0, c0 = oracle.sample_ray(grid, row[:3], row[3:], params)
        assert counts[i] == len(t0)
        assert np.array_equal(cells[i, :counts[i]], c0)
        assert np.array_equal(t[i, :counts[i]], t0)


def test_render_rays_match_oracle(ctx, oracle):
    grid, intr, frames = room_scene()
    ctx.load_grid(grid)
    rays = random_rays(grid, 300, seed=9)
    out = ctx.render_rays(rays)
    for i, row in enumerate(rays):
        r = oracle.render_ray(grid, row[:3], row[3:], RenderParams())
        assert out[i, 5] == r.count and out[i, 6] == r.hit and out[i, 7] == r.terminated_early
        np.testing.assert_allclose(out[i, :3], r.color, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(out[i, 3], r.depth, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(out[i, 4], r.transmittance_terminal, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("stride", [1, 3])
def test_render_image_matches_oracle(ctx, oracle, stride):
    grid, intr, frames = room_scene()
    ctx.load_grid(grid)
    for f in frames:
        img = ctx.render_image(intr, f.gt_pose, RenderParams(), stride)
        c, d = oracle.render_image(grid, intr, f.gt_pose, RenderParams(), stride)
        assert rel_err(img.color, c, 1e-6) < RTOL_RENDER
        assert rel_err(img.depth, d, 1e-6) < RTOL_RENDER
        assert np.array_equal(img.depth > 0, d > 0)


def test_render_image_config1_shape(ctx, oracle):
    """160x120 frame of a 65^3 room grid (config 1 shape)."""
    grid = synth.scene_grid(65, seed=2)
    intr = synth.small_intrinsics()
    pose = synth.look_at((2.0, 1.2, 1.5), (2.0, 3.5, 1.5))
    ctx.load_grid(grid)
    img = ctx.render_image(intr, pose)
    c, d = oracle.render_image(grid, intr, pose, RenderParams())
    assert rel_err(img.color, c, 1e-6) < RTOL_RENDER
    assert rel_err(img.depth, d, 1e-6) < RTOL_RENDER
    # the scene is seen: most pixels hit a surface
    assert (d > 0).mean() > 0.9


def test_render_empty_grid_is_background(ctx):
    grid = VoxelGrid(synth.GridGeometry((4, 4, 4), (0, 0, 0), 0.25), 0.0)
    grid.set_all_active(False)
    ctx.load_grid(grid)
    intr = synth.CameraIntrinsics(60, 60, 16, 12, 32, 24)
    img = ctx.render_image(intr, synth.look_at((0.4, -1.2, 0.4), (0.4, 0.4, 0.4)))
    assert not img.color.any() and not img.depth.any()


@pytest.mark.parametrize("deterministic", [True, False])
def test_mapping_gradient_matches_oracle(ctx, oracle, deterministic):
    grid, intr, frames = room_scene()
    g0 = fresh_grid(grid)
    cfg = MappingConfig(deterministic=deterministic)
    batch = oracle.draw_batch(21, len(frames), intr.width, intr.height, 512)
    ctx.load_grid(g0)
    ctx.load_frames(intr, frames)
    grad, st = ctx.mapping_gradient(cfg, batch)
    _, _, grad_o, st_o = oracle.mapping_step(g0, frames, intr, cfg, batch, apply=False,
                                             want_grad=True)
    assert st.rays_color == st_o.rays_color and st.rays_depth == st_o.rays_depth
    assert st.samples == st_o.samples
    assert abs(st.loss_photometric - st_o.loss_photometric) <= 1e-9 * st_o.loss_photometric
    assert abs(st.loss_geometric - st_o.loss_geometric) <= 1e-9 * max(st_o.loss_geometric, 1e-12)
    touched_o = np.abs(grad_o).sum(1) > 0
    touched = np.abs(grad).sum(1) > 0
    assert np.array_equal(touched, touched_o)
    scale = np.abs(grad_o).max()
    if deterministic:
        # fp64 sorted/segmented reduce in the reference's order: agreement ~1e-12
        assert rel_err(grad, grad_o, 1e-9 * scale) < 1e-9
    else:
        assert rel_err(grad, grad_o, 1e-4 * scale) < RTOL_GRAD


@pytest.mark.parametrize("deterministic", [True, False])
def test_mapping_gradient_with_clamped_colour_and_free_space(ctx, oracle, deterministic):
    """Colours that clamp (SH coefficients up to +-1.5) and samples with sigma_raw
    <= 0 (sigma in [-0.3, 0.6]): the reference gates dL/dc per clamped channel and
    dL/dsigma on sigma_raw > 0 (gradients.cpp:69-97). The fast path carries both
    gates through its sample records (clamp flags in the colour sign bits, the
    sigma gate in the cell word, vrf_internal.h)."""
    grid, intr, frames = room_scene()
    g0 = fresh_grid(grid, seed=8, sh_noise=1.5)
    rng = np.random.default_rng(9)
    g0.data[:, 0] = rng.uniform(-0.3, 0.6, g0.data.shape[0]).astype(np.float32)
    cfg = MappingConfig(deterministic=deterministic)
    batch = oracle.draw_batch(22, len(frames), intr.width, intr.height, 512)
    ctx.load_grid(g0)
    ctx.load_frames(intr, frames)
    grad, st = ctx.mapping_gradient(cfg, batch)
    _, _, grad_o, st_o = oracle.mapping_step(g0, frames, intr, cfg, batch, apply=False,
                                             want_grad=True)
    assert st.rays_color == st_o.rays_color and st.samples == st_o.samples
    # (the fast forward contracts SH in fp32: ~1e-7 per channel at these coefficients)
    ltol = 1e-9 if deterministic else 1e-6
    assert abs(st.loss_photometric - st_o.loss_photometric) <= ltol * st_o.loss_photometric
    # the clamp gate fires: some colour rows of touched vertices are exactly zero in
    # the reference (every contributing sample clamped that channel). Samples with
    # sigma_raw <= 0 have w = 0 and a gated dL/dsigma, so the vertices only they
    # reach stay untouched: the zero patterns below must agree exactly.
    touched_o = np.abs(grad_o).sum(1) > 0
    assert np.any((grad_o[touched_o, 1:10] == 0).all(1))
    assert np.mean(g0.data[:, 0] < 0) > 0.25
    assert np.array_equal(np.abs(grad).sum(1) > 0, touched_o)
    assert np.array_equal(grad == 0, grad_o == 0)
    scale = np.abs(grad_o).max()
    tol = 1e-9 if deterministic else RTOL_GRAD
    assert rel_err(grad, grad_o, (1e-9 if deterministic else 1e-4) * scale) < tol


def test_deterministic_gradient_is_bit_reproducible(ctx, oracle):
    grid, intr, frames = room_scene()
    g0 = fresh_grid(grid, seed=4)
    cfg = MappingConfig(deterministic=True)
    batch = oracle.draw_batch(5, len(frames), intr.width, intr.height, 1024)
    ctx.load_grid(g0)
    ctx.load_frames(intr, frames)
    a, _ = ctx.mapping_gradient(cfg, batch)
    b, _ = ctx.mapping_gradient(cfg, batch)
    assert np.array_equal(a, b)


def test_deterministic_gradient_chunked_equals_unchunked(ctx, oracle, monkeypatch):
    """Deterministic mode split into many ray chunks keeps the single sequential
    accumulation order: bit-identical to the one-chunk result."""
    grid, intr, frames = room_scene()
    g0 = fresh_grid(grid, seed=6)
    cfg = MappingConfig(deterministic=True)
    batch = oracle.draw_batch(8, len(frames), intr.width, intr.height, 700)
    ctx.load_grid(g0)
    ctx.load_frames(intr, frames)
    whole, _ = ctx.mapping_gradient(cfg, batch)
    monkeypatch.setenv("VRF_DET_CHUNK", "500")
    chunked, st = ctx.mapping_gradient(cfg, batch)
    assert st.samples > 5 * 500  # really several chunks
    assert np.array_equal(whole, chunked)


def test_mapping_step_matches_oracle(ctx, oracle):
    """One full mapping_step (RGB+depth loss, RMSProp) vs the oracle, then a second
    step on top (RMSProp state carried on device)."""
    grid, intr, frames = room_scene()
    g0 = fresh_grid(grid)
    cfg = MappingConfig(deterministic=True)
    ctx.load_grid(g0)
    ctx.load_frames(intr, frames)
    ctx.rmsprop_reset()
    data, v = g0.data, None
    gcur = g0
    for step in range(2):
        batch = oracle.draw_batch(100 + step, len(frames), intr.width, intr.height, 512)
        st = ctx.mapping_step(cfg, batch)
        data, v, _, st_o = oracle.mapping_step(gcur, frames, intr, cfg, batch, rms_v=v)
        gcur = VoxelGrid.__new__(VoxelGrid)
        gcur.geom, gcur.data, gcur.active = g0.geom, data, g0.active
        assert st.rays_color == st_o.rays_color
        np.testing.assert_allclose(st.loss_total, st_o.loss_total, rtol=1e-5)
        dev = ctx.download_grid().data
        # device stores fp32 parameters: compare at fp32 resolution of the update
        np.testing.assert_allclose(dev, data, rtol=2e-5, atol=2e-5 * np.abs(data).max())


def test_mapping_errors_follow_the_reference(ctx, oracle):
    grid, intr, frames = room_scene()
    ctx.load_grid(fresh_grid(grid))
    ctx.load_frames(intr, frames)
    with pytest.raises(IndexError):
        ctx.mapping_step(MappingConfig(), np.array([[0, intr.width, 0]]))
    # all rays miss: a grid with every cell inactive
    g = fresh_grid(grid)
    g.set_all_active(False)
    ctx.load_grid(g)
    with pytest.raises(RuntimeError, match="no ray hit the grid"):
        ctx.mapping_step(MappingConfig(), np.array([[0, 1, 1], [1, 2, 2]]))
    assert np.array_equal(ctx.download_grid().data, g.data)
    # an empty batch (rays_per_batch = 0) has no hits either (mapping.cpp:151),
    # in the fast and the deterministic mode, and leaves the grid as it was
    ctx.load_grid(fresh_grid(grid))
    before = ctx.download_grid().data.copy()
    for det in (False, True):
        with pytest.raises(RuntimeError, match="no ray hit the grid"):
            ctx.mapping_step(MappingConfig(deterministic=det), np.zeros((0, 3), np.int32))
    assert np.array_equal(ctx.download_grid().data, before)


def test_pose_gradient_matches_oracle(ctx, oracle):
    grid, intr, frames = room_scene()
    frame = frames[1]
    ctx.load_grid(grid)
    ctx.load_frames(intr, frames)
    rng = np.random.default_rng(3)
    px = np.stack([rng.integers(0, intr.width, 300), rng.integers(0, intr.height, 300)], 1)
    pose = Pose(frame.gt_pose.q, tuple(np.asarray(frame.gt_pose.t) + [0.01, -0.02, 0.005]))
    tc = TrackingConfig()
    g = ctx.pose_gradient(1, intr, pose, px, tc)
    o = oracle.pose_gradient(grid, frame, intr, pose, px, 1.0, 1.0, RenderParams())
    assert g.rays_used == o.rays_used
    ref_vec = np.concatenate([o.d_omega, o.d_tau])
    got = np.concatenate([g.d_omega, g.d_tau])
    assert rel_err(got, ref_vec, 1e-6 * np.abs(ref_vec).max()) < 1e-6
    assert abs(g.loss - o.loss) <= 1e-9 * o.loss
    ne = ctx.pose_normal_equations(1, intr, pose, px, TrackingConfig(lambda_d=0.5))
    no = oracle.normal_eqs(grid, frame, intr, pose, px, 1.0, 0.5, RenderParams())
    from paper_2307_03404_b200.api import unpack_sym6
    jo = unpack_sym6(no.jtj)
    assert rel_err(ne.jtj, jo, 1e-6 * np.abs(jo).max()) < 1e-6
    assert rel_err(ne.jtr, np.array(no.jtr), 1e-6 * np.abs(no.jtr).max()) < 1e-6


def test_track_frame_adam_matches_oracle(ctx, oracle):
    grid, intr, frames = room_scene()
    frame = frames[2]
    ctx.load_grid(grid)
    ctx.load_frames(intr, frames)
    init = Pose(frame.gt_pose.q, tuple(np.asarray(frame.gt_pose.t) + [0.02, 0.0, -0.01]))
    tc = TrackingConfig(rays_per_iteration=256, iterations=10)
    r = ctx.track_frame(2, intr, init, tc)
    o, trace = oracle.track_frame(grid, frame, intr, init, tc)
    assert r.iterations_run == o.iterations_run
    np.testing.assert_allclose(r.loss_trace, trace, rtol=1e-6)
    assert np.linalg.norm(np.asarray(r.pose.t) - np.array(o.pose.t)) < 1e-3  # 1 mm
    dq = abs(float(np.dot(r.pose.q, np.array(o.pose.q))))
    assert 2 * np.degrees(np.arccos(min(1.0, dq))) < 0.05


def test_track_frame_gn_converges(ctx):
    grid, intr, frames = room_scene(res=33, width=64, height=48)
    frame = frames[1]
    ctx.load_grid(grid)
    ctx.load_frames(intr, frames)
    gt = np.asarray(frame.gt_pose.t)
    init = Pose(frame.gt_pose.q, tuple(gt + [0.03, -0.02, 0.01]))
    r = ctx.track_frame_gn(1, intr, init, GNConfig(rays_per_iteration=2048, iterations=8))
    err0 = np.linalg.norm(np.asarray(init.t) - gt)
    err1 = np.linalg.norm(np.asarray(r.pose.t) - gt)
    assert err1 < 0.5 * err0


def test_prune_matches_host_prune(ctx):
    grid = synth.scene_grid(33, seed=2, prune_tau=0.0)
    ctx.load_grid(grid)
    n = ctx.prune(1e-3)
    host = grid.copy()
    n_host = synth.prune(host, 1e-3)
    assert n == n_host
    assert np.array_equal(ctx.download_grid().active, host.active)


def test_upsample_matches_oracle(ctx, oracle):
    """Device VoxelGrid::upsampled: the fp64 trilinear replay over the fp32 payload,
    stored in fp32, equals the reference's double result rounded to fp32; the
    occupancy and geometry match exactly; RMSProp restarts at zero."""
    grid = fresh_grid(synth.scene_grid(17, seed=2, prune_tau=1e-3), sh_noise=0.3)
    ctx.load_grid(grid)
    ctx.upsample(64)
    (res, origin, voxel), data, act = oracle.upsample(grid, 64)
    assert tuple(ctx.geom.res) == res and ctx.geom.voxel_size == voxel
    out = ctx.download_grid()
    assert np.array_equal(out.active, act)
    assert np.array_equal(ctx.download_payload_f32(), data.astype(np.float32))
    assert not ctx.rmsprop_v().any()
    with pytest.raises(RuntimeError, match="exceed configured maximum"):
        ctx.upsample(64)
    # the refined grid renders like the oracle's refined grid
    fine = VoxelGrid(synth.GridGeometry(res, origin, voxel))
    fine.data[:] = data.astype(np.float32)
    fine.active[:] = act
    rays = random_rays(fine, 64)
    rr = ctx.render_rays(rays, RenderParams())
    for i, row in enumerate(rays):
        r0 = oracle.render_ray(fine, row[:3], row[3:], RenderParams())
        assert rel_err(rr[i, 3], r0.depth, 1e-3) < RTOL_RENDER


def test_vxgf_roundtrip_with_reference(ctx, ref, tmp_path):
    """.vxgf written from HBM loads in the reference with the same checksum, and a
    reference-written file loads into HBM bit for bit (voxel_grid.cpp:222-278)."""
    grid = fresh_grid(synth.scene_grid(17, seed=2, prune_tau=1e-3), sh_noise=0.3)
    ctx.load_grid(grid)
    path = tmp_path / "dev.vxgf"
    ctx.save_grid(path)
    h = ref.load(path)
    h0 = ref.grid(grid)
    try:
        assert ref.lib.ref_grid_checksum(h) == ref.lib.ref_grid_checksum(h0)
        rpath = tmp_path / "ref.vxgf"
        ref.save(h0, rpath)
        assert rpath.read_bytes() == path.read_bytes()
    finally:
        ref.lib.ref_grid_destroy(h)
        ref.lib.ref_grid_destroy(h0)
    ctx.init_grid(synth.GridGeometry((5, 5, 5), (0.0, 0.0, 0.0), 0.5), 0.0)
    ctx.load_grid_file(rpath)
    assert tuple(ctx.geom.res) == tuple(grid.geom.res)
    out = ctx.download_grid()
    assert np.array_equal(out.data, grid.data) and np.array_equal(out.active, grid.active)
    # error contract (test_voxel_grid.cpp:386-402)
    bad = tmp_path / "bad.vxgf"
    bad.write_bytes(b"NOPE" + path.read_bytes()[4:])
    with pytest.raises(RuntimeError, match="bad magic"):
        ctx.load_grid_file(bad)
    vers = tmp_path / "vers.vxgf"
    vers.write_bytes(path.read_bytes()[:4] + b"\x02\x00\x00\x00" + path.read_bytes()[8:])
    with pytest.raises(RuntimeError, match="unsupported version"):
        ctx.load_grid_file(vers)
    trunc = tmp_path / "trunc.vxgf"
    trunc.write_bytes(path.read_bytes()[:-3])
    with pytest.raises(RuntimeError, match="truncated payload"):
        ctx.load_grid_file(trunc)
    nan = bytearray(path.read_bytes())
    nan[52:56] = np.array([np.nan], np.float32).tobytes()
    (tmp_path / "nan.vxgf").write_bytes(bytes(nan))
    with pytest.raises(RuntimeError, match="non-finite payload"):
        ctx.load_grid_file(tmp_path / "nan.vxgf")
    with pytest.raises(RuntimeError, match="cannot open"):
        ctx.load_grid_file(tmp_path / "missing.vxgf")


@pytest.mark.parametrize("deterministic", [True, False])
def test_mapping_steps_pipeline_equals_step_loop(ctx, deterministic):
    """vrf_mapping_steps (draw of batch i+1 overlapped with step i) == the plain
    loop of Rng draw + mapping_step (mapping.cpp:302-312)."""
    from paper_2307_03404_b200.api import Rng
    grid, intr, frames = room_scene()
    cfg = MappingConfig(rays_per_batch=700, deterministic=deterministic)
    start = fresh_grid(grid)
    ctx.load_grid(start)
    ctx.load_frames(intr, frames)
    ctx.rmsprop_reset()
    r1 = Rng(5)
    a = ctx.mapping_steps(cfg, r1, len(frames), 4)
    ga = ctx.download_grid().data
    ctx.load_grid(start)
    ctx.rmsprop_reset()
    r2 = Rng(5)
    b = [ctx.mapping_step(cfg, r2.draw_batch(len(frames), intr.width, intr.height, 700))
         for _ in range(4)]
    gb = ctx.download_grid().data
    assert r1.next_u64() == r2.next_u64()
    for x, y in zip(a, b):
        assert x.rays_color == y.rays_color and x.samples == y.samples
        if deterministic:
            assert x.loss_total == y.loss_total
        else:
            assert x.loss_total == pytest.approx(y.loss_total, rel=1e-5)
    if deterministic:
        assert np.array_equal(ga, gb)
    else:
        assert np.max(np.abs(ga - gb)) <= 1e-4 * np.max(np.abs(gb))
    with pytest.raises(ValueError, match="keyframe index out of range"):
        ctx.mapping_steps(cfg, r1, len(frames) + 1, 1)


def test_upsample_far_corner_where_the_reference_throws(ctx, oracle):
    """VoxelGrid::upsampled's world round trip can put the far-corner vertices an
    ulp outside the box, and the reference then throws out_of_range from locate
    (voxel_grid.cpp:203-206, 107-111; e.g. map_scene on room_scene's fitted
    geometry). The device clamps those points to the box instead; with that
    single difference it matches the oracle bit for bit."""
    from paper_2307_03404_b200.api import fit_grid_geometry
    grid, intr, frames = room_scene()
    cfg = MappingConfig(initial_resolution=9)
    geom = fit_grid_geometry(frames, list(range(len(frames))), intr, cfg)
    g0 = fresh_grid(VoxelGrid(geom, 0.0), sigma_init=0.3, sh_noise=0.3)
    with pytest.raises(IndexError):
        oracle.upsample(g0, 64)  # the reference behaviour
    (res, origin, voxel), data, act = oracle.upsample(g0, 64, clamp_outside=True)
    ctx.load_grid(g0)
    ctx.upsample(64)
    assert tuple(ctx.geom.res) == res
    assert np.array_equal(ctx.download_payload_f32(), data.astype(np.float32))


def test_sparse_schedule_with_superblock_jumps_bit_exact(ctx, oracle):
    """Empty-space jumps over 8^3 blocks and 64^3 superblocks leave the sample
    schedule unchanged (renderer.cpp:62-79): a 129^3 grid whose only active cells
    form a thin spherical shell, random rays from inside and outside it."""
    rng = np.random.default_rng(21)
    n = 129
    geom = synth.GridGeometry((n, n, n), (-3.2, -3.2, -3.2), 0.05)
    grid = VoxelGrid(geom, 2.0)
    c = (np.arange(n - 1) + 0.5) * 0.05 - 3.2
    zz, yy, xx = np.meshgrid(c, c, c, indexing="ij")
    r = np.sqrt(xx ** 2 + yy ** 2 + zz ** 2)
    grid.active[:] = (np.abs(r - 1.5) < 0.08).reshape(-1).astype(np.uint8)
    ctx.load_grid(grid)
    o = rng.uniform(-2.5, 2.5, (200, 3))
    d = rng.normal(size=(200, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rays = np.concatenate([o, d], axis=1)
    params = RenderParams(termination_eps=0.0)  # never terminate: walk every segment
    counts, t, delta, cells = ctx.sample_rays(rays, params, cap=4096)
    nonempty = 0
    for i, row in enumerate(rays):
        t0, d0, c0 = oracle.sample_ray(grid, row[:3], row[3:], params, cap=4096)
        assert counts[i] == len(t0)
        assert np.array_equal(t[i, :counts[i]], t0)
        assert np.array_equal(cells[i, :counts[i]], c0)
        nonempty += len(t0) > 0
    assert nonempty > 30


def test_block_sparse_rmsprop_matches_full_scan(tmp_path):
    """The block-sparse RMSProp (touched 8^3-vertex blocks marked by the scatter)
    updates exactly the groups the full scan updates: two fast mapping steps with
    and without VRF_RMSPROP_FULL agree to fp32 atomics-order noise."""
    import subprocess
    import sys as _sys
    script = r'''
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, "."); sys.path.insert(0, "oracle")
from scenes import room_scene, fresh_grid
from paper_2307_03404_b200 import Context, MappingConfig, Rng
grid, intr, frames = room_scene(res=33)
ctx = Context(0)
ctx.load_grid(fresh_grid(grid)); ctx.load_frames(intr, frames); ctx.rmsprop_reset()
ctx.mapping_steps(MappingConfig(rays_per_batch=2000), Rng(3), len(frames), 2)
np.save(sys.argv[1], ctx.download_payload_f32())
'''
    outs = []
    for full in (False, True):
        env = dict(os.environ)
        if full:
            env["VRF_RMSPROP_FULL"] = "1"
        f = tmp_path / f"p{int(full)}.npy"
        subprocess.run([_sys.executable, "-c", script, str(f)], check=True, env=env,
                       cwd=str(Path(__file__).resolve().parent.parent))
        outs.append(np.load(f))
    a, b = outs
    assert np.max(np.abs(a - b)) <= 1e-4 * np.max(np.abs(b))


def test_sensor_format_frames_equal_the_double_path(ctx, oracle):
    """vrf_frame_set_u8u16 (8-bit RGB, 16-bit depth) converts exactly like the
    reference's PNG loaders: tracking on it equals tracking on the double frame
    (including the Adam path's host depth, fetched back from the device)."""
    from paper_2307_03404_b200.api import TrackingConfig
    grid, intr, frames = room_scene()
    ctx.load_grid(grid)
    ctx.reserve_frames(intr, 2)
    f = frames[1]
    rgb = np.clip(np.floor(f.color * 255.0 + 0.5), 0, 255).astype(np.uint8)
    du = np.where(f.depth > 0, np.floor(f.depth * intr.depth_scale + 0.5), 0).astype(np.uint16)
    ctx.set_frame(0, f, f.gt_pose)
    ctx.set_frame_u8u16(1, rgb, du, f.gt_pose)
    cfg = TrackingConfig(rays_per_iteration=256, iterations=5)
    init = frames[0].gt_pose
    a = ctx.track_frame(0, intr, init, cfg)
    b = ctx.track_frame(1, intr, init, cfg)
    assert np.array_equal(np.asarray(a.pose.t), np.asarray(b.pose.t))
    assert a.loss_trace == b.loss_trace


def test_small_batch_group_kernels_equal_thread_kernels(tmp_path):
    """K0g / K2g (8 lanes per ray, small batches) against the thread-per-ray K0 /
    K2 (VRF_FWD_GROUP_MAX=VRF_BWD_GROUP_MAX=0): the same composited samples and hit counts,
    the same loss to the last bits of the fixed-order block sums, and one fast
    mapping step's gradient to fp32 atomics-order noise."""
    import subprocess
    import sys as _sys
    script = r'''
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, "."); sys.path.insert(0, "oracle")
from scenes import room_scene, fresh_grid
from paper_2307_03404_b200 import Context, MappingConfig
import oracle as orc
grid, intr, frames = room_scene(res=33)
ctx = Context(0)
ctx.load_grid(fresh_grid(grid)); ctx.load_frames(intr, frames)
batch = orc.Oracle().draw_batch(5, len(frames), intr.width, intr.height, 3000)
g, st = ctx.mapping_gradient(MappingConfig(), batch)
np.savez(sys.argv[1], g=g, s=np.array([st.samples, st.rays_color, st.rays_depth]),
         l=np.array([st.loss_photometric, st.loss_geometric]))
'''
    outs = []
    for thread in (False, True):
        env = dict(os.environ)
        if thread:
            env["VRF_FWD_GROUP_MAX"] = "0"
            env["VRF_BWD_GROUP_MAX"] = "0"
        f = tmp_path / f"k{int(thread)}.npz"
        subprocess.run([_sys.executable, "-c", script, str(f)], check=True, env=env,
                       cwd=str(Path(__file__).resolve().parent.parent))
        outs.append(np.load(f))
    a, b = outs
    assert np.array_equal(a["s"], b["s"])
    np.testing.assert_allclose(a["l"], b["l"], rtol=1e-13)
    assert np.max(np.abs(a["g"] - b["g"])) <= 1e-4 * np.max(np.abs(b["g"]))


@pytest.mark.parametrize("n_rays", [60000, 200000])
def test_fast_gradient_matches_deterministic_at_larger_batches(ctx, oracle, n_rays):
    """The fast gradient against the deterministic FP64 one at batch sizes where
    the kernel variants switch: 60K rays run K0 (thread) + K2g (8 lanes), 200K
    run K0 + the merged queued K2q. Tolerance: the fast path's fp32 records and
    reductions (1e-3 relative to the gradient scale)."""
    grid, intr, frames = room_scene(res=33, width=64, height=48)
    g0 = fresh_grid(grid, seed=9)
    batch = oracle.draw_batch(21, len(frames), intr.width, intr.height, n_rays)
    ctx.load_grid(g0)
    ctx.load_frames(intr, frames)
    fast, sf = ctx.mapping_gradient(MappingConfig(), batch)
    det, sd = ctx.mapping_gradient(MappingConfig(deterministic=True), batch)
    assert sf.samples == sd.samples and sf.rays_color == sd.rays_color
    scale = np.abs(det).max()
    assert np.max(np.abs(fast - det)) <= 1e-3 * scale
    assert np.array_equal(fast != 0, det != 0)


def test_k2q_three_ctas_per_sm_matches_deterministic(tmp_path):
    """The 3-CTA/SM K2q build that grids of >= 64M vertices run (config 4), forced
    at 200K rays with VRF_K2_MINB3_VERTS=0: the fast gradient against the
    deterministic FP64 one at the same 1e-3 tolerance, same touched set."""
    import subprocess
    import sys as _sys
    script = r'''
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, "."); sys.path.insert(0, "oracle")
from scenes import room_scene, fresh_grid
from paper_2307_03404_b200 import Context, MappingConfig
import oracle as orc
grid, intr, frames = room_scene(res=33, width=64, height=48)
ctx = Context(0)
ctx.load_grid(fresh_grid(grid, seed=9)); ctx.load_frames(intr, frames)
batch = orc.Oracle().draw_batch(21, len(frames), intr.width, intr.height, 200000)
fast, sf = ctx.mapping_gradient(MappingConfig(), batch)
det, sd = ctx.mapping_gradient(MappingConfig(deterministic=True), batch)
np.savez(sys.argv[1], fast=fast, det=det, s=np.array([sf.samples, sd.samples]))
'''
    f = tmp_path / "k2q3.npz"
    env = dict(os.environ, VRF_K2_MINB3_VERTS="0")
    subprocess.run([_sys.executable, "-c", script, str(f)], check=True, env=env,
                   cwd=str(Path(__file__).resolve().parent.parent))
    d = np.load(f)
    assert d["s"][0] == d["s"][1]
    scale = np.abs(d["det"]).max()
    assert np.max(np.abs(d["fast"] - d["det"])) <= 1e-3 * scale
    assert np.array_equal(d["fast"] != 0, d["det"] != 0)


def test_synth_from_grid_matches_oracle_renders(ctx, oracle):
    """synth_from_grid (dataset.cpp:443-462) on the device: the quantised frames
    equal the oracle's render_image quantised the same way (renders agree to
    1e-12, so only exact quantisation ties could differ)."""
    grid, intr, frames = room_scene(res=33, width=64, height=48)
    poses = [f.gt_pose for f in frames]
    got = synth.synth_from_grid(ctx, grid, poses, [0.0, 1.0, 2.0][:len(poses)], intr)
    for f, p in zip(got, poses):
        c, d = oracle.render_image(grid, intr, p, RenderParams())
        cq, dq = synth.quantize_frame(c, d, intr.depth_scale)
        assert np.mean(f.color != cq) < 1e-3 and np.mean(f.depth != dq) < 1e-3
        assert f.gt_pose is p


def test_grid_digest_tracks_mutation_only(ctx, oracle):
    """vrf_grid_digest (device-side integrity check): unchanged by rendering and
    tracking (tracking never mutates the grid), changed by a mapping
    step, an occupancy change or a single payload float."""
    grid, intr, frames = room_scene()
    ctx.load_grid(grid)
    ctx.load_frames(intr, frames)
    d0 = ctx.grid_digest()
    assert d0 == ctx.grid_digest()
    ctx.render_image(intr, frames[1].gt_pose)
    rng = np.random.default_rng(1)
    px = np.stack([rng.integers(0, intr.width, 64), rng.integers(0, intr.height, 64)], 1)
    ctx.pose_gradient(1, intr, frames[1].gt_pose, px, TrackingConfig())
    ctx.track_frame(1, intr, frames[1].gt_pose, TrackingConfig(rays_per_iteration=128,
                                                               iterations=3))
    ctx.track_frame_gn(1, intr, frames[1].gt_pose, GNConfig(rays_per_iteration=256,
                                                            iterations=2))
    assert ctx.grid_digest() == d0
    g = grid.copy()
    g.data[17, 5] = np.float32(g.data[17, 5] + 0.5)
    ctx.load_grid(g)
    assert ctx.grid_digest() != d0
    g2 = grid.copy()
    g2.active[3] = not g2.active[3]
    ctx.load_grid(g2)
    assert ctx.grid_digest() != d0
    ctx.load_grid(grid)
    assert ctx.grid_digest() == d0
    ctx.load_grid(fresh_grid(grid))
    d1 = ctx.grid_digest()
    ctx.mapping_step(MappingConfig(), oracle.draw_batch(3, len(frames), intr.width,
                                                        intr.height, 256))
    assert ctx.grid_digest() != d1
