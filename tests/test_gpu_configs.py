"""Parity at BASELINE.json's own config shapes, on the GPU.

* Config 3's scene (257^3-vertex room, 1200x680 keyframes): the fast mapping
  gradient (K0 records + K2q, and the record-overflow backward) against the
  deterministic FP64 one on a 65,536-ray batch — the regime of the headline
  bench (index widths, record caps, the queued scatter).
* The record-overflow backward (rays longer than the record cap re-march) and
  the record-free configuration, forced with vrf_set_record_limits, on the
  batch sizes where the K2 variants switch (K2g <= 160K rays < K2q).
* Configs 1 and 2 against the reference build (oracle/_ref, the reference's
  own TUs): map_scene + track_sequence at config 1's shapes, and the Adam
  track_frame at config 2's. Reduced iteration counts keep the CPU side to
  seconds; the shapes are the configs'.

Tolerances: the fast path's fp32 records and reductions, 1e-3 relative to the
gradient scale (north_star); trajectories within 1 mm / 0.05 deg.
"""
import math

import numpy as np
import pytest

from paper_2307_03404_b200 import synth
from paper_2307_03404_b200.api import (Frame, GridGeometry, MappingConfig, Pose, TrackingConfig,
                                       VoxelGrid)
import paper_2307_03404_b200.api as api

from scenes import fresh_grid, room_scene

pytestmark = pytest.mark.gpu

RTOL_GRAD = 1e-3


def _render(ctx, intr, poses):
    out = []
    for i, p in enumerate(poses):
        img = ctx.render_image(intr, p)
        c, d = synth.quantize_frame(img.color, img.depth, intr.depth_scale)
        out.append(Frame(c, d, i / 30.0, p))
    return out


def _fast_vs_det(ctx, batch, limits=None):
    if limits is not None:
        ctx.set_record_limits(max_k=limits)
    try:
        fast, sf = ctx.mapping_gradient(MappingConfig(), batch)
    finally:
        ctx.set_record_limits()
    det, sd = ctx.mapping_gradient(MappingConfig(deterministic=True), batch)
    assert sf.samples == sd.samples and sf.rays_color == sd.rays_color
    assert sf.rays_depth == sd.rays_depth
    scale = np.abs(det).max()
    assert np.max(np.abs(fast - det)) <= RTOL_GRAD * scale
    assert np.array_equal(fast != 0, det != 0)
    return sf


@pytest.mark.parametrize("n_rays", [60000, 200000])
@pytest.mark.parametrize("max_k", [4, 0])
def test_record_overflow_and_record_free_backward(ctx, oracle, n_rays, max_k):
    """max_k = 4: most rays of this scene have more samples than 4 and take the
    recompute-march backward (kOverflow), the rest the record walk (K2g at 60K
    rays, K2q at 200K). max_k = 0: no records at all."""
    grid, intr, frames = room_scene(res=33, width=64, height=48)
    g0 = fresh_grid(grid, seed=11)
    batch = oracle.draw_batch(23, len(frames), intr.width, intr.height, n_rays)
    ctx.load_grid(g0)
    ctx.load_frames(intr, frames)
    st = _fast_vs_det(ctx, batch, limits=max_k)
    assert st.samples > 4 * st.rays_color  # rays are longer than the cap on average


@pytest.fixture(scope="module")
def config3(ctx):
    """Config 3's scene: the 257^3 room map renders 1200x680 keyframes; the map
    being trained starts at sigma 0.1 with small SH noise (all cells active)."""
    room = synth.Room().scaled(7.0 / 4.0, 6.0 / 4.0, 1.0)
    gt = synth.scene_grid(257, room, seed=2, prune_tau=1e-3)
    intr = synth.replica_intrinsics()
    poses = synth.room_path(30, room, seed=4)[::10]
    ctx.load_grid(gt)
    frames = _render(ctx, intr, poses)
    g0 = VoxelGrid(gt.geom, 0.1)
    rng = np.random.default_rng(5)
    g0.data[:, 1:] = rng.uniform(-0.05, 0.05, g0.data[:, 1:].shape).astype(np.float32)
    return g0, intr, frames


@pytest.mark.slow
@pytest.mark.parametrize("max_k", [None, 64])
def test_config3_fast_gradient_matches_deterministic(ctx, config3, max_k):
    g0, intr, frames = config3
    ctx.load_grid(g0)
    ctx.load_frames(intr, frames)
    rng = api.Rng(3)
    batch = rng.draw_batch(len(frames), intr.width, intr.height, 65536)
    st = _fast_vs_det(ctx, batch, limits=max_k)
    assert st.samples > 100 * st.rays_color  # the long rays of the headline regime


def _traj_close(a, b, dt_m=1e-3, dr_deg=0.05):
    for x, y in zip(a, b):
        assert np.linalg.norm(np.asarray(x.t) - np.asarray(y.t)) < dt_m
        dq = abs(float(np.dot(x.q, y.q)))
        assert 2 * math.degrees(math.acos(min(1.0, dq))) < dr_deg


@pytest.mark.slow
def test_config1_map_scene_and_track_sequence_match_reference(ctx, ref):
    """Config 1 (65^3, 160x120, 10 frames, keyframe_stride 1, 4096-ray batches):
    map_scene in deterministic mode for 40 iterations, GPU vs the reference's
    own map_scene (1 thread, its deterministic setting); then track_sequence
    (Adam, 2048 x 40, previous-pose init) on the GPU-mapped grid, GPU vs
    reference."""
    room = synth.Room()
    gt = synth.scene_grid(65, room, seed=2, prune_tau=1e-3)
    intr = synth.small_intrinsics()
    poses = synth.circle_trajectory(10, (2.0, 2.0, 0.0), 0.8, 1.5, (2.0, 3.5, 1.5), arc_deg=9.0)
    ctx.load_grid(gt)
    frames = _render(ctx, intr, poses)
    geom = GridGeometry((65, 65, 65), (-0.2, -0.2, -0.7), 4.4 / 64)
    mcfg = MappingConfig(keyframe_stride=1, rays_per_batch=4096, iterations_per_stage=40,
                         upsample_stages=0, sigma_init=0.1, seed=1, deterministic=True)
    grid_gpu, log = api.map_scene(frames, intr, mcfg, geom, ctx=ctx)
    fh = ref.frames(frames, intr)
    try:
        h, cpu_loss, _ = ref.map_scene(fh, intr, mcfg, geom, threads=1)
        cpu_grid = ref.read_grid(h, geom.num_vertices)
        ref.lib.ref_grid_destroy(h)
        np.testing.assert_allclose(log[-1][1].loss_total, cpu_loss, rtol=1e-4)
        # fp32 device parameters against the reference's fp64 ones after 40 steps.
        # RMSProp normalises each update (lr g / sqrt(v + eps)), so a vertex whose
        # gradient is at rounding level in both can take differently signed steps
        # of up to lr: a few outliers are expected, the bulk must agree.
        d = np.abs(grid_gpu.data - cpu_grid)
        scale = np.abs(cpu_grid).max()
        assert np.mean(d <= 1e-4 * scale) >= 0.999, np.quantile(d, [0.5, 0.99, 0.999, 1.0])
        assert np.sqrt(np.mean(d * d)) <= 1e-3 * np.sqrt(np.mean(cpu_grid * cpu_grid))
        tcfg = TrackingConfig()
        gpu_poses, _ = api.track_sequence(grid_gpu, frames, intr, tcfg, ctx=ctx)
        gh = ref.grid(grid_gpu)
        cpu_p, _ = ref.track_sequence(gh, fh, intr, tcfg, len(frames), threads=1)
        ref.lib.ref_grid_destroy(gh)
    finally:
        ref.lib.ref_frames_destroy(fh)
    _traj_close(gpu_poses, [Pose(q, t) for q, t in cpu_p])


@pytest.mark.slow
def test_config2_adam_track_frame_matches_reference(ctx, ref):
    """Config 2 (257^3 map, 1200x680): the reference's Adam tracker (2048 rays x
    40 iterations, its pixel stream) from the previous frame's pose, GPU vs the
    reference build, on three frames."""
    room = synth.Room().scaled(7.0 / 4.0, 6.0 / 4.0, 1.0)
    gt = synth.scene_grid(257, room, seed=2, prune_tau=1e-3)
    intr = synth.replica_intrinsics()
    poses = synth.room_path(4, room, seed=4)
    ctx.load_grid(gt)
    frames = _render(ctx, intr, poses)
    tcfg = TrackingConfig()
    gpu_poses, _ = api.track_sequence(gt, frames, intr, tcfg, ctx=ctx)
    gh = ref.grid(gt)
    fh = ref.frames(frames, intr)
    try:
        cpu_p, _ = ref.track_sequence(gh, fh, intr, tcfg, len(frames), threads=0)
    finally:
        ref.lib.ref_grid_destroy(gh)
        ref.lib.ref_frames_destroy(fh)
    _traj_close(gpu_poses, [Pose(q, t) for q, t in cpu_p])


def test_update_log_and_partial_writes(ctx, oracle):
    """The drop-in's residency primitives: the RMSProp update log holds exactly the
    float4 groups a step changed (with their new theta and v), and partial vertex
    writes land where they should."""
    import ctypes as C
    from paper_2307_03404_b200 import _capi as capi
    grid, intr, frames = room_scene(res=17)
    g0 = fresh_grid(grid, seed=4)
    ctx.load_grid(g0)
    ctx.load_frames(intr, frames)
    ctx.rmsprop_reset()
    lib, h = ctx._lib, ctx._h
    before = ctx.download_payload_f32().reshape(-1, 7, 4).copy()
    assert lib.vrf_track_updates(h, 1) == 0
    try:
        ctx.mapping_step(MappingConfig(), oracle.draw_batch(2, len(frames), intr.width,
                                                            intr.height, 300))
        n = C.c_int64()
        assert lib.vrf_updates_count(h, C.byref(n)) == 0 and n.value > 0
        ids = np.zeros(n.value, np.uint32)
        th = np.zeros((n.value, 4), np.float32)
        vv = np.zeros((n.value, 4), np.float32)
        assert lib.vrf_updates_read(h, n.value, ids.ctypes.data, th.ctypes.data,
                                    vv.ctypes.data) == 0
        # the sorted, ranged read (the drop-in's chunked write-back): the same
        # entries in ascending id order, in two ranges
        k = n.value // 3
        sid = np.zeros(n.value, np.uint32)
        sth = np.zeros((n.value, 4), np.float32)
        svv = np.zeros((n.value, 4), np.float32)
        for a, b in ((0, k), (k, n.value)):
            assert lib.vrf_updates_read_range(h, a, b - a, 1, sid[a:].ctypes.data,
                                              sth[a:].ctypes.data, svv[a:].ctypes.data) == 0
        order = np.argsort(ids)
        assert np.array_equal(sid, ids[order])
        assert np.array_equal(sth, th[order]) and np.array_equal(svv, vv[order])
        part = np.zeros((5, 4), np.float32)
        assert lib.vrf_updates_read_range(h, 1, 5, 0, sid.ctypes.data, part.ctypes.data,
                                          svv.ctypes.data) == 0
        assert np.array_equal(part, th[1:6])
        assert lib.vrf_updates_read_range(h, n.value - 1, 2, 1, sid.ctypes.data,
                                          part.ctypes.data, svv.ctypes.data) != 0
    finally:
        lib.vrf_track_updates(h, 0)
    after = ctx.download_payload_f32().reshape(-1, 7, 4)
    # chunked fp32 state reads (payload and RMSProp v)
    nf = after.size
    got = np.zeros(nf, np.float32)
    for a in range(0, nf, 1000):
        c = min(1000, nf - a)
        assert lib.vrf_state_read_f32(h, 0, a, c, got[a:].ctypes.data) == 0
    assert np.array_equal(got, after.reshape(-1))
    assert lib.vrf_state_read_f32(h, 1, 0, nf, got.ctypes.data) == 0
    np.testing.assert_array_equal(got, ctx.rmsprop_v().reshape(-1).astype(np.float32))
    assert lib.vrf_state_read_f32(h, 2, 0, 1, got.ctypes.data) != 0
    assert lib.vrf_state_read_f32(h, 0, nf - 1, 2, got.ctypes.data) != 0
    flat_b, flat_a = before.reshape(-1, 4), after.reshape(-1, 4)
    assert len(np.unique(ids)) == len(ids)
    np.testing.assert_array_equal(flat_a[ids], th)
    changed = np.nonzero(np.any(flat_a != flat_b, axis=1))[0]
    assert set(changed.tolist()) <= set(ids.tolist())  # every change is logged
    np.testing.assert_array_equal(ctx.rmsprop_v().reshape(-1, 4)[ids].astype(np.float32), vv)
    # partial writes: vertices [5, 9) set on the device, the rest untouched
    src = np.full((4, 28), 0.25)
    assert lib.vrf_grid_write_vertices(h, 5, 4, src.ctypes.data) == 0
    got = ctx.download_payload_f32()
    assert np.all(got[5:9] == np.float32(0.25))
    np.testing.assert_array_equal(got[:5], after.reshape(-1, 28)[:5])
    np.testing.assert_array_equal(got[9:], after.reshape(-1, 28)[9:])
