"""ctypes binding of the CPU oracle — TEST INFRASTRUCTURE ONLY.

* ``Oracle``  -> oracle/liboracle_voxrf.so  (plain-C FP64 restatement, voxrf_oracle.c)
* ``RefLib``  -> oracle/_ref/libvoxrf_ref.so (the reference's own sources compiled
                 unchanged against oracle/shim; built by `make -C oracle ref`)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference arm
may import this module. The product (paper_2307_03404_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle_voxrf.so"
REF_SO = HERE / "_ref" / "libvoxrf_ref.so"
REF_SRC = Path("/root/reference/proj")


class Geometry(C.Structure):
    _fields_ = [("res", C.c_int32 * 3), ("origin", C.c_double * 3), ("voxel_size", C.c_double)]


class Grid(C.Structure):
    _fields_ = [("geom", Geometry), ("data", C.c_void_p), ("active", C.c_void_p)]


class Intr(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("depth_scale", C.c_double)]


class PoseS(C.Structure):
    _fields_ = [("q", C.c_double * 4), ("t", C.c_double * 3)]


class Params(C.Structure):
    _fields_ = [("step", C.c_double), ("t_near", C.c_double), ("t_far", C.c_double),
                ("termination_eps", C.c_double)]


class FrameS(C.Structure):
    _fields_ = [("color", C.c_void_p), ("depth", C.c_void_p), ("pose", PoseS)]


class RayResult(C.Structure):
    _fields_ = [("color", C.c_double * 3), ("depth", C.c_double),
                ("transmittance_terminal", C.c_double), ("count", C.c_int32), ("hit", C.c_int32),
                ("terminated_early", C.c_int32)]


class MapCfg(C.Structure):
    _fields_ = [("lambda_d", C.c_double), ("lr_sigma", C.c_double), ("lr_sh", C.c_double),
                ("rmsprop_decay", C.c_double), ("rmsprop_eps", C.c_double), ("render", Params)]


class MapStats(C.Structure):
    _fields_ = [("loss_photometric", C.c_double), ("loss_geometric", C.c_double),
                ("loss_total", C.c_double), ("rays_color", C.c_int32), ("rays_depth", C.c_int32),
                ("psnr_estimate", C.c_double), ("samples", C.c_int64), ("bad_ray", C.c_int32)]


class TrackLoss(C.Structure):
    _fields_ = [("lambda_p", C.c_double), ("lambda_d", C.c_double), ("render", Params)]


class PoseGrad(C.Structure):
    _fields_ = [("d_omega", C.c_double * 3), ("d_tau", C.c_double * 3), ("loss", C.c_double),
                ("rays_used", C.c_int32)]


class NormalEqs(C.Structure):
    _fields_ = [("jtj", C.c_double * 21), ("jtr", C.c_double * 6), ("loss", C.c_double),
                ("rays_used", C.c_int32)]


class TrackCfg(C.Structure):
    _fields_ = [("rays_per_iteration", C.c_int32), ("iterations", C.c_int32),
                ("lr_omega", C.c_double), ("lr_tau", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("adam_eps", C.c_double), ("lambda_p", C.c_double),
                ("lambda_d", C.c_double), ("convergence_step", C.c_double),
                ("divergence_factor", C.c_double), ("divergence_patience", C.c_int32),
                ("max_redraws", C.c_int32), ("seed", C.c_uint64), ("render", Params)]


class TrackResult(C.Structure):
    _fields_ = [("pose", PoseS), ("failed", C.c_int32), ("iterations_run", C.c_int32),
                ("final_loss", C.c_double)]


def build(ref: bool = True) -> None:
    """make -C oracle (and the reference build when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    if ref and REF_SRC.exists():
        subprocess.run(["make", "-s", "-j8", "-C", str(HERE), "ref"], check=True)


def _ptr(a):
    return C.c_void_p(a.ctypes.data)


def geometry(geom) -> Geometry:
    return Geometry((C.c_int32 * 3)(*map(int, geom.res)), (C.c_double * 3)(*map(float, geom.origin)),
                    float(geom.voxel_size))


def intr_s(i) -> Intr:
    return Intr(i.fx, i.fy, i.cx, i.cy, int(i.width), int(i.height), i.depth_scale)


def pose_s(p) -> PoseS:
    return PoseS((C.c_double * 4)(*map(float, p.q)), (C.c_double * 3)(*map(float, p.t)))


def params_s(p) -> Params:
    return Params(p.step, p.t_near, p.t_far, p.termination_eps)


class _GridHold:
    """Keeps numpy buffers alive while a C struct points at them."""

    def __init__(self, grid):
        self.data = np.ascontiguousarray(grid.data, dtype=np.float64)
        self.active = np.ascontiguousarray(grid.active, dtype=np.uint8)
        self.s = Grid(geometry(grid.geom), self.data.ctypes.data, self.active.ctypes.data)


class _FramesHold:
    def __init__(self, frames):
        self.colors = [np.ascontiguousarray(f.color, np.float64) for f in frames]
        self.depths = [np.ascontiguousarray(f.depth, np.float64) for f in frames]
        self.arr = (FrameS * max(1, len(frames)))(*[
            FrameS(c.ctypes.data, d.ctypes.data, pose_s(f.gt_pose))
            for c, d, f in zip(self.colors, self.depths, frames)])


class OracleError(RuntimeError):
    pass


def _check(rc, what):
    if rc == 1:
        raise ValueError(what)
    if rc == 2:
        raise IndexError(what)
    if rc != 0:
        raise OracleError(what)


class Oracle:
    """The plain-C restatement (voxrf_oracle.c)."""

    def __init__(self):
        if not ORACLE_SO.exists():
            build(ref=False)
        self.lib = C.CDLL(str(ORACLE_SO))

    def generate_ray(self, intr, pose, u, v):
        o = np.zeros(3)
        d = np.zeros(3)
        _check(self.lib.or_generate_ray(C.byref(intr_s(intr)), C.byref(pose_s(pose)),
                                        C.c_double(u), C.c_double(v), _ptr(o), _ptr(d)),
               "generate_ray: pixel outside image")
        return o, d

    def sample_ray(self, grid, o, d, params, cap=4096):
        h = _GridHold(grid)
        t = np.zeros(cap)
        delta = np.zeros(cap)
        cells = np.zeros(cap, np.uint32)
        o = np.ascontiguousarray(o, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        n = self.lib.or_sample_ray(C.byref(h.s), _ptr(o), _ptr(d), C.byref(params_s(params)), cap,
                                   _ptr(t), _ptr(delta), _ptr(cells))
        if n < 0:
            _check(-n, "sample_ray")
        return t[:n], delta[:n], cells[:n]

    def render_ray(self, grid, o, d, params):
        h = _GridHold(grid)
        r = RayResult()
        o = np.ascontiguousarray(o, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        _check(self.lib.or_render_ray(C.byref(h.s), _ptr(o), _ptr(d), C.byref(params_s(params)),
                                      C.byref(r)), "render_ray")
        return r

    def upsample(self, grid, max_resolution, clamp_outside=False):
        """VoxelGrid::upsampled (voxel_grid.cpp:190-220) -> (geometry, data, active).
        clamp_outside: clamp far-corner vertices the reference would throw on."""
        h = _GridHold(grid)
        f = Geometry()
        cl = 1 if clamp_outside else 0
        rc = self.lib.or_upsample(C.byref(h.s), int(max_resolution), cl, C.byref(f), None, None)
        if rc == 3:
            raise OracleError("upsample: resolution would exceed configured maximum")
        res = tuple(f.res)
        nv = res[0] * res[1] * res[2]
        nc = (res[0] - 1) * (res[1] - 1) * (res[2] - 1)
        data = np.zeros((nv, 28))
        act = np.zeros(nc, np.uint8)
        _check(self.lib.or_upsample(C.byref(h.s), int(max_resolution), cl, C.byref(f),
                                    _ptr(data), _ptr(act)),
               "upsample: voxel grid: point outside grid")
        return (res, tuple(f.origin), f.voxel_size), data, act

    def render_image(self, grid, intr, pose, params, stride=1):
        h = _GridHold(grid)
        ow = (intr.width + stride - 1) // stride
        oh = (intr.height + stride - 1) // stride
        color = np.zeros((oh, ow, 3))
        depth = np.zeros((oh, ow))
        _check(self.lib.or_render_image(C.byref(h.s), C.byref(intr_s(intr)), C.byref(pose_s(pose)),
                                        C.byref(params_s(params)), stride, _ptr(color), _ptr(depth)),
               "render_image")
        return color, depth

    def mapping_step(self, grid, frames, intr, cfg, batch, rms_v=None, apply=True, want_grad=False):
        """Returns (new_data, new_rms_v, grad or None, stats). grid is not modified."""
        data = np.ascontiguousarray(grid.data, np.float64).copy()
        active = np.ascontiguousarray(grid.active, np.uint8)
        gs = Grid(geometry(grid.geom), data.ctypes.data, active.ctypes.data)
        fh = _FramesHold(frames)
        v = np.zeros_like(data) if rms_v is None else np.ascontiguousarray(rms_v, np.float64).reshape(data.shape).copy()
        grad = np.zeros_like(data) if want_grad else None
        b = np.ascontiguousarray(batch, np.int32)
        st = MapStats()
        mc = MapCfg(cfg.lambda_d, cfg.lr_sigma, cfg.lr_sh, cfg.rmsprop_decay, cfg.rmsprop_eps,
                    params_s(cfg.render))
        rc = self.lib.or_mapping_step(C.byref(gs), fh.arr, len(frames), C.byref(intr_s(intr)),
                                      C.byref(mc), _ptr(b), b.shape[0], _ptr(v),
                                      _ptr(grad) if want_grad else None, 1 if apply else 0,
                                      C.byref(st))
        _check(rc, f"mapping_step (bad_ray={st.bad_ray}, rays_color={st.rays_color})")
        return data, v, grad, st

    def mapping_grad_global(self, grid, frames, intr, cfg, batch, m_color, m_depth):
        data = np.ascontiguousarray(grid.data, np.float64)
        active = np.ascontiguousarray(grid.active, np.uint8)
        gs = Grid(geometry(grid.geom), data.ctypes.data, active.ctypes.data)
        fh = _FramesHold(frames)
        grad = np.zeros_like(data)
        b = np.ascontiguousarray(batch, np.int32).reshape(-1, 3)
        st = MapStats()
        mc = MapCfg(cfg.lambda_d, cfg.lr_sigma, cfg.lr_sh, cfg.rmsprop_decay, cfg.rmsprop_eps,
                    params_s(cfg.render))
        rc = self.lib.or_mapping_grad_global(C.byref(gs), fh.arr, len(frames),
                                             C.byref(intr_s(intr)), C.byref(mc), _ptr(b),
                                             b.shape[0], int(m_color), int(m_depth), _ptr(grad),
                                             C.byref(st))
        _check(rc, "mapping_grad_global")
        return grad, st

    def pose_gradient(self, grid, frame, intr, pose, pixels, lambda_p, lambda_d, params):
        h = _GridHold(grid)
        fh = _FramesHold([frame])
        px = np.ascontiguousarray(pixels, np.int32)
        out = PoseGrad()
        _check(self.lib.or_pose_gradient(C.byref(h.s), fh.arr, C.byref(intr_s(intr)),
                                         C.byref(pose_s(pose)), _ptr(px), px.shape[0],
                                         C.byref(TrackLoss(lambda_p, lambda_d, params_s(params))),
                                         C.byref(out)), "pose_gradient")
        return out

    def normal_eqs(self, grid, frame, intr, pose, pixels, lambda_p, lambda_d, params):
        h = _GridHold(grid)
        fh = _FramesHold([frame])
        px = np.ascontiguousarray(pixels, np.int32)
        out = NormalEqs()
        _check(self.lib.or_pose_normal_eqs(C.byref(h.s), fh.arr, C.byref(intr_s(intr)),
                                           C.byref(pose_s(pose)), _ptr(px), px.shape[0],
                                           C.byref(TrackLoss(lambda_p, lambda_d, params_s(params))),
                                           C.byref(out)), "normal_eqs")
        return out

    def track_frame(self, grid, frame, intr, init, tcfg):
        h = _GridHold(grid)
        fh = _FramesHold([frame])
        out = TrackResult()
        trace = np.zeros(max(tcfg.iterations, 1))
        _check(self.lib.or_track_frame(C.byref(h.s), fh.arr, C.byref(intr_s(intr)),
                                       C.byref(pose_s(init)), C.byref(track_cfg(tcfg)),
                                       C.byref(out), _ptr(trace)), "track_frame")
        return out, trace[:out.iterations_run]

    def draw_batch(self, seed, n_frames, w, h, n):
        st = (C.c_uint64 * 4)()
        self.lib.or_rng_seed(C.c_uint64(seed), st)
        out = np.zeros((n, 3), np.int32)
        self.lib.or_draw_batch(st, n_frames, w, h, n, _ptr(out))
        return out


def track_cfg(c) -> TrackCfg:
    return TrackCfg(c.rays_per_iteration, c.iterations, c.lr_omega, c.lr_tau, c.beta1, c.beta2,
                    c.adam_eps, c.lambda_p, c.lambda_d, c.convergence_step, c.divergence_factor,
                    c.divergence_patience, c.max_redraws, c.seed & (2**64 - 1), params_s(c.render))


class MapSceneCfg(C.Structure):
    _fields_ = [("keyframe_stride", C.c_int32), ("rays_per_batch", C.c_int32),
                ("iterations_per_stage", C.c_int32), ("initial_resolution", C.c_int32),
                ("upsample_stages", C.c_int32), ("max_resolution", C.c_int32),
                ("prune_every", C.c_int32), ("threads", C.c_int32), ("deterministic", C.c_int32),
                ("pad", C.c_int32), ("lambda_d", C.c_double), ("lr_sigma", C.c_double),
                ("lr_sh", C.c_double), ("rmsprop_decay", C.c_double), ("rmsprop_eps", C.c_double),
                ("prune_threshold", C.c_double), ("sigma_init", C.c_double),
                ("bounds_margin", C.c_double), ("seed", C.c_uint64), ("render", Params)]


class RefLib:
    """The reference's own functions (oracle/_ref/libvoxrf_ref.so)."""

    def __init__(self):
        if not REF_SO.exists():
            if not REF_SRC.exists():
                raise FileNotFoundError("oracle/_ref not built and /root/reference absent")
            build(ref=True)
        lib = C.CDLL(str(REF_SO))
        lib.ref_grid_create.restype = C.c_void_p
        lib.ref_grid_create.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_frames_create.restype = C.c_void_p
        lib.ref_frames_create.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        lib.ref_mapper_create.restype = C.c_void_p
        lib.ref_mapper_create.argtypes = [C.c_uint64]
        lib.ref_last_error.restype = C.c_char_p
        for n in ["ref_grid_destroy", "ref_frames_destroy", "ref_mapper_destroy"]:
            getattr(lib, n).argtypes = [C.c_void_p]
        lib.ref_grid_read.argtypes = [C.c_void_p, C.c_void_p]
        lib.ref_grid_occupancy.argtypes = [C.c_void_p, C.c_void_p]
        lib.ref_grid_upsampled.restype = C.c_void_p
        lib.ref_grid_upsampled.argtypes = [C.c_void_p, C.c_int]
        lib.ref_grid_save.argtypes = [C.c_void_p, C.c_char_p]
        lib.ref_grid_load.restype = C.c_void_p
        lib.ref_grid_load.argtypes = [C.c_char_p]
        lib.ref_grid_checksum.restype = C.c_uint64
        lib.ref_grid_checksum.argtypes = [C.c_void_p]
        lib.ref_mapper_rms.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
        lib.ref_mapping_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                         C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        lib.ref_mapping_grad.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        lib.ref_render_image.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                         C.c_int, C.c_void_p, C.c_void_p]
        lib.ref_render_ray.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_sample_ray.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                       C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_pose_gradient.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p]
        lib.ref_pose_normal_eqs.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        lib.ref_track_frame.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        # eval.cpp / trajectory.cpp
        vp = C.c_void_p
        lib.ref_ate_rmse.argtypes = [vp, vp, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp]
        lib.ref_rpe.argtypes = [vp, vp, C.c_int, vp, vp, C.c_int, C.c_double, vp, vp, vp]
        lib.ref_psnr.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                 C.c_uint64, vp, vp]
        lib.ref_depth_l1.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp]
        lib.ref_evaluate_map_quality.argtypes = [vp, vp, vp, vp, C.c_int, vp, C.c_int, C.c_int,
                                                 C.c_uint64, C.c_int, vp, vp, vp, vp]
        lib.ref_save_tum.argtypes = [C.c_char_p, vp, vp, C.c_int]
        lib.ref_load_tum.argtypes = [C.c_char_p, C.c_int, vp, vp]
        self.lib = lib

    def _err(self, rc, what):
        if rc != 0:
            msg = self.lib.ref_last_error().decode()
            _check(rc, f"{what}: {msg}")

    def grid(self, grid):
        g = geometry(grid.geom)
        data = np.ascontiguousarray(grid.data, np.float64)
        act = np.ascontiguousarray(grid.active, np.uint8)
        return self.lib.ref_grid_create(C.byref(g), _ptr(data), _ptr(act))

    def fit_grid_geometry(self, frames_h, intr, initial_resolution, bounds_margin):
        g = Geometry()
        self.lib.ref_fit_grid_geometry.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_double,
                                                   C.c_void_p]
        self._err(self.lib.ref_fit_grid_geometry(frames_h, C.byref(intr_s(intr)),
                                                 int(initial_resolution), float(bounds_margin),
                                                 C.byref(g)), "fit_grid_geometry")
        return tuple(g.res), tuple(g.origin), g.voxel_size

    def map_scene(self, frames_h, intr, cfg, geometry=None, threads=0):
        """The reference's map_scene (mapping.cpp:278-316) -> (grid handle, final loss, ms)."""
        c = MapSceneCfg(cfg.keyframe_stride, cfg.rays_per_batch, cfg.iterations_per_stage,
                        cfg.initial_resolution, cfg.upsample_stages, cfg.max_resolution,
                        cfg.prune_every, threads, 1 if cfg.deterministic else 0, 0, cfg.lambda_d,
                        cfg.lr_sigma, cfg.lr_sh, cfg.rmsprop_decay, cfg.rmsprop_eps,
                        cfg.prune_threshold, cfg.sigma_init, cfg.bounds_margin,
                        cfg.seed & (2**64 - 1), params_s(cfg.render))
        loss, ms = C.c_double(), C.c_double()
        self.lib.ref_map_scene.restype = C.c_void_p
        self.lib.ref_map_scene.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p]
        g = None if geometry is None else globals()["geometry"](geometry)
        h = self.lib.ref_map_scene(frames_h, C.byref(intr_s(intr)), C.byref(c),
                                   None if g is None else C.byref(g), C.byref(loss), C.byref(ms))
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return h, loss.value, ms.value

    def track_sequence(self, grid_h, frames_h, intr, tcfg, n_frames, threads=0,
                       constant_velocity=False):
        """The reference's track_sequence (tracking.cpp:254-295) -> (poses [(q, t)], ms)."""
        out = (PoseS * n_frames)()
        ms = C.c_double()
        self.lib.ref_track_sequence.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        self._err(self.lib.ref_track_sequence(grid_h, frames_h, C.byref(intr_s(intr)),
                                              C.byref(track_cfg(tcfg)), threads,
                                              1 if constant_velocity else 0, out, C.byref(ms)),
                  "track_sequence")
        return [(tuple(p.q), tuple(p.t)) for p in out], ms.value

    def read_occupancy(self, handle, ncells):
        out = np.zeros(ncells, np.uint8)
        self.lib.ref_grid_occupancy(handle, _ptr(out))
        return out

    def upsampled(self, handle, max_resolution):
        """VoxelGrid::upsampled (voxel_grid.cpp:190-220) -> new handle."""
        h = self.lib.ref_grid_upsampled(handle, int(max_resolution))
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return h

    def save(self, handle, path):
        self._err(self.lib.ref_grid_save(handle, str(path).encode()), "save")

    def load(self, path):
        h = self.lib.ref_grid_load(str(path).encode())
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return h

    def frames(self, frames, intr):
        fh = _FramesHold(frames)
        return self.lib.ref_frames_create(fh.arr, len(frames), intr.width, intr.height)

    def read_grid(self, handle, nv):
        out = np.zeros((nv, 28))
        self.lib.ref_grid_read(handle, _ptr(out))
        return out

    def render_image(self, grid_h, intr, pose, params, stride=1, threads=1):
        ow = (intr.width + stride - 1) // stride
        oh = (intr.height + stride - 1) // stride
        color = np.zeros((oh, ow, 3))
        depth = np.zeros((oh, ow))
        self._err(self.lib.ref_render_image(grid_h, C.byref(intr_s(intr)), C.byref(pose_s(pose)),
                                            C.byref(params_s(params)), stride, threads,
                                            _ptr(color), _ptr(depth)), "render_image")
        return color, depth

    def render_ray(self, grid_h, o, d, params):
        r = RayResult()
        o = np.ascontiguousarray(o, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        self._err(self.lib.ref_render_ray(grid_h, _ptr(o), _ptr(d), C.byref(params_s(params)),
                                          C.byref(r)), "render_ray")
        return r

    def sample_ray(self, grid_h, o, d, params, cap=4096):
        t = np.zeros(cap)
        delta = np.zeros(cap)
        n = C.c_int()
        o = np.ascontiguousarray(o, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        self._err(self.lib.ref_sample_ray(grid_h, _ptr(o), _ptr(d), C.byref(params_s(params)), cap,
                                          _ptr(t), _ptr(delta), C.byref(n)), "sample_ray")
        return t[:n.value], delta[:n.value]

    def mapping_step(self, grid_h, frames_h, intr, cfg, n_rays, threads, deterministic, mapper):
        st = MapStats()
        mc = MapCfg(cfg.lambda_d, cfg.lr_sigma, cfg.lr_sh, cfg.rmsprop_decay, cfg.rmsprop_eps,
                    params_s(cfg.render))
        self._err(self.lib.ref_mapping_step(grid_h, frames_h, C.byref(intr_s(intr)), C.byref(mc),
                                            n_rays, threads, 1 if deterministic else 0, mapper,
                                            C.byref(st)), "mapping_step")
        return st

    def mapping_grad(self, grid_h, frames_h, intr, cfg, batch, nv):
        b = np.ascontiguousarray(batch, np.int32)
        out = np.zeros((nv, 28))
        samples = C.c_int64()
        mc = MapCfg(cfg.lambda_d, cfg.lr_sigma, cfg.lr_sh, cfg.rmsprop_decay, cfg.rmsprop_eps,
                    params_s(cfg.render))
        self._err(self.lib.ref_mapping_grad(grid_h, frames_h, C.byref(intr_s(intr)), C.byref(mc),
                                            _ptr(b), b.shape[0], _ptr(out), C.byref(samples)),
                  "mapping_grad")
        return out, samples.value

    def pose_gradient(self, grid_h, frames_h, intr, pose, pixels, lambda_p, lambda_d, params,
                      threads=1):
        px = np.ascontiguousarray(pixels, np.int32)
        out = PoseGrad()
        self._err(self.lib.ref_pose_gradient(grid_h, frames_h, C.byref(intr_s(intr)),
                                             C.byref(pose_s(pose)), _ptr(px), px.shape[0],
                                             C.byref(TrackLoss(lambda_p, lambda_d, params_s(params))),
                                             threads, C.byref(out)), "pose_gradient")
        return out

    def normal_eqs(self, grid_h, frames_h, intr, pose, pixels, lambda_p, lambda_d, params):
        px = np.ascontiguousarray(pixels, np.int32)
        out = NormalEqs()
        self._err(self.lib.ref_pose_normal_eqs(grid_h, frames_h, C.byref(intr_s(intr)),
                                               C.byref(pose_s(pose)), _ptr(px), px.shape[0],
                                               C.byref(TrackLoss(lambda_p, lambda_d,
                                                                 params_s(params))),
                                               C.byref(out)), "normal_eqs")
        return out

    def track_frame(self, grid_h, frames_h, intr, init, tcfg, threads=1):
        out = TrackResult()
        trace = np.zeros(max(tcfg.iterations, 1))
        self._err(self.lib.ref_track_frame(grid_h, frames_h, C.byref(intr_s(intr)),
                                           C.byref(pose_s(init)), C.byref(track_cfg(tcfg)), threads,
                                           C.byref(out), _ptr(trace)), "track_frame")
        return out, trace[:out.iterations_run]

    # ---- eval.cpp / trajectory.cpp
    @staticmethod
    def _traj(poses, ts):
        arr = (PoseS * max(len(poses), 1))(*[pose_s(p) for p in poses])
        return np.ascontiguousarray(ts, np.float64), arr

    def ate_rmse(self, est, est_ts, ref, ref_ts, align=True):
        """eval.cpp:140-172 -> (rmse, pairs)."""
        et, ea = self._traj(est, est_ts)
        rt, ra = self._traj(ref, ref_ts)
        out, pairs = C.c_double(), C.c_int()
        self._err(self.lib.ref_ate_rmse(_ptr(et), ea, len(est), _ptr(rt), ra, len(ref),
                                        1 if align else 0, C.byref(out), C.byref(pairs)),
                  "ate_rmse")
        return out.value, pairs.value

    def rpe(self, est, est_ts, ref, ref_ts, interval_m=1.0):
        """eval.cpp:174-208 -> (rpe_t, rpe_r_deg, pairs)."""
        et, ea = self._traj(est, est_ts)
        rt, ra = self._traj(ref, ref_ts)
        t, r, n = C.c_double(), C.c_double(), C.c_int()
        self._err(self.lib.ref_rpe(_ptr(et), ea, len(est), _ptr(rt), ra, len(ref),
                                   float(interval_m), C.byref(t), C.byref(r), C.byref(n)), "rpe")
        return t.value, r.value, n.value

    def psnr(self, rendered, reference, masks=None, images=10, pixels_per_image=10000, seed=0):
        """eval.cpp:64-97 -> (psnr_db, samples)."""
        a = np.ascontiguousarray(np.stack(rendered), np.float64)
        b = np.ascontiguousarray(np.stack(reference), np.float64)
        m = None if masks is None else np.ascontiguousarray(np.stack(masks), np.float64)
        n, h, w = a.shape[:3]
        out, cnt = C.c_double(), C.c_int()
        self._err(self.lib.ref_psnr(_ptr(a), _ptr(b), None if m is None else _ptr(m), n, w, h,
                                    images, pixels_per_image, seed & (2**64 - 1), C.byref(out),
                                    C.byref(cnt)), "psnr")
        return out.value, cnt.value

    def depth_l1(self, rendered, reference, masks=None):
        """eval.cpp:99-122 -> (l1_m, pixels)."""
        a = np.ascontiguousarray(np.stack(rendered), np.float64)
        b = np.ascontiguousarray(np.stack(reference), np.float64)
        m = None if masks is None else np.ascontiguousarray(np.stack(masks), np.float64)
        n, h, w = a.shape
        out, cnt = C.c_double(), C.c_int()
        self._err(self.lib.ref_depth_l1(_ptr(a), _ptr(b), None if m is None else _ptr(m), n, w,
                                        h, C.byref(out), C.byref(cnt)), "depth_l1")
        return out.value, cnt.value

    def evaluate_map_quality(self, grid_h, frames_h, intr, indices, params, images=10,
                             pixels_per_image=10000, seed=0, threads=0):
        """eval.cpp:210-240 -> (psnr_db, depth_l1_m, color_samples, depth_pixels)."""
        idx = np.ascontiguousarray(indices, np.int32)
        p, l1 = C.c_double(), C.c_double()
        ns, npx = C.c_int(), C.c_int()
        self._err(self.lib.ref_evaluate_map_quality(
            grid_h, frames_h, C.byref(intr_s(intr)), _ptr(idx), len(idx),
            C.byref(params_s(params)), images, pixels_per_image, seed & (2**64 - 1), threads,
            C.byref(p), C.byref(l1), C.byref(ns), C.byref(npx)), "evaluate_map_quality")
        return p.value, l1.value, ns.value, npx.value

    def save_tum(self, path, poses, ts):
        """trajectory.cpp:10-23."""
        t, a = self._traj(poses, ts)
        self._err(self.lib.ref_save_tum(str(path).encode(), _ptr(t), a, len(poses)), "save_tum")

    def load_tum(self, path, cap=100000):
        """trajectory.cpp:25-46 -> (poses [(q, t)], timestamps)."""
        ts = np.zeros(cap)
        arr = (PoseS * cap)()
        n = self.lib.ref_load_tum(str(path).encode(), cap, _ptr(ts), arr)
        if n < 0:
            _check(-n, "load_tum: " + self.lib.ref_last_error().decode())
        return [(tuple(arr[i].q), tuple(arr[i].t)) for i in range(min(n, cap))], ts[:n]
