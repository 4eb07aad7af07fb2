"""Python mirror of the reference's hot-path API (proj/include/voxrf/*.hpp).

Two layers:

* :class:`Context` — one device session (one GPU): the grid, its RMSProp state
  and the keyframes stay resident in HBM between calls. This is what bench.py,
  the multi-GPU driver and long-running callers use.
* Reference-named functions — :func:`render_image`, :func:`mapping_step`,
  :func:`pose_gradient`, :func:`track_frame`, :func:`track_sequence` — with the
  reference's argument meaning and error behaviour (ValueError for
  std::invalid_argument, IndexError for std::out_of_range, RuntimeError for
  std::runtime_error, same messages). They run on a default context and sync
  host objects in and out, like the in-place VoxelGrid semantics of
  mapping_step (mapping.hpp:80-82).

All computation runs in libvoxrf_b200.so on the GPU; nothing here computes a
rendering or a gradient on the CPU.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _capi as capi

SH_COEFFS = 9
PAYLOAD = 28


class VoxrfError(RuntimeError):
    pass


def _raise(code: int, msg: str):
    if code == capi.VRF_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if code == capi.VRF_ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    raise RuntimeError(msg)


# ---------------------------------------------------------------- value types
@dataclass
class GridGeometry:
    """GridGeometry — voxel_grid.hpp:20-63 (res counts vertices per axis)."""
    res: tuple = (0, 0, 0)
    origin: tuple = (0.0, 0.0, 0.0)
    voxel_size: float = 0.0

    def validate(self):
        if min(self.res) < 2:
            raise ValueError("grid: resolution must be >= 2 per axis")
        if not self.voxel_size > 0.0:
            raise ValueError("grid: voxel_size must be > 0")

    @property
    def num_vertices(self) -> int:
        return int(self.res[0]) * int(self.res[1]) * int(self.res[2])

    @property
    def num_cells(self) -> int:
        return (int(self.res[0]) - 1) * (int(self.res[1]) - 1) * (int(self.res[2]) - 1)

    def world_min(self):
        return np.asarray(self.origin, dtype=np.float64)

    def world_max(self):
        return np.asarray(self.origin, np.float64) + (np.asarray(self.res, np.float64) - 1.0) * self.voxel_size

    def to_world(self, g):
        return np.asarray(self.origin, np.float64) + np.asarray(g, np.float64) * self.voxel_size

    def vertex_index(self, ix, iy, iz) -> int:
        return int(ix + self.res[0] * (iy + self.res[1] * iz))

    def cell_index(self, cx, cy, cz) -> int:
        return int(cx + (self.res[0] - 1) * (cy + (self.res[1] - 1) * cz))

    def _c(self):
        return capi.GridGeometry_c((C.c_int32 * 3)(*[int(r) for r in self.res]),
                                   (C.c_double * 3)(*[float(o) for o in self.origin]),
                                   float(self.voxel_size))


class VoxelGrid:
    """Host VoxelGrid (voxel_grid.hpp:112-175): float64 [V][28] + uint8 occupancy."""

    def __init__(self, geom: GridGeometry, sigma_init: float = 0.0):
        geom.validate()
        self.geom = geom
        self.data = np.zeros((geom.num_vertices, PAYLOAD), dtype=np.float64)
        if sigma_init != 0.0:
            self.data[:, 0] = sigma_init
        self.active = np.ones(geom.num_cells, dtype=np.uint8)

    def geometry(self) -> GridGeometry:
        return self.geom

    def vertex(self, index: int):
        return self.data[index]

    def set_all_active(self, on: bool):
        self.active[:] = 1 if on else 0

    def set_cell_active(self, cx, cy, cz, on: bool):
        self.active[self.geom.cell_index(cx, cy, cz)] = 1 if on else 0

    def cell_active(self, cx, cy, cz) -> bool:
        return bool(self.active[self.geom.cell_index(cx, cy, cz)])

    def active_cell_count(self) -> int:
        return int(self.active.sum())

    def copy(self) -> "VoxelGrid":
        g = VoxelGrid.__new__(VoxelGrid)
        g.geom = self.geom
        g.data = self.data.copy()
        g.active = self.active.copy()
        return g


@dataclass
class CameraIntrinsics:
    """CameraIntrinsics — camera.hpp:11-24."""
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    width: int = 0
    height: int = 0
    depth_scale: float = 1000.0

    def validate(self):
        if self.fx <= 0.0 or self.fy <= 0.0:
            raise ValueError("intrinsics: fx, fy must be > 0")
        if self.width <= 0 or self.height <= 0:
            raise ValueError("intrinsics: empty image size")
        if self.cx <= 0.0 or self.cx >= self.width or self.cy <= 0.0 or self.cy >= self.height:
            raise ValueError("intrinsics: principal point outside image")
        if self.depth_scale <= 0.0:
            raise ValueError("intrinsics: depth_scale must be > 0")

    def _c(self):
        return capi.Intrinsics_c(self.fx, self.fy, self.cx, self.cy, int(self.width),
                                 int(self.height), self.depth_scale)


@dataclass
class Pose:
    """Pose — pose.hpp:11-24; q = (w, x, y, z)."""
    q: tuple = (1.0, 0.0, 0.0, 0.0)
    t: tuple = (0.0, 0.0, 0.0)

    def _c(self):
        return capi.Pose_c((C.c_double * 4)(*map(float, self.q)), (C.c_double * 3)(*map(float, self.t)))

    @staticmethod
    def _from_c(p) -> "Pose":
        return Pose(tuple(p.q), tuple(p.t))

    def rotation(self) -> np.ndarray:
        w, x, y, z = self.q
        return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                         [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                         [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


@dataclass
class RenderParams:
    """RenderParams — renderer.hpp:12-24."""
    step: float = 0.0
    t_near: float = 0.05
    t_far: float = 0.0
    termination_eps: float = 1e-4

    def _c(self):
        return capi.RenderParams_c(self.step, self.t_near, self.t_far, self.termination_eps)


@dataclass
class Frame:
    """Frame — frame.hpp:10-19: colour HxWx3 in [0,1], depth HxW along-ray metres (0 = invalid)."""
    color: np.ndarray
    depth: np.ndarray
    timestamp: float = 0.0
    gt_pose: Optional[Pose] = None
    # optional sensor-format copies (8-bit RGB, 16-bit depth units) for the cheap
    # upload path (Context.set_frame_u8u16)
    color_u8: Optional[np.ndarray] = None
    depth_u16: Optional[np.ndarray] = None

    def depth_valid(self, x: int, y: int) -> bool:
        return bool(self.depth[y, x] > 0.0)


@dataclass
class MappingConfig:
    """MappingConfig — mapping.hpp:19-41."""
    lambda_d: float = 1.0
    rays_per_batch: int = 4096
    iterations_per_stage: int = 2000
    lr_sigma: float = 30.0
    lr_sh: float = 1e-2
    rmsprop_decay: float = 0.95
    rmsprop_eps: float = 1e-8
    keyframe_stride: int = 10
    initial_resolution: int = 33
    upsample_stages: int = 2
    max_resolution: int = 513
    prune_threshold: float = 1e-3
    prune_every: int = 0
    sigma_init: float = 0.1
    bounds_margin: float = 0.05
    seed: int = 1
    threads: int = 0
    deterministic: bool = False
    render: RenderParams = field(default_factory=RenderParams)

    def _c(self):
        return capi.MappingConfig_c(self.lambda_d, self.lr_sigma, self.lr_sh, self.rmsprop_decay,
                                    self.rmsprop_eps, 1 if self.deterministic else 0, 0,
                                    self.render._c())


@dataclass
class MapStepStats:
    """MapStepStats — mapping.hpp:68-75 (+ composited sample count)."""
    loss_photometric: float = 0.0
    loss_geometric: float = 0.0
    loss_total: float = 0.0
    rays_color: int = 0
    rays_depth: int = 0
    psnr_estimate: float = 0.0
    samples: int = 0


@dataclass
class TrackingConfig:
    """TrackingConfig — tracking.hpp:29-51."""
    rays_per_iteration: int = 2048
    iterations: int = 40
    lr_omega: float = 1e-3
    lr_tau: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    lambda_p: float = 1.0
    lambda_d: float = 1.0
    init_policy: str = "previous"  # or "constant_velocity"
    convergence_step: float = 0.0
    divergence_factor: float = 10.0
    divergence_patience: int = 20
    max_redraws: int = 50
    seed: int = 7
    threads: int = 0
    deterministic: bool = False
    render: RenderParams = field(default_factory=RenderParams)

    def _loss_c(self):
        return capi.TrackingLoss_c(self.lambda_p, self.lambda_d, self.render._c())

    def _c(self):
        return capi.TrackingConfig_c(self.rays_per_iteration, self.iterations, self.lr_omega,
                                     self.lr_tau, self.beta1, self.beta2, self.adam_eps,
                                     self.lambda_p, self.lambda_d, self.convergence_step,
                                     self.divergence_factor, self.divergence_patience,
                                     self.max_redraws, self.seed & (2**64 - 1), self.render._c())


@dataclass
class GNConfig:
    """Gauss-Newton / LM tracker settings (new; the reference only has Adam).

    Every iteration evaluates exactly rays_per_iteration stratified pixel draws."""
    rays_per_iteration: int = 16384
    iterations: int = 10
    lambda_p: float = 1.0
    lambda_d: float = 1.0
    damping: float = 1e-4
    max_redraws: int = 50
    seed: int = 7
    render: RenderParams = field(default_factory=RenderParams)
    # capi.POSE_KERNEL_GN (k_pose_group_u) or POSE_KERNEL_GN_CHECK (its checker)
    kernel: int = capi.POSE_KERNEL_GN

    def _c(self):
        return capi.GnConfig_c(self.rays_per_iteration, self.iterations, self.lambda_p,
                               self.lambda_d, self.damping, self.max_redraws, self.kernel,
                               self.seed & (2**64 - 1), self.render._c())


@dataclass
class PoseGradient:
    """PoseGradient — tracking.hpp:60-65."""
    d_omega: np.ndarray
    d_tau: np.ndarray
    loss: float
    rays_used: int
    samples: int = 0


@dataclass
class NormalEquations:
    jtj: np.ndarray  # 6x6 symmetric
    jtr: np.ndarray  # 6
    loss: float      # un-normalised sum
    rays_used: int
    samples: int = 0


@dataclass
class TrackFrameResult:
    """TrackFrameResult — tracking.hpp:75-80."""
    pose: Pose
    loss_trace: list
    failed: bool = False
    iterations_run: int = 0


class Rng:
    """The reference Rng stream (rng.hpp:13-81, xoshiro256** via splitmix64)."""

    def __init__(self, seed: int):
        self.state = (C.c_uint64 * 4)()
        capi.load().vrf_rng_seed(seed & (2**64 - 1), self.state)

    def next_u64(self) -> int:
        return int(capi.load().vrf_rng_next(self.state))

    def uniform_index(self, n: int) -> int:
        return (self.next_u64() * n) >> 64

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def draw_batch(self, n_frames: int, width: int, height: int, n: int,
                   out: np.ndarray = None) -> np.ndarray:
        """mapping.cpp:121-128 — n (frame, px, py) triples; into `out` (a C-contiguous
        int32 (n, 3) array, e.g. a pinned host buffer) when given."""
        if out is None:
            out = np.empty((n, 3), dtype=np.int32)
        elif out.dtype != np.int32 or out.shape != (n, 3) or not out.flags.c_contiguous:
            raise ValueError("draw_batch: out must be a C-contiguous int32 array of shape (n, 3)")
        capi.load().vrf_rng_draw_batch(self.state, n_frames, width, height, n,
                                       out.ctypes.data_as(C.c_void_p))
        return out

    def draw_eval_samples(self, n_images: int, width: int, height: int, images: int,
                          pixels_per_image: int) -> np.ndarray:
        """eval.cpp:72-83's draws: (image, x, y) rows, images x pixels_per_image."""
        out = np.zeros((images * pixels_per_image, 3), np.int32)
        capi.load().vrf_rng_draw_eval_samples(self.state, n_images, width, height, images,
                                              pixels_per_image, out.ctypes.data_as(C.c_void_p))
        return out

    def draw_valid_pixels(self, depth: np.ndarray, count: int, max_redraws: int) -> np.ndarray:
        """tracking.cpp:147-166."""
        d = np.ascontiguousarray(depth, dtype=np.float64)
        out = np.empty((count, 2), dtype=np.int32)
        n = capi.load().vrf_rng_draw_valid_pixels(self.state, d.ctypes.data_as(C.c_void_p),
                                                  d.shape[1], d.shape[0], count, max_redraws,
                                                  out.ctypes.data_as(C.c_void_p))
        return out[:n]


class RmspropState:
    """RmspropState — mapping.hpp:48-52. Device-resident inside a Context; the
    host copy is materialised on demand."""

    def __init__(self):
        self.v: Optional[np.ndarray] = None
        self._ctx: Optional["Context"] = None

    def reset(self, num_params: int):
        self.v = np.zeros(num_params)
        if self._ctx is not None:
            self._ctx.rmsprop_reset()


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- device session
class Context:
    """One GPU session of libvoxrf_b200 (vrf_context)."""

    def __init__(self, device: int = 0, shard_multiple: int = 1):
        self._lib = capi.load()
        h = C.c_void_p()
        rc = self._lib.vrf_context_create(device, C.byref(h))
        if rc != capi.VRF_OK:
            raise RuntimeError(f"voxrf_b200: cannot create a CUDA context on device {device} "
                               f"(status {rc}); a B200 is required — there is no CPU fallback")
        self._h = h
        self.device = device
        self.geom: Optional[GridGeometry] = None
        self.intrinsics: Optional[CameraIntrinsics] = None
        self.n_frames = 0
        if shard_multiple != 1:
            self._check(self._lib.vrf_set_shard_multiple(self._h, shard_multiple))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.vrf_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != capi.VRF_OK:
            _raise(rc, self._lib.vrf_last_error(self._h).decode())

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.vrf_kernel_launch_count(self._h))

    PROFILE_SLOTS = ("map_forward", "map_backward", "rmsprop", "misc", "pose_forward",
                     "pose_backward", "render", "deterministic_reduce")

    def set_record_limits(self, budget_gb: float = -1.0, max_k: int = -1):
        """Sample-record sizing of the fast mapping path (vrf_set_record_limits):
        max_k = 0 disables records, max_k >= 4 caps records per ray (longer rays
        take the recompute-march backward); negative values are automatic."""
        self._check(self._lib.vrf_set_record_limits(self._h, float(budget_gb), int(max_k)))

    def profile_enable(self, on: bool = True):
        self._check(self._lib.vrf_profile_enable(self._h, 1 if on else 0))

    def profile_read(self) -> dict:
        out = {}
        for i, name in enumerate(self.PROFILE_SLOTS):
            ms, n = C.c_double(), C.c_int64()
            self._check(self._lib.vrf_profile_read(self._h, i, C.byref(ms), C.byref(n)))
            out[name] = (ms.value, n.value)
        out["touched_groups"] = int(self._lib.vrf_profile_touched_groups(self._h))
        out["track_samples"] = int(self._lib.vrf_profile_track_samples(self._h))
        return out

    def set_stream(self, stream_ptr: int):
        """Run on an external CUDA stream, e.g. torch.cuda.current_stream().cuda_stream.
        Handle 0 (torch's default stream) means the legacy default stream, passed as
        cudaStreamLegacy (1): NULL would select the context's own non-blocking stream,
        which does not order itself with torch's work."""
        ptr = int(stream_ptr) if stream_ptr else 1  # cudaStreamLegacy
        self._check(self._lib.vrf_set_stream(self._h, C.c_void_p(ptr)))

    def device_buffers(self):
        b = capi.DeviceBuffers_c()
        self._check(self._lib.vrf_get_device_buffers(self._h, C.byref(b)))
        return b

    # ---- grid
    def init_grid(self, geom: GridGeometry, sigma_init: float = 0.0):
        g = geom._c()
        self._check(self._lib.vrf_grid_init(self._h, C.byref(g), float(sigma_init)))
        self.geom = geom

    def fill_grid(self, sigma_init: float):
        """Payload := VoxelGrid(geom, sigma_init)'s, occupancy kept (vrf_grid_fill)."""
        self._check(self._lib.vrf_grid_fill(self._h, float(sigma_init)))

    def load_grid(self, grid: VoxelGrid):
        data = np.ascontiguousarray(grid.data, dtype=np.float64)
        occ = np.ascontiguousarray(grid.active, dtype=np.uint8)
        g = grid.geom._c()
        self._check(self._lib.vrf_grid_upload(self._h, C.byref(g), _ptr(data), _ptr(occ)))
        self.geom = grid.geom

    def load_grid_f32(self, geom: GridGeometry, payload: np.ndarray, occupancy_bits=None):
        data = np.ascontiguousarray(payload, dtype=np.float32)
        g = geom._c()
        bits = None if occupancy_bits is None else np.ascontiguousarray(occupancy_bits, np.uint8)
        self._check(self._lib.vrf_grid_upload_f32(self._h, C.byref(g), _ptr(data),
                                                  None if bits is None else _ptr(bits)))
        self.geom = geom

    def download_grid(self) -> VoxelGrid:
        grid = VoxelGrid.__new__(VoxelGrid)
        grid.geom = self.geom
        grid.data = np.empty((self.geom.num_vertices, PAYLOAD), dtype=np.float64)
        grid.active = np.empty(self.geom.num_cells, dtype=np.uint8)
        self._check(self._lib.vrf_grid_download(self._h, _ptr(grid.data), _ptr(grid.active)))
        return grid

    def grid_digest(self) -> int:
        """Device-side integrity digest of the resident grid (vrf_grid_digest)."""
        out = C.c_uint64()
        self._check(self._lib.vrf_grid_digest(self._h, C.byref(out)))
        return int(out.value)

    def download_payload_f32(self) -> np.ndarray:
        out = np.empty((self.geom.num_vertices, PAYLOAD), dtype=np.float32)
        self._check(self._lib.vrf_grid_download_f32(self._h, _ptr(out)))
        return out

    def upsample(self, max_resolution: int = 1024):
        """VoxelGrid::upsampled (voxel_grid.cpp:190-220) in place on the device."""
        self._check(self._lib.vrf_grid_upsample(self._h, int(max_resolution)))
        g = self.geom
        self.geom = GridGeometry(tuple(2 * int(r) - 1 for r in g.res), g.origin, g.voxel_size * 0.5)

    def save_grid(self, path):
        """VoxelGrid::save (voxel_grid.cpp:222-239) straight from HBM."""
        self._check(self._lib.vrf_grid_save(self._h, str(path).encode()))

    def load_grid_file(self, path):
        """VoxelGrid::load (voxel_grid.cpp:241-278) straight into HBM."""
        self._check(self._lib.vrf_grid_load(self._h, str(path).encode()))
        g = capi.GridGeometry_c()
        self._lib.vrf_grid_get_geometry(self._h, C.byref(g))
        self.geom = GridGeometry(tuple(g.res), tuple(g.origin), g.voxel_size)

    def prune(self, tau: float) -> int:
        n = C.c_int64()
        self._check(self._lib.vrf_grid_prune(self._h, tau, C.byref(n)))
        return int(n.value)

    # ---- frames
    def load_frames(self, intrinsics: CameraIntrinsics, frames: Sequence[Frame]):
        n = len(frames)
        colors = [np.ascontiguousarray(f.color, dtype=np.float64) for f in frames]
        depths = [np.ascontiguousarray(f.depth, dtype=np.float64) for f in frames]
        for c_, d_ in zip(colors, depths):
            if c_.shape != (intrinsics.height, intrinsics.width, 3) or d_.shape != (intrinsics.height, intrinsics.width):
                raise ValueError("frame size does not match the intrinsics")
        cp = (C.c_void_p * max(n, 1))(*[c_.ctypes.data for c_ in colors])
        dp = (C.c_void_p * max(n, 1))(*[d_.ctypes.data for d_ in depths])
        poses = (capi.Pose_c * max(n, 1))(*[(f.gt_pose or Pose())._c() for f in frames])
        ic = intrinsics._c()
        self._check(self._lib.vrf_frames_upload(self._h, C.byref(ic), n, cp, dp, poses))
        self.intrinsics = intrinsics
        self.n_frames = n

    def reserve_frames(self, intrinsics: CameraIntrinsics, capacity: int):
        """Slot store for online use (see vrf_frames_reserve)."""
        ic = intrinsics._c()
        self._check(self._lib.vrf_frames_reserve(self._h, C.byref(ic), int(capacity)))
        self.intrinsics = intrinsics
        self.n_frames = 0

    def set_frame(self, slot: int, frame: Frame, pose: Optional[Pose] = None):
        """Write one frame slot; pose defaults to frame.gt_pose."""
        h, w = self.intrinsics.height, self.intrinsics.width
        c_ = np.ascontiguousarray(frame.color, dtype=np.float64)
        d_ = np.ascontiguousarray(frame.depth, dtype=np.float64)
        if c_.shape != (h, w, 3) or d_.shape != (h, w):
            raise ValueError("frame size does not match the intrinsics")
        pc = (pose or frame.gt_pose or Pose())._c()
        self._check(self._lib.vrf_frame_set(self._h, int(slot), _ptr(c_), _ptr(d_), C.byref(pc)))
        self.n_frames = max(self.n_frames, int(slot) + 1)

    def set_frame_u8u16(self, slot: int, rgb: np.ndarray, depth_units: np.ndarray,
                        pose: Pose):
        """Write one frame slot from sensor data: uint8 RGB (H, W, 3) and uint16 depth
        units (H, W), converted on the device like the reference's PNG loaders."""
        h, w = self.intrinsics.height, self.intrinsics.width
        c_ = np.ascontiguousarray(rgb, dtype=np.uint8)
        d_ = np.ascontiguousarray(depth_units, dtype=np.uint16)
        if c_.shape != (h, w, 3) or d_.shape != (h, w):
            raise ValueError("frame size does not match the intrinsics")
        pc = pose._c()
        self._check(self._lib.vrf_frame_set_u8u16(self._h, int(slot), _ptr(c_), _ptr(d_),
                                                  C.byref(pc)))
        self.n_frames = max(self.n_frames, int(slot) + 1)

    def set_frame_pose(self, slot: int, pose: Pose):
        pc = pose._c()
        self._check(self._lib.vrf_frame_set_pose(self._h, int(slot), C.byref(pc)))

    # ---- renderer
    def render_image(self, intr: CameraIntrinsics, pose: Pose, params: RenderParams = None,
                     stride: int = 1) -> Frame:
        params = params or RenderParams()
        if stride < 1:
            raise ValueError("render_image: stride must be >= 1")
        ow = (intr.width + stride - 1) // stride
        oh = (intr.height + stride - 1) // stride
        color = np.zeros((oh, ow, 3))
        depth = np.zeros((oh, ow))
        ic, pc, rp = intr._c(), pose._c(), params._c()
        self._check(self._lib.vrf_render_image(self._h, C.byref(ic), C.byref(pc), C.byref(rp),
                                               stride, _ptr(color), _ptr(depth)))
        return Frame(color, depth, 0.0, pose)

    def sample_rays(self, rays: np.ndarray, params: RenderParams = None, cap: int = 4096):
        params = params or RenderParams()
        rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 6)
        n = rays.shape[0]
        counts = np.zeros(n, np.int32)
        t = np.zeros((n, cap))
        delta = np.zeros((n, cap))
        cells = np.zeros((n, cap), np.uint32)
        rp = params._c()
        self._check(self._lib.vrf_debug_sample_rays(self._h, _ptr(rays), n, C.byref(rp), cap,
                                                    _ptr(counts), _ptr(t), _ptr(delta),
                                                    _ptr(cells)))
        return counts, t, delta, cells

    def render_rays(self, rays: np.ndarray, params: RenderParams = None) -> np.ndarray:
        """(n, 8): r, g, b, depth, T_terminal, count, hit, terminated_early."""
        params = params or RenderParams()
        rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 6)
        out = np.zeros((rays.shape[0], 8))
        rp = params._c()
        self._check(self._lib.vrf_debug_render_rays(self._h, _ptr(rays), rays.shape[0],
                                                    C.byref(rp), _ptr(out)))
        return out

    # ---- mapping
    def mapping_step(self, config: MappingConfig, batch: np.ndarray) -> MapStepStats:
        b = np.ascontiguousarray(batch, dtype=np.int32).reshape(-1, 3)
        st = capi.MapStepStats_c()
        cc = config._c()
        self._check(self._lib.vrf_mapping_step(self._h, C.byref(cc), _ptr(b), b.shape[0],
                                               C.byref(st)))
        return _stats(st)

    def mapping_steps(self, config: MappingConfig, rng: "Rng", n_keyframes: int, n_steps: int):
        """n_steps mapping_step calls with batches drawn from rng (map_scene's inner
        loop, mapping.cpp:302-312), host draws overlapped with device steps."""
        st = (capi.MapStepStats_c * max(n_steps, 1))()
        cc = config._c()
        self._check(self._lib.vrf_mapping_steps(self._h, C.byref(cc), rng.state, int(n_keyframes),
                                                int(config.rays_per_batch), int(n_steps), st))
        return [_stats(st[i]) for i in range(n_steps)]

    def mapping_step_device(self, config: MappingConfig, batch_dev_ptr: int, n: int) -> MapStepStats:
        st = capi.MapStepStats_c()
        cc = config._c()
        self._check(self._lib.vrf_mapping_step_device(self._h, C.byref(cc),
                                                      C.c_void_p(batch_dev_ptr), n, C.byref(st)))
        return _stats(st)

    def mapping_gradient(self, config: MappingConfig, batch: np.ndarray):
        b = np.ascontiguousarray(batch, dtype=np.int32).reshape(-1, 3)
        grad = np.empty((self.geom.num_vertices, PAYLOAD))
        st = capi.MapStepStats_c()
        cc = config._c()
        self._check(self._lib.vrf_mapping_gradient(self._h, C.byref(cc), _ptr(b), b.shape[0],
                                                   _ptr(grad), C.byref(st)))
        return grad, _stats(st)

    def rmsprop_reset(self):
        self._check(self._lib.vrf_rmsprop_reset(self._h))

    def rmsprop_upload(self, v: np.ndarray):
        vv = np.ascontiguousarray(v, dtype=np.float64).reshape(-1)
        if vv.size != self.geom.num_vertices * PAYLOAD:
            raise ValueError("rmsprop state size does not match the grid")
        self._check(self._lib.vrf_rmsprop_upload(self._h, _ptr(vv)))

    def rmsprop_v(self) -> np.ndarray:
        v = np.empty((self.geom.num_vertices, PAYLOAD))
        self._check(self._lib.vrf_rmsprop_download(self._h, _ptr(v)))
        return v

    def map_forward(self, config: MappingConfig, batch_dev_ptr: int, n: int):
        out = capi.MapPartials_c()
        cc = config._c()
        self._check(self._lib.vrf_map_forward(self._h, C.byref(cc), C.c_void_p(batch_dev_ptr), n,
                                              C.byref(out)))
        return out

    def map_backward(self, config: MappingConfig, rays_color: int, rays_depth: int):
        cc = config._c()
        self._check(self._lib.vrf_map_backward(self._h, C.byref(cc), rays_color, rays_depth))

    def map_apply(self, config: MappingConfig, v_begin: int, v_end: int):
        cc = config._c()
        self._check(self._lib.vrf_map_apply(self._h, C.byref(cc), v_begin, v_end))

    # ---- tracking
    # ---- block-sparse multi-GPU exchange (device pointers; see distributed.py)
    def blocks_count(self) -> int:
        n = C.c_int32()
        self._check(self._lib.vrf_blocks_count(self._h, C.byref(n)))
        return int(n.value)

    def blocks_touched(self, flags_ptr: int):
        self._check(self._lib.vrf_blocks_touched(self._h, C.c_void_p(flags_ptr)))

    def blocks_pack(self, ids_ptr: int, n: int, which: int, out_ptr: int):
        self._check(self._lib.vrf_blocks_pack(self._h, C.c_void_p(ids_ptr), int(n), int(which),
                                              C.c_void_p(out_ptr)))

    def blocks_unpack_payload(self, ids_ptr: int, n: int, in_ptr: int):
        self._check(self._lib.vrf_blocks_unpack_payload(self._h, C.c_void_p(ids_ptr), int(n),
                                                        C.c_void_p(in_ptr)))

    def blocks_apply(self, config: MappingConfig, ids_ptr: int, n: int, grad_ptr: int):
        cc = config._c()
        self._check(self._lib.vrf_blocks_apply(self._h, C.byref(cc), C.c_void_p(ids_ptr), int(n),
                                               C.c_void_p(grad_ptr)))

    def grad_clear(self):
        self._check(self._lib.vrf_grad_clear(self._h))

    # ---- fused peer-memory exchange (vrf_exchange_p2p)
    def peer_buffers(self):
        b = capi.PeerBuffers_c()
        self._check(self._lib.vrf_peer_buffers_get(self._h, C.byref(b)))
        return b

    def peers_set(self, rank: int, peers) -> None:
        """peers: one PeerBuffers_c per rank (rank order), valid on this device."""
        arr = (capi.PeerBuffers_c * len(peers))(*peers)
        self._check(self._lib.vrf_peers_set(self._h, len(peers), int(rank), arr))

    def ipc_export(self) -> bytes:
        buf = (C.c_uint8 * capi.IPC_HANDLE_BYTES)()
        self._check(self._lib.vrf_ipc_export(self._h, buf))
        return bytes(buf)

    def peers_open_ipc(self, rank: int, handles) -> None:
        """handles: every rank's ipc_export() bytes, rank order."""
        blob = b"".join(handles)
        if len(blob) != capi.IPC_HANDLE_BYTES * len(handles):
            raise ValueError("peers_open_ipc: malformed handles")
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        self._check(self._lib.vrf_peers_open_ipc(self._h, len(handles), int(rank), buf))

    def exchange_p2p(self, config: MappingConfig):
        cc = config._c()
        self._check(self._lib.vrf_exchange_p2p(self._h, C.byref(cc)))

    def pose_gradient(self, frame: int, intr: CameraIntrinsics, pose: Pose, pixels: np.ndarray,
                      config: TrackingConfig) -> PoseGradient:
        px = np.ascontiguousarray(pixels, dtype=np.int32).reshape(-1, 2)
        out = capi.PoseGradient_c()
        ic, pc, lc = intr._c(), pose._c(), config._loss_c()
        self._check(self._lib.vrf_pose_gradient(self._h, frame, C.byref(ic), C.byref(pc),
                                                _ptr(px), px.shape[0], C.byref(lc), C.byref(out)))
        return PoseGradient(np.array(out.d_omega), np.array(out.d_tau), out.loss, out.rays_used,
                            out.samples)

    def pose_normal_equations(self, frame: int, intr: CameraIntrinsics, pose: Pose,
                              pixels: np.ndarray, config: TrackingConfig,
                              kernel: int = capi.POSE_KERNEL_PARITY) -> NormalEquations:
        """JᵀJ / Jᵀr over the given pixels; kernel selects the pose kernel
        (POSE_KERNEL_PARITY: FP64, POSE_KERNEL_GN: the Gauss-Newton tracker's)."""
        px = np.ascontiguousarray(pixels, dtype=np.int32).reshape(-1, 2)
        out = capi.NormalEquations_c()
        ic, pc, lc = intr._c(), pose._c(), config._loss_c()
        self._check(self._lib.vrf_pose_normal_equations_ex(self._h, frame, C.byref(ic),
                                                           C.byref(pc), _ptr(px), px.shape[0],
                                                           C.byref(lc), kernel, C.byref(out)))
        return NormalEquations(unpack_sym6(out.jtj), np.array(out.jtr), out.loss, out.rays_used,
                               out.samples)

    def evaluate_views(self, intr: CameraIntrinsics, poses: Sequence[Pose], colors, depths,
                       samples: np.ndarray, params: Optional[RenderParams] = None):
        """vrf_evaluate_views: renders each view on the device and scores it there
        against (colors[v], depths[v]). Returns (sum_sq_color, color_samples,
        sum_abs_depth, depth_pixels)."""
        n = len(poses)
        h, w = intr.height, intr.width
        cs = [np.ascontiguousarray(c, np.float64) for c in colors]
        ds = [np.ascontiguousarray(d, np.float64) for d in depths]
        for c, d in zip(cs, ds):
            if c.shape != (h, w, 3) or d.shape != (h, w):
                raise ValueError("evaluate_map_quality: image dimensions differ")
        pa = (capi.Pose_c * n)(*[p._c() for p in poses])
        cp = (C.c_void_p * n)(*[c.ctypes.data for c in cs])
        dp = (C.c_void_p * n)(*[d.ctypes.data for d in ds])
        smp = np.ascontiguousarray(samples, np.int32).reshape(-1, 3)
        out = capi.ViewMetrics_c()
        ic, rp = intr._c(), (params or RenderParams())._c()
        self._check(self._lib.vrf_evaluate_views(self._h, C.byref(ic), n, pa, cp, dp,
                                                 C.byref(rp), _ptr(smp), smp.shape[0],
                                                 C.byref(out)))
        return out.sum_sq_color, out.color_samples, out.sum_abs_depth, out.depth_pixels

    def track_frame(self, frame: int, intr: CameraIntrinsics, init: Pose,
                    config: TrackingConfig) -> TrackFrameResult:
        out = capi.TrackFrameResult_c()
        trace = np.zeros(max(config.iterations, 1))
        ic, pc, tc = intr._c(), init._c(), config._c()
        self._check(self._lib.vrf_track_frame(self._h, frame, C.byref(ic), C.byref(pc),
                                              C.byref(tc), C.byref(out), _ptr(trace)))
        return TrackFrameResult(Pose._from_c(out.pose), list(trace[:out.iterations_run]),
                                bool(out.failed), out.iterations_run)

    def track_frame_gn(self, frame: int, intr: CameraIntrinsics, init: Pose,
                       config: GNConfig) -> TrackFrameResult:
        out = capi.TrackFrameResult_c()
        ic, pc, gc = intr._c(), init._c(), config._c()
        self._check(self._lib.vrf_track_frame_gn(self._h, frame, C.byref(ic), C.byref(pc),
                                                 C.byref(gc), C.byref(out)))
        return TrackFrameResult(Pose._from_c(out.pose), [out.final_loss], bool(out.failed),
                                out.iterations_run)

    def track_frame_gn_history(self) -> np.ndarray:
        """(loss/m, m, samples) per iteration of the last track_frame_gn call."""
        n = self._lib.vrf_track_frame_gn_history(self._h, None, 0)
        h = np.zeros(3 * max(n, 1))
        self._lib.vrf_track_frame_gn_history(self._h, h.ctypes.data_as(C.POINTER(C.c_double)),
                                             3 * n)
        return h[:3 * n].reshape(n, 3)


def unpack_sym6(packed) -> np.ndarray:
    m = np.zeros((6, 6))
    k = 0
    for a in range(6):
        for b in range(a, 6):
            m[a, b] = m[b, a] = packed[k]
            k += 1
    return m


def _stats(st) -> MapStepStats:
    return MapStepStats(st.loss_photometric, st.loss_geometric, st.loss_total, st.rays_color,
                        st.rays_depth, st.psnr_estimate, st.samples)


# ---------------------------------------------------------------- reference-named functions
_DEFAULT: Optional[Context] = None


def default_context() -> Context:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Context(0)
    return _DEFAULT


def render_image(grid: VoxelGrid, intr: CameraIntrinsics, pose: Pose,
                 params: RenderParams = None, stride: int = 1, threads: int = 0) -> Frame:
    """render_image — renderer.hpp:83-84."""
    ctx = default_context()
    ctx.load_grid(grid)
    return ctx.render_image(intr, pose, params or RenderParams(), stride)


def mapping_step(grid: VoxelGrid, keyframes: Sequence[Frame], intrinsics: CameraIntrinsics,
                 config: MappingConfig, rmsprop: RmspropState, rng: Rng) -> MapStepStats:
    """mapping_step — mapping.hpp:80-82: draws the batch from rng, renders, applies
    the RGB+depth gradient through sparse RMSProp, mutates grid and rmsprop."""
    if not keyframes:
        raise RuntimeError("mapping_step: no keyframes")
    ctx = default_context()
    ctx.load_grid(grid)
    ctx.load_frames(intrinsics, keyframes)
    if rmsprop.v is None or rmsprop.v.size != grid.data.size:
        rmsprop.v = np.zeros(grid.data.size)
    _upload_rms(ctx, rmsprop.v)
    batch = rng.draw_batch(len(keyframes), intrinsics.width, intrinsics.height,
                           config.rays_per_batch)
    stats = ctx.mapping_step(config, batch)
    grid.data[:] = ctx.download_grid().data
    rmsprop.v = ctx.rmsprop_v().reshape(-1)
    return stats


def _upload_rms(ctx: Context, v: np.ndarray):
    """Seed the device RMSProp state from the host copy (stored fp32 on device)."""
    ctx.rmsprop_upload(v)


def pose_gradient(grid: VoxelGrid, frame: Frame, intrinsics: CameraIntrinsics, pose: Pose,
                  pixels: np.ndarray, config: TrackingConfig) -> PoseGradient:
    """pose_gradient — tracking.hpp:70-73."""
    ctx = default_context()
    ctx.load_grid(grid)
    ctx.load_frames(intrinsics, [frame])
    return ctx.pose_gradient(0, intrinsics, pose, pixels, config)


def track_frame(grid: VoxelGrid, frame: Frame, intrinsics: CameraIntrinsics, init: Pose,
                config: TrackingConfig) -> TrackFrameResult:
    """track_frame — tracking.hpp:82-84 (Adam, reference pixel stream)."""
    ctx = default_context()
    ctx.load_grid(grid)
    ctx.load_frames(intrinsics, [frame])
    return ctx.track_frame(0, intrinsics, init, config)


def pose_compose(a: Pose, b: Pose) -> Pose:
    """operator* — pose.hpp:27-29."""
    aw, ax, ay, az = a.q
    bw, bx, by, bz = b.q
    q = np.array([aw * bw - ax * bx - ay * by - az * bz,
                  aw * bx + ax * bw + ay * bz - az * by,
                  aw * by + ay * bw + az * bx - ax * bz,
                  aw * bz + az * bw + ax * by - ay * bx])
    q /= math.sqrt(float(q @ q))
    t = a.rotation() @ np.asarray(b.t) + np.asarray(a.t)
    return Pose(tuple(q), tuple(t))


def pose_inverse(p: Pose) -> Pose:
    w, x, y, z = p.q
    qi = Pose((w, -x, -y, -z), (0.0, 0.0, 0.0))
    return Pose(qi.q, tuple(-(qi.rotation() @ np.asarray(p.t))))


def track_sequence(grid: VoxelGrid, frames: Sequence[Frame], intrinsics: CameraIntrinsics,
                   config: TrackingConfig, ctx: Optional[Context] = None):
    """track_sequence — tracking.hpp:102-103 (tracking.cpp:254-295). Returns
    (poses, status) with status rows (frame, iterations, final_loss, elapsed_ms, failed)."""
    import time
    if not frames:
        raise RuntimeError("track_sequence: empty dataset")
    if frames[0].gt_pose is None:
        raise RuntimeError("track_sequence: first frame needs a pose")
    ctx = ctx if ctx is not None else default_context()
    ctx.load_grid(grid)
    ctx.load_frames(intrinsics, frames)
    first = frames[0].gt_pose
    poses = [first]
    status = [(0, 0, 0.0, 0.0, False)]
    prev = prev_prev = first
    have_two = False
    for i in range(1, len(frames)):
        init = prev
        if config.init_policy == "constant_velocity" and have_two:
            init = pose_compose(prev, pose_compose(pose_inverse(prev_prev), prev))
        fc = TrackingConfig(**{**config.__dict__})
        fc.seed = (config.seed + 0x9E3779B9 * i) & (2**64 - 1)
        t0 = time.perf_counter()
        tf = ctx.track_frame(i, intrinsics, init, fc)
        ms = (time.perf_counter() - t0) * 1e3
        poses.append(tf.pose)
        status.append((i, tf.iterations_run, tf.loss_trace[-1] if tf.loss_trace else 0.0, ms,
                       tf.failed))
        if not tf.failed:
            prev_prev, prev, have_two = prev, tf.pose, True
    return poses, status


def generate_ray(intr: CameraIntrinsics, pose: Pose, px: float, py: float):
    """generate_ray — camera.hpp:33-41 (host helper for geometry fitting)."""
    v = np.array([(px - intr.cx) / intr.fx, (py - intr.cy) / intr.fy, 1.0])
    v = v / math.sqrt(float(v @ v))
    return np.asarray(pose.t, np.float64), pose.rotation() @ v


def fit_grid_geometry(frames: Sequence[Frame], keyframes: Sequence[int],
                      intrinsics: CameraIntrinsics, config: MappingConfig) -> GridGeometry:
    """fit_grid_geometry — mapping.cpp:235-276: bounds of the back-projected valid
    depth (every 8th pixel) and camera centres, plus the margin."""
    lo = np.full(3, np.inf)
    hi = -lo
    ys = np.arange(0, intrinsics.height, 8)
    xs = np.arange(0, intrinsics.width, 8)
    for k in keyframes:
        f = frames[k]
        if f.gt_pose is None:
            continue
        t = np.asarray(f.gt_pose.t, np.float64)
        lo, hi = np.minimum(lo, t), np.maximum(hi, t)
        d = np.asarray(f.depth)[np.ix_(ys, xs)]
        yy, xx = np.meshgrid(ys, xs, indexing="ij")
        ok = d > 0.0
        if not ok.any():
            continue
        cam = np.stack([(xx[ok] - intrinsics.cx) / intrinsics.fx,
                        (yy[ok] - intrinsics.cy) / intrinsics.fy, np.ones(int(ok.sum()))], 1)
        cam /= np.sqrt(np.sum(cam * cam, 1, keepdims=True))
        p = t + d[ok][:, None] * (cam @ f.gt_pose.rotation().T)
        lo, hi = np.minimum(lo, p.min(0)), np.maximum(hi, p.max(0))
    if not (np.all(np.isfinite(lo)) and np.all(np.isfinite(hi))):
        raise RuntimeError("fit_grid_geometry: no valid depth to bound the scene")
    margin = (hi - lo) * config.bounds_margin
    lo, hi = lo - margin, hi + margin
    voxel = float(np.max(hi - lo)) / float(config.initial_resolution - 1)
    res, origin = [], []
    for a in range(3):
        cells = max(1, int(math.ceil((hi[a] - lo[a]) / voxel - 1e-9)))
        res.append(cells + 1)
        origin.append(float(lo[a] - 0.5 * (cells * voxel - (hi[a] - lo[a]))))
    g = GridGeometry(tuple(res), tuple(origin), voxel)
    g.validate()
    return g


def map_scene(frames: Sequence[Frame], intrinsics: CameraIntrinsics, config: MappingConfig,
              geometry: Optional[GridGeometry] = None, ctx: Optional[Context] = None):
    """map_scene — mapping.hpp:98-99 (mapping.cpp:278-316). The grid, RMSProp state
    and keyframes stay in HBM for the whole stage schedule (device upsampling
    between stages); returns (grid, log rows (iteration, stats, elapsed_ms))."""
    import time
    if not frames:
        raise RuntimeError("map_scene: empty dataset")
    keys = list(range(0, len(frames), config.keyframe_stride))
    for i in keys:
        if frames[i].gt_pose is None:
            raise RuntimeError(f"map_scene: keyframe {i} has no pose")
    geom = geometry or fit_grid_geometry(frames, keys, intrinsics, config)
    ctx = ctx or default_context()
    ctx.init_grid(geom, config.sigma_init)
    ctx.load_frames(intrinsics, [frames[i] for i in keys])
    rng = Rng(config.seed)
    log = []
    t0 = time.perf_counter()
    it_global = 0
    for stage in range(config.upsample_stages + 1):
        if stage > 0:
            ctx.upsample(config.max_resolution)
        left = config.iterations_per_stage
        while left > 0:
            # run up to the next prune point in one pipelined call
            n = left
            if config.prune_every > 0:
                n = min(n, config.prune_every - it_global % config.prune_every)
            stats = ctx.mapping_steps(config, rng, len(keys), n)
            ms = (time.perf_counter() - t0) * 1e3
            for st in stats:
                log.append((it_global, st, ms))
                it_global += 1
            left -= n
            if config.prune_every > 0 and it_global % config.prune_every == 0:
                ctx.prune(config.prune_threshold)
    return ctx.download_grid(), log
