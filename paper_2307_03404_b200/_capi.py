"""ctypes binding of the C-ABI in include/voxrf_b200.h.

Loading fails loudly when libvoxrf_b200.so is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# VRF_LIB: another build of this same library (A/B experiments, tools/ab/).
_LIB_PATH = Path(os.environ.get("VRF_LIB") or
                 Path(__file__).resolve().parent / "_lib" / "libvoxrf_b200.so")

VRF_OK = 0
VRF_ERR_INVALID_ARGUMENT = 1
VRF_ERR_OUT_OF_RANGE = 2
VRF_ERR_RUNTIME = 3
VRF_ERR_CUDA = 4

# pose kernels (include/voxrf_b200.h VRF_POSE_KERNEL_*)
POSE_KERNEL_PARITY = 0
POSE_KERNEL_GN = 1
POSE_KERNEL_GN_CHECK = 2


class GridGeometry_c(C.Structure):
    _fields_ = [("res", C.c_int32 * 3), ("origin", C.c_double * 3), ("voxel_size", C.c_double)]


class Intrinsics_c(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("depth_scale", C.c_double)]


class Pose_c(C.Structure):
    _fields_ = [("q", C.c_double * 4), ("t", C.c_double * 3)]


class RenderParams_c(C.Structure):
    _fields_ = [("step", C.c_double), ("t_near", C.c_double), ("t_far", C.c_double),
                ("termination_eps", C.c_double)]


class MappingConfig_c(C.Structure):
    _fields_ = [("lambda_d", C.c_double), ("lr_sigma", C.c_double), ("lr_sh", C.c_double),
                ("rmsprop_decay", C.c_double), ("rmsprop_eps", C.c_double),
                ("deterministic", C.c_int32), ("reserved", C.c_int32),
                ("render", RenderParams_c)]


class MapStepStats_c(C.Structure):
    _fields_ = [("loss_photometric", C.c_double), ("loss_geometric", C.c_double),
                ("loss_total", C.c_double), ("rays_color", C.c_int32),
                ("rays_depth", C.c_int32), ("psnr_estimate", C.c_double),
                ("samples", C.c_int64), ("bad_ray", C.c_int32), ("reserved", C.c_int32)]


class TrackingLoss_c(C.Structure):
    _fields_ = [("lambda_p", C.c_double), ("lambda_d", C.c_double), ("render", RenderParams_c)]


class PoseGradient_c(C.Structure):
    _fields_ = [("d_omega", C.c_double * 3), ("d_tau", C.c_double * 3), ("loss", C.c_double),
                ("rays_used", C.c_int32), ("reserved", C.c_int32), ("samples", C.c_int64)]


class NormalEquations_c(C.Structure):
    _fields_ = [("jtj", C.c_double * 21), ("jtr", C.c_double * 6), ("loss", C.c_double),
                ("rays_used", C.c_int32), ("reserved", C.c_int32), ("samples", C.c_int64)]


class TrackingConfig_c(C.Structure):
    _fields_ = [("rays_per_iteration", C.c_int32), ("iterations", C.c_int32),
                ("lr_omega", C.c_double), ("lr_tau", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("adam_eps", C.c_double), ("lambda_p", C.c_double),
                ("lambda_d", C.c_double), ("convergence_step", C.c_double),
                ("divergence_factor", C.c_double), ("divergence_patience", C.c_int32),
                ("max_redraws", C.c_int32), ("seed", C.c_uint64), ("render", RenderParams_c)]


class TrackFrameResult_c(C.Structure):
    _fields_ = [("pose", Pose_c), ("failed", C.c_int32), ("iterations_run", C.c_int32),
                ("final_loss", C.c_double)]


class GnConfig_c(C.Structure):
    _fields_ = [("rays_per_iteration", C.c_int32), ("iterations", C.c_int32),
                ("lambda_p", C.c_double), ("lambda_d", C.c_double), ("damping", C.c_double),
                ("max_redraws", C.c_int32), ("kernel", C.c_int32), ("seed", C.c_uint64),
                ("render", RenderParams_c)]


class ViewMetrics_c(C.Structure):
    _fields_ = [("sum_sq_color", C.c_double), ("color_samples", C.c_int64),
                ("sum_abs_depth", C.c_double), ("depth_pixels", C.c_int64)]


class DeviceBuffers_c(C.Structure):
    _fields_ = [("payload", C.c_void_p), ("grad", C.c_void_p), ("rms_v", C.c_void_p),
                ("num_vertices", C.c_int64), ("padded_vertices", C.c_int64),
                ("stream", C.c_void_p)]


class PeerBuffers_c(C.Structure):
    _fields_ = [("grad", C.c_uint64), ("payload", C.c_uint64), ("tb", C.c_uint64)]


IPC_HANDLE_BYTES = 192
MAX_PEERS = 8


class MapPartials_c(C.Structure):
    _fields_ = [("rays_color", C.c_int32), ("rays_depth", C.c_int32),
                ("sum_photometric", C.c_double), ("sum_geometric", C.c_double),
                ("samples", C.c_int64), ("bad_ray", C.c_int32), ("reserved", C.c_int32)]


P = C.POINTER
vp = C.c_void_p
_SIGS = {
    "vrf_abi_version": (C.c_int, []),
    "vrf_context_create": (C.c_int, [C.c_int, P(vp)]),
    "vrf_context_destroy": (None, [vp]),
    "vrf_last_error": (C.c_char_p, [vp]),
    "vrf_set_shard_multiple": (C.c_int, [vp, C.c_int]),
    "vrf_set_stream": (C.c_int, [vp, vp]),
    "vrf_set_record_limits": (C.c_int, [vp, C.c_double, C.c_int]),
    "vrf_grid_write_vertices": (C.c_int, [vp, C.c_int64, C.c_int64, vp]),
    "vrf_rmsprop_write_vertices": (C.c_int, [vp, C.c_int64, C.c_int64, vp]),
    "vrf_grid_set_occupancy": (C.c_int, [vp, vp]),
    "vrf_track_updates": (C.c_int, [vp, C.c_int]),
    "vrf_updates_count": (C.c_int, [vp, P(C.c_int64)]),
    "vrf_updates_read": (C.c_int, [vp, C.c_int64, vp, vp, vp]),
    "vrf_updates_read_range": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int, vp, vp, vp]),
    "vrf_state_read_f32": (C.c_int, [vp, C.c_int, C.c_int64, C.c_int64, vp]),
    "vrf_host_alloc": (vp, [C.c_size_t]),
    "vrf_host_free": (None, [vp]),
    "vrf_get_device_buffers": (C.c_int, [vp, P(DeviceBuffers_c)]),
    "vrf_kernel_launch_count": (C.c_int64, [vp]),
    "vrf_profile_enable": (C.c_int, [vp, C.c_int]),
    "vrf_profile_read": (C.c_int, [vp, C.c_int, P(C.c_double), P(C.c_int64)]),
    "vrf_profile_touched_groups": (C.c_int64, [vp]),
    "vrf_profile_track_samples": (C.c_int64, [vp]),
    "vrf_grid_init": (C.c_int, [vp, P(GridGeometry_c), C.c_double]),
    "vrf_grid_fill": (C.c_int, [vp, C.c_double]),
    "vrf_grid_upload": (C.c_int, [vp, P(GridGeometry_c), vp, vp]),
    "vrf_grid_upload_f32": (C.c_int, [vp, P(GridGeometry_c), vp, vp]),
    "vrf_grid_download": (C.c_int, [vp, vp, vp]),
    "vrf_grid_download_f32": (C.c_int, [vp, vp]),
    "vrf_grid_get_geometry": (C.c_int, [vp, P(GridGeometry_c)]),
    "vrf_grid_prune": (C.c_int, [vp, C.c_double, P(C.c_int64)]),
    "vrf_grid_digest": (C.c_int, [vp, P(C.c_uint64)]),
    "vrf_grid_upsample": (C.c_int, [vp, C.c_int]),
    "vrf_grid_save": (C.c_int, [vp, C.c_char_p]),
    "vrf_grid_load": (C.c_int, [vp, C.c_char_p]),
    "vrf_frames_upload": (C.c_int, [vp, P(Intrinsics_c), C.c_int, P(vp), P(vp), P(Pose_c)]),
    "vrf_frames_count": (C.c_int, [vp]),
    "vrf_frames_reserve": (C.c_int, [vp, P(Intrinsics_c), C.c_int]),
    "vrf_frame_set": (C.c_int, [vp, C.c_int, vp, vp, P(Pose_c)]),
    "vrf_frame_set_pose": (C.c_int, [vp, C.c_int, P(Pose_c)]),
    "vrf_frame_set_u8u16": (C.c_int, [vp, C.c_int, vp, vp, P(Pose_c)]),
    "vrf_render_image": (C.c_int, [vp, P(Intrinsics_c), P(Pose_c), P(RenderParams_c), C.c_int,
                                   vp, vp]),
    "vrf_mapping_step": (C.c_int, [vp, P(MappingConfig_c), vp, C.c_int, P(MapStepStats_c)]),
    "vrf_mapping_steps": (C.c_int, [vp, P(MappingConfig_c), P(C.c_uint64), C.c_int, C.c_int,
                                    C.c_int, P(MapStepStats_c)]),
    "vrf_mapping_step_device": (C.c_int, [vp, P(MappingConfig_c), vp, C.c_int,
                                          P(MapStepStats_c)]),
    "vrf_mapping_gradient": (C.c_int, [vp, P(MappingConfig_c), vp, C.c_int, vp,
                                       P(MapStepStats_c)]),
    "vrf_rmsprop_reset": (C.c_int, [vp]),
    "vrf_rmsprop_download": (C.c_int, [vp, vp]),
    "vrf_rmsprop_upload": (C.c_int, [vp, vp]),
    "vrf_map_forward": (C.c_int, [vp, P(MappingConfig_c), vp, C.c_int, P(MapPartials_c)]),
    "vrf_map_backward": (C.c_int, [vp, P(MappingConfig_c), C.c_int32, C.c_int32]),
    "vrf_map_apply": (C.c_int, [vp, P(MappingConfig_c), C.c_int64, C.c_int64]),
    "vrf_blocks_count": (C.c_int, [vp, P(C.c_int32)]),
    "vrf_blocks_touched": (C.c_int, [vp, vp]),
    "vrf_blocks_pack": (C.c_int, [vp, vp, C.c_int, C.c_int, vp]),
    "vrf_blocks_unpack_payload": (C.c_int, [vp, vp, C.c_int, vp]),
    "vrf_blocks_apply": (C.c_int, [vp, P(MappingConfig_c), vp, C.c_int, vp]),
    "vrf_grad_clear": (C.c_int, [vp]),
    "vrf_peer_buffers_get": (C.c_int, [vp, P(PeerBuffers_c)]),
    "vrf_peers_set": (C.c_int, [vp, C.c_int, C.c_int, P(PeerBuffers_c)]),
    "vrf_ipc_export": (C.c_int, [vp, vp]),
    "vrf_peers_open_ipc": (C.c_int, [vp, C.c_int, C.c_int, vp]),
    "vrf_exchange_p2p": (C.c_int, [vp, P(MappingConfig_c)]),
    "vrf_pose_gradient": (C.c_int, [vp, C.c_int, P(Intrinsics_c), P(Pose_c), vp, C.c_int,
                                    P(TrackingLoss_c), P(PoseGradient_c)]),
    "vrf_pose_normal_equations": (C.c_int, [vp, C.c_int, P(Intrinsics_c), P(Pose_c), vp,
                                            C.c_int, P(TrackingLoss_c), P(NormalEquations_c)]),
    "vrf_pose_normal_equations_ex": (C.c_int, [vp, C.c_int, P(Intrinsics_c), P(Pose_c), vp,
                                               C.c_int, P(TrackingLoss_c), C.c_int,
                                               P(NormalEquations_c)]),
    "vrf_track_frame": (C.c_int, [vp, C.c_int, P(Intrinsics_c), P(Pose_c),
                                  P(TrackingConfig_c), P(TrackFrameResult_c), vp]),
    "vrf_track_frame_gn": (C.c_int, [vp, C.c_int, P(Intrinsics_c), P(Pose_c), P(GnConfig_c),
                                     P(TrackFrameResult_c)]),
    "vrf_track_frame_gn_history": (C.c_int, [vp, P(C.c_double), C.c_int]),
    "vrf_evaluate_views": (C.c_int, [vp, P(Intrinsics_c), C.c_int, vp, vp, vp,
                                     P(RenderParams_c), vp, C.c_int, P(ViewMetrics_c)]),
    "vrf_rng_draw_eval_samples": (None, [P(C.c_uint64), C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, vp]),
    "vrf_rng_seed": (None, [C.c_uint64, P(C.c_uint64)]),
    "vrf_rng_next": (C.c_uint64, [P(C.c_uint64)]),
    "vrf_rng_draw_batch": (None, [P(C.c_uint64), C.c_int, C.c_int, C.c_int, C.c_int, vp]),
    "vrf_rng_draw_valid_pixels": (C.c_int, [P(C.c_uint64), vp, C.c_int, C.c_int, C.c_int,
                                            C.c_int, vp]),
    "vrf_debug_sample_rays": (C.c_int, [vp, vp, C.c_int, P(RenderParams_c), C.c_int, vp, vp, vp,
                                        vp]),
    "vrf_debug_render_rays": (C.c_int, [vp, vp, C.c_int, P(RenderParams_c), vp]),
}

EXPORTED = tuple(_SIGS)
_lib = None


def lib_path() -> Path:
    return _LIB_PATH


def load() -> C.CDLL:
    """Load libvoxrf_b200.so; raise if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise RuntimeError(
            f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(str(_LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
