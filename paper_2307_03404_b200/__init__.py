"""B200-native per-ray hot path of Plenoxel RGB-D mapping and tracking
(arXiv 2307.03404): sm_100a CUDA kernels behind a C-ABI (include/voxrf_b200.h),
with a Python mirror of the reference's render/map/track API."""
from .api import (  # noqa: F401
    CameraIntrinsics, Context, Frame, GNConfig, GridGeometry, MappingConfig, MapStepStats,
    NormalEquations, Pose, PoseGradient, RenderParams, Rng, RmspropState, TrackFrameResult,
    TrackingConfig, VoxelGrid, default_context, mapping_step, pose_gradient, render_image,
    track_frame, track_sequence,
)

__all__ = [
    "CameraIntrinsics", "Context", "Frame", "GNConfig", "GridGeometry", "MappingConfig",
    "MapStepStats", "NormalEquations", "Pose", "PoseGradient", "RenderParams", "Rng",
    "RmspropState", "TrackFrameResult", "TrackingConfig", "VoxelGrid", "default_context",
    "mapping_step", "pose_gradient", "render_image", "track_frame", "track_sequence",
]
