"""B200-native multi-depth-camera renderer (RPL distillation-stage depth path).

Drop-in for the renderer API of the reference package ``multidepth``
(/root/reference/pkg/src/multidepth/__init__.py:14-82) restricted to the hot
path: mesh registration, camera intrinsics/extrinsics, per-step pose updates,
``render`` returning an [envs, cams, H, W] depth tensor, and the sensor model
(noise, dropout, latency, downsampling). Rendering runs in hand-written CUDA
kernels for sm_100a (libmdrt.so, C ABI in include/mdrt.h); there is no CPU
backend.
"""

from .transforms import (RigidPose, Ray, quat_identity, quat_normalize, quat_mul, quat_conjugate,
                         quat_rotate, quat_to_matrix, quat_from_matrix, quat_from_axis_angle,
                         quat_from_euler, quat_yaw, world_to_body_ray, body_to_world_ray)
from .mesh import TriMesh, load_obj, save_obj, make_box, make_plane, make_icosphere, merge_meshes
from .bvh import BVH, build_bvh, query_bvh, validate_bvh
from .camera import CameraModel, build_depth_ray, look_at_pose
from .scene import Scene, Body, DepthFrame, render, render_naive_baseline, depth_to_z
from .kernels import BACKENDS, default_backend, resolve_threads
from .sensor import (SensorConfig, CameraRandomization, FrameBuffer, apply_noise_dropout,
                     downsample_min, sample_latencies, sample_camera_offsets, randomize_scene_cameras,
                     randomized_camera)
from .perception import (RsmConfig, RSM_MODES, DEFAULT_RSM_PROBS, rsm_sample_modes, rsm_mask_columns,
                         rsm_apply)
from .pipeline import CapturedStep, render_pipeline
from .frameio import (FormatError, FrameWriter, write_frames, read_frames, write_grid, read_grid, depth_to_u8,
                      write_pgm, read_pgm)

__version__ = "0.1.0"

__all__ = [
    "RigidPose", "Ray", "quat_identity", "quat_normalize", "quat_mul", "quat_conjugate",
    "quat_rotate", "quat_to_matrix", "quat_from_matrix", "quat_from_axis_angle", "quat_from_euler",
    "quat_yaw", "world_to_body_ray", "body_to_world_ray",
    "BVH", "build_bvh", "query_bvh", "validate_bvh",
    "TriMesh", "load_obj", "save_obj", "make_box", "make_plane", "make_icosphere", "merge_meshes",
    "CameraModel", "build_depth_ray", "look_at_pose",
    "Scene", "Body", "DepthFrame", "render", "render_naive_baseline", "depth_to_z",
    "BACKENDS", "default_backend", "resolve_threads",
    "SensorConfig", "CameraRandomization", "FrameBuffer", "apply_noise_dropout", "downsample_min",
    "sample_latencies", "sample_camera_offsets", "randomize_scene_cameras", "randomized_camera",
    "RsmConfig", "RSM_MODES", "DEFAULT_RSM_PROBS", "rsm_sample_modes", "rsm_mask_columns", "rsm_apply",
    "render_pipeline", "CapturedStep", "FormatError", "FrameWriter", "write_frames", "read_frames",
    "write_grid", "read_grid", "depth_to_u8", "write_pgm", "read_pgm", "__version__",
]
