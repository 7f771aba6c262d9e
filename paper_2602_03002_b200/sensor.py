"""Depth-sensor model on the GPU: noise, dropout, latency, downsampling.

Mirror of the reference ``multidepth.sensor`` (/root/reference/pkg/src/multidepth/sensor.py).
Per-pixel work runs in CUDA kernels of libmdrt.so; the random streams are the
reference's own counter-based generator (rng.py), evaluated on the device, so
dropout masks are bit-identical to the reference and noise agrees to the last
float32 bit up to libm ulp differences in log/cos.

Small per-env draws (latencies, camera offsets) stay on the host in
``rng.py`` exactly as in the reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native, rng
from .camera import CameraModel
from .scene import DepthFrame, Scene, _cuda_device
from .transforms import RigidPose, quat_from_euler

NATIVE_RESOLUTION = (240, 135)
POLICY_RESOLUTION = (48, 27)
DOWNSAMPLE_FACTOR = 5
DEFAULT_NOISE_SCALE = 0.1
DEFAULT_DROPOUT_P = 0.05
DEFAULT_MAX_DELAY = 0.100
DEPTH_FLOOR = 1e-6


@dataclass(frozen=True)
class SensorConfig:
    noise_scale: float = DEFAULT_NOISE_SCALE
    dropout_p: float = DEFAULT_DROPOUT_P
    max_delay: float = DEFAULT_MAX_DELAY
    dropout_fill: float | None = None   # None -> camera far limit
    seed: int = 0

    def __post_init__(self):
        if self.noise_scale < 0:
            raise ValueError("noise_scale must be >= 0")
        if not 0.0 <= self.dropout_p < 1.0:
            raise ValueError("dropout_p must be in [0, 1)")
        if self.max_delay < 0:
            raise ValueError("max_delay must be >= 0")

    @property
    def key(self) -> int:
        return int(rng.stream_key(self.seed, "sensor"))


def _to_cuda(depth, device=None):
    """(tensor on GPU, was_numpy)."""
    if isinstance(depth, torch.Tensor):
        if depth.device.type != "cuda":
            return depth.to(_cuda_device(device), torch.float32).contiguous(), "torch-cpu"
        return depth.to(torch.float32).contiguous(), None
    arr = np.ascontiguousarray(np.asarray(depth), dtype=np.float32)
    return torch.from_numpy(arr).to(_cuda_device(device)), "numpy"


def _back(t: torch.Tensor, kind):
    if kind == "numpy":
        return t.cpu().numpy()
    if kind == "torch-cpu":
        return t.cpu()
    return t


def _stream(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def apply_noise_dropout(depth, config: SensorConfig, *, d_max, step: int = 0, env_offset: int = 0):
    """Drop (p) to the fill value or scale by 1 + sigma*g, clamp to [1e-6, d_max] (sensor.py:55-82).

    ``depth`` (N,C,H,W): CUDA tensor (result stays on the device) or numpy
    (computed on the GPU, returned as numpy). ``env_offset`` shifts the env
    counter for env-sliced multi-GPU runs.
    """
    if len(depth.shape) != 4:
        raise ValueError(f"expected (N, C, H, W) depth, got shape {tuple(depth.shape)}")
    t, kind = _to_cuda(depth)
    n, c, h, w = t.shape
    dm = np.ascontiguousarray(np.broadcast_to(np.asarray(d_max, dtype=np.float64), (c,)))
    fill = dm if config.dropout_fill is None else np.full(c, float(config.dropout_fill))
    fill = np.ascontiguousarray(fill, dtype=np.float64)
    out = torch.empty_like(t)
    _native.check(_native.lib().mdrt_noise_dropout(
        ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(out.data_ptr()), n, c, h, w, int(env_offset),
        _native.dptr(dm), _native.dptr(fill), float(config.noise_scale), float(config.dropout_p),
        config.key, int(step), _stream(t)))
    return _back(out, kind)


def downsample_min(depth, factor: int = DOWNSAMPLE_FACTOR):
    """Block-minimum pooling over the trailing (H, W) (sensor.py:85-100)."""
    if factor < 1:
        raise ValueError("factor must be >= 1")
    t, kind = _to_cuda(depth)
    h, w = t.shape[-2:]
    if h % factor or w % factor:
        raise ValueError(f"resolution {w}x{h} not divisible by downsample factor {factor}")
    planes = int(np.prod(t.shape[:-2])) if t.dim() > 2 else 1
    out = torch.empty(tuple(t.shape[:-2]) + (h // factor, w // factor), dtype=torch.float32,
                      device=t.device)
    _native.check(_native.lib().mdrt_downsample_min(
        ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(out.data_ptr()), planes, h, w, factor, _stream(t)))
    return _back(out, kind)


class FrameBuffer:
    """Latency buffer keyed by timestamp, frames resident in HBM (sensor.py:103-150).

    A ring of ``capacity`` device frames. ``fetch_delayed`` returns the newest
    frame with timestamp <= now - delay, else the oldest retained one; the
    batch form selects per env on the device and gathers row e of each
    selected frame. ``render_pipeline`` writes into the ring from inside the
    traversal kernel (no extra pass).
    """

    def __init__(self, capacity: int = 16):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        if capacity > 32:
            raise ValueError("capacity must be <= 32")
        self.capacity = int(capacity)
        self._times: list[float] = []
        self._slots: list[int] = []
        self._ring: torch.Tensor | None = None
        self._slot_buf: torch.Tensor | None = None

    def __len__(self) -> int:
        return len(self._slots)

    @property
    def ring(self) -> torch.Tensor | None:
        """(capacity, N, C, H, W) device storage (for checkpointing)."""
        return self._ring

    def _ensure(self, shape, device) -> None:
        if self._ring is None:
            self._ring = torch.empty((self.capacity,) + tuple(shape), dtype=torch.float32, device=device)
        elif tuple(self._ring.shape[1:]) != tuple(shape) or self._ring.device != device:
            raise ValueError(f"frame shape {tuple(shape)} does not match buffer {tuple(self._ring.shape[1:])}")

    def _reserve(self, timestamp: float) -> int:
        """Register a new newest frame; returns its ring slot (evicts the oldest when full)."""
        if self._times and timestamp <= self._times[-1]:
            raise ValueError(f"timestamps must be strictly increasing; got {timestamp} "
                             f"after {self._times[-1]}")
        if len(self._slots) < self.capacity:
            used = set(self._slots)
            slot = next(s for s in range(self.capacity) if s not in used)
        else:
            slot = self._slots.pop(0)
            self._times.pop(0)
        self._times.append(float(timestamp))
        self._slots.append(slot)
        return slot

    def push(self, frame: DepthFrame) -> None:
        t, _ = _to_cuda(frame.data)
        self._ensure(t.shape, t.device)
        slot = self._reserve(frame.timestamp)
        self._ring[slot].copy_(t)

    def fetch_delayed(self, now: float, delay: float) -> DepthFrame:
        if not self._slots:
            raise LookupError("frame buffer is empty")
        if delay < 0:
            raise ValueError("delay must be >= 0")
        k = int(np.searchsorted(np.asarray(self._times), now - delay, side="right")) - 1
        k = max(k, 0)
        return DepthFrame(self._ring[self._slots[k]], self._times[k])

    def select_slots(self, now: float, delays) -> torch.Tensor:
        """Per-env ring slot on the device (int32 (N,))."""
        if not self._slots:
            raise LookupError("frame buffer is empty")
        d = _delays_tensor(delays, self._ring.device)
        n = d.shape[0]
        if self._slot_buf is None or self._slot_buf.shape[0] != n:
            self._slot_buf = torch.empty(n, dtype=torch.int32, device=self._ring.device)
        times = np.ascontiguousarray(self._times, dtype=np.float64)
        order = np.ascontiguousarray(self._slots, dtype=np.int32)
        _native.check(_native.lib().mdrt_select_slots(
            _native.dptr(times), order.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(times),
            float(now), ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(self._slot_buf.data_ptr()), n,
            _stream(d)))
        return self._slot_buf

    def fetch_delayed_batch(self, now: float, delays):
        """Row e of the frame selected for delay[e]; (N, C, H, W) CUDA tensor."""
        d = _delays_tensor(delays, self._ring.device if self._ring is not None else None)
        if d.dim() != 1:
            raise ValueError("delays must be 1-D over environments")
        slot = self.select_slots(now, d)
        n = d.shape[0]
        if n > self._ring.shape[1]:
            raise ValueError("more delays than environments in the buffered frames")
        per_env = int(np.prod(self._ring.shape[2:]))
        out = torch.empty((n,) + tuple(self._ring.shape[2:]), dtype=torch.float32, device=self._ring.device)
        frames = (ctypes.c_void_p * self.capacity)(*[self._ring[i].data_ptr() for i in range(self.capacity)])
        _native.check(_native.lib().mdrt_gather_delayed(
            frames, self.capacity, ctypes.c_void_p(slot.data_ptr()), ctypes.c_void_p(out.data_ptr()), n,
            per_env, _stream(out)))
        return out


def _delays_tensor(delays, device) -> torch.Tensor:
    if isinstance(delays, torch.Tensor):
        d = delays.to(dtype=torch.float64)
        if device is not None:
            d = d.to(device)
        elif d.device.type != "cuda":
            d = d.to(_cuda_device(None))
        return d.contiguous()
    arr = np.asarray(delays, dtype=np.float64)
    if arr.ndim != 1:
        raise ValueError("delays must be 1-D over environments")
    if np.any(arr < 0):
        raise ValueError("delay must be >= 0")
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device if device is not None else _cuda_device(None))


def sample_latencies(config: SensorConfig, num_envs: int, *, episode: int = 0) -> np.ndarray:
    """Per-env delay ~ U[0, max_delay] from stream "latency" (sensor.py:153-158)."""
    key = rng.stream_key(config.seed, "latency")
    return rng.uniform(key, episode, np.arange(num_envs), low=0.0, high=config.max_delay)


@dataclass(frozen=True)
class CameraRandomization:
    translation: float = 0.025
    rot_roll_deg: float = 2.5
    rot_pitch_deg: float = 3.0
    rot_yaw_deg: float = 2.5
    fov_deg: float = 2.0
    seed: int = 0

    def __post_init__(self):
        for name in ("translation", "rot_roll_deg", "rot_pitch_deg", "rot_yaw_deg", "fov_deg"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0")


def sample_camera_offsets(config: CameraRandomization, num_envs: int, num_cameras: int, *,
                          episode: int = 0):
    """(offset_pos (N,C,3), offset_rot (N,C,4), fov_delta (N,C)) (sensor.py:183-211)."""
    key = rng.stream_key(config.seed, "camera")
    env = np.arange(num_envs).reshape(-1, 1)
    cam = np.arange(num_cameras).reshape(1, -1)
    t = config.translation
    pos = np.stack([rng.uniform(key, 0, a, episode, env, cam, low=-t, high=t) for a in range(3)], axis=-1)
    bounds = (config.rot_roll_deg, config.rot_pitch_deg, config.rot_yaw_deg)
    euler = np.stack([np.radians(rng.uniform(key, 1, a, episode, env, cam, low=-b, high=b))
                      for a, b in enumerate(bounds)], axis=-1)
    rot = np.empty((num_envs, num_cameras, 4))
    for e in range(num_envs):
        for c in range(num_cameras):
            rot[e, c] = quat_from_euler(*euler[e, c])
    fov = rng.uniform(key, 2, 0, episode, env, cam, low=-config.fov_deg, high=config.fov_deg)
    return pos, rot, fov


def randomize_scene_cameras(scene: Scene, config: CameraRandomization, *, episode: int = 0) -> None:
    scene.set_camera_randomization(*sample_camera_offsets(config, scene.num_envs, scene.num_cameras,
                                                          episode=episode))


def randomized_camera(camera: CameraModel, offset_pos, offset_rot, fov_delta: float) -> CameraModel:
    off = RigidPose(np.asarray(offset_pos, dtype=np.float64), np.asarray(offset_rot, dtype=np.float64))
    return camera.with_mount(camera.mount.compose(off)).with_fov_delta(fov_delta)
