"""Random side masking (RSM) of depth observations, on the GPU.

Mirror of the reference's RSM (/root/reference/pkg/src/multidepth/perception.py:
120-202): per (env, camera) a mode (none / small / large) is drawn from the
terrain-kind distribution; the side bands of ``int(f * W)`` columns are
overwritten with U[fill_low, fill_high) fills from the counter stream
"rsm-fill" keyed (step, env, cam, row, col). The fill arithmetic is the
reference's (f64, then cast to float32), so outputs are bit-identical.

``rsm_apply`` runs the standalone kernel; ``render_pipeline(..., rsm=cfg,
rsm_modes=modes)`` applies the same masking inside the fused traversal
kernel's epilogue.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native, rng
from .sensor import _back, _stream, _to_cuda

RSM_MODES = ("none", "small", "large")
DEFAULT_RSM_PROBS = {
    "flat": (0.2, 0.4, 0.4),
    "slope_pyramid": (0.2, 0.4, 0.4),
    "stairs_up": (0.2, 0.4, 0.4),
    "stairs_down": (0.2, 0.4, 0.4),
    "stepping_stones": (0.6, 0.3, 0.1),
}


@dataclass(frozen=True)
class RsmConfig:
    f_small: float = 0.125
    f_large: float = 0.25
    probs: dict = field(default_factory=lambda: dict(DEFAULT_RSM_PROBS))
    fill_low: float = 0.3
    fill_high: float | None = None   # None -> camera far limit
    seed: int = 0

    def __post_init__(self):
        if not (0.0 <= self.f_small <= 0.5 and 0.0 <= self.f_large <= 0.5):
            raise ValueError("mask fractions must be in [0, 0.5]")
        for kind, p in self.probs.items():
            arr = np.asarray(p, dtype=np.float64)
            if arr.shape != (3,) or np.any(arr < 0) or not np.isclose(arr.sum(), 1.0):
                raise ValueError(f"probs[{kind!r}] must be 3 nonnegative values summing to 1")

    def probs_for(self, kind: str):
        try:
            return self.probs[kind]
        except KeyError:
            raise KeyError(f"no side-mask probabilities for terrain kind {kind!r}") from None

    @property
    def fill_key(self) -> int:
        return int(rng.stream_key(self.seed, "rsm-fill"))


def rsm_sample_modes(config: RsmConfig, kind: str, num_envs: int, num_cameras: int, *,
                     episode: int = 0) -> np.ndarray:
    """Mask mode per (env, cam): 0 none, 1 small, 2 large (perception.py:150-157)."""
    probs = np.asarray(config.probs_for(kind), dtype=np.float64)
    key = rng.stream_key(config.seed, "rsm-mode")
    return rng.categorical(key, probs, episode, np.arange(num_envs).reshape(-1, 1),
                           np.arange(num_cameras).reshape(1, -1))


def rsm_mask_columns(config: RsmConfig, mode: int, width: int) -> int:
    """Columns masked on each side for a mode (perception.py:160-166)."""
    if mode == 0:
        return 0
    return int((config.f_small if mode == 1 else config.f_large) * width)


def _fill_high(config: RsmConfig, d_max, c: int) -> np.ndarray:
    return np.ascontiguousarray(np.broadcast_to(
        np.asarray(d_max if config.fill_high is None else config.fill_high, dtype=np.float64), (c,)))


def _modes_tensor(modes, n: int, c: int, device) -> torch.Tensor:
    t = torch.as_tensor(np.asarray(modes) if not isinstance(modes, torch.Tensor) else modes)
    if tuple(t.shape) != (n, c):
        raise ValueError(f"modes shape {tuple(t.shape)} does not match (N, C)=({n}, {c})")
    return t.to(device=device, dtype=torch.int32).contiguous()


def rsm_apply(depth, modes, config: RsmConfig, *, d_max, step: int = 0, env_offset: int = 0):
    """Overwrite side bands of (N, C, H, W) depth with random fill (perception.py:169-202).

    CUDA tensor in -> CUDA tensor out; numpy in -> numpy out (computed on the GPU).
    """
    if len(depth.shape) != 4:
        raise ValueError(f"expected (N, C, H, W) depth, got shape {tuple(depth.shape)}")
    t, kind = _to_cuda(depth)
    n, c, h, w = t.shape
    m = _modes_tensor(modes, n, c, t.device)
    k = np.array([0, rsm_mask_columns(config, 1, w), rsm_mask_columns(config, 2, w)], dtype=np.int32)
    high = _fill_high(config, d_max, c)
    out = torch.empty_like(t)
    _native.check(_native.lib().mdrt_rsm_apply(
        ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(out.data_ptr()), n, c, h, w, ctypes.c_void_p(m.data_ptr()),
        k.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), config.fill_key, int(step), int(env_offset),
        float(config.fill_low), _native.dptr(high), _stream(t)))
    return _back(out, kind)
