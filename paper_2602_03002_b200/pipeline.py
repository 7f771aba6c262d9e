"""The fused per-step depth pipeline: render + sensor + latency in one kernel.

Semantically identical to the reference sequence

    frame = render(scene, timestamp=t)                                   # scene.py:332-348
    noisy = apply_noise_dropout(frame.data, cfg, d_max=..., step=step)   # sensor.py:55-82
    buf.push(DepthFrame(noisy, t))                                       # sensor.py:122-131
    obs = buf.fetch_delayed_batch(t, delays)                             # sensor.py:141-150

but executed as two launches (prologue + traversal) with the noise/dropout
epilogue and the latency-ring write/read fused into the traversal kernel's
tail, so each pixel's range is written to HBM once (ring) and the delayed
observation once (obs).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native
from .scene import Scene
from .perception import RsmConfig, _fill_high, _modes_tensor, rsm_mask_columns
from .sensor import FrameBuffer, SensorConfig, _delays_tensor


def _set_downsample(a, scene: Scene, ds_out: torch.Tensor, f: int) -> None:
    n, c, h, w = scene.frame_shape
    if f < 1 or h % f or w % f:
        raise ValueError(f"resolution {w}x{h} not divisible by downsample factor {f}")
    shape = (n, c, h // f, w // f)
    if (not isinstance(ds_out, torch.Tensor) or ds_out.device != scene.device or ds_out.dtype != torch.float32
            or tuple(ds_out.shape) != shape or not ds_out.is_contiguous()):
        raise ValueError(f"ds_out must be a contiguous float32 CUDA tensor of shape {shape}")
    a.ds_out = ds_out.data_ptr()
    a.ds_factor = int(f)


def _set_rsm(a, scene: Scene, rsm: RsmConfig, rsm_modes, keep: list) -> None:
    if rsm_modes is None:
        raise ValueError("rsm needs rsm_modes (N, C)")
    m = _modes_tensor(rsm_modes, scene.num_envs, scene.num_cameras, scene.device)
    high = _fill_high(rsm, scene.d_max_per_camera, scene.num_cameras)
    keep += [m, high]
    a.flags |= _native.RSM
    a.rsm_modes = m.data_ptr()
    a.rsm_k1 = rsm_mask_columns(rsm, 1, scene.width)
    a.rsm_k2 = rsm_mask_columns(rsm, 2, scene.width)
    a.rsm_key = rsm.fill_key
    a.rsm_fill_low = float(rsm.fill_low)
    a.rsm_fill_high = _native.dptr(high)


def render_pipeline(scene: Scene, *, sensor: SensorConfig | None = None, step: int = 0,
                    frame_buffer: FrameBuffer | None = None, timestamp: float | None = None,
                    delays=None, early_termination: bool = True, out: torch.Tensor | None = None,
                    clean_out: torch.Tensor | None = None,
                    counters: torch.Tensor | None = None,
                    host_out: torch.Tensor | None = None, rsm: RsmConfig | None = None,
                    rsm_modes=None, ds_out: torch.Tensor | None = None,
                    downsample_factor: int = 5, host_ds_out: torch.Tensor | None = None) -> torch.Tensor:
    """One simulation step of the multi-depth pipeline; returns the observation (N,C,H,W).

    * ``sensor``: apply noise/dropout/clamp with counters (step, global env, cam, row, col).
    * ``frame_buffer`` + ``timestamp`` + ``delays`` (N,): push the noisy frame
      and return, per env, the newest frame with ts <= timestamp - delay.
    * ``clean_out``: optionally also store the noise-free range image.
    * ``host_out``: pinned CPU tensor that receives the observation asynchronously
      (side copy stream, overlaps the next step; ``scene.host_sync()`` before use).
    * ``rsm`` + ``rsm_modes`` (N, C): random side masking of the observation
      (perception.py:169-202), i.e. ``rsm_apply(obs, rsm_modes, rsm, step=step)``.
    * ``ds_out`` (N, C, H/f, W/f): also write ``downsample_min(obs, f)``
      (sensor.py:85-100) from the same kernel, f = ``downsample_factor``;
      ``host_ds_out`` (pinned CPU, same shape) receives it like ``host_out``
      (the paper's policy reads the 48x27 block minimum, not the native frame).
    """
    data = scene._new_frame(out)
    scene._guard_out(data)
    a, keep = _pipeline_args(scene, data, sensor=sensor, step=step, frame_buffer=frame_buffer, timestamp=timestamp,
                             delays=delays, early_termination=early_termination, clean_out=clean_out,
                             counters=counters, rsm=rsm, rsm_modes=rsm_modes, ds_out=ds_out,
                             downsample_factor=downsample_factor, host_ds_out=host_ds_out)
    scene._launch(a)
    if host_out is not None:
        scene._deliver(data, host_out)
    if host_ds_out is not None:
        scene._deliver(ds_out, host_ds_out)
    return data


def _pipeline_args(scene: Scene, data: torch.Tensor, *, sensor, step, frame_buffer, timestamp, delays,
                   early_termination, clean_out, counters, rsm, rsm_modes, ds_out, downsample_factor,
                   host_ds_out):
    """StepArgs of one render_pipeline step (advances the FrameBuffer bookkeeping);
    returns (args, keep-alive list)."""
    a = scene._step_args(data, early_termination)
    if clean_out is not None:
        scene._new_frame(clean_out)
        a.out_clean = clean_out.data_ptr()
    keep = []
    a.step = int(step)
    if ds_out is not None:
        _set_downsample(a, scene, ds_out, downsample_factor)
        scene._guard_out(ds_out)
    elif host_ds_out is not None:
        raise ValueError("host_ds_out needs ds_out")
    if rsm is not None:
        _set_rsm(a, scene, rsm, rsm_modes, keep)
    if sensor is not None:
        a.flags |= _native.SENSOR
        a.noise_scale = float(sensor.noise_scale)
        a.dropout_p = float(sensor.dropout_p)
        a.sensor_key = sensor.key
        a.step = int(step)
        if sensor.dropout_fill is not None:
            fill = np.full(scene.num_cameras, float(sensor.dropout_fill), dtype=np.float64)
            keep.append(fill)
            a.fill = _native.dptr(fill)
    if frame_buffer is not None:
        if timestamp is None or delays is None:
            raise ValueError("frame_buffer needs timestamp and delays")
        d = _delays_tensor(delays, scene.device)
        if tuple(d.shape) != (scene.num_envs,):
            raise ValueError(f"delays must have shape ({scene.num_envs},)")
        frame_buffer._ensure(scene.frame_shape, scene.device)
        slot = frame_buffer._reserve(float(timestamp))
        times = np.ascontiguousarray(frame_buffer._times, dtype=np.float64)
        order = np.ascontiguousarray(frame_buffer._slots, dtype=np.int32)
        keep += [times, order, d]
        if frame_buffer._slot_buf is None or frame_buffer._slot_buf.shape[0] != scene.num_envs:
            frame_buffer._slot_buf = torch.empty(scene.num_envs, dtype=torch.int32, device=scene.device)
        a.flags |= _native.LATENCY
        a.ring = frame_buffer._ring.data_ptr()
        a.ring_slots = frame_buffer.capacity
        a.write_slot = slot
        a.ring_count = len(times)
        a.ring_times = _native.dptr(times)
        a.ring_order = order.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        a.now = float(timestamp)
        a.delays = d.data_ptr()
        a.read_slot = frame_buffer._slot_buf.data_ptr()
    if counters is not None:
        a.flags |= _native.COUNT
        a.counters = counters.data_ptr()
    return a, keep


class CapturedStep:
    """``render_pipeline`` captured once as a CUDA graph and replayed per step.

    The graph is advance -> prologue -> render (three kernels, no host
    arguments): the step counter, timestamp ``t0 + k*dt``, sensor-stream
    prefix and latency-ring push live in device memory and are advanced by the
    first kernel (MDRT_DEVICE_STATE), so a replay needs no host work beyond
    ``cudaGraphLaunch``. Poses are read from ``scene.body_positions`` /
    ``scene.body_rotations`` (write them in place, e.g. from the simulator).
    Replays produce exactly the observations of the eager sequence
    ``render_pipeline(step=k, timestamp=t0 + k*dt)`` for k = first_step, ...
    (tests/test_gpu_parity.py::test_captured_step_matches_eager). The paper's
    renderer is likewise captured in a graph.
    """

    # Lifetime and ownership: the graph holds raw device pointers, so the step keeps
    # every tensor it recorded alive (out, ds_out, delays, RSM modes, camera
    # randomisation, bound link states) and refuses to replay once the scene
    # replaced one of them (scene._ptr_version; re-randomising cameras writes in
    # place and is fine). The context has one device step state: a newer
    # CapturedStep on the same scene takes it over and the older one refuses to
    # replay; close() releases it. Replays are ordered against other renders of
    # the scene on any stream (mdrt_order_begin/end).

    def __init__(self, scene: Scene, *, sensor: SensorConfig | None = None,
                 frame_buffer: FrameBuffer | None = None, delays=None, dt: float = 0.02, t0: float = 0.0,
                 first_step: int = 0, out: torch.Tensor | None = None, early_termination: bool = True,
                 rsm: RsmConfig | None = None, rsm_modes=None, ds_out: torch.Tensor | None = None,
                 downsample_factor: int = 5):
        if frame_buffer is not None and (delays is None or not dt > 0):
            raise ValueError("frame_buffer needs delays and dt > 0")
        self.scene = scene
        self.frame_buffer = frame_buffer
        self.dt, self.t0 = float(dt), float(t0)
        self.next_step = int(first_step)
        self.out = scene._new_frame(out)
        a = scene._step_args(self.out, early_termination)
        a.flags |= _native.DEVICE_STATE
        # every tensor whose pointer the graph records (see the class comment)
        self._keep = [self.out, scene.body_positions, scene.body_rotations, scene._rand_pos, scene._rand_rot,
                      scene._rand_fov, scene._link_states]
        key = 0
        if rsm is not None:
            _set_rsm(a, scene, rsm, rsm_modes, self._keep)
        if ds_out is not None:
            _set_downsample(a, scene, ds_out, downsample_factor)
            self._keep.append(ds_out)
            self.ds_out = ds_out
        if sensor is not None:
            a.flags |= _native.SENSOR
            a.noise_scale = float(sensor.noise_scale)
            a.dropout_p = float(sensor.dropout_p)
            key = sensor.key
            if sensor.dropout_fill is not None:
                fill = np.full(scene.num_cameras, float(sensor.dropout_fill), dtype=np.float64)
                self._keep.append(fill)
                a.fill = _native.dptr(fill)
        times, order, slots = np.zeros(0), np.zeros(0, np.int32), 0
        if frame_buffer is not None:
            d = _delays_tensor(delays, scene.device)
            if tuple(d.shape) != (scene.num_envs,):
                raise ValueError(f"delays must have shape ({scene.num_envs},)")
            frame_buffer._ensure(scene.frame_shape, scene.device)
            if frame_buffer._slot_buf is None or frame_buffer._slot_buf.shape[0] != scene.num_envs:
                frame_buffer._slot_buf = torch.empty(scene.num_envs, dtype=torch.int32, device=scene.device)
            times = np.asarray(frame_buffer._times, dtype=np.float64)
            order = np.asarray(frame_buffer._slots, dtype=np.int32)
            slots = frame_buffer.capacity
            self._keep += [d, frame_buffer._ring, frame_buffer._slot_buf]
            a.flags |= _native.LATENCY
            a.ring = frame_buffer._ring.data_ptr()
            a.ring_slots = frame_buffer.capacity
            a.delays = d.data_ptr()
            a.read_slot = frame_buffer._slot_buf.data_ptr()
        scene._ctx.state_set(scene.num_envs, key, self.t0, self.dt, self.next_step, slots, times, order,
                             rsm_key=rsm.fill_key if rsm is not None else 0)
        scene._state_owner = self          # a previous CapturedStep of this scene stops replaying
        self._version = scene._ptr_version
        self._args = a
        # warm the launch path (occupancy query) outside capture, then capture
        plain = scene._step_args(self.out, early_termination)
        side = torch.cuda.Stream(scene.device)
        side.wait_stream(torch.cuda.current_stream(scene.device))
        with torch.cuda.stream(side):
            scene._launch(plain)
        torch.cuda.current_stream(scene.device).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            scene._launch(a)

    def replay(self) -> torch.Tensor:
        """Run step ``next_step`` on the current stream; returns the observation tensor."""
        sc = self.scene
        if sc._state_owner is not self:
            raise RuntimeError("this CapturedStep no longer owns the scene's device step state "
                               "(a newer CapturedStep took it over, or close() was called)")
        if sc._ptr_version != self._version:
            raise RuntimeError("the scene's pose / camera-randomisation buffers were replaced after capture "
                               "(bind_link_states, set_body_poses after a bind, or camera randomisation "
                               "set / cleared): capture a new CapturedStep")
        stream = torch.cuda.current_stream(sc.device).cuda_stream
        sc._ctx.order_begin(stream)
        self.graph.replay()
        sc._ctx.order_end(stream)
        if self.frame_buffer is not None:   # host shadow of the device ring bookkeeping
            self.frame_buffer._reserve(self.t0 + float(self.next_step) * self.dt)
        self.next_step += 1
        return self.out

    def device_state(self) -> dict:
        return self.scene._ctx.state_get()

    def close(self) -> None:
        """Release the scene's device step state and the recorded buffers."""
        if self.scene._state_owner is self:
            self.scene._state_owner = None
        self.graph = None
        self._keep = []
