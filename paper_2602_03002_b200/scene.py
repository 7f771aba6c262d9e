"""Batched multi-environment scenes rendered on a B200.

Mirror of the reference ``multidepth.scene`` (/root/reference/pkg/src/multidepth/scene.py)
with the state moved to the GPU:

* geometry (body meshes in link frames + world terrain) is registered once;
  the native library builds one SAH BVH per mesh and uploads it
  (``mdrt_add_body``/``mdrt_set_terrain``/``mdrt_commit``) -- never rebuilt;
* per-env body poses and camera randomisation live in CUDA tensors;
* ``render`` launches the prologue (camera poses, intrinsics, link culling)
  and the traversal kernel on the current torch stream and returns a CUDA
  tensor ``[N, C, H, W]`` float32 of Euclidean range (misses read exactly
  ``float32(d_max)``).

There is no CPU path: constructing a Scene without a CUDA device raises.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .camera import CameraModel
from .mesh import TriMesh
from .transforms import RigidPose, quat_identity


@dataclass(frozen=True)
class Body:
    name: str
    mesh: TriMesh
    body_id: int = -1   # index in the native context (its BVH is built once)


@dataclass
class DepthFrame:
    """Range depth [env, camera, row, col] in metres (scene.py:33-46)."""

    data: object          # torch.Tensor (CUDA) or np.ndarray
    timestamp: float = 0.0

    def __post_init__(self):
        if len(self.data.shape) != 4:
            raise ValueError(f"depth data must be 4-D (N,C,H,W), got {tuple(self.data.shape)}")

    @property
    def shape(self) -> tuple[int, int, int, int]:
        return tuple(self.data.shape)


def _cuda_device(device) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("a CUDA device is required: the B200 renderer has no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    return torch.device("cuda", dev.index if dev.index is not None else torch.cuda.current_device())


def _as_device_f32(x, device, shape=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=torch.float32)
    else:
        t = torch.as_tensor(np.asarray(x, dtype=np.float64), dtype=torch.float32).to(device)
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"expected shape {tuple(shape)}, got {tuple(t.shape)}")
    return t.contiguous()


class Scene:
    """Shared immutable geometry + per-environment poses (scene.py:150-330).

    ``env_offset`` is the global index of environment 0 of this scene; it keys
    the sensor RNG so an env-sliced multi-GPU run reproduces the single-GPU
    stream bit-for-bit.
    """

    def __init__(self, num_envs: int, bodies=(), cameras=(), terrain: TriMesh | None = None, *,
                 device=None, env_offset: int = 0):
        if num_envs < 1:
            raise ValueError("num_envs must be >= 1")
        self.num_envs = int(num_envs)
        self.env_offset = int(env_offset)
        entries = []
        for i, entry in enumerate(bodies):
            if isinstance(entry, Body):
                name, mesh = entry.name, entry.mesh
            elif isinstance(entry, tuple):
                name, mesh = entry
            else:
                name, mesh = f"body{i}", entry
            if mesh.num_faces == 0:
                raise ValueError(f"body {name!r} has no triangles")
            entries.append((str(name), mesh))
        cams = tuple(cameras)
        if not cams:
            raise ValueError("scene needs at least one camera")
        h, w = cams[0].height, cams[0].width
        for cam in cams:
            if (cam.height, cam.width) != (h, w):
                raise ValueError("all cameras in a scene must share one resolution")
            if cam.parent_body is not None and not 0 <= cam.parent_body < len(entries):
                raise ValueError(f"camera {cam.name!r} parent_body {cam.parent_body} out of range")
        if len(cams) > 64:
            raise ValueError("at most 64 cameras per scene")
        if terrain is not None and terrain.num_faces == 0:
            raise ValueError("terrain mesh has no triangles")

        self.device = _cuda_device(device)
        self._ctx = _native.Context(self.device.index)
        body_list = []
        for name, mesh in entries:
            body_list.append(Body(name, mesh, self._ctx.add_body(mesh.vertices, mesh.faces)))
        self.bodies: tuple[Body, ...] = tuple(body_list)
        self.terrain = terrain
        if terrain is not None:
            self._ctx.set_terrain(terrain.vertices, terrain.faces)
        self.cameras: tuple[CameraModel, ...] = cams
        self.height, self.width = h, w
        self._ctx.set_cameras(
            w, h, [c.hfov_deg for c in cams], [c.vfov_deg for c in cams], [c.d_max for c in cams],
            [-1 if c.parent_body is None else c.parent_body for c in cams],
            np.stack([c.mount.translation for c in cams]), np.stack([c.mount.rotation for c in cams]))
        self._ctx.commit()
        self.geometry_stats = self._ctx.stats()

        n, b = self.num_envs, len(self.bodies)
        self.body_positions = torch.zeros((n, b, 3), dtype=torch.float32, device=self.device)
        self.body_rotations = torch.zeros((n, b, 4), dtype=torch.float32, device=self.device)
        self.body_rotations[..., 0] = 1.0
        self._rand_pos: torch.Tensor | None = None
        self._rand_rot: torch.Tensor | None = None
        self._rand_fov: torch.Tensor | None = None
        self._link_states = None
        # bumped whenever a device buffer the kernels read by pointer is replaced
        # (camera randomisation allocated/cleared, link states bound/unbound), so a
        # CapturedStep recorded against the old pointers refuses to replay
        self._ptr_version = 0
        self._state_owner = None       # the CapturedStep that owns the device step state
        self.debug_flags = 0           # extra MDRT_* flags for A/B runs (e.g. _native.NO_TILE_ENTRY)
        self.d_max_per_camera = np.array([c.d_max for c in cams], dtype=np.float64)

    # -- sizes -------------------------------------------------------------
    @property
    def num_bodies(self) -> int:
        return len(self.bodies)

    @property
    def num_cameras(self) -> int:
        return len(self.cameras)

    @property
    def frame_shape(self) -> tuple[int, int, int, int]:
        return (self.num_envs, self.num_cameras, self.height, self.width)

    # -- pose state (scene.py:227-253) --------------------------------------
    def set_body_pose(self, env: int, body: int, pose: RigidPose) -> None:
        if not 0 <= env < self.num_envs:
            raise ValueError(f"env {env} out of range [0, {self.num_envs})")
        if not 0 <= body < self.num_bodies:
            raise ValueError(f"body {body} out of range [0, {self.num_bodies})")
        self.body_positions[env, body] = torch.as_tensor(pose.translation, dtype=torch.float32)
        self.body_rotations[env, body] = torch.as_tensor(pose.rotation, dtype=torch.float32)

    def set_body_poses(self, positions, rotations, *, validate: bool = True) -> None:
        """positions (N,B,3), rotations (N,B,4) wxyz; numpy or torch (any device).

        Quaternions are normalised on the device (in f64) by the prologue
        kernel, so any nonzero norm is accepted as in the reference.
        Pinned host tensors are uploaded asynchronously on the scene's upload
        stream (overlapping kernels already queued), ordered before the next
        render on the current stream.
        ``validate=False`` skips the finite/zero-norm checks (for CUDA inputs
        they need a device->host read).
        """
        n, b = self.num_envs, self.num_bodies
        self.unbind_link_states()
        srcs = []
        for x, k in ((positions, 3), (rotations, 4)):
            if isinstance(x, torch.Tensor):
                t = x if x.dtype == torch.float32 else x.to(torch.float32)
            else:
                t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64), dtype=np.float32))
            if tuple(t.shape) != (n, b, k):
                raise ValueError(f"expected poses shaped {(n, b, 3)} / {(n, b, 4)}, "
                                 f"got {tuple(torch.as_tensor(positions).shape)} / "
                                 f"{tuple(torch.as_tensor(rotations).shape)}")
            srcs.append(t)
        pos, rot = srcs
        if validate and pos.numel():
            finite = torch.isfinite(pos).all() & torch.isfinite(rot).all()
            small = (rot.double().norm(dim=-1) < 1e-12).any()
            if not bool(finite.item()):
                raise ValueError("poses must be finite")
            if bool(small.item()):
                raise ValueError("zero quaternion in body rotations")
        if pos.device.type == "cpu" and pos.is_pinned() and rot.is_pinned() and pos.numel():
            self._upload_poses(pos, rot)
            return
        for dst, src in ((self.body_positions, pos), (self.body_rotations, rot)):
            dst.copy_(src, non_blocking=src.device.type == "cpu" and src.is_pinned())

    def _upload_poses(self, pos: torch.Tensor, rot: torch.Tensor) -> None:
        """Pinned host poses: H2D on the scene's upload stream into one of two
        staging buffers, so the PCIe transfer overlaps the previous step's
        kernels; the current stream then waits for it and copies staging ->
        body_positions/body_rotations device-to-device (fixed pointers, so
        captured graphs keep working). The caller must not modify ``pos``/``rot``
        until that copy ran (as for any non_blocking copy)."""
        if not hasattr(self, "_up_stream"):
            self._up_stream = torch.cuda.Stream(self.device)
            self._up_pos = [torch.empty_like(self.body_positions) for _ in range(2)]
            self._up_rot = [torch.empty_like(self.body_rotations) for _ in range(2)]
            self._up_free = [None, None]
            self._up_slot = 0
        j = self._up_slot = self._up_slot ^ 1
        cur = torch.cuda.current_stream(self.device)
        up = self._up_stream
        if self._up_free[j] is not None:
            up.wait_event(self._up_free[j])        # previous D2D copy out of slot j was enqueued
        with torch.cuda.stream(up):
            self._up_pos[j].copy_(pos, non_blocking=True)
            self._up_rot[j].copy_(rot, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(up)
        cur.wait_event(ready)
        self.body_positions.copy_(self._up_pos[j])
        self.body_rotations.copy_(self._up_rot[j])
        free = torch.cuda.Event()
        free.record(cur)
        self._up_free[j] = free

    def bind_link_states(self, states: torch.Tensor, link_map, *, pos_offset: int = 0, rot_offset: int = 3,
                         quat_order: str = "xyzw") -> None:
        """Read body poses straight from a simulator's link-state tensor (zero copy).

        ``states``: CUDA float32, shape (N, L, R) (or (N*L, R)), one R-float record
        per (env, simulator link), e.g. R = 13: position, quaternion, linear and
        angular velocity. ``link_map[b]`` is the simulator link index of body b.
        Every render (and every ``CapturedStep`` replay) reads the tensor's
        current contents in the prologue kernel, so there is no per-step pose
        copy; keep the tensor alive and write it in place. ``set_body_poses``
        unbinds it. Quaternions may be unnormalised (normalised on the device).
        """
        if quat_order not in ("xyzw", "wxyz"):
            raise ValueError("quat_order must be 'xyzw' or 'wxyz'")
        if not isinstance(states, torch.Tensor) or states.device != self.device or states.dtype != torch.float32:
            raise ValueError(f"states must be a float32 tensor on {self.device}")
        if not states.is_contiguous():
            raise ValueError("states must be contiguous")
        n = self.num_envs
        if states.dim() == 2:
            if states.shape[0] % n:
                raise ValueError(f"{states.shape[0]} records do not split into {n} envs")
            links, rec = states.shape[0] // n, states.shape[1]
        elif states.dim() == 3 and states.shape[0] == n:
            links, rec = states.shape[1], states.shape[2]
        else:
            raise ValueError(f"states must be (N, L, R) or (N*L, R) with N={n}, got {tuple(states.shape)}")
        lm = np.asarray(link_map, dtype=np.int64).reshape(-1)
        if lm.shape != (self.num_bodies,) or (lm.size and (lm.min() < 0 or lm.max() >= links)):
            raise ValueError(f"link_map must hold {self.num_bodies} link indices in [0, {links})")
        if not (0 <= pos_offset <= rec - 3 and 0 <= rot_offset <= rec - 4):
            raise ValueError(f"pos/rot offsets outside the {rec}-float record")
        lmap = torch.as_tensor(lm.astype(np.int32), device=self.device)
        self._link_states = (states, lmap, links, rec, int(pos_offset), int(rot_offset), quat_order == "xyzw")
        self._ptr_version += 1

    def unbind_link_states(self) -> None:
        if self._link_states is not None:
            self._link_states = None
            self._ptr_version += 1

    def _host_poses(self) -> tuple[np.ndarray, np.ndarray]:
        """(N,B,3), (N,B,4) wxyz f64 host copies of the pose source the prologue reads."""
        ls = getattr(self, "_link_states", None)
        if ls is None:
            return self.body_positions.double().cpu().numpy(), self.body_rotations.double().cpu().numpy()
        states, lmap, links, rec, po, ro, xyzw = ls
        r = states.reshape(self.num_envs, links, rec)[:, lmap.long()].double().cpu().numpy()
        q = r[..., ro:ro + 4]
        return r[..., po:po + 3], (q[..., [3, 0, 1, 2]] if xyzw else q)

    def body_pose(self, env: int, body: int) -> RigidPose:
        bp, bq = self._host_poses()
        return RigidPose(bp[env, body], bq[env, body])

    # -- camera randomisation (scene.py:256-277) -----------------------------
    def set_camera_randomization(self, offset_pos, offset_rot, fov_delta) -> None:
        n, c = self.num_envs, self.num_cameras
        p = _as_device_f32(offset_pos, self.device)
        r = _as_device_f32(offset_rot, self.device)
        f = _as_device_f32(fov_delta, self.device)
        if tuple(p.shape) != (n, c, 3) or tuple(r.shape) != (n, c, 4) or tuple(f.shape) != (n, c):
            raise ValueError("camera randomization arrays have wrong shapes")
        if self._rand_pos is not None:
            # re-randomisation (e.g. per episode) writes the scene's own buffers in
            # place, so captured graphs keep reading valid memory and see the new offsets
            self._rand_pos.copy_(p)
            self._rand_rot.copy_(r)
            self._rand_fov.copy_(f)
            return
        # fresh buffers owned by the scene (never the caller's tensors)
        self._rand_pos, self._rand_rot, self._rand_fov = p.clone(), r.clone(), f.clone()
        self._ptr_version += 1

    def clear_camera_randomization(self) -> None:
        if self._rand_pos is not None:
            self._rand_pos = self._rand_rot = self._rand_fov = None
            self._ptr_version += 1

    # -- host-side views of the derived state (API parity) --------------------
    def camera_world_poses(self) -> tuple[np.ndarray, np.ndarray]:
        """(N,C,3), (N,C,4): parent pose o mount o offset, as the prologue computes it."""
        from .transforms import quat_mul, quat_normalize, quat_rotate
        bp, bq = self._host_poses()
        rp = None if self._rand_pos is None else self._rand_pos.double().cpu().numpy()
        rq = None if self._rand_rot is None else self._rand_rot.double().cpu().numpy()
        n, c = self.num_envs, self.num_cameras
        pos, rot = np.empty((n, c, 3)), np.empty((n, c, 4))
        for ci, cam in enumerate(self.cameras):
            for e in range(n):
                t, q = cam.mount.translation, cam.mount.rotation
                if cam.parent_body is not None:
                    pq = quat_normalize(bq[e, cam.parent_body])
                    t, q = bp[e, cam.parent_body] + quat_rotate(pq, t), quat_mul(pq, q)
                if rp is not None:
                    t, q = t + quat_rotate(q, rp[e, ci]), quat_mul(q, quat_normalize(rq[e, ci]))
                pos[e, ci], rot[e, ci] = t, q
        return pos, rot

    def ray_grids(self) -> tuple[np.ndarray, np.ndarray]:
        """Host copy of the ray grids the device generates on the fly (scene.py:304-329)."""
        if self._rand_fov is None:
            g = [cam.ray_grid() for cam in self.cameras]
            return np.stack([d for d, _ in g])[None], np.stack([s for _, s in g])[None]
        fov = self._rand_fov.double().cpu().numpy()
        n, c, h, w = self.frame_shape
        dirs, scale = np.empty((n, c, h, w, 3)), np.empty((n, c, h, w))
        for ci, cam in enumerate(self.cameras):
            for e in range(n):
                dirs[e, ci], scale[e, ci] = cam.with_fov_delta(float(fov[e, ci])).ray_grid()
        return dirs, scale

    # -- native step ---------------------------------------------------------
    def _step_args(self, out: torch.Tensor, early_termination: bool) -> _native.StepArgs:
        a = _native.StepArgs()
        a.num_envs = self.num_envs
        a.flags = (_native.EARLY_TERMINATION if early_termination else 0) | self.debug_flags
        a.env_offset = self.env_offset
        a.body_pos = self.body_positions.data_ptr() if self.num_bodies else None
        a.body_rot = self.body_rotations.data_ptr() if self.num_bodies else None
        ls = getattr(self, "_link_states", None)
        if ls is not None and self.num_bodies:
            states, lmap, env_stride, rec, po, ro, xyzw = ls
            a.link_states = states.data_ptr()
            a.env_stride, a.record_stride, a.pos_offset, a.rot_offset = env_stride, rec, po, ro
            a.link_map = lmap.data_ptr()
            if xyzw:
                a.flags |= _native.ROT_XYZW
        if self._rand_pos is not None:
            a.cam_off_pos = self._rand_pos.data_ptr()
            a.cam_off_rot = self._rand_rot.data_ptr()
            a.fov_delta = self._rand_fov.data_ptr()
        a.ray_envs = 1
        a.out = out.data_ptr()
        if _native.is_remote(a.out):
            a.flags |= _native.WIDE_STORES
        return a

    def _launch(self, args: _native.StepArgs) -> None:
        # mdrt_render orders the context's shared scratch across streams itself
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self._ctx.render(args, stream)

    # -- asynchronous host delivery ------------------------------------------
    def _guard_out(self, out: torch.Tensor) -> None:
        """Make the current stream wait until a pending host copy of ``out`` finished."""
        ev = self._copy_events.get(out.data_ptr()) if hasattr(self, "_copy_events") else None
        if ev is not None:
            torch.cuda.current_stream(self.device).wait_event(ev)

    def _deliver(self, out: torch.Tensor, host_out: torch.Tensor) -> None:
        """Queue out -> host_out (pinned) on the scene's copy stream, ordered after the kernel."""
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = torch.cuda.Stream(self.device)
            self._copy_events = {}
        if host_out.device.type != "cpu" or tuple(host_out.shape) != tuple(out.shape) or \
                host_out.dtype != torch.float32 or not host_out.is_pinned():
            raise ValueError(f"host_out must be a pinned float32 CPU tensor of shape {tuple(out.shape)}")
        cur = torch.cuda.current_stream(self.device)
        done = torch.cuda.Event()
        done.record(cur)
        self._copy_stream.wait_event(done)
        with torch.cuda.stream(self._copy_stream):
            host_out.copy_(out, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self._copy_stream)
        out.record_stream(self._copy_stream)
        self._copy_events[out.data_ptr()] = ev
        self._last_copy = ev

    def host_sync(self) -> None:
        """Block until every queued host delivery has landed."""
        ev = getattr(self, "_last_copy", None)
        if ev is not None:
            ev.synchronize()

    def _new_frame(self, out):
        if out is None:
            return torch.empty(self.frame_shape, dtype=torch.float32, device=self.device)
        if (not isinstance(out, torch.Tensor) or out.device != self.device or out.dtype != torch.float32
                or tuple(out.shape) != self.frame_shape or not out.is_contiguous()):
            raise ValueError(f"out must be a contiguous float32 CUDA tensor of shape {self.frame_shape}")
        return out


def _check_backend(backend, threads):
    from . import kernels
    kernels.resolve_backend(backend)
    if threads is not None:
        kernels.resolve_threads(threads)


def render(scene: Scene, *, early_termination: bool = True, backend: str | None = None,
           threads: int | None = None, timestamp: float = 0.0, out=None,
           counters: torch.Tensor | None = None, host_out: torch.Tensor | None = None) -> DepthFrame:
    """One ray per (env, camera, pixel); returns range depth (scene.py:332-348).

    Bodies are queried in their link frames (never rebuilt), then terrain in
    the world frame bounded by the best body hit when early_termination is on.
    ``host_out`` (pinned CPU tensor): the frame is also copied to the host on a
    side stream, overlapping the next step's kernels (call ``scene.host_sync()``
    before reading it). ``counters`` (int64 CUDA tensor of 2) accumulates BVH node-record fetches
    and triangle tests (the algorithmic-bytes denominator); with 4 slots it
    also splits out link-tree node fetches and link traversals started.
    """
    _check_backend(backend, threads)
    data = scene._new_frame(out)
    scene._guard_out(data)
    args = scene._step_args(data, early_termination)
    if counters is not None:
        args.flags |= _native.COUNT
        if counters.numel() >= 4:
            args.flags |= _native.COUNT_DETAIL
        args.counters = counters.data_ptr()
    scene._launch(args)
    if host_out is not None:
        scene._deliver(data, host_out)
    return DepthFrame(data, timestamp)


class _FlatTris:
    """The FlatGeometry fields the CUDA seam reads (scene.py:49-78)."""

    def __init__(self, body_tris, terrain_tris):
        empty = np.zeros((0, 3))
        cat = (lambda k: np.concatenate([t[:, k] for t in body_tris])) if body_tris else (lambda k: empty)
        self.tri_v0, self.tri_v1, self.tri_v2 = cat(0), cat(1), cat(2)
        self.body_tri_offsets = np.cumsum([0] + [len(t) for t in body_tris])
        self.body_root = np.zeros(len(body_tris), np.int32)
        g = terrain_tris if terrain_tris is not None else np.zeros((0, 3, 3))
        self.g_tri_v0, self.g_tri_v1, self.g_tri_v2 = g[:, 0], g[:, 1], g[:, 2]


def render_naive_baseline(scene: Scene, *, early_termination: bool = True, backend: str | None = None,
                          threads: int | None = None, timestamp: float = 0.0) -> DepthFrame:
    """The reference's refit path (scene.py:351-378), kept as its comparison foil:
    per environment every link mesh is transformed to world coordinates and gets
    freshly built BVHs, queried with identity poses through the backend seam. The
    terrain (static in both paths) is traced once for all envs and the closest
    hit of the two kept. Output matches ``render`` to float32 precision; its cost
    (host BVH builds per env and link) does not."""
    _check_backend(backend, threads)
    from .kernels import cuda_backend
    n, c = scene.num_envs, scene.num_cameras
    cam_pos, cam_rot = scene.camera_world_poses()
    dirs, scale = scene.ray_grids()
    d_max = scene.d_max_per_camera
    out = torch.full(scene.frame_shape, 0.0, dtype=torch.float32, device=scene.device)
    shared = dirs.shape[0] == 1
    if scene.terrain is not None:
        flat_t = _FlatTris([], scene.terrain.triangles())
        cuda_backend.render_batch(flat_t, np.zeros((n, 0, 3)), np.zeros((n, 0, 4)), cam_pos, cam_rot, dirs, scale,
                                  d_max, early_termination, out)
    else:
        out[:] = torch.as_tensor(np.asarray(d_max, np.float32), device=scene.device).view(1, c, 1, 1)
    if scene.num_bodies:
        bp, bq = scene._host_poses()
        nb = scene.num_bodies
        id_pos, id_rot = np.zeros((1, nb, 3)), np.tile(quat_identity(), (1, nb, 1))
        part = torch.empty((1,) + scene.frame_shape[1:], dtype=torch.float32, device=scene.device)
        for e in range(n):
            world = [b.mesh.transformed(RigidPose(bp[e, k], bq[e, k])).triangles() for k, b in enumerate(scene.bodies)]
            er = 0 if shared else e
            cuda_backend.render_batch(_FlatTris(world, None), id_pos, id_rot, cam_pos[e:e + 1], cam_rot[e:e + 1],
                                      dirs[er:er + 1], scale[er:er + 1], d_max, early_termination, part)
            torch.minimum(out[e:e + 1], part, out=out[e:e + 1])
    return DepthFrame(out, timestamp)


def depth_to_z(frame, scale):
    """range / |K^-1 p| (scene.py:381-387); works on numpy or torch."""
    if isinstance(frame, torch.Tensor):
        return frame / torch.as_tensor(scale, dtype=frame.dtype, device=frame.device)
    return np.asarray(frame) / np.asarray(scale)
