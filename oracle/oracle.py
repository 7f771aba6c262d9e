"""CPU oracle for the depth path -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu-baseline /
``--impl reference`` leg may import this module. The product package
(``paper_2602_03002_b200``) never imports it and has no CPU fallback.

The arithmetic lives in ``oracle.c`` (plain C, f64, no FMA contraction); this
module is the numpy glue that restates the reference's host-side steps
(paths relative to /root/reference/pkg/src/multidepth):

* ``filter_degenerate``   mesh.py:47-56     (drop faces with area < 1e-12)
* ``build_bvh``           bvh.py:68-136     (C: orc_build_bvh)
* ``flatten``             scene.py:89-147   (flatten_geometry)
* ``quat_*``/``compose``  transforms.py:32-58,151-156
* ``camera_world_poses``  scene.py:279-295
* ``ray_grid``            camera.py:51-90   (+ with_fov_delta camera.py:92-95)
* ``render``              scene.py:332-348 -> numba_backend.py:155-219 (C: orc_render)
* ``apply_noise_dropout`` sensor.py:55-82   (C: orc_noise_dropout)
* ``stream_key/uniform/normal`` rng.py:30-99
* ``sample_latencies``    sensor.py:153-158
* ``frame_select``        sensor.py:133-150 (C: orc_frame_select)
* ``downsample_min``      sensor.py:85-100  (C: orc_downsample_min)
* ``rsm_*``               perception.py:150-202 (C: orc_rsm_apply; modes via categorical)
* ``depth_to_u8``/``mdpt_bytes`` frameio.py:21-38, 81-86 (numpy)

Pinned against the live reference by tests/golden/make_golden.py.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
_lock = threading.Lock()

DEGENERATE_AREA = 1e-12
LEAF_SIZE = 4
DEPTH_FLOOR = 1e-6

_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64


def build_lib(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "oracle.c")):
        subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build_lib()
            L = ctypes.CDLL(_LIB_PATH)
            L.orc_build_bvh.restype = _i64
            L.orc_build_bvh.argtypes = [_dp, _i64, ctypes.c_int, _dp, _dp, _i32p, _i32p, _i32p,
                                        _i32p, _i64p]
            L.orc_render.restype = None
            L.orc_render.argtypes = ([_i64] * 6 + [_dp, _dp, _dp, _dp, _dp, _dp, _i32p, _dp, _dp]
                                     + [_i32p] * 4 + [_dp] * 3 + [_i64, _dp, _dp] + [_i32p] * 4
                                     + [_dp] * 3 + [_dp, ctypes.c_int, _fp, ctypes.c_int, _i64p])
            L.orc_set_bary_eps.restype = None
            L.orc_set_bary_eps.argtypes = [ctypes.c_double]
            L.orc_mix64.restype = _u64
            L.orc_mix64.argtypes = [_u64]
            L.orc_absorb.restype = _u64
            L.orc_absorb.argtypes = [_u64, _u64]
            L.orc_stream_key.restype = _u64
            L.orc_stream_key.argtypes = [_i64, ctypes.c_char_p, _i64]
            L.orc_uniform.restype = None
            L.orc_uniform.argtypes = [_u64, _i64p, _i64, _i64, ctypes.c_double, ctypes.c_double, _dp]
            L.orc_normal.restype = None
            L.orc_normal.argtypes = [_u64, _i64p, _i64, _i64, _dp]
            L.orc_noise_dropout.restype = None
            L.orc_noise_dropout.argtypes = [_fp, _i64, _i64, _i64, _i64, _i64, _dp, _dp,
                                            ctypes.c_double, ctypes.c_double, _u64, _i64, _fp,
                                            ctypes.c_int]
            L.orc_frame_select.restype = None
            L.orc_frame_select.argtypes = [_dp, _i64, ctypes.c_double, _dp, _i64, _i64p]
            L.orc_downsample_min.restype = None
            L.orc_downsample_min.argtypes = [_fp, _i64, _i64, _i64, _i64, _fp]
            L.orc_max_threads.restype = ctypes.c_int
            L.orc_rsm_apply.restype = None
            L.orc_rsm_apply.argtypes = [_fp, _i64, _i64, _i64, _i64, _i32p, _i64p, _u64, _i64, _i64,
                                        ctypes.c_double, _dp, _fp]
            _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ct)


def max_threads() -> int:
    """All host cores this process may run on (launchers such as torchrun set
    OMP_NUM_THREADS=1, which would make the CPU baseline single-threaded)."""
    try:
        import os
        return max(len(os.sched_getaffinity(0)), 1)
    except (AttributeError, OSError):
        return int(lib().orc_max_threads())


# ---------------------------------------------------------------------------
# meshes / BVH (mesh.py:47-56, bvh.py:68-136, scene.py:89-147)
# ---------------------------------------------------------------------------

def filter_degenerate(vertices, faces):
    v = np.ascontiguousarray(vertices, dtype=np.float64)
    f = np.ascontiguousarray(faces, dtype=np.int64)
    if f.size == 0:
        return v, f
    tri = v[f]
    areas = 0.5 * np.linalg.norm(np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]), axis=1)
    keep = areas >= DEGENERATE_AREA
    return v, np.ascontiguousarray(f[keep])


def build_bvh(tris: np.ndarray, leaf_size: int = LEAF_SIZE) -> dict:
    tris = np.ascontiguousarray(tris, dtype=np.float64).reshape(-1, 3, 3)
    F = tris.shape[0]
    if F == 0:
        raise ValueError("cannot build a BVH over an empty mesh")
    mcap = 2 * F
    node_min = np.empty((mcap, 3))
    node_max = np.empty((mcap, 3))
    left = np.empty(mcap, np.int32)
    right = np.empty(mcap, np.int32)
    start = np.empty(mcap, np.int32)
    count = np.empty(mcap, np.int32)
    tri_index = np.empty(F, np.int64)
    M = lib().orc_build_bvh(_p(tris, _dp), F, leaf_size, _p(node_min, _dp), _p(node_max, _dp),
                            _p(left, _i32p), _p(right, _i32p), _p(start, _i32p),
                            _p(count, _i32p), _p(tri_index, _i64p))
    v = tris[tri_index]
    return dict(node_min=node_min[:M].copy(), node_max=node_max[:M].copy(),
                left=left[:M].copy(), right=right[:M].copy(), start=start[:M].copy(),
                count=count[:M].copy(), tri_v0=np.ascontiguousarray(v[:, 0]),
                tri_v1=np.ascontiguousarray(v[:, 1]), tri_v2=np.ascontiguousarray(v[:, 2]),
                tri_index=tri_index)


def flatten(body_bvhs: list, terrain_bvh: dict | None) -> dict:
    out = {}
    if body_bvhs:
        roots, nmin, nmax, lf, rt, st, ct, v0, v1, v2 = ([] for _ in range(10))
        node_off = tri_off = 0
        for b in body_bvhs:
            roots.append(node_off)
            nmin.append(b["node_min"]); nmax.append(b["node_max"])
            l = b["left"].copy(); r = b["right"].copy()
            l[l >= 0] += node_off; r[r >= 0] += node_off
            lf.append(l); rt.append(r)
            st.append(b["start"] + np.int32(tri_off)); ct.append(b["count"])
            v0.append(b["tri_v0"]); v1.append(b["tri_v1"]); v2.append(b["tri_v2"])
            node_off += len(b["node_min"]); tri_off += len(b["tri_v0"])
        out.update(body_root=np.asarray(roots, np.int32), node_min=np.vstack(nmin),
                   node_max=np.vstack(nmax), left=np.concatenate(lf), right=np.concatenate(rt),
                   start=np.concatenate(st), count=np.concatenate(ct), tri_v0=np.vstack(v0),
                   tri_v1=np.vstack(v1), tri_v2=np.vstack(v2))
    else:
        out.update(body_root=np.zeros(0, np.int32), node_min=np.zeros((0, 3)),
                   node_max=np.zeros((0, 3)), left=np.zeros(0, np.int32),
                   right=np.zeros(0, np.int32), start=np.zeros(0, np.int32),
                   count=np.zeros(0, np.int32), tri_v0=np.zeros((0, 3)),
                   tri_v1=np.zeros((0, 3)), tri_v2=np.zeros((0, 3)))
    keys = ("node_min", "node_max", "left", "right", "start", "count", "tri_v0", "tri_v1", "tri_v2")
    if terrain_bvh is not None:
        for k in keys:
            out["g_" + k] = terrain_bvh[k]
    else:
        for k in keys:
            out["g_" + k] = np.zeros((0, 3)) if k in ("node_min", "node_max") or k.startswith("tri") \
                else np.zeros(0, np.int32)
    return {k: np.ascontiguousarray(v) for k, v in out.items()}


# ---------------------------------------------------------------------------
# pose / camera math (transforms.py, camera.py, scene.py:279-329)
# ---------------------------------------------------------------------------

def quat_normalize(q):
    q = np.asarray(q, dtype=np.float64)
    return q / float(np.linalg.norm(q))


def quat_mul(a, b):
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return quat_normalize(np.array([aw * bw - ax * bx - ay * by - az * bz,
                                    aw * bx + ax * bw + ay * bz - az * by,
                                    aw * by - ax * bz + ay * bw + az * bx,
                                    aw * bz + ax * by - ay * bx + az * bw]))


def quat_rotate(q, v):
    qv = np.asarray(q, dtype=np.float64)[1:]
    t = 2.0 * np.cross(qv, v)
    return np.asarray(v, dtype=np.float64) + float(q[0]) * t + np.cross(qv, t)


def compose(ta, qa, tb, qb):
    # RigidPose.compose then RigidPose.__post_init__ renormalizes once more
    return ta + quat_rotate(qa, tb), quat_normalize(quat_mul(qa, qb))


def camera_world_poses(cameras, body_pos, body_rot, rand_pos=None, rand_rot=None):
    """cameras: list of dicts with mount_pos, mount_rot, parent (int|None)."""
    n = body_pos.shape[0]
    c = len(cameras)
    pos = np.empty((n, c, 3))
    rot = np.empty((n, c, 4))
    for ci, cam in enumerate(cameras):
        # mount_rot is a RigidPose rotation (already unit); used as-is
        mt = np.asarray(cam["mount_pos"], np.float64)
        mq = np.asarray(cam["mount_rot"], np.float64)
        for e in range(n):
            if cam.get("parent") is None:
                t, q = mt, mq
            else:
                b = cam["parent"]
                t, q = compose(body_pos[e, b], quat_normalize(body_rot[e, b]), mt, mq)
            if rand_pos is not None:
                t, q = compose(t, q, rand_pos[e, ci], quat_normalize(rand_rot[e, ci]))
            pos[e, ci] = t
            rot[e, ci] = q
    return pos, rot


def intrinsics(width, height, hfov_deg, vfov_deg):
    fx = (width / 2.0) / math.tan(math.radians(hfov_deg) / 2.0)
    fy = (height / 2.0) / math.tan(math.radians(vfov_deg) / 2.0)
    return fx, fy, width / 2.0, height / 2.0


def ray_grid(width, height, hfov_deg, vfov_deg):
    fx, fy, cx, cy = intrinsics(width, height, hfov_deg, vfov_deg)
    u = (np.arange(width) + 0.5 - cx) / fx
    v = (np.arange(height) + 0.5 - cy) / fy
    dirs = np.empty((height, width, 3))
    dirs[:, :, 0] = u[None, :]
    dirs[:, :, 1] = v[:, None]
    dirs[:, :, 2] = 1.0
    scale = np.sqrt(dirs[:, :, 0] ** 2 + dirs[:, :, 1] ** 2 + 1.0)
    return dirs, scale


def ray_grids(cameras, n_envs, fov_delta=None):
    h, w = cameras[0]["height"], cameras[0]["width"]
    c = len(cameras)
    if fov_delta is None:
        grids = [ray_grid(w, h, cam["hfov_deg"], cam["vfov_deg"]) for cam in cameras]
        return (np.ascontiguousarray(np.stack([g[0] for g in grids])[None]),
                np.ascontiguousarray(np.stack([g[1] for g in grids])[None]))
    dirs = np.empty((n_envs, c, h, w, 3))
    scale = np.empty((n_envs, c, h, w))
    for ci, cam in enumerate(cameras):
        for e in range(n_envs):
            d = float(fov_delta[e, ci])
            dirs[e, ci], scale[e, ci] = ray_grid(w, h, cam["hfov_deg"] + d, cam["vfov_deg"] + d)
    return dirs, scale


# ---------------------------------------------------------------------------
# render (scene.py:332-348 -> numba_backend.py:155-219)
# ---------------------------------------------------------------------------

class OracleScene:
    """Geometry prepared once (like Scene.__init__ + flat_geometry)."""

    def __init__(self, bodies, terrain, cameras):
        """bodies: list of (verts, faces); terrain: (verts, faces) or None;
        cameras: list of dicts (width, height, hfov_deg, vfov_deg, d_max,
        mount_pos, mount_rot, parent)."""
        bvhs = []
        for verts, faces in bodies:
            v, f = filter_degenerate(verts, faces)
            bvhs.append(build_bvh(v[f]))
        tb = None
        if terrain is not None:
            v, f = filter_degenerate(*terrain)
            tb = build_bvh(v[f])
        self.flat = flatten(bvhs, tb)
        self.cameras = list(cameras)
        self.num_bodies = len(bodies)

    def render(self, body_pos, body_rot, *, rand_pos=None, rand_rot=None, fov_delta=None,
               early_termination=True, threads=0, counters=None, cam_pose=None, grids=None):
        body_pos = np.ascontiguousarray(body_pos, np.float64)
        body_rot = np.asarray(body_rot, np.float64)
        n = body_pos.shape[0]
        if self.num_bodies:
            body_rot = body_rot / np.linalg.norm(body_rot, axis=-1, keepdims=True)
        body_rot = np.ascontiguousarray(body_rot)
        if rand_rot is not None:  # Scene.set_camera_randomization (scene.py:269-271)
            rand_rot = np.asarray(rand_rot, np.float64)
            rand_rot = rand_rot / np.linalg.norm(rand_rot, axis=-1, keepdims=True)
        if cam_pose is None:
            cam_pos, cam_rot = camera_world_poses(self.cameras, body_pos, body_rot, rand_pos,
                                                  rand_rot)
        else:
            cam_pos, cam_rot = cam_pose
        if grids is None:
            dirs, scale = ray_grids(self.cameras, n, fov_delta)
        else:
            dirs, scale = grids
        return render_flat(self.flat, body_pos, body_rot, cam_pos, cam_rot, dirs, scale,
                           np.array([c["d_max"] for c in self.cameras], np.float64),
                           early_termination, threads=threads, counters=counters)


def set_bary_eps(eps: float) -> None:
    """Barycentric margin of the oracle's triangle test (0 = the reference's exact
    test). Only for classifying GPU/oracle hit-miss flips."""
    lib().orc_set_bary_eps(float(eps))


def render_flat(flat, body_pos, body_rot, cam_pos, cam_rot, ray_dirs, ray_scale, d_max,
                early_termination=True, threads=0, counters=None):
    """Exactly the backend seam render_batch (numba_backend.py:222-234)."""
    f = flat
    cam_pos = np.ascontiguousarray(cam_pos, np.float64)
    cam_rot = np.ascontiguousarray(cam_rot, np.float64)
    ray_dirs = np.ascontiguousarray(ray_dirs, np.float64)
    ray_scale = np.ascontiguousarray(ray_scale, np.float64)
    body_pos = np.ascontiguousarray(body_pos, np.float64)
    body_rot = np.ascontiguousarray(body_rot, np.float64)
    d_max = np.ascontiguousarray(d_max, np.float64)
    n, c = cam_pos.shape[:2]
    rn, _, h, w = ray_scale.shape
    b = len(f["body_root"])
    out = np.empty((n, c, h, w), np.float32)
    ctr = np.zeros(2, np.int64)
    L = lib()
    L.orc_render(n, c, h, w, b, rn, _p(cam_pos, _dp), _p(cam_rot, _dp), _p(ray_dirs, _dp),
                 _p(ray_scale, _dp), _p(body_pos, _dp), _p(body_rot, _dp),
                 _p(f["body_root"], _i32p), _p(f["node_min"], _dp), _p(f["node_max"], _dp),
                 _p(f["left"], _i32p), _p(f["right"], _i32p), _p(f["start"], _i32p),
                 _p(f["count"], _i32p), _p(f["tri_v0"], _dp), _p(f["tri_v1"], _dp),
                 _p(f["tri_v2"], _dp), len(f["g_node_min"]), _p(f["g_node_min"], _dp),
                 _p(f["g_node_max"], _dp), _p(f["g_left"], _i32p), _p(f["g_right"], _i32p),
                 _p(f["g_start"], _i32p), _p(f["g_count"], _i32p), _p(f["g_tri_v0"], _dp),
                 _p(f["g_tri_v1"], _dp), _p(f["g_tri_v2"], _dp), _p(d_max, _dp),
                 int(bool(early_termination)), _p(out, _fp), int(threads),
                 _p(ctr, _i64p) if counters is not None else None)
    if counters is not None:
        counters[:] = ctr
    return out


# ---------------------------------------------------------------------------
# RNG + sensor (rng.py, sensor.py)
# ---------------------------------------------------------------------------

def stream_key(seed: int, name: str) -> int:
    data = name.encode("utf-8")
    return int(lib().orc_stream_key(int(seed), data, len(data)))


def _counters(*counters):
    arrs = np.broadcast_arrays(*[np.asarray(c, dtype=np.int64) for c in counters])
    shape = arrs[0].shape
    mat = np.ascontiguousarray(np.stack([a.ravel() for a in arrs], axis=1))
    return shape, mat


def uniform(key, *counters, low=0.0, high=1.0):
    shape, mat = _counters(*counters)
    out = np.empty(mat.shape[0])
    lib().orc_uniform(int(key), _p(mat, _i64p), mat.shape[0], mat.shape[1], low, high,
                      _p(out, _dp))
    return out.reshape(shape)


def normal(key, *counters):
    shape, mat = _counters(*counters)
    out = np.empty(mat.shape[0])
    lib().orc_normal(int(key), _p(mat, _i64p), mat.shape[0], mat.shape[1], _p(out, _dp))
    return out.reshape(shape)


def apply_noise_dropout(depth, *, noise_scale, dropout_p, seed, d_max, step=0,
                        dropout_fill=None, env_offset=0, threads=0):
    depth = np.ascontiguousarray(depth, np.float32)
    n, c, h, w = depth.shape
    dm = np.ascontiguousarray(np.broadcast_to(np.asarray(d_max, np.float64), (c,)))
    fill = dm if dropout_fill is None else np.full(c, float(dropout_fill))
    fill = np.ascontiguousarray(fill, np.float64)
    out = np.empty_like(depth)
    lib().orc_noise_dropout(_p(depth, _fp), n, c, h, w, int(env_offset), _p(dm, _dp),
                            _p(fill, _dp), float(noise_scale), float(dropout_p),
                            stream_key(seed, "sensor"), int(step), _p(out, _fp), int(threads))
    return out


def sample_latencies(max_delay: float, seed: int, num_envs: int, episode: int = 0):
    return uniform(stream_key(seed, "latency"), episode, np.arange(num_envs), low=0.0,
                   high=max_delay)


def frame_select(times, now, delays):
    times = np.ascontiguousarray(times, np.float64)
    delays = np.ascontiguousarray(delays, np.float64)
    idx = np.empty(len(delays), np.int64)
    lib().orc_frame_select(_p(times, _dp), len(times), float(now), _p(delays, _dp), len(delays),
                           _p(idx, _i64p))
    return idx


def downsample_min(depth, factor):
    depth = np.ascontiguousarray(depth, np.float32)
    h, w = depth.shape[-2:]
    if h % factor or w % factor:
        raise ValueError("not divisible")
    planes = int(np.prod(depth.shape[:-2]))
    out = np.empty(depth.shape[:-2] + (h // factor, w // factor), np.float32)
    lib().orc_downsample_min(_p(depth, _fp), planes, h, w, factor, _p(out, _fp))
    return out


def depth_to_u8(depth, d_max):
    """frameio.py:81-86: f64 ratio, clip to [0, 1], round-half-even of 255 * (1 - frac)."""
    frac = np.clip(np.asarray(depth, np.float64) / float(d_max), 0.0, 1.0)
    return np.rint(255.0 * (1.0 - frac)).astype(np.uint8)


def mdpt_bytes(depth):
    """frameio.py:21-38: '<4sHIIII' header (MDPT, 1, N, C, H, W) + little-endian float32 payload."""
    import struct
    a = np.ascontiguousarray(depth, np.float32)
    return struct.pack("<4sHIIII", b"MDPT", 1, *a.shape) + a.astype("<f4").tobytes()


def categorical(key, probs, *counters):
    """rng.py:102-116."""
    probs = np.asarray(probs, dtype=np.float64)
    edges = np.cumsum(probs)
    u = np.asarray(uniform(key, *counters)) * edges[-1]
    return np.minimum(np.searchsorted(edges, u, side="right"), len(probs) - 1).astype(np.int64)


def rsm_sample_modes(probs, seed, num_envs, num_cameras, episode=0):
    """perception.py:150-157."""
    return categorical(stream_key(seed, "rsm-mode"), probs, episode, np.arange(num_envs).reshape(-1, 1),
                       np.arange(num_cameras).reshape(1, -1))


def rsm_apply(depth, modes, *, f_small, f_large, fill_low, fill_high, seed, d_max, step=0, env_offset=0):
    """perception.py:169-202 (k = int(f * W) per side, fill uniform [fill_low, fill_high or d_max])."""
    depth = np.ascontiguousarray(depth, np.float32)
    n, c, h, w = depth.shape
    modes = np.ascontiguousarray(modes, np.int32)
    high = np.ascontiguousarray(np.broadcast_to(np.asarray(d_max if fill_high is None else fill_high,
                                                           np.float64), (c,)))
    ks = np.array([0, int(f_small * w), int(f_large * w)], np.int64)
    out = np.empty_like(depth)
    lib().orc_rsm_apply(_p(depth, _fp), n, c, h, w, _p(modes, _i32p), _p(ks, _i64p), stream_key(seed, "rsm-fill"),
                        int(step), int(env_offset), float(fill_low), _p(high, _dp), _p(out, _fp))
    return out
