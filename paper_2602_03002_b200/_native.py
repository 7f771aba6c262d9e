"""ctypes binding of libmdrt.so (C ABI in include/mdrt.h).

There is no fallback: if the library is missing or no CUDA device is visible
every entry point raises. The library is loaded from this package directory
(built in-tree by ``paper_2602_03002_b200.build``).
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# MDRT_LIB: load an alternative in-tree build (kernel-variant experiments only)
LIB_PATH = os.environ.get("MDRT_LIB") or os.path.join(_HERE, "libmdrt.so")

MDRT_OK = 0
MDRT_EINVAL = -1
MDRT_ECUDA = -2
MDRT_ESTATE = -3

ABI_VERSION = 2            # include/mdrt.h MDRT_ABI_VERSION (StepArgs layout below)
EARLY_TERMINATION = 0x1
SENSOR = 0x2
LATENCY = 0x4
COUNT = 0x8
NO_CULL = 0x10
PHASE_PROLOGUE = 0x20
PHASE_TRACE = 0x40
COUNT_DETAIL = 0x80
DEVICE_STATE = 0x100
RSM = 0x200
ROT_XYZW = 0x400
WIDE_STORES = 0x800
NO_TILE_ENTRY = 0x1000
TILE_ENTRY = 0x2000

_c_dp = ctypes.POINTER(ctypes.c_double)
_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_i32p = ctypes.POINTER(ctypes.c_int32)


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "num_bodies", "body_triangles", "body_nodes", "terrain_triangles", "terrain_nodes",
        "terrain_depth", "body_max_depth", "node_bytes", "tri_bytes", "node_record_size",
        "tri_record_size")]

    def as_dict(self) -> dict:
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class StepArgs(ctypes.Structure):
    _fields_ = [
        ("num_envs", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("env_offset", ctypes.c_int64),
        ("body_pos", ctypes.c_void_p),
        ("body_rot", ctypes.c_void_p),
        ("cam_off_pos", ctypes.c_void_p),
        ("cam_off_rot", ctypes.c_void_p),
        ("fov_delta", ctypes.c_void_p),
        ("cam_pos", ctypes.c_void_p),
        ("cam_rot", ctypes.c_void_p),
        ("ray_dirs", ctypes.c_void_p),
        ("ray_scale", ctypes.c_void_p),
        ("ray_envs", ctypes.c_int32),
        ("noise_scale", ctypes.c_double),
        ("dropout_p", ctypes.c_double),
        ("fill", _c_dp),
        ("sensor_key", ctypes.c_uint64),
        ("step", ctypes.c_int64),
        ("ring", ctypes.c_void_p),
        ("ring_slots", ctypes.c_int32),
        ("write_slot", ctypes.c_int32),
        ("ring_count", ctypes.c_int32),
        ("ring_times", _c_dp),
        ("ring_order", _c_i32p),
        ("now", ctypes.c_double),
        ("delays", ctypes.c_void_p),
        ("read_slot", ctypes.c_void_p),
        ("out_clean", ctypes.c_void_p),
        ("out", ctypes.c_void_p),
        ("counters", ctypes.c_void_p),
        ("rsm_modes", ctypes.c_void_p),
        ("rsm_k1", ctypes.c_int32),
        ("rsm_k2", ctypes.c_int32),
        ("rsm_key", ctypes.c_uint64),
        ("rsm_fill_low", ctypes.c_double),
        ("rsm_fill_high", _c_dp),
        ("ds_out", ctypes.c_void_p),
        ("ds_factor", ctypes.c_int32),
        ("link_states", ctypes.c_void_p),
        ("env_stride", ctypes.c_int64),
        ("record_stride", ctypes.c_int32),
        ("pos_offset", ctypes.c_int32),
        ("rot_offset", ctypes.c_int32),
        ("link_map", ctypes.c_void_p),
    ]


class MdrtError(RuntimeError):
    pass


_lib = None
_lock = threading.Lock()


def lib():
    """Load libmdrt.so (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2602_03002_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        sig = {
            "mdrt_abi_version": (ctypes.c_int, []),
            "mdrt_last_error": (ctypes.c_char_p, []),
            "mdrt_device_count": (ctypes.c_int, [_c_i32p]),
            "mdrt_create": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(vp)]),
            "mdrt_destroy": (ctypes.c_int, [vp]),
            "mdrt_add_body": (ctypes.c_int, [vp, _c_dp, ctypes.c_int64, _c_i64p, ctypes.c_int64, _c_i32p]),
            "mdrt_set_terrain": (ctypes.c_int, [vp, _c_dp, ctypes.c_int64, _c_i64p, ctypes.c_int64]),
            "mdrt_set_cameras": (ctypes.c_int, [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _c_dp,
                                                _c_dp, _c_dp, _c_i32p, _c_dp, _c_dp]),
            "mdrt_commit": (ctypes.c_int, [vp]),
            "mdrt_get_stats": (ctypes.c_int, [vp, ctypes.POINTER(Stats)]),
            "mdrt_render": (ctypes.c_int, [vp, ctypes.POINTER(StepArgs), vp]),
            "mdrt_noise_dropout": (ctypes.c_int, [vp, vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                  ctypes.c_int32, ctypes.c_int64, _c_dp, _c_dp,
                                                  ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
                                                  ctypes.c_int64, vp]),
            "mdrt_gather_delayed": (ctypes.c_int, [ctypes.POINTER(vp), ctypes.c_int32, vp, vp,
                                                   ctypes.c_int64, ctypes.c_int64, vp]),
            "mdrt_select_slots": (ctypes.c_int, [_c_dp, _c_i32p, ctypes.c_int32, ctypes.c_double, vp, vp,
                                                 ctypes.c_int64, vp]),
            "mdrt_downsample_min": (ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                                   ctypes.c_int32, vp]),
            "mdrt_depth_to_u8": (ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_double, vp]),
            "mdrt_bvh_build": (ctypes.c_int, [_c_dp, ctypes.c_int64, _c_i64p, ctypes.c_int64, ctypes.c_int32, vp,
                                              ctypes.c_int64, vp, ctypes.c_int64, _c_i64p, _c_i64p]),
            "mdrt_query_rays": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_int64, ctypes.c_float, vp, vp, vp]),
            "mdrt_bvh_check": (ctypes.c_int, [_c_dp, ctypes.c_int64, _c_i64p, ctypes.c_int64, _c_i64p]),
            "mdrt_probe_read": (ctypes.c_int, [vp, ctypes.c_int64, ctypes.c_int32, vp, vp]),
            "mdrt_state_set": (ctypes.c_int, [vp, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double,
                                              ctypes.c_double, ctypes.c_int64, ctypes.c_int32, _c_dp, _c_i32p,
                                              ctypes.c_int32]),
            "mdrt_rsm_apply": (ctypes.c_int, [vp, vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                              vp, _c_i32p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_double, _c_dp, vp]),
            "mdrt_state_get": (ctypes.c_int, [vp, _c_i64p, _c_dp, _c_i32p, _c_i32p, _c_dp, _c_i32p]),
            "mdrt_peer_alloc": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(vp), ctypes.c_char_p]),
            "mdrt_peer_open": (ctypes.c_int, [ctypes.c_int32, ctypes.c_char_p, ctypes.POINTER(vp)]),
            "mdrt_peer_close": (ctypes.c_int, [vp]),
            "mdrt_peer_free": (ctypes.c_int, [vp]),
            "mdrt_sync": (ctypes.c_int, [vp]),
            "mdrt_host_touch": (ctypes.c_int, [vp, ctypes.c_int64, ctypes.c_int32]),
            "mdrt_host_copy": (ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_int32]),
            "mdrt_order_begin": (ctypes.c_int, [vp, vp]),
            "mdrt_order_end": (ctypes.c_int, [vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.mdrt_abi_version() != ABI_VERSION:
            raise ImportError(f"{LIB_PATH} has ABI {L.mdrt_abi_version()}, this package needs {ABI_VERSION}: "
                              "rebuild with `python -m paper_2602_03002_b200.build --force`")
        _lib = L
        return _lib


# symbols declared by include/mdrt.h (checked by tests/test_abi.py)
EXPORTS = ("mdrt_abi_version", "mdrt_last_error", "mdrt_device_count", "mdrt_create", "mdrt_destroy",
           "mdrt_add_body", "mdrt_set_terrain", "mdrt_set_cameras", "mdrt_commit", "mdrt_get_stats",
           "mdrt_render", "mdrt_noise_dropout", "mdrt_gather_delayed", "mdrt_select_slots",
           "mdrt_downsample_min", "mdrt_depth_to_u8", "mdrt_bvh_build", "mdrt_query_rays", "mdrt_bvh_check", "mdrt_probe_read", "mdrt_state_set", "mdrt_state_get", "mdrt_rsm_apply", "mdrt_peer_alloc",
           "mdrt_peer_open", "mdrt_peer_close", "mdrt_peer_free", "mdrt_sync", "mdrt_order_begin",
           "mdrt_order_end", "mdrt_host_touch", "mdrt_host_copy")


# Device address ranges that are remote memory (peer mappings of another GPU's
# buffer, distributed.PeerFrameSink): a render whose `out` lies in one gets
# MDRT_WIDE_STORES so its epilogue writes NVLink in whole 32 B sectors.
_remote: dict[int, int] = {}


def register_remote(base: int, nbytes: int) -> None:
    _remote[int(base)] = int(nbytes)


def unregister_remote(base: int) -> None:
    _remote.pop(int(base), None)


def is_remote(ptr: int) -> bool:
    p = int(ptr)
    return any(b <= p < b + n for b, n in _remote.items())


def check(rc: int) -> None:
    if rc == MDRT_OK:
        return
    msg = lib().mdrt_last_error().decode("utf-8", "replace")
    if rc == MDRT_EINVAL:
        raise ValueError(msg)
    raise MdrtError(f"mdrt error {rc}: {msg}")


def device_count() -> int:
    n = ctypes.c_int32(0)
    check(lib().mdrt_device_count(ctypes.byref(n)))
    return int(n.value)


def dptr(a) -> ctypes.Array:
    return a.ctypes.data_as(_c_dp)


def bvh_check(verts, faces) -> dict:
    """Host-only build + invariant check of one mesh's packed BVH (no GPU needed)."""
    import numpy as np
    v = np.ascontiguousarray(verts, dtype=np.float64)
    f = np.ascontiguousarray(faces, dtype=np.int64)
    info = np.zeros(4, np.int64)
    check(lib().mdrt_bvh_check(dptr(v), len(v), f.ctypes.data_as(_c_i64p), len(f),
                               info.ctypes.data_as(_c_i64p)))
    return dict(nodes=int(info[0]), triangles=int(info[1]), depth=int(info[2]), leaves=int(info[3]))


class Context:
    """Owns one mdrt_ctx (geometry + camera rig on one device)."""

    def __init__(self, device: int):
        self._ptr = ctypes.c_void_p()
        check(lib().mdrt_create(int(device), ctypes.byref(self._ptr)))
        self.device = int(device)

    def __del__(self):
        ptr = getattr(self, "_ptr", None)
        if ptr and ptr.value and _lib is not None:
            _lib.mdrt_destroy(ptr)
            self._ptr = ctypes.c_void_p()

    @property
    def ptr(self):
        return self._ptr

    def add_body(self, verts, faces) -> int:
        import numpy as np
        v = np.ascontiguousarray(verts, dtype=np.float64)
        f = np.ascontiguousarray(faces, dtype=np.int64)
        bid = ctypes.c_int32(-1)
        check(lib().mdrt_add_body(self._ptr, dptr(v), len(v), f.ctypes.data_as(_c_i64p), len(f),
                                  ctypes.byref(bid)))
        return int(bid.value)

    def set_terrain(self, verts, faces) -> None:
        import numpy as np
        v = np.ascontiguousarray(verts, dtype=np.float64)
        f = np.ascontiguousarray(faces, dtype=np.int64)
        check(lib().mdrt_set_terrain(self._ptr, dptr(v), len(v), f.ctypes.data_as(_c_i64p), len(f)))

    def set_cameras(self, width, height, hfov, vfov, d_max, parent, mount_pos, mount_rot) -> None:
        import numpy as np
        hf = np.ascontiguousarray(hfov, np.float64)
        vf = np.ascontiguousarray(vfov, np.float64)
        dm = np.ascontiguousarray(d_max, np.float64)
        pa = np.ascontiguousarray(parent, np.int32)
        mp = np.ascontiguousarray(mount_pos, np.float64)
        mr = np.ascontiguousarray(mount_rot, np.float64)
        check(lib().mdrt_set_cameras(self._ptr, len(hf), int(width), int(height), dptr(hf), dptr(vf),
                                     dptr(dm), pa.ctypes.data_as(_c_i32p), dptr(mp), dptr(mr)))

    def commit(self) -> None:
        check(lib().mdrt_commit(self._ptr))

    def stats(self) -> dict:
        s = Stats()
        check(lib().mdrt_get_stats(self._ptr, ctypes.byref(s)))
        return s.as_dict()

    def render(self, args: StepArgs, stream: int) -> None:
        check(lib().mdrt_render(self._ptr, ctypes.byref(args), ctypes.c_void_p(stream)))

    def sync(self) -> None:
        check(lib().mdrt_sync(self._ptr))

    def order_begin(self, stream: int) -> None:
        check(lib().mdrt_order_begin(self._ptr, ctypes.c_void_p(stream)))

    def order_end(self, stream: int) -> None:
        check(lib().mdrt_order_end(self._ptr, ctypes.c_void_p(stream)))

    def state_set(self, num_envs, key, t0, dt, next_step, ring_slots, times, order, rsm_key=0) -> None:
        import numpy as np
        t = np.ascontiguousarray(times, dtype=np.float64)
        o = np.ascontiguousarray(order, dtype=np.int32)
        check(lib().mdrt_state_set(self._ptr, int(num_envs), int(key), int(rsm_key), float(t0), float(dt),
                                   int(next_step),
                                   int(ring_slots), dptr(t), o.ctypes.data_as(_c_i32p), len(t)))

    def state_get(self) -> dict:
        import numpy as np
        ns = ctypes.c_int64()
        now = ctypes.c_double()
        ws = ctypes.c_int32()
        cnt = ctypes.c_int32()
        t = np.zeros(32)
        o = np.zeros(32, np.int32)
        check(lib().mdrt_state_get(self._ptr, ctypes.byref(ns), ctypes.byref(now), ctypes.byref(ws),
                                   ctypes.byref(cnt), dptr(t), o.ctypes.data_as(_c_i32p)))
        n = int(cnt.value)
        return dict(next_step=int(ns.value), now=float(now.value), write_slot=int(ws.value),
                    times=t[:n].tolist(), order=o[:n].tolist())
