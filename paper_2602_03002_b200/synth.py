"""Synthetic workloads of BASELINE.json's configs (terrain, G1 proxy, camera rig, poses).

The reference ships no G1 asset and its terrain generator (terrain.py) is out
of scope for the renderer, so this module produces deterministic stand-ins of
the named shapes:

* terrain: 0.05 m height-grid tiles (slope pyramid, stairs up/down, rolling),
  stepping stones as boxes over a recessed floor -- same construction rules as
  terrain.py:218-360 (grid meshes, box stones), re-derived here; the config 1,
  2 and 3 meshes equal the reference generator's bit for bit (stairs tiles
  centred in their 6 m tile: x shifted by 1.08 m), pinned by
  tests/test_host_api.py against checksums written by the live reference;
* G1 proxy: 30 rigid links (pelvis, 2x6 leg, 3 waist, 2x7 arm) meshed as
  ellipsoids/boxes in their link frames (~8.7k triangles), posed by forward
  kinematics with per-step joint perturbations from the counter RNG stream
  "motion" keyed (step, env, joint) like bench.pose_trajectory (bench.py:66-86);
* cameras: torso-parented 64x48 depth cameras, 101 x 69 deg FOV,
  front mount (+0.12, 0, +0.15) pitched 45 deg down, back mirrored, optional
  left/right.

Everything is plain numpy so the CPU oracle and the GPU see identical inputs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import rng
from .camera import CameraModel, look_at_pose
from .mesh import TriMesh, make_box, make_icosphere, make_plane, merge_meshes
from .transforms import RigidPose

CELL = 0.05


# ---------------------------------------------------------------------------
# terrain
# ---------------------------------------------------------------------------

def grid_mesh(xs: np.ndarray, ys: np.ndarray, heights: np.ndarray) -> TriMesh:
    """Height grid -> 2 triangles per cell (heights[iy, ix])."""
    ny, nx = heights.shape
    gx, gy = np.meshgrid(xs, ys)
    verts = np.column_stack([gx.ravel(), gy.ravel(), heights.ravel()])
    iy, ix = np.meshgrid(np.arange(ny - 1), np.arange(nx - 1), indexing="ij")
    a = (iy * nx + ix).ravel()
    faces = np.empty((2 * a.size, 3), dtype=np.int64)
    faces[0::2] = np.column_stack([a, a + 1, a + nx + 1])
    faces[1::2] = np.column_stack([a, a + nx + 1, a + nx])
    return TriMesh(verts, faces)


def _axis(lo: float, hi: float, cell: float = CELL) -> np.ndarray:
    n = int(round((hi - lo) / cell)) + 1
    return lo + np.arange(n) * cell


@dataclass
class Terrain:
    mesh: TriMesh
    height: callable            # (x, y) arrays -> ground height
    bounds: tuple               # (xmin, xmax, ymin, ymax) usable for robot placement
    name: str = ""


def slope_pyramid_height(x, y, size=6.0, incline_deg=20.0, platform=1.0):
    cheb = np.maximum(np.abs(x), np.abs(y))
    return math.tan(math.radians(incline_deg)) * np.clip(size / 2 - np.maximum(cheb, platform / 2), 0.0, None)


def stairs_height(x, y, down=False, size=6.0, step_length=0.27, step_height=0.12, num_steps=8):
    run = num_steps * step_length
    x0 = -run / 2.0                                  # stairs centred in the tile
    k = np.clip(np.floor((x - x0) / step_length + 1e-9).astype(np.int64) + 1, 0, num_steps)
    h = k * step_height
    return -h if down else h


def tile_field(kinds, tile=6.0, cell=CELL) -> Terrain:
    """len(kinds)=k*k tiles on a square grid, each a height-grid mesh (config 2)."""
    k = int(round(math.sqrt(len(kinds))))
    assert k * k == len(kinds)
    parts = []
    funcs = {}
    for idx, kind in enumerate(kinds):
        i, j = idx % k, idx // k
        cx, cy = (i - (k - 1) / 2) * tile, (j - (k - 1) / 2) * tile
        xs = _axis(-tile / 2, tile / 2, cell)
        gx, gy = np.meshgrid(xs, xs)
        f = _tile_func(kind, tile)
        parts.append(grid_mesh(xs + cx, xs + cy, f(gx, gy)))
        funcs[(i, j)] = (cx, cy, f)

    def height(x, y):
        x = np.asarray(x, np.float64)
        y = np.asarray(y, np.float64)
        i = np.clip(np.floor(x / tile + k / 2).astype(int), 0, k - 1)
        j = np.clip(np.floor(y / tile + k / 2).astype(int), 0, k - 1)
        out = np.zeros(np.broadcast(x, y).shape)
        for (ii, jj), (cx, cy, f) in funcs.items():
            m = (i == ii) & (j == jj)
            out[m] = f(np.broadcast_to(x, out.shape)[m] - cx, np.broadcast_to(y, out.shape)[m] - cy)
        return out

    half = k * tile / 2
    return Terrain(merge_meshes(parts), height, (-half + 0.5, half - 0.5, -half + 0.5, half - 0.5),
                   name="tiles:" + ",".join(kinds))


def _tile_func(kind, tile):
    if kind == "slope_pyramid":
        return lambda x, y: slope_pyramid_height(x, y, size=tile)
    if kind == "stairs_up":
        return lambda x, y: stairs_height(x, y, size=tile)
    if kind == "stairs_down":
        return lambda x, y: stairs_height(x, y, down=True, size=tile)
    if kind == "flat":
        return lambda x, y: np.zeros(np.broadcast(x, y).shape)
    raise ValueError(kind)


def stairs_terrain(cell=CELL, width=3.0, platform=1.0, step_length=0.27, step_height=0.12,
                   num_steps=8) -> Terrain:
    """Single stairs_up patch like TerrainSpec(kind="stairs_up") defaults (config 1)."""
    run = num_steps * step_length
    xs = _axis(-platform, run + platform, cell)
    ys = _axis(-width / 2, width / 2, cell)
    gx, gy = np.meshgrid(xs, ys)

    def height(x, y):
        k = np.clip(np.floor(np.asarray(x) / step_length + 1e-9).astype(np.int64) + 1, 0, num_steps)
        return k * step_height + 0.0 * np.asarray(y)

    return Terrain(grid_mesh(xs, ys, height(gx, gy)), height,
                   (-platform + 0.3, run + platform - 0.3, -width / 2 + 0.3, width / 2 - 0.3), "stairs_up")


def stepping_stones(size=24.0, stone=0.25, gap=0.60, floor_depth=0.5, variation=0.02, seed=0) -> Terrain:
    """Boxes over a recessed floor plane (config 3: 729 stones, 8,750 triangles)."""
    pitch = stone + gap
    imax = int(math.floor((size / 2 - stone / 2) / pitch + 1e-9))
    key = rng.stream_key(seed, "terrain")
    parts = [make_plane(size=(size, size), center=(0.0, 0.0, -floor_depth))]
    tops = {}
    for i in range(-imax, imax + 1):
        for j in range(-imax, imax + 1):
            top = float(rng.uniform(key, i, j, low=-variation, high=variation))
            tops[(i, j)] = top
            parts.append(make_box(size=(stone, stone, top + floor_depth),
                                  center=(i * pitch, j * pitch, (top - floor_depth) / 2)))

    def height(x, y):
        x = np.asarray(x, np.float64)
        y = np.asarray(y, np.float64)
        si = np.rint(x / pitch).astype(int)
        sj = np.rint(y / pitch).astype(int)
        on = (np.abs(x - si * pitch) <= stone / 2) & (np.abs(y - sj * pitch) <= stone / 2) & \
             (np.abs(si) <= imax) & (np.abs(sj) <= imax)
        out = np.full(np.broadcast(x, y).shape, -floor_depth)
        for idx in zip(*np.nonzero(on)):
            out[idx] = tops[(int(si[idx]), int(sj[idx]))]
        return out

    half = imax * pitch
    return Terrain(merge_meshes(parts), height, (-half, half, -half, half), "stepping_stones")


def rolling_terrain(nodes=1300, cell=CELL, amp=0.35, seed=5) -> Terrain:
    """Random rolling height grid (tests/scenes.py:31-46 pattern), (nodes-1)^2*2 triangles (config 5).

    BASELINE config 5 names a 1M-triangle terrain whose BVH exceeds L2; with
    this framework's 80 B/triangle BVH footprint 1M triangles (708 nodes) would
    still fit the 126 MB L2, so the default follows SURVEY.md 8(d) ("otherwise
    increase nodes"): 1300 x 1300 nodes = 3.37M triangles, ~270 MB of BVH
    (>= 2x L2). ``nodes=708`` gives the literal 999,698-triangle variant."""
    r = np.random.default_rng(seed)
    ext = (nodes - 1) * cell
    xs = -ext / 2 + np.arange(nodes) * cell
    fx, px, fy, py = r.uniform(0.5, 1.5), r.uniform(0, 6), r.uniform(0.5, 1.5), r.uniform(0, 6)
    gx, gy = np.meshgrid(xs, xs)
    jitter = r.uniform(-0.05, 0.05, size=gx.shape)

    def smooth(x, y):
        return amp * np.sin(np.asarray(x) * fx + px) * np.cos(np.asarray(y) * fy + py)

    hz = smooth(gx, gy) + jitter
    return Terrain(grid_mesh(xs, xs, hz), lambda x, y: smooth(x, y) + 0.05,
                   (-ext / 2 + 1, ext / 2 - 1, -ext / 2 + 1, ext / 2 - 1), "rolling")


# ---------------------------------------------------------------------------
# G1 proxy (30 links)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Link:
    name: str
    parent: int
    offset: tuple           # joint origin in the parent frame
    axis: int               # joint axis (0=x, 1=y, 2=z) in this link's frame
    q0: float               # default joint angle (standing)
    shape: str              # "ellipsoid" | "box"
    center: tuple           # mesh centre in the link frame
    size: tuple             # radii (ellipsoid) or full extents (box)


def _leg(side: int, base: int) -> list[Link]:
    s = 1.0 if side > 0 else -1.0
    nm = "left" if side > 0 else "right"
    return [
        Link(f"{nm}_hip_pitch", 0, (0.0, 0.09 * s, -0.05), 1, -0.15, "ellipsoid", (0, 0, 0), (0.05, 0.05, 0.05)),
        Link(f"{nm}_hip_roll", base + 0, (0.0, 0.03 * s, -0.02), 0, 0.0, "ellipsoid", (0, 0, -0.02), (0.05, 0.045, 0.06)),
        Link(f"{nm}_hip_yaw", base + 1, (0.0, 0.0, -0.06), 2, 0.0, "ellipsoid", (0, 0, -0.13), (0.065, 0.065, 0.17)),
        Link(f"{nm}_knee", base + 2, (0.0, 0.0, -0.28), 1, 0.35, "ellipsoid", (0, 0, -0.14), (0.055, 0.055, 0.17)),
        Link(f"{nm}_ankle_pitch", base + 3, (0.0, 0.0, -0.30), 1, -0.2, "ellipsoid", (0, 0, 0), (0.035, 0.035, 0.035)),
        Link(f"{nm}_ankle_roll", base + 4, (0.0, 0.0, -0.02), 0, 0.0, "box", (0.03, 0, -0.03), (0.22, 0.09, 0.04)),
    ]


def _arm(side: int, base: int, torso: int) -> list[Link]:
    s = 1.0 if side > 0 else -1.0
    nm = "left" if side > 0 else "right"
    return [
        Link(f"{nm}_shoulder_pitch", torso, (0.0, 0.16 * s, 0.28), 1, 0.25, "ellipsoid", (0, 0.02 * s, 0), (0.05, 0.05, 0.05)),
        Link(f"{nm}_shoulder_roll", base + 0, (0.0, 0.04 * s, 0.0), 0, 0.15 * s, "ellipsoid", (0, 0, -0.03), (0.045, 0.045, 0.06)),
        Link(f"{nm}_shoulder_yaw", base + 1, (0.0, 0.0, -0.06), 2, 0.0, "ellipsoid", (0, 0, -0.08), (0.045, 0.045, 0.11)),
        Link(f"{nm}_elbow", base + 2, (0.0, 0.0, -0.17), 1, -0.9, "ellipsoid", (0, 0, -0.07), (0.04, 0.04, 0.1)),
        Link(f"{nm}_wrist_roll", base + 3, (0.0, 0.0, -0.15), 2, 0.0, "ellipsoid", (0, 0, -0.02), (0.035, 0.035, 0.04)),
        Link(f"{nm}_wrist_pitch", base + 4, (0.0, 0.0, -0.04), 1, 0.0, "ellipsoid", (0, 0, -0.01), (0.03, 0.03, 0.03)),
        Link(f"{nm}_wrist_yaw", base + 5, (0.0, 0.0, -0.03), 2, 0.0, "box", (0, 0, -0.05), (0.05, 0.08, 0.1)),
    ]


def g1_links(arms_raised: bool = False) -> list[Link]:
    links = [Link("pelvis", -1, (0.0, 0.0, 0.0), 2, 0.0, "ellipsoid", (0, 0, 0), (0.09, 0.14, 0.08))]
    links += _leg(+1, 1)           # 1..6
    links += _leg(-1, 7)           # 7..12
    links += [
        Link("waist_yaw", 0, (0.0, 0.0, 0.06), 2, 0.0, "ellipsoid", (0, 0, 0.02), (0.06, 0.08, 0.04)),      # 13
        Link("waist_roll", 13, (0.0, 0.0, 0.04), 0, 0.0, "ellipsoid", (0, 0, 0.02), (0.06, 0.08, 0.04)),    # 14
        Link("torso", 14, (0.0, 0.0, 0.04), 1, 0.0, "box", (0, 0, 0.2), (0.18, 0.28, 0.34)),               # 15
    ]
    links += _arm(+1, 16, 15)      # 16..22
    links += _arm(-1, 23, 15)      # 23..29
    if arms_raised:
        # shoulders pitched forward/up, elbows bent: hands cross the lower front FOV (config 3)
        upd = {"left_shoulder_pitch": -0.9, "right_shoulder_pitch": -0.9, "left_elbow": -0.6, "right_elbow": -0.6}
        links = [Link(**{**l.__dict__, "q0": upd.get(l.name, l.q0)}) for l in links]
    assert len(links) == 30
    return links


TORSO = 15


def _ellipsoid(center, radii, subdivisions=2) -> TriMesh:
    m = make_icosphere(1.0, subdivisions=subdivisions)
    return TriMesh(m.vertices * np.asarray(radii) + np.asarray(center), m.faces, frame="body-local")


def link_mesh(l: Link) -> TriMesh:
    if l.shape == "box":
        b = make_box(size=l.size, center=l.center)
        return TriMesh(b.vertices, b.faces, frame="body-local")
    return _ellipsoid(l.center, l.size)


# ---- batched quaternion helpers (wxyz, numpy) ----
def qmul(a, b):
    aw, ax, ay, az = np.moveaxis(a, -1, 0)
    bw, bx, by, bz = np.moveaxis(b, -1, 0)
    return np.stack([aw * bw - ax * bx - ay * by - az * bz, aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx, aw * bz + ax * by - ay * bx + az * bw], -1)


def qrot(q, v):
    w = q[..., :1]
    u = q[..., 1:]
    t = 2.0 * np.cross(u, v)
    return v + w * t + np.cross(u, t)


def axis_quat(axis: int, angle):
    angle = np.asarray(angle, np.float64)
    q = np.zeros(angle.shape + (4,))
    q[..., 0] = np.cos(angle / 2)
    q[..., 1 + axis] = np.sin(angle / 2)
    return q


def forward_kinematics(links, root_pos, root_quat, joint_q):
    """root_pos (N,3), root_quat (N,4), joint_q (N,B) -> link poses (N,B,3), (N,B,4)."""
    n, b = joint_q.shape
    pos = np.empty((n, b, 3))
    rot = np.empty((n, b, 4))
    for i, l in enumerate(links):
        if l.parent < 0:
            p, q = root_pos, root_quat
        else:
            pp, pq = pos[:, l.parent], rot[:, l.parent]
            p = pp + qrot(pq, np.broadcast_to(np.asarray(l.offset, np.float64), pp.shape))
            q = pq
        q = qmul(q, axis_quat(l.axis, joint_q[:, i]))
        pos[:, i] = p
        rot[:, i] = q / np.linalg.norm(q, axis=-1, keepdims=True)
    return pos, rot


# ---------------------------------------------------------------------------
# cameras
# ---------------------------------------------------------------------------

def torso_cameras(num_cams: int = 2, width: int = 64, height: int = 48, hfov: float = 101.0,
                  vfov: float = 69.0, d_max: float = 10.0) -> list[CameraModel]:
    """Depth cameras on the torso link: front (+x), back, left, right; 45 deg down."""
    mounts = [((0.12, 0.0, 0.15), (1.0, 0.0)), ((-0.12, 0.0, 0.15), (-1.0, 0.0)),
              ((0.0, 0.16, 0.15), (0.0, 1.0)), ((0.0, -0.16, 0.15), (0.0, -1.0))]
    names = ["front", "back", "left", "right"]
    cams = []
    for k in range(num_cams):
        (x, y, z), (fx, fy) = mounts[k]
        pos = np.array([x, y, z])
        pose = look_at_pose(pos, pos + np.array([fx, fy, -1.0]))
        cams.append(CameraModel(width=width, height=height, hfov_deg=hfov, vfov_deg=vfov, d_max=d_max,
                                mount=pose, parent_body=TORSO, name=names[k]))
    return cams


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------

@dataclass
class Workload:
    name: str
    terrain: Terrain
    links: list
    cameras: list
    num_envs: int
    roots: np.ndarray = field(default=None)       # (N,3) pelvis positions
    yaws: np.ndarray = field(default=None)        # (N,)
    seed: int = 0
    joint_sigma: float = 0.15

    @property
    def bodies(self):
        return [(l.name, link_mesh(l)) for l in self.links]

    def poses(self, step: int, envs: slice | None = None):
        """Per-step link poses (N,B,3), (N,B,4) f64, deterministic in (seed, step, env, joint)."""
        sl = envs if envs is not None else slice(0, self.num_envs)
        env = np.arange(self.num_envs)[sl]
        key = rng.stream_key(self.seed, "motion")
        q0 = np.array([l.q0 for l in self.links])
        noise = rng.normal(key, step, env.reshape(-1, 1), np.arange(len(self.links)).reshape(1, -1))
        jq = q0[None, :] + self.joint_sigma * noise
        jq[:, 0] = 0.0
        rq = axis_quat(2, self.yaws[sl])
        return forward_kinematics(self.links, self.roots[sl], rq, jq)


def _place(terrain: Terrain, n: int, seed: int, height: float = 0.75):
    r = np.random.default_rng(seed)
    x0, x1, y0, y1 = terrain.bounds
    x = r.uniform(x0, x1, n)
    y = r.uniform(y0, y1, n)
    yaw = r.uniform(-math.pi, math.pi, n)
    z = terrain.height(x, y) + height
    return np.column_stack([x, y, z]), yaw


def config(name: str, num_envs: int | None = None) -> Workload:
    """BASELINE.json configs: cfg1 (1 env stairs), cfg2 (4096x2 tiles), cfg3 (4096x4 stones),
    cfg4 (32768x2 tiles), cfg5 (4096x2 160x120 rolling 1M tris)."""
    if name == "cfg1":
        t = stairs_terrain()
        w = Workload("cfg1", t, g1_links(), torso_cameras(1), num_envs or 1, joint_sigma=0.0)
        w.roots = np.array([[-0.8 + 0.27 * 0, 0.0, 0.75]])
        w.roots = np.repeat(w.roots, w.num_envs, 0)
        w.yaws = np.zeros(w.num_envs)
        return w
    if name in ("cfg2", "cfg4"):
        kinds = ["slope_pyramid", "stairs_up", "stairs_down"] * 3
        t = tile_field(kinds)
        n = num_envs or (4096 if name == "cfg2" else 32768)
        w = Workload(name, t, g1_links(), torso_cameras(2), n)
    elif name == "paper":
        # the paper's training resolution: 1024 envs, 240x135 native depth per camera,
        # min-pooled 5x to the 48x27 policy input (sensor.py:27-29)
        kinds = ["slope_pyramid", "stairs_up", "stairs_down"] * 3
        t = tile_field(kinds)
        n = num_envs or 1024
        w = Workload(name, t, g1_links(), torso_cameras(2, width=240, height=135), n)
    elif name == "cfg3":
        t = stepping_stones()
        n = num_envs or 4096
        w = Workload(name, t, g1_links(arms_raised=True), torso_cameras(4), n)
    elif name in ("cfg5", "cfg5_1m"):
        t = rolling_terrain(nodes=708 if name == "cfg5_1m" else 1300)
        n = num_envs or 4096
        w = Workload(name, t, g1_links(), torso_cameras(2, width=160, height=120), n)
    else:
        raise ValueError(f"unknown config {name!r}")
    w.roots, w.yaws = _place(t, n, seed=0)
    return w
