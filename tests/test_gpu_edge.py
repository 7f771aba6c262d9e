"""Edge cases of the CUDA path against the CPU oracle (reference semantics,
numba_backend.py:155-219): more links than a warp has lanes, a camera inside a
closed link mesh, single-triangle links (one-leaf trees), degenerate and
non-tile-multiple resolutions, empty scenes, everything culled, many cameras
with different ranges, parented cameras on a moving link.
"""

import numpy as np
import torch
import pytest

from test_gpu_acceptance import f32, random_scene

pytestmark = pytest.mark.gpu


def _cams_dict(cams):
    return [dict(width=c.width, height=c.height, hfov_deg=c.hfov_deg, vfov_deg=c.vfov_deg, d_max=c.d_max,
                 mount_pos=c.mount.translation, mount_rot=c.mount.rotation, parent=c.parent_body) for c in cams]


def _check(md, orc, bodies, terrain, cams, pos, rot, n, tol=1e-4, max_bad=0):
    scene = md.Scene(n, bodies=[(f"b{k}", m) for k, m in enumerate(bodies)], cameras=cams, terrain=terrain)
    if bodies:
        scene.set_body_poses(pos, rot)
    out = md.render(scene).data.cpu().numpy().astype(np.float64)
    osc = orc.OracleScene([(m.vertices, m.faces) for m in bodies],
                          None if terrain is None else (terrain.vertices, terrain.faces), _cams_dict(cams))
    ref = osc.render(pos if bodies else np.zeros((n, 0, 3)), rot if bodies else np.zeros((n, 0, 4)))
    d = np.abs(out - ref)
    assert int((d > tol).sum()) <= max_bad, (d.max(), int((d > tol).sum()))
    miss = ref == np.asarray([c.d_max for c in cams], np.float32).reshape(1, -1, 1, 1)
    assert np.array_equal(out[miss], ref[miss])          # misses are exactly d_max
    return out, ref


def test_more_links_than_warp_lanes(pkg, oracle):
    g = np.random.default_rng(41)
    bodies, terrain, cams, pos, rot, _ = random_scene(pkg, g, num_envs=3, num_cams=3, num_bodies=45)
    _check(pkg, oracle, bodies, terrain, cams, pos, rot, 3, max_bad=2)


def test_camera_inside_closed_link(pkg, oracle):
    """Rays start inside a link's box: the cull rectangle must be the whole image
    and the (double-sided) inner walls are hit at their exact distance."""
    box = pkg.make_box(size=(1.0, 1.0, 1.0))
    bodies = [pkg.TriMesh(f32(box.vertices), box.faces, frame="body-local")]
    cam = pkg.CameraModel(width=21, height=13, hfov_deg=90.0, vfov_deg=70.0, d_max=5.0,
                          mount=pkg.look_at_pose([0.0, 0.0, 0.0], [1.0, 0.0, 0.0]))
    pos = f32(np.array([[[0.1, -0.05, 0.02]], [[0.0, 0.0, 0.0]]]))
    rot = f32(np.array([[[1.0, 0.0, 0.0, 0.0]], [[np.cos(0.3), 0.0, 0.0, np.sin(0.3)]]]))
    out, ref = _check(pkg, oracle, bodies, None, [cam], pos, rot, 2)
    assert out.max() < 1.0                                        # every ray hits a wall
    assert abs(out[1, 0, 6, 10] - 0.5 / np.cos(0.6)) < 1e-5       # centre ray; quat half-angle 0.3 = yaw 0.6


def test_single_triangle_links_and_tiny_images(pkg, oracle):
    tri = pkg.TriMesh(f32(np.array([[0.0, -0.5, -0.5], [0.0, 0.5, -0.5], [0.0, 0.0, 0.6]])),
                      np.array([[0, 1, 2]]), frame="body-local")
    plane = pkg.make_plane(size=(8.0, 8.0), center=(0.0, 0.0, -0.3))
    for w, h in ((1, 1), (1, 17), (33, 1), (13, 5), (65, 3)):
        cam = pkg.CameraModel(width=w, height=h, hfov_deg=80.0, vfov_deg=60.0, d_max=6.0,
                              mount=pkg.look_at_pose([-2.0, 0.2, 0.5], [0.0, 0.0, 0.0]))
        pos = f32(np.array([[[0.0, 0.0, 0.0], [0.3, 0.1, 0.0]]]))
        rot = f32(np.array([[[1.0, 0, 0, 0], [np.cos(0.2), 0, 0, np.sin(0.2)]]]))
        _check(pkg, oracle, [tri, tri], plane, [cam], pos, rot, 1)


def test_empty_scene_and_everything_culled(pkg, oracle):
    cams = [pkg.CameraModel(width=16, height=9, hfov_deg=70.0, vfov_deg=50.0, d_max=d,
                            mount=pkg.look_at_pose([0.0, 0.0, 1.0], [1.0, 0.0, 1.0])) for d in (3.0, 7.5)]
    scene = pkg.Scene(2, bodies=[], cameras=cams, terrain=None)
    out = pkg.render(scene).data.cpu().numpy()
    assert np.array_equal(out[:, 0], np.full((2, 9, 16), np.float32(3.0)))
    assert np.array_equal(out[:, 1], np.full((2, 9, 16), np.float32(7.5)))
    box = pkg.make_box(size=(0.4, 0.4, 0.4))
    bodies = [pkg.TriMesh(f32(box.vertices), box.faces, frame="body-local")] * 3
    far = f32(np.array([[[50.0, 0, 1], [0, 60.0, 1], [-1.5, 0, 1]]] * 2))   # behind / out of range
    rot = f32(np.tile(np.array([1.0, 0, 0, 0]), (2, 3, 1)))
    out, _ = _check(pkg, oracle, bodies, None, cams, far, rot, 2)
    assert np.array_equal(out[:, 0], np.full((2, 9, 16), np.float32(3.0)))


def test_many_cameras_parented_to_moving_link(pkg, oracle):
    g = np.random.default_rng(5)
    bodies, terrain, _, pos, rot, _ = random_scene(pkg, g, num_envs=2, num_cams=1, num_bodies=6)
    cams = []
    for c in range(6):
        yaw = 2 * np.pi * c / 6
        mount = pkg.RigidPose(np.array([0.3 * np.cos(yaw), 0.3 * np.sin(yaw), 0.4]),
                              pkg.quat_from_euler(0.0, 0.5 + 0.1 * c, yaw))
        cams.append(pkg.CameraModel(width=24, height=16, hfov_deg=70.0 + 5 * c, vfov_deg=50.0, d_max=2.0 + c,
                                    mount=mount, parent_body=c % 6))
    # mounts rounded to what crosses the ABI (f64 mounts, f32 poses)
    _check(pkg, oracle, bodies, terrain, cams, pos, rot, 2, max_bad=2)


_SCHED_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[2])
import paper_2602_03002_b200 as md
from paper_2602_03002_b200 import synth
w = synth.config("cfg2", 512)
f32 = lambda x: np.asarray(x, np.float64).astype(np.float32).astype(np.float64)
bodies = [(nm, md.TriMesh(f32(m.vertices), m.faces, frame="body-local")) for nm, m in w.bodies]
scene = md.Scene(w.num_envs, bodies=bodies, cameras=w.cameras,
                 terrain=md.TriMesh(f32(w.terrain.mesh.vertices), w.terrain.mesh.faces))
p, q = w.poses(1)
scene.set_body_poses(p, q)
out = md.render_pipeline(scene, sensor=md.SensorConfig(seed=2), step=1)
np.save(sys.argv[1], out.cpu().numpy())
"""


@pytest.mark.parametrize("frac", ["0.5", "0.95", "1.0"])
def test_sm_local_tile_schedule_is_bitwise_identical(tmp_path, frac):
    """The SM-local tile schedule (chunks + pool + stealing) renders every tile exactly once."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for f in ("0", frac):
        path = tmp_path / f"o{f}.npy"
        env = dict(os.environ, MDRT_LOCAL_FRAC=f)
        subprocess.run([sys.executable, "-c", _SCHED_SCRIPT, str(path), root], check=True, env=env, timeout=300)
        outs[f] = np.load(path)
    assert np.array_equal(outs["0"], outs[frac])


def test_high_resolution_camera(pkg, oracle):
    """A 320x240 camera (8x4 tiles, 2400 tiles per view) against the oracle."""
    g = np.random.default_rng(8)
    bodies, terrain, cams, pos, rot, _ = random_scene(pkg, g, num_envs=2, num_cams=1, num_bodies=6)
    cam = cams[0]
    hi = pkg.CameraModel(width=320, height=240, hfov_deg=cam.hfov_deg, vfov_deg=cam.vfov_deg, d_max=cam.d_max,
                         mount=cam.mount)
    _check(pkg, oracle, bodies, terrain, [hi], pos, rot, 2, max_bad=int(1e-4 * 2 * 320 * 240) + 1)


def test_two_scenes_alternating(pkg, oracle):
    """Two live scenes with different image widths (4x8 and 8x4 tiles, separate
    native contexts) rendered alternately stay independent and match the oracle."""
    g = np.random.default_rng(12)
    bodies, terrain, cams, pos, rot, _ = random_scene(pkg, g, num_envs=2, num_cams=1, num_bodies=4)
    cam = cams[0]
    narrow = pkg.CameraModel(width=48, height=32, hfov_deg=cam.hfov_deg, vfov_deg=cam.vfov_deg,
                             d_max=cam.d_max, mount=cam.mount)
    wide = pkg.CameraModel(width=160, height=96, hfov_deg=cam.hfov_deg, vfov_deg=cam.vfov_deg,
                           d_max=cam.d_max, mount=cam.mount)
    sa = pkg.Scene(2, bodies=[(f"b{k}", m) for k, m in enumerate(bodies)], cameras=[narrow], terrain=terrain)
    sb = pkg.Scene(2, bodies=[(f"b{k}", m) for k, m in enumerate(bodies)], cameras=[wide], terrain=terrain)
    for s in (sa, sb):
        s.set_body_poses(pos, rot)
    first = [pkg.render(sa).data.clone(), pkg.render(sb).data.clone()]
    for _ in range(3):
        assert torch.equal(pkg.render(sb).data, first[1])
        assert torch.equal(pkg.render(sa).data, first[0])
    for s, out in ((sa, first[0]), (sb, first[1])):
        c = s.cameras[0]
        osc = oracle.OracleScene([(m.vertices, m.faces) for m in bodies], (terrain.vertices, terrain.faces),
                                 [dict(width=c.width, height=c.height, hfov_deg=c.hfov_deg, vfov_deg=c.vfov_deg,
                                       d_max=c.d_max, mount_pos=c.mount.translation, mount_rot=c.mount.rotation,
                                       parent=None)])
        ref = osc.render(pos, rot)
        d = np.abs(out.cpu().numpy().astype(np.float64) - ref)
        assert int((d > 1e-4).sum()) <= max(1, int(1e-4 * d.size))
