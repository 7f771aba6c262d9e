"""Acceptance-style sweep (reference tests/test_acceptance.py:62-90, criterion 1):
100 random scenes (2 envs x 4 cams x 32x24, 8 bodies of boxes/icospheres/
triangle soups over a rolling 10x10-node terrain, look-at cameras on a ring,
random per-env poses, half of them with camera randomisation) rendered on the
GPU and by the CPU oracle on identical float32-representable inputs.

Bar (BASELINE.json): |depth - oracle| <= 1e-4 m except grazing-edge pixels,
which are counted and must stay <= 0.01 % of all pixels.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def random_scene(md, g, num_envs=2, num_cams=4, width=32, height=24, num_bodies=8, camrand=False):
    bodies = []
    for _ in range(num_bodies):
        kind = g.integers(0, 3)
        if kind == 0:
            m = md.make_box(size=tuple(g.uniform(0.15, 0.5, size=3)))
        elif kind == 1:
            m = md.make_icosphere(radius=g.uniform(0.1, 0.3), subdivisions=int(g.integers(0, 2)))
        else:
            k = int(g.integers(4, 21))
            base = np.repeat(g.uniform(-0.25, 0.25, size=(k, 3)), 3, axis=0)
            m = md.TriMesh(base + g.uniform(-0.15, 0.15, size=base.shape), np.arange(3 * k).reshape(-1, 3))
        bodies.append(md.TriMesh(f32(m.vertices), m.faces, frame="body-local"))
    xs = np.linspace(-3.0, 3.0, 10)
    gx, gy = np.meshgrid(xs, xs)
    gz = 0.35 * np.sin(gx * g.uniform(0.5, 1.5) + g.uniform(0, 6)) * np.cos(gy * g.uniform(0.5, 1.5) +
                                                                             g.uniform(0, 6)) \
        + g.uniform(-0.05, 0.05, size=gx.shape)
    iy, ix = np.meshgrid(np.arange(9), np.arange(9), indexing="ij")
    a = (iy * 10 + ix).ravel()
    faces = np.concatenate([np.column_stack([a, a + 1, a + 11]), np.column_stack([a, a + 11, a + 10])])
    terrain = md.TriMesh(f32(np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])), faces)
    cams = []
    for c in range(num_cams):
        ang = 2 * np.pi * (c + g.uniform(0, 0.5)) / num_cams
        r = g.uniform(2.2, 3.5)
        pos = np.array([r * np.cos(ang), r * np.sin(ang), g.uniform(0.6, 2.2)])
        tgt = g.uniform(-0.5, 0.5, size=3) + np.array([0, 0, 0.4])
        cams.append(md.CameraModel(width=width, height=height, hfov_deg=float(g.uniform(60, 100)),
                                   vfov_deg=float(g.uniform(45, 75)), d_max=float(g.uniform(4, 12)),
                                   mount=md.look_at_pose(pos, tgt)))
    pos = np.stack([g.uniform(-1.5, 1.5, (num_envs, num_bodies)), g.uniform(-1.5, 1.5, (num_envs, num_bodies)),
                    g.uniform(0.0, 1.5, (num_envs, num_bodies))], -1)
    rot = g.standard_normal((num_envs, num_bodies, 4))
    rot = f32(rot / np.linalg.norm(rot, axis=-1, keepdims=True))
    rand = None
    if camrand:
        p, q, f = md.sample_camera_offsets(md.CameraRandomization(seed=int(g.integers(0, 1000))), num_envs,
                                           num_cams)
        rand = (f32(p), f32(q / np.linalg.norm(q, axis=-1, keepdims=True)), f32(f))
    return bodies, terrain, cams, f32(pos), rot, rand


def test_hundred_random_scenes_vs_oracle(pkg, oracle):
    g = np.random.default_rng(20260816)
    bad = total = 0
    worst = 0.0
    for i in range(100):
        bodies, terrain, cams, pos, rot, rand = random_scene(pkg, g, camrand=(i % 2 == 1))
        scene = pkg.Scene(2, bodies=[(f"b{k}", m) for k, m in enumerate(bodies)], cameras=cams, terrain=terrain)
        scene.set_body_poses(pos, rot)
        if rand is not None:
            scene.set_camera_randomization(*rand)
        out = pkg.render(scene).data.cpu().numpy().astype(np.float64)
        cd = [dict(width=c.width, height=c.height, hfov_deg=c.hfov_deg, vfov_deg=c.vfov_deg, d_max=c.d_max,
                   mount_pos=c.mount.translation, mount_rot=c.mount.rotation, parent=None) for c in cams]
        osc = oracle.OracleScene([(m.vertices, m.faces) for m in bodies], (terrain.vertices, terrain.faces), cd)
        ref = osc.render(pos, rot, rand_pos=None if rand is None else rand[0],
                         rand_rot=None if rand is None else rand[1], fov_delta=None if rand is None else rand[2])
        d = np.abs(out - ref)
        bad += int((d > 1e-4).sum())
        total += d.size
        worst = max(worst, float(d[d <= 1e-4].max()))
    print(f"100 scenes: {bad}/{total} pixels outside 1e-4 m ({bad / total:.2e}), max |d| inside {worst:.2e} m")
    assert worst <= 1e-4
    assert bad <= 1e-4 * total
