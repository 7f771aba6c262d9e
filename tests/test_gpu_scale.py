"""CUDA path vs the CPU oracle on the BASELINE workload shapes (synthetic G1 proxy + terrain).

Identical float32-rounded meshes and poses go to both sides. Sizes are cut so
the oracle finishes in seconds; the full 4096-env configuration is covered by
size-independent properties (slice equivalence, determinism, range bounds)
plus an oracle spot check on a random subset of its environments.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL_M = 1e-4
MAX_BAD_FRACTION = 1e-4


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def rounded_workload(pkg, name, n):
    from paper_2602_03002_b200 import synth
    w = synth.config(name, n)
    bodies = [(nm, pkg.TriMesh(f32(m.vertices), m.faces, frame="body-local")) for nm, m in w.bodies]
    terrain = pkg.TriMesh(f32(w.terrain.mesh.vertices), w.terrain.mesh.faces)
    return w, bodies, terrain


def poses32(w, step, sl=None):
    p, q = w.poses(step, sl)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    return f32(p), f32(q)


def oracle_scene(oracle, bodies, terrain, cams):
    cd = [dict(width=c.width, height=c.height, hfov_deg=c.hfov_deg, vfov_deg=c.vfov_deg, d_max=c.d_max,
               mount_pos=c.mount.translation, mount_rot=c.mount.rotation,
               parent=c.parent_body) for c in cams]
    return oracle.OracleScene([(m.vertices, m.faces) for _, m in bodies],
                              (terrain.vertices, terrain.faces), cd)


def compare(out, ref):
    d = np.abs(np.asarray(out, np.float64) - np.asarray(ref, np.float64))
    bad = d > TOL_M
    return int(bad.sum()), float(d[~bad].max()) if (~bad).any() else 0.0, d.size


@pytest.mark.parametrize("name,n,camrand", [("cfg2", 96, True), ("cfg3", 48, False), ("cfg5", 6, False)])
def test_workload_vs_oracle(pkg, oracle, name, n, camrand):
    w, bodies, terrain = rounded_workload(pkg, name, n)
    scene = pkg.Scene(n, bodies=bodies, cameras=w.cameras, terrain=terrain)
    osc = oracle_scene(oracle, bodies, terrain, w.cameras)
    rand = None
    if camrand:
        p, q, f = pkg.sample_camera_offsets(pkg.CameraRandomization(seed=3), n, len(w.cameras))
        q = q / np.linalg.norm(q, axis=-1, keepdims=True)
        rand = (f32(p), f32(q), f32(f))
        scene.set_camera_randomization(*rand)
    for step in (0, 5):
        bp, bq = poses32(w, step)
        scene.set_body_poses(bp, bq)
        out = pkg.render(scene).data.cpu().numpy()
        ref = osc.render(bp, bq, rand_pos=None if rand is None else rand[0],
                         rand_rot=None if rand is None else rand[1],
                         fov_delta=None if rand is None else rand[2])
        nbad, maxd, npx = compare(out, ref)
        hit = float(np.mean(ref < np.asarray([c.d_max for c in w.cameras])[None, :, None, None]))
        print(f"{name} step {step}: bad {nbad}/{npx} ({nbad / npx:.2e}), max|d| {maxd:.2e}, hit {hit:.3f}")
        assert maxd <= TOL_M
        assert nbad <= MAX_BAD_FRACTION * npx + 1


def test_sensor_statistics_vs_oracle(pkg, oracle):
    """Noise/dropout on a rendered cfg2 frame: dropout mask bit-exact, residual stats within 1 %."""
    w, bodies, terrain = rounded_workload(pkg, "cfg2", 128)
    scene = pkg.Scene(128, bodies=bodies, cameras=w.cameras, terrain=terrain)
    scene.set_body_poses(*poses32(w, 1))
    cfg = pkg.SensorConfig(noise_scale=0.1, dropout_p=0.05, seed=11)
    clean = torch.empty(scene.frame_shape, device="cuda")
    obs = pkg.render_pipeline(scene, sensor=cfg, step=7, clean_out=clean).cpu().numpy()
    c = clean.cpu().numpy()
    ref = oracle.apply_noise_dropout(c, noise_scale=0.1, dropout_p=0.05, seed=11, d_max=scene.d_max_per_camera,
                                     step=7)
    dmax = np.float32(10.0)
    sub = c < 10.0 / (1 + 5 * 0.1)             # noise alone cannot reach d_max here
    drop_gpu, drop_ref = (obs == dmax) & sub, (ref == dmax) & sub
    assert np.array_equal(drop_gpu, drop_ref)
    rate_g, rate_r = drop_gpu.sum() / sub.sum(), drop_ref.sum() / sub.sum()
    assert abs(rate_g - rate_r) <= 0.01 * rate_r
    keep = sub & ~drop_gpu
    zg = (obs[keep].astype(np.float64) / c[keep] - 1) / 0.1
    zr = (ref[keep].astype(np.float64) / c[keep] - 1) / 0.1
    assert abs(zg.mean() - zr.mean()) < 0.01
    assert abs(zg.std() / zr.std() - 1) < 0.01
    ul = np.abs(obs.view(np.int32).astype(np.int64) - ref.view(np.int32).astype(np.int64))
    print(f"sensor: dropout {rate_g:.5f}, exact {np.mean(ul == 0):.7f}, max ulp {ul.max()}")
    assert ul.max() <= 1


def test_full_size_properties(pkg, oracle):
    """4096 envs x 2 cams (config 2): slice equivalence, determinism, bounds, oracle spot check."""
    n = 4096
    w, bodies, terrain = rounded_workload(pkg, "cfg2", n)
    scene = pkg.Scene(n, bodies=bodies, cameras=w.cameras, terrain=terrain)
    bp, bq = poses32(w, 2)
    scene.set_body_poses(bp, bq)
    cfg = pkg.SensorConfig(seed=1)
    a = pkg.render_pipeline(scene, sensor=cfg, step=2)
    b = pkg.render_pipeline(scene, sensor=cfg, step=2)
    assert torch.equal(a, b)
    assert float(a.min()) >= 1e-6 and float(a.max()) <= 10.0
    clean = pkg.render(scene).data
    assert torch.all(clean <= 10.0)
    # spot check 24 random envs against the oracle
    idx = np.sort(np.random.default_rng(0).choice(n, 24, replace=False))
    osc = oracle_scene(oracle, bodies, terrain, w.cameras)
    ref = osc.render(bp[idx], bq[idx])
    nbad, maxd, npx = compare(clean.cpu().numpy()[idx], ref)
    assert maxd <= TOL_M and nbad <= MAX_BAD_FRACTION * npx + 1
    # env-slice equivalence (sharding): envs [1000, 1064) rendered as their own scene
    sub = pkg.Scene(64, bodies=bodies, cameras=w.cameras, terrain=terrain, env_offset=1000)
    sub.set_body_poses(bp[1000:1064], bq[1000:1064])
    assert torch.equal(pkg.render_pipeline(sub, sensor=cfg, step=2), a[1000:1064])
