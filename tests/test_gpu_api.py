"""Reference API behaviour on the GPU path: validation errors (reference
tests/test_render.py:214-238, scene.py:159-250), DepthFrame/depth_to_z
(test_render.py:241-248), geometry never rebuilt on pose updates
(test_render.py:251-265), backend/threads selection (kernels/__init__.py:38-75)
and the caller-supplied output contract (scene.py:344-347)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def down_camera(md, **kw):
    args = dict(width=9, height=7, hfov_deg=70.0, vfov_deg=55.0, d_max=5.0,
                mount=md.look_at_pose([0.0, 0.0, 1.0], [0.0, 0.0, 0.0]))
    args.update(kw)
    return md.CameraModel(**args)


def test_scene_validation(pkg):
    cam = down_camera(pkg)
    with pytest.raises(ValueError):
        pkg.Scene(0, cameras=[cam])
    with pytest.raises(ValueError):
        pkg.Scene(1, cameras=[])
    with pytest.raises(ValueError):
        pkg.Scene(1, cameras=[cam, pkg.CameraModel(width=4, height=4, hfov_deg=60.0, vfov_deg=60.0)])
    with pytest.raises(ValueError):
        pkg.Scene(1, cameras=[down_camera(pkg, parent_body=0)])


def test_set_body_poses_validation(pkg):
    scene = pkg.Scene(2, bodies=[("b", pkg.make_box(size=(0.1, 0.1, 0.1)))], cameras=[down_camera(pkg)])
    with pytest.raises(ValueError):
        scene.set_body_poses(np.zeros((2, 2, 3)), np.zeros((2, 2, 4)))
    with pytest.raises(ValueError):
        scene.set_body_poses(np.zeros((2, 1, 3)), np.zeros((2, 1, 4)))          # zero quaternion
    with pytest.raises(ValueError):
        scene.set_body_poses(np.full((2, 1, 3), np.nan), np.tile([1.0, 0, 0, 0], (2, 1, 1)))
    with pytest.raises(ValueError):
        scene.set_body_pose(5, 0, pkg.RigidPose.identity())
    with pytest.raises(ValueError):
        scene.set_camera_randomization(np.zeros((2, 1, 3)), np.zeros((2, 2, 4)), np.zeros((2, 1)))
    # unnormalised quaternions are accepted and normalised (scene.py:246-250)
    scene.set_body_poses(np.zeros((2, 1, 3)), np.tile([3.0, 0, 0, 0], (2, 1, 1)))
    a = pkg.render(scene).data
    scene.set_body_poses(np.zeros((2, 1, 3)), np.tile([1.0, 0, 0, 0], (2, 1, 1)))
    assert torch.equal(a, pkg.render(scene).data)


def test_depth_frame_and_z_conversion(pkg):
    scene = pkg.Scene(1, cameras=[down_camera(pkg)], terrain=pkg.make_plane(size=(10.0, 10.0)))
    frame = pkg.render(scene, timestamp=2.5)
    assert frame.timestamp == 2.5 and frame.shape == (1, 1, 7, 9)
    _, scales = scene.cameras[0].ray_grid()
    z = pkg.depth_to_z(frame.data[0, 0].cpu().numpy(), scales)
    assert np.allclose(z, 1.0, atol=1e-5)
    zt = pkg.depth_to_z(frame.data[0, 0], scales)
    assert torch.allclose(zt.cpu(), torch.ones(7, 9, dtype=torch.float32), atol=1e-5)


def test_geometry_not_rebuilt_on_pose_change(pkg):
    rng = np.random.default_rng(107)
    scene = pkg.Scene(3, bodies=[("a", pkg.make_icosphere(0.2, 1)), ("b", pkg.make_box(size=(0.3, 0.2, 0.1)))],
                      cameras=[down_camera(pkg)], terrain=pkg.make_plane(size=(6.0, 6.0)))
    stats = dict(scene.geometry_stats)
    ctx = scene._ctx
    before = pkg.render(scene).data.clone()
    scene.set_body_poses(rng.uniform(-1, 1, size=(3, 2, 3)) * [1, 1, 0.2] + [0, 0, 0.5],
                         rng.standard_normal((3, 2, 4)))
    after = pkg.render(scene).data
    assert scene._ctx is ctx and dict(scene.geometry_stats) == stats
    assert not torch.equal(before, after)


def test_backend_threads_and_out_contract(pkg):
    scene = pkg.Scene(2, cameras=[down_camera(pkg)], terrain=pkg.make_plane(size=(10.0, 10.0)))
    with pytest.raises(ValueError):
        pkg.render(scene, backend="numba")
    with pytest.raises(ValueError):
        pkg.render(scene, threads="four")
    ref = pkg.render(scene, backend="cuda", threads=4).data
    out = torch.empty(scene.frame_shape, device="cuda")
    got = pkg.render(scene, out=out).data
    assert got.data_ptr() == out.data_ptr() and torch.equal(out, ref)
    for bad in (torch.empty((2, 1, 7, 8), device="cuda"), torch.empty(scene.frame_shape),
                torch.empty(scene.frame_shape, device="cuda", dtype=torch.float64),
                torch.empty((2, 1, 9, 7), device="cuda").transpose(2, 3)):
        with pytest.raises(ValueError):
            pkg.render(scene, out=bad)


def test_naive_baseline_matches_render(pkg):
    """render_naive_baseline (scene.py:351-378: world-space link BVHs rebuilt per env)
    equals render() to float32 precision (test_acceptance.py criterion 2's premise)."""
    rng = np.random.default_rng(21)
    cams = [pkg.CameraModel(width=24, height=16, hfov_deg=80.0, vfov_deg=60.0, d_max=6.0,
                            mount=pkg.look_at_pose([2.5 * np.cos(a), 2.5 * np.sin(a), 1.5], [0.0, 0.0, 0.3]))
            for a in (0.3, 2.4)]
    scene = pkg.Scene(3, bodies=[("a", pkg.make_icosphere(0.3, 1)), ("b", pkg.make_box(size=(0.5, 0.3, 0.2)))],
                      cameras=cams, terrain=pkg.make_plane(size=(8.0, 8.0)))
    scene.set_body_poses(rng.uniform(-0.8, 0.8, size=(3, 2, 3)) * [1, 1, 0.3] + [0, 0, 0.4],
                         rng.standard_normal((3, 2, 4)))
    scene.set_camera_randomization(*pkg.sample_camera_offsets(pkg.CameraRandomization(seed=2), 3, 2))
    fast = pkg.render(scene, timestamp=1.5)
    naive = pkg.render_naive_baseline(scene, timestamp=1.5)
    assert naive.timestamp == 1.5 and naive.shape == fast.shape
    d = torch.abs(naive.data - fast.data)
    assert float(d.max()) < 1e-4 and int((d > 1e-5).sum()) <= 2


def test_optimized_beats_naive_refit(pkg):
    """test_acceptance.py:106-126 (criterion 2): the no-refit render is >= 2x the
    refit baseline on 32 envs x 2 cams with 8 bodies (here by orders of magnitude)."""
    import time
    rng = np.random.default_rng(5)
    bodies = [(f"b{k}", pkg.make_icosphere(0.15, 2)) for k in range(8)]
    cams = [pkg.CameraModel(width=64, height=36, hfov_deg=80.0, vfov_deg=55.0, d_max=6.0,
                            mount=pkg.look_at_pose([3.0 * np.cos(a), 3.0 * np.sin(a), 1.2], [0.0, 0.0, 0.3]))
            for a in (0.0, 3.0)]
    scene = pkg.Scene(32, bodies=bodies, cameras=cams, terrain=pkg.make_plane(size=(8.0, 8.0)))
    scene.set_body_poses(rng.uniform(-1, 1, size=(32, 8, 3)) * [1, 1, 0.3] + [0, 0, 0.5],
                         rng.standard_normal((32, 8, 4)))
    pkg.render(scene)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        pkg.render(scene)
    torch.cuda.synchronize()
    fast = (time.perf_counter() - t0) / 5
    t0 = time.perf_counter()
    naive = pkg.render_naive_baseline(scene)
    torch.cuda.synchronize()
    slow = time.perf_counter() - t0
    assert torch.max(torch.abs(naive.data - pkg.render(scene).data)).item() < 1e-4
    print(f"optimized {fast * 1e3:.2f} ms, naive refit {slow * 1e3:.1f} ms ({slow / fast:.0f}x)")
    assert slow >= 2.0 * fast
