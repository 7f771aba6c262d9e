"""Host-side mirror of the reference API (no GPU): transforms, meshes, cameras,
counter RNG, per-env draws, FrameBuffer bookkeeping. Expectations follow the
reference's own unit tests (tests/test_transforms.py, test_camera.py,
test_mesh.py, test_rng.py, test_sensor.py) and the golden vectors."""

import math
import os

import numpy as np
import pytest

import casefile
from conftest import GOLDEN
from paper_2602_03002_b200 import rng
from paper_2602_03002_b200.camera import CameraModel, build_depth_ray, look_at_pose
from paper_2602_03002_b200.mesh import TriMesh, load_obj, make_box, make_icosphere, make_plane, merge_meshes, save_obj
from paper_2602_03002_b200.sensor import (CameraRandomization, FrameBuffer, SensorConfig, sample_camera_offsets,
                                          sample_latencies)
from paper_2602_03002_b200.transforms import (Ray, RigidPose, quat_conjugate, quat_from_axis_angle, quat_from_euler,
                                              quat_from_matrix, quat_identity, quat_mul, quat_normalize, quat_rotate,
                                              quat_to_matrix, world_to_body_ray)


def rq(g):
    q = g.standard_normal(4)
    return q / np.linalg.norm(q)


def test_quaternion_identities():
    g = np.random.default_rng(0)
    for _ in range(50):
        q1, q2, v = rq(g), rq(g), g.standard_normal(3)
        assert np.allclose(quat_rotate(q1, v), quat_to_matrix(q1) @ v, atol=1e-12)
        assert np.allclose(quat_rotate(quat_mul(q1, q2), v), quat_rotate(q1, quat_rotate(q2, v)), atol=1e-12)
        assert np.allclose(quat_rotate(quat_conjugate(q1), quat_rotate(q1, v)), v, atol=1e-12)
        m = quat_to_matrix(q1)
        q = quat_from_matrix(m)
        assert np.allclose(quat_to_matrix(q), m, atol=1e-12)
    with pytest.raises(ValueError):
        quat_normalize(np.zeros(4))
    with pytest.raises(ValueError):
        quat_normalize(np.ones(3))


def test_euler_order_is_z_y_x():
    r, p, y = 0.3, -0.2, 0.9
    q = quat_from_euler(r, p, y)
    ref = quat_mul(quat_from_axis_angle([0, 0, 1], y), quat_mul(quat_from_axis_angle([0, 1, 0], p),
                                                                 quat_from_axis_angle([1, 0, 0], r)))
    assert np.allclose(q, ref)


def test_pose_compose_and_body_ray():
    g = np.random.default_rng(1)
    a = RigidPose(g.standard_normal(3), rq(g))
    b = RigidPose(g.standard_normal(3), rq(g))
    p = g.standard_normal(3)
    assert np.allclose(a.compose(b).apply(p), a.apply(b.apply(p)))
    assert np.allclose(a.inverse().apply(a.apply(p)), p)
    ray = Ray(np.array([0.0, 0.0, 2.0]), np.array([0.1, 0.0, -1.0]), 1.3)
    br = world_to_body_ray(ray, a)
    t = 0.7
    assert np.allclose(a.apply(br.origin + t * br.direction), ray.origin + t * ray.direction)
    assert br.scale == ray.scale


def test_camera_intrinsics_and_grid():
    cam = CameraModel(width=48, height=27, hfov_deg=87.0, vfov_deg=58.0)
    assert cam.fx == pytest.approx(24 / math.tan(math.radians(87) / 2))
    assert cam.cx == 24.0 and cam.cy == 13.5
    assert np.allclose(np.linalg.inv(cam.k_matrix()), cam.k_inv(), atol=1e-12)
    c9 = CameraModel(width=9, height=7, hfov_deg=90.0, vfov_deg=70.0)
    d, s = c9.ray_grid()
    assert np.allclose(d[3, 4], [0, 0, 1]) and s[3, 4] == pytest.approx(1.0)
    assert np.allclose(s, np.linalg.norm(d, axis=-1))
    assert d[3, 8, 0] > 0 and d[6, 4, 1] > 0
    with pytest.raises(ValueError):
        CameraModel(width=0, height=1, hfov_deg=60, vfov_deg=60)
    with pytest.raises(ValueError):
        CameraModel(width=4, height=4, hfov_deg=180, vfov_deg=60)


def test_look_at_conventions():
    pose = look_at_pose([0.0, 0.0, 1.0], [0.0, 0.0, 0.0])
    assert np.allclose(quat_rotate(pose.rotation, [0, 0, 1]), [0, 0, -1])     # +z forward
    pose2 = look_at_pose([0, 0, 0], [1.0, 0, 0])
    assert np.allclose(quat_rotate(pose2.rotation, [0, 1, 0]), [0, 0, -1])    # +y down
    r = build_depth_ray(pose, CameraModel(width=9, height=7, hfov_deg=70, vfov_deg=55).k_inv(), 4, 3)
    assert np.allclose(r.direction, [0, 0, -1]) and r.scale == pytest.approx(1.0)


def test_mesh_primitives_and_degenerates(tmp_path):
    m = TriMesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [2, 0, 0.]]), np.array([[0, 1, 2], [0, 1, 3]]))
    assert m.num_faces == 1 and m.dropped_degenerate == 1
    b = make_box(size=(2, 4, 6), center=(1, 0, -1))
    lo, hi = b.bounds()
    assert b.num_faces == 12 and np.allclose(lo, [0, -2, -4]) and np.allclose(hi, [2, 2, 2])
    s = make_icosphere(2.0, subdivisions=2)
    assert s.num_faces == 320 and np.allclose(np.linalg.norm(s.vertices, axis=1), 2.0)
    assert make_plane(size=(4, 2), center=(0, 0, 0.5)).num_faces == 2
    mm = merge_meshes([b, s])
    assert mm.num_faces == 332 and mm.faces.max() == mm.num_vertices - 1
    save_obj(tmp_path / "b.obj", b)
    bb = load_obj(tmp_path / "b.obj")
    assert np.allclose(bb.vertices, b.vertices) and np.array_equal(bb.faces, b.faces)
    with pytest.raises(ValueError):
        TriMesh(np.zeros((3, 3)), np.array([[0, 1, 5]]))


@pytest.fixture(scope="module")
def sens():
    return casefile.load(os.path.join(GOLDEN, "sensor.npz"))


def test_host_rng_bit_exact_with_reference(sens):
    names = ["sensor", "sensor", "latency", "a-much-longer-stream-name"]
    for seed, name, val in zip(sens["keys_seed"], names, sens["keys_val"]):
        assert int(rng.stream_key(int(seed), name)) == int(val)
    key = rng.stream_key(5, "demo")
    c = sens["rng_counters"]
    assert np.array_equal(rng.uniform(key, c[:, 0], c[:, 1]), sens["rng_uniform"])
    assert np.array_equal(rng.normal(key, c[:, 0], c[:, 1]), sens["rng_normal"])


def test_rng_slicing_commutes_and_streams_differ():
    key = rng.stream_key(9, "batch")
    env, pix = np.arange(64).reshape(-1, 1), np.arange(33).reshape(1, -1)
    assert np.array_equal(rng.normal(key, env, pix)[10:20, 4:9], rng.normal(key, env[10:20], pix[:, 4:9]))
    assert rng.uniform(rng.stream_key(0, "a"), 0) != rng.uniform(rng.stream_key(0, "b"), 0)
    assert rng.uniform(key, 1, 2) != rng.uniform(key, 2, 1)


def test_per_env_draws_match_reference(sens):
    assert np.array_equal(sample_latencies(SensorConfig(max_delay=0.1, seed=5), 100, episode=2),
                          sens["latencies_ep2"])
    p, q, f = sample_camera_offsets(CameraRandomization(seed=4), 16, 2, episode=1)
    assert np.array_equal(p, sens["camoff_pos"])
    assert np.allclose(q, sens["camoff_rot"], rtol=0, atol=1e-15)
    assert np.array_equal(f, sens["camoff_fov"])


def test_sensor_config_validation():
    with pytest.raises(ValueError):
        SensorConfig(noise_scale=-1)
    with pytest.raises(ValueError):
        SensorConfig(dropout_p=1.0)
    with pytest.raises(ValueError):
        CameraRandomization(fov_deg=-1)


def test_frame_buffer_host_bookkeeping():
    """Slot assignment / eviction of the HBM ring follows FrameBuffer (sensor.py:122-131)."""
    buf = FrameBuffer(capacity=3)
    slots = [buf._reserve(float(i)) for i in range(6)]
    assert slots == [0, 1, 2, 0, 1, 2]
    assert buf._times == [3.0, 4.0, 5.0] and len(buf) == 3
    with pytest.raises(ValueError, match="increasing"):
        buf._reserve(5.0)
    with pytest.raises(ValueError):
        FrameBuffer(capacity=0)


def test_rsm_host_side(sens):
    from paper_2602_03002_b200.perception import RSM_MODES, RsmConfig, rsm_mask_columns, rsm_sample_modes
    assert RSM_MODES == ("none", "small", "large")
    cfg = RsmConfig()
    assert [rsm_mask_columns(cfg, m, 48) for m in (0, 1, 2)] == [0, 6, 12]
    assert rsm_mask_columns(cfg, 1, 30) == 3
    assert np.array_equal(rsm_sample_modes(RsmConfig(seed=3), "stepping_stones", 64, 2, episode=1),
                          sens["rsm_modes_stones"])
    modes = rsm_sample_modes(RsmConfig(seed=0), "stepping_stones", 100_000, 1)
    freqs = np.bincount(modes.ravel(), minlength=3) / modes.size
    assert np.all(np.abs(freqs - np.array([0.6, 0.3, 0.1])) < 0.01)
    with pytest.raises(KeyError):
        cfg.probs_for("volcano")
    with pytest.raises(ValueError):
        RsmConfig(probs={"flat": (0.5, 0.5, 0.5)})


def test_benchmark_terrains_are_the_reference_generators():
    """synth.py's config 1/2/3 terrains reproduce the reference generator's meshes
    (terrain.py:278-360) bit for bit (stairs tiles up to their placement shift)."""
    import hashlib
    from paper_2602_03002_b200 import synth
    ref = np.load(os.path.join(GOLDEN, "terrain.npz"))

    def check(name, mesh):
        v = np.array(mesh.vertices, np.float64)
        assert [len(v), len(mesh.faces)] == ref[name + "_shape"].tolist()
        assert hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() == str(ref[name + "_vsha"])
        assert hashlib.sha256(np.ascontiguousarray(mesh.faces, np.int64).tobytes()).hexdigest() == \
            str(ref[name + "_fsha"])

    check("cfg1_stairs", synth.stairs_terrain().mesh)
    check("tile_slope_pyramid", synth.tile_field(["slope_pyramid"]).mesh)
    check("tile_stairs_up", synth.tile_field(["stairs_up"]).mesh)       # fixture: reference x - 1.08
    check("tile_stairs_down", synth.tile_field(["stairs_down"]).mesh)
    check("cfg3_stones", synth.stepping_stones().mesh)
