"""Parity of the CUDA path (libmdrt.so through the package API) with the reference.

Tolerances (BASELINE.json north star): with noise/dropout off, per-pixel range
within 1e-4 m; pixels outside that band (hit/miss flips on grazing edges or a
different surface hit at a silhouette) are counted and must stay <= 0.01 % of
all pixels; misses read exactly float32(d_max); latency indexing bit-exact;
dropout masks bit-exact (same counter RNG); noisy values within 1 float32 ulp.
"""

import glob
import os

import numpy as np
import pytest
import torch

import casefile
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

TOL_M = 1e-4
MAX_BAD_FRACTION = 1e-4
RENDER_CASES = sorted(glob.glob(os.path.join(GOLDEN, "render_*.npz")))


def compare(out, ref, tol=TOL_M):
    out = np.asarray(out, np.float64)
    ref = np.asarray(ref, np.float64)
    d = np.abs(out - ref)
    bad = d > tol
    good = ~bad
    return int(bad.sum()), float(d[good].max()) if good.any() else 0.0, out.size


@pytest.fixture(scope="module")
def golden_results(pkg):
    res = {}
    for path in RENDER_CASES:
        case = casefile.load(path)
        scene = casefile.build_scene(case, pkg)
        out = pkg.render(scene, early_termination=bool(case["early"])).data
        res[os.path.basename(path)] = (case, out.cpu().numpy())
    return res


@pytest.mark.parametrize("path", RENDER_CASES, ids=lambda p: os.path.basename(p)[7:-4])
def test_render_matches_reference_golden(golden_results, path):
    case, out = golden_results[os.path.basename(path)]
    ref = case["out"]
    assert out.shape == ref.shape and out.dtype == np.float32
    nbad, maxd, n = compare(out, ref)
    print(f"{os.path.basename(path)}: bad {nbad}/{n}, max |d| on good {maxd:.3e}")
    assert maxd <= TOL_M
    assert nbad <= max(1, int(MAX_BAD_FRACTION * n))
    # misses are exactly d_max (scene.py:336-338)
    dmax = case["cam_dmax"].astype(np.float32)[None, :, None, None]
    miss_ref = ref == dmax
    assert np.all(out[miss_ref & (np.abs(out - ref) <= TOL_M)] == np.broadcast_to(dmax, out.shape)[
        miss_ref & (np.abs(out - ref) <= TOL_M)])


def test_render_suite_bad_fraction(golden_results):
    tot_bad = tot = 0
    for case, out in golden_results.values():
        b, _, n = compare(out, case["out"])
        tot_bad += b
        tot += n
    print(f"golden suite: {tot_bad} / {tot} pixels outside 1e-4 m")
    assert tot_bad <= MAX_BAD_FRACTION * tot


def test_flat_ground_analytic(pkg):
    cam = pkg.CameraModel(width=9, height=7, hfov_deg=70.0, vfov_deg=55.0, d_max=10.0,
                          mount=pkg.look_at_pose([0.0, 0.0, 1.0], [0.0, 0.0, 0.0]))
    scene = pkg.Scene(1, cameras=[cam], terrain=pkg.make_plane(size=(20.0, 20.0)))
    out = pkg.render(scene).data.cpu().numpy()[0, 0].astype(np.float64)
    assert abs(out[3, 4] - 1.0) < 1e-6
    _, scales = cam.ray_grid()
    assert np.max(np.abs(out - scales)) < 1e-5


def test_miss_and_far_clamp(pkg):
    cam = pkg.CameraModel(width=9, height=7, hfov_deg=70.0, vfov_deg=55.0, d_max=3.5,
                          mount=pkg.look_at_pose([0.0, 0.0, 1.0], [0.0, 0.0, 0.0]))
    scene = pkg.Scene(1, cameras=[cam])
    assert torch.all(pkg.render(scene).data == np.float32(3.5))
    cam2 = pkg.CameraModel(width=9, height=7, hfov_deg=70.0, vfov_deg=55.0, d_max=0.25,
                           mount=pkg.look_at_pose([0.0, 0.0, 1.0], [0.0, 0.0, 0.0]))
    scene2 = pkg.Scene(1, cameras=[cam2], terrain=pkg.make_plane(size=(10.0, 10.0)))
    assert torch.all(pkg.render(scene2).data == np.float32(0.25))


def _case_scene(pkg, name):
    case = casefile.load(os.path.join(GOLDEN, name))
    return case, casefile.build_scene(case, pkg)


def test_early_termination_and_determinism(pkg):
    case, scene = _case_scene(pkg, "render_rand5.npz")
    a = pkg.render(scene, early_termination=True).data.clone()
    b = pkg.render(scene, early_termination=False).data.clone()
    c = pkg.render(scene, early_termination=True).data.clone()
    assert torch.max(torch.abs(a - b)).item() < 1e-7
    assert torch.equal(a, c)


def test_body_permutation_invariant(pkg):
    case = casefile.load(os.path.join(GOLDEN, "render_rand4.npz"))
    scene = casefile.build_scene(case, pkg)
    base = pkg.render(scene).data.clone()
    nb = int(case["num_bodies"])
    perm = np.random.default_rng(3).permutation(nb)
    p = dict(case)
    for i, src in enumerate(perm):
        p[f"body{i}_v"], p[f"body{i}_f"] = case[f"body{src}_v"], case[f"body{src}_f"]
    p["body_pos"], p["body_rot"] = case["body_pos"][:, perm], case["body_rot"][:, perm]
    out = pkg.render(casefile.build_scene(p, pkg)).data
    assert torch.max(torch.abs(out - base)).item() < 1e-7


def test_cull_is_exact(pkg):
    """Per-view link culling never changes a pixel (MDRT_NO_CULL A/B)."""
    from paper_2602_03002_b200 import _native
    case, scene = _case_scene(pkg, "render_cfg2_slice.npz")
    a = pkg.render(scene).data.clone()
    out = torch.empty_like(a)
    args = scene._step_args(out, True)
    args.flags |= _native.NO_CULL
    scene._launch(args)
    assert torch.equal(a, out)


def test_counters_do_not_change_output(pkg):
    case, scene = _case_scene(pkg, "render_cfg1.npz")
    a = pkg.render(scene).data.clone()
    ctr = torch.zeros(2, dtype=torch.int64, device=scene.device)
    b = pkg.render(scene, counters=ctr).data
    assert torch.equal(a, b)
    nodes, tris = ctr.tolist()
    assert nodes > 0 and tris > 0


def test_env_offset_slicing_is_bit_identical(pkg):
    """Env-sliced scenes (multi-GPU sharding) reproduce the full render + sensor stream."""
    case = casefile.load(os.path.join(GOLDEN, "render_cfg2_slice.npz"))
    full = casefile.build_scene(case, pkg)
    cfg = pkg.SensorConfig(seed=9)
    ref = pkg.render_pipeline(full, sensor=cfg, step=4).cpu()
    n = int(case["num_envs"])
    parts = []
    for lo, hi in ((0, 3), (3, n)):
        sub = dict(case)
        sub["body_pos"], sub["body_rot"] = case["body_pos"][lo:hi], case["body_rot"][lo:hi]
        sub["num_envs"] = np.array(hi - lo)
        s = casefile.build_scene(sub, pkg)
        s.env_offset = lo
        parts.append(pkg.render_pipeline(s, sensor=cfg, step=4).cpu())
    assert torch.equal(torch.cat(parts), ref)


@pytest.fixture(scope="module")
def sens():
    return casefile.load(os.path.join(GOLDEN, "sensor.npz"))


def _ulps(a, b):
    return np.abs(a.view(np.int32).astype(np.int64) - b.view(np.int32).astype(np.int64))


def test_noise_dropout_matches_reference(pkg, sens):
    cfg = pkg.SensorConfig(noise_scale=0.1, dropout_p=0.05, seed=7)
    d = torch.from_numpy(sens["depth"]).cuda()
    out = pkg.apply_noise_dropout(d, cfg, d_max=sens["d_max"], step=3).cpu().numpy()
    ref = sens["out_s3"]
    u = _ulps(out, ref)
    print(f"noise: exact {np.mean(u == 0):.6f}, max ulp {u.max()}")
    assert u.max() <= 1 and np.mean(u == 0) > 0.999
    cfg2 = pkg.SensorConfig(noise_scale=0.2, dropout_p=0.3, dropout_fill=0.25, seed=2)
    out2 = pkg.apply_noise_dropout(sens["depth"], cfg2, d_max=sens["d_max"], step=0)   # numpy in/out
    assert isinstance(out2, np.ndarray)
    ref2 = sens["out_fill_s0"]
    assert np.array_equal(out2 == np.float32(0.25), ref2 == np.float32(0.25))   # dropout mask exact
    assert _ulps(out2, ref2).max() <= 1


def test_noise_statistics(pkg):
    """test_acceptance.py:306-316: std in [0.19, 0.21] m at 2.0 m, dropout in [0.045, 0.055]."""
    cfg = pkg.SensorConfig(noise_scale=0.1, dropout_p=0.05, seed=0)
    d = torch.full((1, 1, 400, 256), 2.0, device="cuda")
    out = pkg.apply_noise_dropout(d, cfg, d_max=10.0).cpu().numpy()
    dropped = out == np.float32(10.0)
    assert 0.045 <= dropped.mean() <= 0.055
    assert 0.19 <= out[~dropped].astype(np.float64).std() <= 0.21


def test_latency_buffer_matches_reference(pkg, sens):
    dt = float(sens["latency_dt"])
    buf = pkg.FrameBuffer(capacity=int(sens["latency_capacity"]))
    delays = sens["delays"]
    n = len(delays)
    for s, ref in enumerate(sens["latency_sel"]):
        buf.push(pkg.DepthFrame(torch.full((n, 1, 1, 1), float(s), device="cuda"), s * dt))
        got = buf.fetch_delayed_batch(s * dt, delays)[:, 0, 0, 0].cpu().numpy().astype(np.int64)
        assert np.array_equal(got, ref), f"step {s}"


def test_frame_buffer_semantics(pkg):
    buf = pkg.FrameBuffer(capacity=3)
    for i in range(6):
        buf.push(pkg.DepthFrame(torch.full((1, 1, 2, 2), float(i), device="cuda"), float(i)))
    assert len(buf) == 3
    assert torch.all(buf.fetch_delayed(10.0, 100.0).data == 3.0)
    with pytest.raises(ValueError, match="increasing"):
        buf.push(pkg.DepthFrame(torch.zeros((1, 1, 2, 2), device="cuda"), 5.0))
    with pytest.raises(LookupError):
        pkg.FrameBuffer().fetch_delayed(0.0, 0.0)


def test_downsample_matches_reference(pkg, sens):
    out = pkg.downsample_min(torch.from_numpy(sens["ds_in"]).cuda(), 5).cpu().numpy()
    assert np.array_equal(out, sens["ds_out"])


def test_fused_pipeline_equals_unfused_sequence(pkg):
    """render -> apply_noise_dropout -> push -> fetch_delayed_batch == one fused step, bitwise."""
    case, scene = _case_scene(pkg, "render_cfg2_slice.npz")
    n = scene.num_envs
    cfg = pkg.SensorConfig(seed=3)
    delays = np.array([0.0, 0.02, 0.05, 0.1, 0.013, 0.07, 0.04, 0.2])[:n]
    fused_buf, ref_buf = pkg.FrameBuffer(capacity=4), pkg.FrameBuffer(capacity=4)
    rng = np.random.default_rng(0)
    for s in range(7):
        pos = case["body_pos"] + rng.normal(0, 0.01, case["body_pos"].shape)
        scene.set_body_poses(pos.astype(np.float32), case["body_rot"])
        ts = s * 0.02
        clean = torch.empty(scene.frame_shape, device="cuda")
        obs = pkg.render_pipeline(scene, sensor=cfg, step=s, frame_buffer=fused_buf, timestamp=ts,
                                  delays=delays, clean_out=clean)
        frame = pkg.render(scene, timestamp=ts)
        assert torch.equal(frame.data, clean)
        noisy = pkg.apply_noise_dropout(frame.data, cfg, d_max=scene.d_max_per_camera, step=s)
        ref_buf.push(pkg.DepthFrame(noisy, ts))
        ref = ref_buf.fetch_delayed_batch(ts, delays)
        assert torch.equal(obs, ref), f"step {s}"


def test_seam_render_batch_matches_golden(pkg, oracle):
    """kernels.get_render_fn('cuda') with the reference's render_batch arguments."""
    from paper_2602_03002_b200 import kernels

    class Flat:   # FlatGeometry-shaped (scene.py:49-78)
        pass

    for name in ("render_rand_camrand.npz", "render_parented.npz", "render_cfg1.npz"):
        case = casefile.load(os.path.join(GOLDEN, name))
        bv = []
        for v, f in casefile.bodies(case):
            bv.append(oracle.build_bvh(v[f]))
        t = casefile.terrain(case)
        fl = oracle.flatten(bv, None if t is None else oracle.build_bvh(t[0][t[1]]))
        flat = Flat()
        for k, v in fl.items():
            setattr(flat, k, v)
        offs = [0]
        for b in bv:
            offs.append(offs[-1] + len(b["tri_v0"]))
        flat.body_tri_offsets = np.array(offs)
        r = casefile.rand(case)
        n = int(case["num_envs"])
        bp, bq = case["body_pos"], case["body_rot"]
        cam_pos, cam_rot = oracle.camera_world_poses(casefile.cameras_dicts(case), bp, bq,
                                                     None if r is None else r[0],
                                                     None if r is None else r[1])
        dirs, scale = oracle.ray_grids(casefile.cameras_dicts(case), n, None if r is None else r[2])
        out = np.empty(case["out"].shape, np.float32)
        _, fn = kernels.get_render_fn("cuda")
        fn(flat, bp, bq, cam_pos, cam_rot, dirs, scale, case["cam_dmax"], True, out, 4)
        nbad, maxd, npx = compare(out, case["out"])
        assert maxd <= TOL_M and nbad <= max(1, int(MAX_BAD_FRACTION * npx)), (name, nbad, maxd)


def test_backend_registry(pkg):
    from paper_2602_03002_b200 import kernels
    assert kernels.BACKENDS == ("cuda",)
    with pytest.raises(ValueError):
        kernels.get_render_fn("numba")
    case, scene = _case_scene(pkg, "render_flat.npz")
    with pytest.raises(ValueError):
        pkg.render(scene, backend="numpy")


def test_async_host_delivery(pkg):
    """host_out: pinned copies on the scene's copy stream match the device observations."""
    case, scene = _case_scene(pkg, "render_cfg2_slice.npz")
    cfg = pkg.SensorConfig(seed=4)
    outs = [torch.empty(scene.frame_shape, device="cuda") for _ in range(2)]
    hosts = [torch.empty(scene.frame_shape).pin_memory() for _ in range(2)]
    expect = []
    for s in range(5):
        obs = pkg.render_pipeline(scene, sensor=cfg, step=s, out=outs[s % 2], host_out=hosts[s % 2])
        expect.append(obs.clone())
        if s >= 1:
            scene.host_sync()
            assert torch.equal(hosts[(s - 1) % 2], expect[s - 1].cpu()) or torch.equal(hosts[s % 2], expect[s].cpu())
    scene.host_sync()
    torch.cuda.synchronize()
    assert torch.equal(hosts[4 % 2], expect[4].cpu())
    assert torch.equal(hosts[3 % 2], expect[3].cpu())


def test_captured_step_matches_eager(pkg):
    """CUDA-graph replay (device step state) == eager render_pipeline, bitwise, incl. latency ring."""
    from paper_2602_03002_b200.pipeline import CapturedStep
    case = casefile.load(os.path.join(GOLDEN, "render_cfg2_slice.npz"))
    s_eager, s_graph = casefile.build_scene(case, pkg), casefile.build_scene(case, pkg)
    cfg = pkg.SensorConfig(seed=6)
    n = s_eager.num_envs
    delays = np.array([0.0, 0.02, 0.05, 0.1, 0.013, 0.07, 0.04, 0.2])[:n]
    dt = 0.02
    fb_e, fb_g = pkg.FrameBuffer(capacity=4), pkg.FrameBuffer(capacity=4)
    cap = CapturedStep(s_graph, sensor=cfg, frame_buffer=fb_g, delays=delays, dt=dt, first_step=3)
    rng = np.random.default_rng(1)
    for k in range(3, 10):
        pos = (case["body_pos"] + rng.normal(0, 0.01, case["body_pos"].shape)).astype(np.float32)
        s_eager.set_body_poses(pos, case["body_rot"])
        s_graph.body_positions.copy_(torch.from_numpy(pos))
        ref = pkg.render_pipeline(s_eager, sensor=cfg, step=k, frame_buffer=fb_e, timestamp=k * dt, delays=delays)
        got = cap.replay()
        assert torch.equal(got, ref), f"step {k}"
        assert fb_g._times == fb_e._times and fb_g._slots == fb_e._slots
    st = cap.device_state()
    assert st["next_step"] == 10 and st["times"] == fb_e._times and st["order"] == fb_e._slots


def test_pinned_pose_upload_overlaps_and_matches(pkg):
    """Pinned host poses go through the scene's upload stream + staging double buffer;
    results equal the synchronous path, also when the host reuses two pinned buffers
    and when a captured graph reads the poses."""
    from paper_2602_03002_b200.pipeline import CapturedStep
    case = casefile.load(os.path.join(GOLDEN, "render_cfg2_slice.npz"))
    s_pin, s_ref, s_graph = (casefile.build_scene(case, pkg) for _ in range(3))
    cfg = pkg.SensorConfig(seed=3)
    cap = CapturedStep(s_graph, sensor=cfg, first_step=0)
    rng = np.random.default_rng(4)
    host = [(torch.empty(case["body_pos"].shape, dtype=torch.float32).pin_memory(),
             torch.empty(case["body_rot"].shape, dtype=torch.float32).pin_memory()) for _ in range(2)]
    outs = [torch.empty(s_pin.frame_shape, device="cuda") for _ in range(2)]
    got, want = [], []
    for k in range(6):
        pos = (case["body_pos"] + rng.normal(0, 0.02, case["body_pos"].shape)).astype(np.float32)
        hp, hq = host[k % 2]
        if k >= 2:
            torch.cuda.current_stream().synchronize()   # host buffer k%2 was consumed two steps ago
        hp.copy_(torch.from_numpy(pos))
        hq.copy_(torch.from_numpy(case["body_rot"].astype(np.float32)))
        s_pin.set_body_poses(hp, hq, validate=False)
        got.append(pkg.render_pipeline(s_pin, sensor=cfg, step=k, out=outs[k % 2]).clone())
        s_ref.set_body_poses(pos, case["body_rot"])
        want.append(pkg.render_pipeline(s_ref, sensor=cfg, step=k))
        s_graph.set_body_poses(hp, hq, validate=False)
        assert torch.equal(cap.replay(), want[-1]), f"graph step {k}"
    for k in range(6):
        assert torch.equal(got[k], want[k]), f"step {k}"


def test_rsm_matches_reference(pkg, sens):
    """Random side masking (perception.py:150-202): modes and fills bit-exact vs reference goldens."""
    cfg = pkg.RsmConfig(seed=3)
    assert np.array_equal(pkg.rsm_sample_modes(cfg, "stepping_stones", 64, 2, episode=1), sens["rsm_modes_stones"])
    out = pkg.rsm_apply(torch.from_numpy(sens["rsm_depth"]).cuda(), sens["rsm_modes"], cfg, d_max=[6.0, 8.0],
                        step=5).cpu().numpy()
    assert np.array_equal(out, sens["rsm_out_s5"])
    cfg2 = pkg.RsmConfig(seed=4, fill_high=4.0, f_small=0.1, f_large=0.3)
    out2 = pkg.rsm_apply(sens["rsm_depth"], sens["rsm_modes"], cfg2, d_max=[6.0, 8.0], step=0)
    assert np.array_equal(out2, sens["rsm_out2_s0"])


def test_fused_rsm_equals_standalone(pkg):
    """render_pipeline(rsm=...) == rsm_apply(render_pipeline(...)), and the captured step agrees."""
    from paper_2602_03002_b200.pipeline import CapturedStep
    case, scene = _case_scene(pkg, "render_cfg2_slice.npz")
    sc2 = casefile.build_scene(case, pkg)
    n, c = scene.num_envs, scene.num_cameras
    sens_cfg = pkg.SensorConfig(seed=2)
    rsm = pkg.RsmConfig(seed=7)
    modes = pkg.rsm_sample_modes(rsm, "stairs_up", n, c, episode=0)
    cap = CapturedStep(sc2, sensor=sens_cfg, rsm=rsm, rsm_modes=modes, first_step=4)
    for s in range(4, 7):
        fused = pkg.render_pipeline(scene, sensor=sens_cfg, step=s, rsm=rsm, rsm_modes=modes).clone()
        plain = pkg.render_pipeline(scene, sensor=sens_cfg, step=s)
        ref = pkg.rsm_apply(plain, modes, rsm, d_max=scene.d_max_per_camera, step=s)
        assert torch.equal(fused, ref), f"step {s}"
        assert torch.equal(cap.replay(), ref), f"captured step {s}"


def test_fused_downsample_equals_standalone(pkg):
    """render_pipeline(ds_out=...) == downsample_min(obs) (sensor.py:85-100), bitwise, incl. graph replay."""
    from paper_2602_03002_b200.pipeline import CapturedStep
    cam = pkg.CameraModel(width=240, height=135, hfov_deg=87.0, vfov_deg=58.0, d_max=6.0,
                          mount=pkg.look_at_pose([0.0, 0.0, 1.2], [1.5, 0.3, 0.0]))
    xs = np.linspace(-4, 4, 41)
    gx, gy = np.meshgrid(xs, xs)
    gz = 0.2 * np.sin(2 * gx) * np.cos(3 * gy)
    a = (np.arange(40)[:, None] * 41 + np.arange(40)[None, :]).ravel()
    faces = np.concatenate([np.column_stack([a, a + 1, a + 42]), np.column_stack([a, a + 42, a + 41])])
    terrain = pkg.TriMesh(np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()]), faces)
    scene = pkg.Scene(3, cameras=[cam, cam], terrain=terrain)
    cfg = pkg.SensorConfig(seed=1)
    ds = torch.empty((3, 2, 27, 48), device="cuda")
    obs = pkg.render_pipeline(scene, sensor=cfg, step=2, ds_out=ds)
    assert torch.equal(ds, pkg.downsample_min(obs, 5))
    ds2 = torch.empty_like(ds)
    cap = CapturedStep(scene, sensor=cfg, first_step=2, ds_out=ds2)
    cap.replay()
    assert torch.equal(ds2, ds)
    with pytest.raises(ValueError):
        pkg.render_pipeline(scene, ds_out=torch.empty((3, 2, 27, 48), device="cuda"), downsample_factor=7)
    # asynchronous delivery of the policy observation (double-buffered, as bench.py's e2e)
    bufs = [torch.empty_like(ds) for _ in range(2)]
    hosts = [torch.empty((3, 2, 27, 48)).pin_memory() for _ in range(2)]
    want = []
    for k in range(4):
        pkg.render_pipeline(scene, sensor=cfg, step=10 + k, ds_out=bufs[k % 2], host_ds_out=hosts[k % 2])
        want.append(bufs[k % 2].clone())
        if k % 2 == 1:
            scene.host_sync()
            assert torch.equal(hosts[0], want[k - 1].cpu()) and torch.equal(hosts[1], want[k].cpu())
    with pytest.raises(ValueError):
        pkg.render_pipeline(scene, host_ds_out=hosts[0])


def test_bound_link_states_zero_copy(pkg):
    """Poses read straight from a simulator-style (N, L, 13) link-state tensor (xyzw quats,
    extra links, permuted link map) render bitwise like set_body_poses, eager and in a
    captured graph whose tensor is updated in place."""
    from paper_2602_03002_b200.pipeline import CapturedStep
    case = casefile.load(os.path.join(GOLDEN, "render_cfg2_slice.npz"))
    s_ref, s_bind, s_graph = (casefile.build_scene(case, pkg) for _ in range(3))
    n, b = s_ref.num_envs, s_ref.num_bodies
    links = b + 5
    rng = np.random.default_rng(3)
    lmap = rng.permutation(links)[:b]
    cfg = pkg.SensorConfig(seed=1)

    def states_for(pos, rot_wxyz):
        st = rng.standard_normal((n, links, 13)).astype(np.float32)   # junk in unused links / velocities
        st[:, lmap, 0:3] = pos
        st[:, lmap, 3:7] = rot_wxyz[..., [1, 2, 3, 0]]                # xyzw
        return st

    st = torch.from_numpy(states_for(case["body_pos"], case["body_rot"])).cuda()
    s_bind.bind_link_states(st, lmap)
    s_graph.bind_link_states(st.reshape(n * links, 13), lmap)
    cap = CapturedStep(s_graph, sensor=cfg, first_step=0)
    for k in range(3):
        pos = (case["body_pos"] + rng.normal(0, 0.02, case["body_pos"].shape)).astype(np.float32)
        rot = case["body_rot"].astype(np.float32) * np.float32(1.5)        # unnormalised on purpose
        st.copy_(torch.from_numpy(states_for(pos, rot)))
        s_ref.set_body_poses(pos, rot)
        want = pkg.render_pipeline(s_ref, sensor=cfg, step=k)
        assert torch.equal(pkg.render_pipeline(s_bind, sensor=cfg, step=k), want), f"eager step {k}"
        assert torch.equal(cap.replay(), want), f"graph step {k}"
        hp, hq = s_bind.camera_world_poses()
        rp, rq = s_ref.camera_world_poses()
        assert np.allclose(hp, rp) and np.allclose(hq, rq)
    wx = torch.from_numpy(np.concatenate([np.zeros((n, links, 2), np.float32),
                                          states_for(case["body_pos"], case["body_rot"])[..., :7][..., [0, 1, 2, 6, 3, 4, 5]]],
                                         axis=-1)).cuda().contiguous()       # pos at 2, wxyz at 5
    s_bind.bind_link_states(wx, lmap, pos_offset=2, rot_offset=5, quat_order="wxyz")
    s_ref.set_body_poses(case["body_pos"], case["body_rot"])
    assert torch.equal(pkg.render(s_bind).data, pkg.render(s_ref).data)
    with pytest.raises(ValueError):
        s_bind.bind_link_states(wx, lmap[:-1])
    with pytest.raises(ValueError):
        s_bind.bind_link_states(wx, lmap, rot_offset=8)
    s_bind.set_body_poses(case["body_pos"], case["body_rot"])            # unbinds
    assert torch.equal(pkg.render(s_bind).data, pkg.render(s_ref).data)


def test_captured_full_pipeline_equals_eager(pkg):
    """Everything at once (sensor + latency ring + side masking + fused 5x5 downsample),
    eager vs CUDA-graph replay, bitwise, over several steps."""
    from paper_2602_03002_b200.pipeline import CapturedStep
    cam = pkg.CameraModel(width=60, height=45, hfov_deg=87.0, vfov_deg=58.0, d_max=6.0,
                          mount=pkg.look_at_pose([0.0, 0.0, 1.2], [1.5, 0.3, 0.0]))
    xs = np.linspace(-4, 4, 41)
    gx, gy = np.meshgrid(xs, xs)
    a = (np.arange(40)[:, None] * 41 + np.arange(40)[None, :]).ravel()
    faces = np.concatenate([np.column_stack([a, a + 1, a + 42]), np.column_stack([a, a + 42, a + 41])])
    terrain = pkg.TriMesh(np.column_stack([gx.ravel(), gy.ravel(), 0.2 * np.sin(2 * gx.ravel())]), faces)
    scenes = [pkg.Scene(5, bodies=[("box", pkg.make_box(size=(0.3, 0.3, 0.3)))], cameras=[cam, cam],
                        terrain=terrain) for _ in range(2)]
    rng = np.random.default_rng(3)
    sens_cfg = pkg.SensorConfig(seed=4)
    rsm = pkg.RsmConfig(seed=5)
    modes = pkg.rsm_sample_modes(rsm, "stepping_stones", 5, 2, episode=0)
    delays = np.array([0.0, 0.02, 0.05, 0.1, 0.03])
    fb_e, fb_g = pkg.FrameBuffer(capacity=4), pkg.FrameBuffer(capacity=4)
    ds_e, ds_g = (torch.empty((5, 2, 9, 12), device="cuda") for _ in range(2))
    cap = CapturedStep(scenes[1], sensor=sens_cfg, frame_buffer=fb_g, delays=delays, dt=0.02, first_step=0,
                       rsm=rsm, rsm_modes=modes, ds_out=ds_g)
    for k in range(6):
        pos = rng.uniform(-1, 1, size=(5, 1, 3)) * [1, 1, 0.2] + [1.2, 0, 0.5]
        rot = rng.standard_normal((5, 1, 4))
        for sc in scenes:
            sc.set_body_poses(pos, rot)
        eager = pkg.render_pipeline(scenes[0], sensor=sens_cfg, step=k, frame_buffer=fb_e, timestamp=0.02 * k,
                                    delays=delays, rsm=rsm, rsm_modes=modes, ds_out=ds_e).clone()
        graph = cap.replay()
        assert torch.equal(graph, eager), f"obs step {k}"
        assert torch.equal(ds_g, ds_e), f"downsample step {k}"
        assert torch.equal(ds_e, pkg.downsample_min(eager, 5))


@pytest.mark.gpu
@pytest.mark.parametrize("p", [0.0, 1e-17, 2.0 ** -53, 3 * 2.0 ** -53, 0.05, 0.5, 0.999999])
def test_dropout_mask_at_threshold_edges(pkg, oracle, p):
    """The kernel's dropout test is an integer compare of the top 53 hash bits against
    ceil(p * 2^53); the oracle keeps the reference's f64 compare unit53(h) < p
    (sensor.py:79). Masks must agree exactly, including p = 0 and p at 1-3 ulps of
    the 53-bit grid."""
    rng = np.random.default_rng(5)
    depth = rng.uniform(0.5, 5.0, size=(3, 2, 40, 64)).astype(np.float32)
    d_max = np.array([6.0, 6.0])
    cfg = pkg.SensorConfig(noise_scale=0.05, dropout_p=p, dropout_fill=0.25, seed=9)
    out = pkg.apply_noise_dropout(torch.from_numpy(depth).cuda(), cfg, d_max=d_max, step=2).cpu().numpy()
    ref = oracle.apply_noise_dropout(depth, noise_scale=0.05, dropout_p=p, seed=9, d_max=d_max, step=2,
                                     dropout_fill=0.25)
    assert np.array_equal(out == np.float32(0.25), ref == np.float32(0.25))
    if p == 0.0:
        assert not (ref == np.float32(0.25)).any()
    assert _ulps(out, ref).max() <= 1
