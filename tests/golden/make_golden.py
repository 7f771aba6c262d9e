"""Generate golden vectors from the LIVE reference implementation.

Run in a container where the reference is importable (it is read-only at
/root/reference; it does not exist on GPU boxes):

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

Every input is rounded to float32-representable values first (meshes, poses,
camera offsets) so the reference (f64) and the GPU (f32 storage) see the same
geometry; camera mounts and intrinsics stay f64 on both sides (they cross the
C ABI as doubles). Outputs are written next to this script as .npz and are the
fixtures that pin both the CPU oracle (tests/test_oracle_golden.py) and the
CUDA path (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import argparse
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def unit_f32(q):
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    return f32(q)


def case_from_reference(md, bodies, terrain, cameras, body_pos, body_rot, rand=None, early=True,
                        num_envs=None):
    """bodies: list of (V,F); terrain: (V,F) or None; cameras: list of CameraModel (md).
    Returns the case dict including the reference output."""
    bmeshes = [md.TriMesh(f32(v), f, frame="body-local") for v, f in bodies]
    tmesh = None if terrain is None else md.TriMesh(f32(terrain[0]), terrain[1])
    n = num_envs if num_envs is not None else body_pos.shape[0]
    scene = md.Scene(num_envs=n, bodies=[(f"b{i}", m) for i, m in enumerate(bmeshes)],
                     cameras=cameras, terrain=tmesh)
    case = {"num_bodies": np.array(len(bmeshes)), "num_envs": np.array(n)}
    for i, m in enumerate(bmeshes):
        case[f"body{i}_v"] = m.vertices
        case[f"body{i}_f"] = m.faces
    if tmesh is not None:
        case["terrain_v"] = tmesh.vertices
        case["terrain_f"] = tmesh.faces
    if bmeshes:
        bp, bq = f32(body_pos), unit_f32(body_rot)
        scene.set_body_poses(bp, bq)
        case["body_pos"], case["body_rot"] = bp, bq
    else:
        case["body_pos"] = np.zeros((n, 0, 3))
        case["body_rot"] = np.zeros((n, 0, 4))
    if rand is not None:
        rp, rq, rf = f32(rand[0]), unit_f32(rand[1]), f32(rand[2])
        scene.set_camera_randomization(rp, rq, rf)
        case["rand_pos"], case["rand_rot"], case["rand_fov"] = rp, rq, rf
    case["cam_w"] = np.array(cameras[0].width)
    case["cam_h"] = np.array(cameras[0].height)
    case["cam_hfov"] = np.array([c.hfov_deg for c in cameras])
    case["cam_vfov"] = np.array([c.vfov_deg for c in cameras])
    case["cam_dmax"] = np.array([c.d_max for c in cameras])
    case["cam_parent"] = np.array([-1 if c.parent_body is None else c.parent_body for c in cameras])
    case["cam_mpos"] = np.stack([c.mount.translation for c in cameras])
    case["cam_mrot"] = np.stack([c.mount.rotation for c in cameras])
    case["early"] = np.array(bool(early))
    case["out"] = md.render(scene, early_termination=early, backend="numba").data
    return case


def random_case(md, rng, num_envs=2, num_cams=2, width=32, height=24, num_bodies=3, parented=False,
                camrand=False):
    """Random scene in the style of the reference fixture (tests/scenes.py:58-108)."""
    def body_mesh():
        kind = rng.integers(0, 3)
        if kind == 0:
            m = md.make_box(size=tuple(rng.uniform(0.15, 0.5, size=3)))
        elif kind == 1:
            m = md.make_icosphere(radius=rng.uniform(0.1, 0.3), subdivisions=int(rng.integers(0, 2)))
        else:
            k = int(rng.integers(4, 21))
            base = np.repeat(rng.uniform(-0.25, 0.25, size=(k, 3)), 3, axis=0)
            v = base + rng.uniform(-0.15, 0.15, size=base.shape)
            m = md.TriMesh(v, np.arange(3 * k).reshape(-1, 3))
        return m.vertices, m.faces

    bodies = [body_mesh() for _ in range(num_bodies)]
    nodes, ext, amp = 10, 6.0, 0.35
    xs = np.linspace(-ext / 2, ext / 2, nodes)
    gx, gy = np.meshgrid(xs, xs)
    gz = amp * np.sin(gx * rng.uniform(0.5, 1.5) + rng.uniform(0, 6)) * \
        np.cos(gy * rng.uniform(0.5, 1.5) + rng.uniform(0, 6)) + rng.uniform(-0.05, 0.05, size=gx.shape)
    verts = np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])
    iy, ix = np.meshgrid(np.arange(nodes - 1), np.arange(nodes - 1), indexing="ij")
    a = (iy * nodes + ix).ravel()
    faces = np.concatenate([np.column_stack([a, a + 1, a + nodes + 1]),
                            np.column_stack([a, a + nodes + 1, a + nodes])]).astype(np.int64)
    cams = []
    for c in range(num_cams):
        ang = 2 * np.pi * (c + rng.uniform(0, 0.5)) / num_cams
        r = rng.uniform(2.2, 3.5)
        pos = np.array([r * np.cos(ang), r * np.sin(ang), rng.uniform(0.6, 2.2)])
        tgt = rng.uniform(-0.5, 0.5, size=3) + np.array([0, 0, 0.4])
        parent = None
        mount = md.look_at_pose(pos, tgt)
        if parented and c == 0:
            # mount relative to body 0 (camera rides the body, test_render.py:131-155)
            parent = 0
            mount = md.RigidPose(np.array([0.0, 0.0, 0.35]),
                                 md.look_at_pose(np.zeros(3), np.array([0.3, 0.1, -1.0])).rotation)
        cams.append(md.CameraModel(width=width, height=height, hfov_deg=float(rng.uniform(60, 100)),
                                   vfov_deg=float(rng.uniform(45, 75)), d_max=float(rng.uniform(4, 12)),
                                   mount=mount, parent_body=parent, name=f"c{c}"))
    pos = np.empty((num_envs, num_bodies, 3))
    pos[..., 0] = rng.uniform(-1.5, 1.5, size=(num_envs, num_bodies))
    pos[..., 1] = rng.uniform(-1.5, 1.5, size=(num_envs, num_bodies))
    pos[..., 2] = rng.uniform(0.0, 1.5, size=(num_envs, num_bodies))
    rot = rng.standard_normal((num_envs, num_bodies, 4))
    rand = None
    if camrand:
        off_rot = np.stack([[md.quat_from_euler(*rng.uniform(-0.04, 0.04, 3)) for _ in range(num_cams)]
                            for _ in range(num_envs)])
        rand = (rng.uniform(-0.02, 0.02, size=(num_envs, num_cams, 3)), off_rot,
                rng.uniform(-2.0, 2.0, size=(num_envs, num_cams)))
    return case_from_reference(md, bodies, (verts, faces), cams, pos, rot, rand=rand)


def make_frameio(md):
    """MDPT / PGM bytes and depth_to_u8 vectors from the reference frameio.py."""
    g = np.random.default_rng(5)
    depth = g.uniform(-0.5, 11.0, size=(3, 2, 27, 48)).astype(np.float32)
    depth[0, 0, 0, :8] = np.float32([0.0, 10.0, 5.0, 2.5, 7.5, 1.25, 8.75, 3.75])   # exact half-way grays
    fio = {"depth": depth}
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "f.mdpt")
        md.write_frames(path, depth)
        fio["mdpt_bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
        md.write_grid(path, depth[1, 1].astype(np.float64))
        fio["grid_bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
        for k, dmax in enumerate((10.0, 8.0, 0.7)):
            fio[f"u8_{k}"] = md.depth_to_u8(depth, dmax)
        fio["u8_dmax"] = np.array([10.0, 8.0, 0.7])
        pgm = os.path.join(tmp, "p.pgm")
        md.write_pgm(pgm, fio["u8_0"][0, 1])
        fio["pgm_bytes"] = np.frombuffer(open(pgm, "rb").read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "frameio.npz"), **fio)


def make_terrain(md):
    """Checksums of the reference generator's meshes for the benchmark terrains
    (terrain.py:278-360): synth.py's tiles must reproduce them bit for bit."""
    import hashlib
    from multidepth.terrain import TerrainSpec, generate_terrain
    plat = (6 - 8 * 0.27) / 2
    specs = {"cfg1_stairs": TerrainSpec(kind="stairs_up"),
             "tile_slope_pyramid": TerrainSpec(kind="slope_pyramid", size=(6.0, 6.0), incline_deg=20.0),
             "tile_stairs_up": TerrainSpec(kind="stairs_up", width=6.0, platform_length=plat),
             "tile_stairs_down": TerrainSpec(kind="stairs_down", width=6.0, platform_length=plat),
             "cfg3_stones": TerrainSpec(kind="stepping_stones", stone_size=0.25, stone_gap=0.60, size=(24, 24))}
    out = {}
    shift = {"tile_stairs_up": 1.08, "tile_stairs_down": 1.08}   # stairs tiles are centred in synth.py
    for name, spec in specs.items():
        m, _ = generate_terrain(spec)
        v = np.array(m.vertices, np.float64)
        v[:, 0] -= shift.get(name, 0.0)
        out[name + "_vsha"] = np.array(hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest())
        out[name + "_fsha"] = np.array(hashlib.sha256(np.ascontiguousarray(m.faces, np.int64).tobytes()).hexdigest())
        out[name + "_shape"] = np.array([len(m.vertices), len(m.faces)])
    np.savez_compressed(os.path.join(HERE, "terrain.npz"), **out)


def make_seam(md):
    """The exact arguments the live reference hands its backend seam: render() is run
    with get_render_fn wrapped so the numba render_batch call (numba_backend.py:222-234)
    is recorded -- the real FlatGeometry (median-split forest, leaf-ordered triangles),
    f64 body/camera poses, the per-env FOV-randomised ray grids, d_max, and the output
    it wrote (scene.py:332-348)."""
    from multidepth import kernels as mk
    from paper_2602_03002_b200 import synth
    w = synth.config("cfg1", 4)
    n = 4
    rng = np.random.default_rng(31)
    bp, bq = w.poses(0)
    bp = f32(bp + rng.normal(0.0, 0.05, bp.shape) * np.array([1.0, 1.0, 0.2]))
    bq = unit_f32(bq)
    bodies = [(nm, md.TriMesh(f32(m.vertices), m.faces, frame="body-local")) for nm, m in w.bodies]
    cams = [md.CameraModel(width=c.width, height=c.height, hfov_deg=c.hfov_deg, vfov_deg=c.vfov_deg, d_max=c.d_max,
                           mount=md.RigidPose(c.mount.translation, c.mount.rotation), parent_body=c.parent_body)
            for c in synth.torso_cameras(2)]
    scene = md.Scene(num_envs=n, bodies=bodies, cameras=cams,
                     terrain=md.TriMesh(f32(w.terrain.mesh.vertices), w.terrain.mesh.faces))
    scene.set_body_poses(bp, bq)
    po, ro, fo = md.sample_camera_offsets(md.CameraRandomization(seed=5), n, 2)
    scene.set_camera_randomization(f32(po), unit_f32(ro), f32(fo))
    captured = {}
    real = mk.get_render_fn

    def spy(backend=None):
        name, fn = real(backend)

        def rec(flat, body_pos, body_rot, cam_pos, cam_rot, ray_dirs, ray_scale, d_max, early, out, threads):
            fn(flat, body_pos, body_rot, cam_pos, cam_rot, ray_dirs, ray_scale, d_max, early, out, threads)
            for f in ("body_root", "node_min", "node_max", "left", "right", "start", "count", "tri_v0", "tri_v1",
                      "tri_v2", "body_tri_offsets", "g_node_min", "g_node_max", "g_left", "g_right", "g_start",
                      "g_count", "g_tri_v0", "g_tri_v1", "g_tri_v2"):
                captured["flat_" + f] = np.asarray(getattr(flat, f)).copy()
            captured.update(body_pos=np.array(body_pos), body_rot=np.array(body_rot), cam_pos=np.array(cam_pos),
                            cam_rot=np.array(cam_rot), ray_dirs=np.array(ray_dirs), ray_scale=np.array(ray_scale),
                            d_max=np.array(d_max), early=np.array(bool(early)), out=out.copy())
        return name, rec

    mk.get_render_fn = spy
    try:
        frame = md.render(scene, backend="numba")
    finally:
        mk.get_render_fn = real
    assert np.array_equal(frame.data, captured["out"])
    np.savez_compressed(os.path.join(HERE, "seam_capture.npz"), **captured)
    print("seam", captured["out"].shape, "ray_dirs", captured["ray_dirs"].shape,
          "hits", int((captured["out"] < 10.0).sum()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default=os.environ.get("MULTIDEPTH_REF", "/root/reference/pkg/src"))
    ap.add_argument("--only", choices=["frameio", "terrain", "seam"], default=None,
                    help="regenerate one fixture group")
    args = ap.parse_args()
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "numba_cache_golden"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, args.ref)
    sys.path.insert(0, ROOT)
    import multidepth as md
    from multidepth import rng as mrng
    from paper_2602_03002_b200 import synth

    if args.only in (None, "frameio"):
        make_frameio(md)
    if args.only in (None, "terrain"):
        make_terrain(md)
    if args.only in (None, "seam"):
        make_seam(md)
    if args.only is not None:
        print("done")
        return
    out = {}
    rng = np.random.default_rng(20261018)
    for k in range(6):
        out[f"rand{k}"] = random_case(md, rng, num_envs=2, num_cams=2 + (k % 3), num_bodies=3 + k)
    out["rand_camrand"] = random_case(md, rng, num_envs=3, num_cams=2, camrand=True)
    out["parented"] = random_case(md, rng, num_envs=2, num_cams=2, parented=True, camrand=True)
    c = random_case(md, np.random.default_rng(7), num_envs=2, num_cams=2, num_bodies=5)
    out["rand_noet"] = c
    # early termination off on the same scene
    # (rebuild through the reference with early=False)
    # analytic flat ground (test_render.py:23-32) and an empty view (test_render.py:35-39)
    down = md.CameraModel(width=9, height=7, hfov_deg=70.0, vfov_deg=55.0, d_max=5.0,
                          mount=md.look_at_pose([0.0, 0.0, 1.0], [0.0, 0.0, 0.0]))
    plane = md.make_plane(size=(10.0, 10.0))
    out["flat"] = case_from_reference(md, [], (plane.vertices, plane.faces), [down], None, None, num_envs=1)
    box = md.make_box(size=(0.3, 0.3, 0.3), center=(5.0, 5.0, 5.0))
    miss_cam = md.CameraModel(width=9, height=7, hfov_deg=70.0, vfov_deg=55.0, d_max=3.5,
                              mount=md.look_at_pose([0.0, 0.0, 1.0], [0.0, 0.0, 0.0]))
    out["miss"] = case_from_reference(md, [(box.vertices, box.faces)], None, [miss_cam],
                                      np.zeros((1, 1, 3)), np.array([[[1.0, 0, 0, 0]]]))
    # config 1: stairs terrain + G1 proxy at default pose, one front camera 64x48
    w = synth.config("cfg1")
    bp, bq = w.poses(0)
    out["cfg1"] = case_from_reference(md, [(m.vertices, m.faces) for _, m in w.bodies],
                                      (w.terrain.mesh.vertices, w.terrain.mesh.faces), w.cameras, bp, bq)
    # a small cfg2-shaped slice (8 envs, 2 cams, 64x48) on one 6 m stairs/slope strip
    t2 = synth.tile_field(["slope_pyramid", "stairs_up", "stairs_down", "slope_pyramid"], tile=3.0)
    w2 = synth.Workload("cfg2_slice", t2, synth.g1_links(), synth.torso_cameras(2), 8)
    w2.roots, w2.yaws = synth._place(t2, 8, seed=1)
    bp2, bq2 = w2.poses(3)
    strip = w2.terrain.mesh
    out["cfg2_slice"] = case_from_reference(md, [(m.vertices, m.faces) for _, m in w2.bodies],
                                            (strip.vertices, strip.faces), w2.cameras, bp2, bq2)
    for name, case in out.items():
        np.savez_compressed(os.path.join(HERE, f"render_{name}.npz"), **case)
        print(name, case["out"].shape, "hits", int((case["out"] < case["cam_dmax"].max()).sum()))

    # early termination off: same scene as rand_noet, reference with early=False
    sc = out["rand_noet"]
    # ---- sensor stage (sensor.py:55-82) ----
    g = np.random.default_rng(11)
    depth = g.uniform(0.3, 9.5, size=(4, 2, 48, 64)).astype(np.float32)
    depth[0, 0, :4] = np.float32(8.0)
    depth[1, 1, :4] = np.float32(10.0)
    dmax = np.array([8.0, 10.0])
    sens = {"depth": depth, "d_max": dmax}
    cfg = md.SensorConfig(noise_scale=0.1, dropout_p=0.05, seed=7)
    sens["out_s3"] = md.apply_noise_dropout(depth, cfg, d_max=dmax, step=3)
    cfg_fill = md.SensorConfig(noise_scale=0.2, dropout_p=0.3, dropout_fill=0.25, seed=2)
    sens["out_fill_s0"] = md.apply_noise_dropout(depth, cfg_fill, d_max=dmax, step=0)
    # env-offset slice: envs 2..3 of the full block equal a 2-env block with env offset 2
    sens["out_s3_full8"] = md.apply_noise_dropout(np.concatenate([depth, depth]), cfg, d_max=dmax, step=3)
    # rng vectors
    keys = [(0, "sensor"), (7, "sensor"), (3, "latency"), (123456789, "a-much-longer-stream-name")]
    sens["keys_seed"] = np.array([k[0] for k in keys])
    sens["keys_val"] = np.array([int(mrng.stream_key(s, n)) for s, n in keys], dtype=np.uint64)
    ctr = np.stack(np.meshgrid(np.arange(5), np.arange(7), indexing="ij"), -1).reshape(-1, 2)
    key = mrng.stream_key(5, "demo")
    sens["rng_counters"] = ctr
    sens["rng_uniform"] = mrng.uniform(key, ctr[:, 0], ctr[:, 1])
    sens["rng_normal"] = mrng.normal(key, ctr[:, 0], ctr[:, 1])
    # latency: pushes at k*dt, capacity 8, per-env delays (sensor.py:103-158)
    dt = 0.02
    lat_cfg = md.SensorConfig(max_delay=0.1, seed=3)
    delays = md.sample_latencies(lat_cfg, 64, episode=0)
    delays[:6] = [0.0, 0.02, 0.04, 0.1, 1.0, 0.06]   # exact multiples and beyond history
    sens["delays"] = delays
    sel = []
    buf = md.FrameBuffer(capacity=8)
    for s in range(12):
        fr = np.full((64, 1, 1, 1), float(s), dtype=np.float32)
        buf.push(md.scene.DepthFrame(fr, s * dt))
        got = buf.fetch_delayed_batch(s * dt, delays)
        sel.append(got[:, 0, 0, 0].astype(np.int64))
    sens["latency_dt"] = np.array(dt)
    sens["latency_capacity"] = np.array(8)
    sens["latency_sel"] = np.stack(sel)
    sens["latencies_ep2"] = md.sample_latencies(md.SensorConfig(max_delay=0.1, seed=5), 100, episode=2)
    # downsample (sensor.py:85-100)
    frames = g.uniform(0.1, 6.0, size=(1, 2, 135, 240)).astype(np.float32)
    sens["ds_in"] = frames
    sens["ds_out"] = md.downsample_min(frames, 5)
    # camera offsets (sensor.py:183-211)
    p, q, f = md.sample_camera_offsets(md.CameraRandomization(seed=4), 16, 2, episode=1)
    sens["camoff_pos"], sens["camoff_rot"], sens["camoff_fov"] = p, q, f
    # random side masking (perception.py:150-202)
    from multidepth import perception as mp
    rcfg = mp.RsmConfig(seed=3)
    sens["rsm_modes_stones"] = mp.rsm_sample_modes(rcfg, "stepping_stones", 64, 2, episode=1)
    rdepth = g.uniform(0.5, 5.0, size=(4, 2, 27, 48)).astype(np.float32)
    rmodes = np.array([[0, 1], [2, 0], [1, 2], [2, 2]])
    sens["rsm_depth"], sens["rsm_modes"] = rdepth, rmodes
    sens["rsm_out_s5"] = mp.rsm_apply(rdepth, rmodes, rcfg, d_max=np.array([6.0, 8.0]), step=5)
    rcfg2 = mp.RsmConfig(seed=4, fill_high=4.0, f_small=0.1, f_large=0.3)
    sens["rsm_out2_s0"] = mp.rsm_apply(rdepth, rmodes, rcfg2, d_max=np.array([6.0, 8.0]), step=0)
    np.savez_compressed(os.path.join(HERE, "sensor.npz"), **sens)

    # early-termination-off render of rand_noet
    bm = [md.TriMesh(sc[f"body{i}_v"], sc[f"body{i}_f"]) for i in range(int(sc["num_bodies"]))]
    cams = [md.CameraModel(width=int(sc["cam_w"]), height=int(sc["cam_h"]), hfov_deg=float(sc["cam_hfov"][c]),
                           vfov_deg=float(sc["cam_vfov"][c]), d_max=float(sc["cam_dmax"][c]),
                           mount=md.RigidPose(sc["cam_mpos"][c], sc["cam_mrot"][c]),
                           parent_body=None if sc["cam_parent"][c] < 0 else int(sc["cam_parent"][c]))
            for c in range(len(sc["cam_hfov"]))]
    scene = md.Scene(num_envs=2, bodies=[(f"b{i}", m) for i, m in enumerate(bm)], cameras=cams,
                     terrain=md.TriMesh(sc["terrain_v"], sc["terrain_f"]))
    scene.set_body_poses(sc["body_pos"], sc["body_rot"])
    noet = dict(sc)
    noet["early"] = np.array(False)
    noet["out"] = md.render(scene, early_termination=False, backend="numba").data
    np.savez_compressed(os.path.join(HERE, "render_rand_noet.npz"), **noet)
    print("done")


if __name__ == "__main__":
    main()
