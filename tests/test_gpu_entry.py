"""Per-tile terrain entry nodes (entry_kernel, csrc/mdrt_kernels.cu) change no result.

The prologue's frustum descent lets every ray of a pixel tile start its terrain
traversal below the tree's top levels. The closest hit must be identical to a
traversal from the root (MDRT_NO_TILE_ENTRY): bitwise, on the golden scenes and
on samples of the benchmark workloads, while counting fewer node fetches.
"""

import os

import numpy as np
import pytest
import torch

import casefile
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _pair(pkg, scene, **kw):
    from paper_2602_03002_b200 import _native
    scene.debug_flags = _native.NO_TILE_ENTRY
    ctr_root = torch.zeros(4, dtype=torch.int64, device=scene.device)
    ref = pkg.render(scene, counters=ctr_root, **kw).data.clone()
    scene.debug_flags = _native.TILE_ENTRY
    ctr = torch.zeros(4, dtype=torch.int64, device=scene.device)
    got = pkg.render(scene, counters=ctr, **kw).data.clone()
    plain = pkg.render(scene, **kw).data
    assert torch.equal(plain, got)
    scene.debug_flags = 0
    assert torch.equal(pkg.render(scene, **kw).data, got)       # the size heuristic's choice, same image
    return got, ref, ctr.tolist(), ctr_root.tolist()


@pytest.mark.parametrize("name", ["cfg1", "cfg2_slice", "rand0", "rand3", "rand_camrand", "parented", "flat", "miss"])
def test_entry_equals_root_on_goldens(pkg, name):
    case = casefile.load(os.path.join(GOLDEN, f"render_{name}.npz"))
    scene = casefile.build_scene(case, pkg)
    got, ref, ctr, ctr_root = _pair(pkg, scene)
    assert torch.equal(got, ref)
    assert ctr[0] <= ctr_root[0] and ctr[1] == ctr_root[1]       # same triangle tests, fewer node fetches


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3", "cfg5"])
def test_entry_equals_root_on_workloads(pkg, cfg):
    from paper_2602_03002_b200 import synth
    n = 64
    w = synth.config(cfg, 4096)
    f32 = lambda x: np.asarray(x, np.float64).astype(np.float32).astype(np.float64)  # noqa: E731
    bodies = [(nm, pkg.TriMesh(f32(m.vertices), m.faces, frame="body-local")) for nm, m in w.bodies]
    scene = pkg.Scene(n, bodies=bodies, cameras=w.cameras,
                      terrain=pkg.TriMesh(f32(w.terrain.mesh.vertices), w.terrain.mesh.faces))
    off = pkg.sample_camera_offsets(pkg.CameraRandomization(seed=3), 4096, len(w.cameras))
    scene.set_camera_randomization(*(np.asarray(a)[:n] for a in off))
    for step in (0, 5):
        bp, bq = w.poses(step, slice(0, n))
        scene.set_body_poses(f32(bp), f32(bq))
        got, ref, ctr, ctr_root = _pair(pkg, scene)
        assert torch.equal(got, ref), f"{cfg} step {step}: {(got != ref).sum().item()} pixels differ"
        assert ctr[1] == ctr_root[1]
        assert ctr[0] < ctr_root[0], (ctr, ctr_root)


def test_entry_with_wide_tiles_and_no_early_termination(pkg):
    from paper_2602_03002_b200 import _native
    case = casefile.load(os.path.join(GOLDEN, "render_cfg2_slice.npz"))
    scene = casefile.build_scene(case, pkg)
    got, ref, _, _ = _pair(pkg, scene, early_termination=False)
    assert torch.equal(got, ref)
    scene.debug_flags = _native.WIDE_STORES | _native.TILE_ENTRY  # 8-wide tiles: entries per 8x4 tile
    wide = pkg.render(scene).data.clone()
    scene.debug_flags = _native.WIDE_STORES | _native.NO_TILE_ENTRY
    assert torch.equal(wide, pkg.render(scene).data)


@pytest.mark.parametrize("seed", range(3))
def test_entry_equals_root_on_random_cameras(pkg, seed):
    """Random camera poses (looking up, sideways, from below the terrain), fields of view
    from 10 to 170 degrees and far limits from 0.3 to 200 m over a 160k-triangle rolling
    terrain: the per-tile entry never changes a pixel."""
    from paper_2602_03002_b200 import synth
    rng = np.random.default_rng(seed)
    t = synth.rolling_terrain(nodes=280, seed=seed)              # 14 m x 14 m, 155,682 triangles
    mesh = pkg.TriMesh(np.asarray(t.mesh.vertices, np.float64).astype(np.float32).astype(np.float64), t.mesh.faces)
    cams = []
    for k in range(4):
        eye = rng.uniform([-7, -7, -0.5], [7, 7, 3.0])
        look = eye + rng.normal(size=3)
        fov = float(rng.uniform(10, 170))
        cams.append(pkg.CameraModel(width=int(rng.integers(7, 70)) if k == 0 else 37, height=29 if k else 23,
                                    hfov_deg=fov, vfov_deg=float(np.clip(fov * rng.uniform(0.5, 1.0), 5, 170)),
                                    d_max=float(10 ** rng.uniform(-0.5, 2.3)), mount=pkg.look_at_pose(eye, look)))
    for cam in cams:
        scene = pkg.Scene(3, cameras=[cam], terrain=mesh)
        off = pkg.sample_camera_offsets(pkg.CameraRandomization(seed=seed + 7), 3, 1)
        scene.set_camera_randomization(*off)
        got, ref, ctr, ctr_root = _pair(pkg, scene)
        assert torch.equal(got, ref), f"{(got != ref).sum().item()} pixels differ ({cam})"
        assert ctr[1] == ctr_root[1] and ctr[0] <= ctr_root[0]


def test_trace_only_call_never_reads_stale_entries(pkg):
    """PHASE_PROLOGUE with entries off, then PHASE_TRACE with them on: the trace-only call
    must not use entries the prologue never computed (it falls back to the root)."""
    from paper_2602_03002_b200 import _native
    case = casefile.load(os.path.join(GOLDEN, "render_cfg2_slice.npz"))
    scene = casefile.build_scene(case, pkg)
    ref = pkg.render(scene).data.clone()
    out = torch.full(scene.frame_shape, -1.0, device=scene.device)
    a = scene._step_args(out, True)
    a.flags |= _native.PHASE_PROLOGUE | _native.NO_TILE_ENTRY
    scene._launch(a)
    b = scene._step_args(out, True)
    b.flags |= _native.PHASE_TRACE | _native.TILE_ENTRY
    scene._launch(b)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
