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
