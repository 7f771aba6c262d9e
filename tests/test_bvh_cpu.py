"""Host-side checks of the GPU BVH builder/packer (no device needed).

mdrt_bvh_check builds a mesh's packed tree exactly as mdrt_add_body /
mdrt_set_terrain do and verifies: every triangle in exactly one leaf, every
decoded (16-bit grid) child box inside its parent's, every vertex inside its
leaf box with the fp32 decode slack, leaf size <= 4, depth <= the GPU stack.
"""

import numpy as np
import pytest

from paper_2602_03002_b200 import _native, synth
from paper_2602_03002_b200.mesh import TriMesh, make_box, make_icosphere, make_plane, merge_meshes


def soup(rng, n, spread=2.0, jitter=0.4, offset=0.0):
    base = np.repeat(rng.uniform(-spread, spread, size=(n, 3)), 3, axis=0) + offset
    v = base + rng.uniform(-jitter, jitter, size=base.shape)
    return v, np.arange(3 * n).reshape(-1, 3)


@pytest.mark.parametrize("seed", range(6))
def test_random_soups(seed):
    rng = np.random.default_rng(seed)
    for n in (1, 2, 3, 5, 17, 300, 2000):
        v, f = soup(rng, n)
        info = _native.bvh_check(v, f)
        assert info["triangles"] == n
        assert info["depth"] <= 24


def test_far_from_origin_and_tiny():
    rng = np.random.default_rng(9)
    v, f = soup(rng, 500, spread=0.5, jitter=0.01, offset=1000.0)   # 1 km away, cm-sized tris
    _native.bvh_check(v, f)
    v, f = soup(rng, 200, spread=1e-3, jitter=1e-4)                 # sub-mm geometry
    _native.bvh_check(v, f)


def test_primitives_and_flat_terrain():
    for m in (make_box(size=(1, 2, 3)), make_icosphere(0.5, subdivisions=3), make_plane(size=(24.0, 24.0)),
              merge_meshes([make_plane(size=(24, 24)), make_box(size=(0.25, 0.25, 0.5))])):
        info = _native.bvh_check(m.vertices, m.faces)
        assert info["triangles"] == m.num_faces


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_workload_terrains_and_links(name):
    w = synth.config(name, 2)
    info = _native.bvh_check(w.terrain.mesh.vertices, w.terrain.mesh.faces)
    assert info["triangles"] == w.terrain.mesh.num_faces
    for _, m in w.bodies:
        assert _native.bvh_check(m.vertices, m.faces)["triangles"] == m.num_faces


def test_degenerate_split_all_centroids_equal():
    # many triangles sharing one centroid: SAH finds no split, median fallback must still bound depth
    v = np.tile(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], dtype=np.float64), (4000, 1))
    f = np.arange(12000).reshape(-1, 3)
    info = _native.bvh_check(v, f)
    assert info["depth"] <= 24


def test_bad_input_rejected():
    with pytest.raises(ValueError):
        _native.bvh_check(np.zeros((3, 3)), np.array([[0, 1, 5]]))


def test_non_finite_vertices_rejected():
    v = np.array([[0, 0, 0], [1, 0, 0], [0, np.nan, 0]], dtype=np.float64)
    with pytest.raises(ValueError, match="finite"):
        _native.bvh_check(v, np.array([[0, 1, 2]]))
    v[1, 2] = np.inf
    with pytest.raises(ValueError, match="finite"):
        _native.bvh_check(v, np.array([[0, 1, 2]]))


def test_oversize_mesh_rejected_before_build():
    """A mesh the 24-entry traversal stack cannot hold (more than leaf_max * 2^23
    triangles) is refused with MDRT_EINVAL by the builder every geometry entry
    point goes through (mdrt_add_body / mdrt_set_terrain / mdrt_bvh_build), before
    any face is read: the faces array below is calloc-backed and never touched."""
    import ctypes
    nf = 4 * (1 << 23) + 1
    faces = np.zeros((nf, 3), dtype=np.int64)            # lazily zero-filled pages
    verts = np.zeros((3, 3), dtype=np.float64)
    counts = np.zeros(3, np.int64)
    i64p = ctypes.POINTER(ctypes.c_int64)
    rc = _native.lib().mdrt_bvh_build(_native.dptr(verts), 3, faces.ctypes.data_as(i64p), nf, 4, None, 0, None, 0,
                                      None, counts.ctypes.data_as(i64p))
    assert rc == _native.MDRT_EINVAL
    assert b"traversal stack" in _native.lib().mdrt_last_error()
    # leaf size 1: the limit is 2^23 triangles
    rc = _native.lib().mdrt_bvh_build(_native.dptr(verts), 3, faces.ctypes.data_as(i64p), (1 << 23) + 1, 1, None, 0,
                                      None, 0, None, counts.ctypes.data_as(i64p))
    assert rc == _native.MDRT_EINVAL
