"""Per-mesh BVH: build, flat view, validation and ray queries.

Mirror of the reference's ``multidepth.bvh`` API (/root/reference/pkg/src/
multidepth/bvh.py:34-260): ``build_bvh(mesh) -> BVH`` with the same flat
arrays (``node_min/node_max/left/right/start/count/tri_v0/tri_v1/tri_v2/
tri_index``), ``validate_bvh`` and ``query_bvh``.

The tree is not the reference's median split: it is the renderer's own
binned-SAH build (``mdrt_bvh_build``, C++), i.e. exactly the tree the GPU
traverses. Its packed records (64 B nodes holding both children's fp32 boxes,
48 B triangles) are kept on the object (``packed_nodes``/``packed_tris``) and
the reference-format arrays are derived from them: node bounds are the packed
fp32 boxes (padded outward, so every triangle lies inside its leaf), triangle
corners are the original f64 vertices in leaf order. ``query_bvh`` runs on the
GPU (``mdrt_query_rays``) against the same records; there is no CPU traversal.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .mesh import TriMesh

LEAF_SIZE = 4          # bvh.py:26 (the builder's default leaf bound)
RAY_EPSILON = 1e-6     # bvh.py:29: hits need t > RAY_EPSILON
NODE_RECORD = np.dtype([("c0x", "<f4", 2), ("c0y", "<f4", 2), ("c1x", "<f4", 2), ("c1y", "<f4", 2),
                        ("c0z", "<f4", 2), ("c1z", "<f4", 2), ("ref", "<i4", 2), ("pad", "<i4", 2)])
TRI_RECORD = np.dtype([("v0", "<f4", 3), ("id", "<i4"), ("e1", "<f4", 3), ("pad1", "<f4"),
                       ("e2", "<f4", 3), ("pad2", "<f4")])
assert NODE_RECORD.itemsize == 64 and TRI_RECORD.itemsize == 48


@dataclass(frozen=True)
class BVH:
    node_min: np.ndarray
    node_max: np.ndarray
    left: np.ndarray
    right: np.ndarray
    start: np.ndarray
    count: np.ndarray
    tri_v0: np.ndarray
    tri_v1: np.ndarray
    tri_v2: np.ndarray
    tri_index: np.ndarray
    packed_nodes: np.ndarray = field(repr=False, default=None)   # NODE_RECORD, root = 0
    packed_tris: np.ndarray = field(repr=False, default=None)    # TRI_RECORD, leaf order
    _device: dict = field(repr=False, default_factory=dict, compare=False)

    @property
    def num_nodes(self) -> int:
        return len(self.node_min)

    @property
    def num_triangles(self) -> int:
        return len(self.tri_v0)

    @property
    def max_depth(self) -> int:
        depth = np.zeros(self.num_nodes, dtype=np.int64)
        for i in range(self.num_nodes):       # parents precede children (DFS order)
            if self.left[i] >= 0:
                depth[self.left[i]] = depth[self.right[i]] = depth[i] + 1
        return int(depth.max()) if self.num_nodes else 0

    def device_records(self, device=None) -> tuple[torch.Tensor, torch.Tensor]:
        """The packed node / triangle records as CUDA byte tensors (uploaded once per device)."""
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        key = str(dev)
        if key not in self._device:
            self._device[key] = (torch.from_numpy(self.packed_nodes.view(np.uint8).copy()).to(dev),
                                 torch.from_numpy(self.packed_tris.view(np.uint8).copy()).to(dev))
        return self._device[key]


def _decode_leaf(ref: int) -> tuple[int, int]:
    v = ~int(ref)
    return v >> 3, (v & 7) + 1


def build_bvh(mesh: TriMesh, leaf_size: int = LEAF_SIZE) -> BVH:
    """Binned-SAH build (the renderer's tree), deterministic; leaves hold <= leaf_size triangles."""
    if mesh.num_faces == 0:
        raise ValueError("cannot build a BVH over an empty mesh")
    if not 1 <= int(leaf_size) <= 8:
        raise ValueError("leaf_size must be in [1, 8]")
    verts = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
    faces = np.ascontiguousarray(mesh.faces, dtype=np.int64)
    nf = len(faces)
    nodes = np.zeros(max(nf, 1), dtype=NODE_RECORD)
    tris = np.zeros(nf, dtype=TRI_RECORD)
    tri_index = np.zeros(nf, dtype=np.int64)
    counts = np.zeros(3, dtype=np.int64)
    i64p = ctypes.POINTER(ctypes.c_int64)
    _native.check(_native.lib().mdrt_bvh_build(
        verts.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(verts), faces.ctypes.data_as(i64p), nf,
        int(leaf_size), nodes.ctypes.data_as(ctypes.c_void_p), len(nodes), tris.ctypes.data_as(ctypes.c_void_p),
        nf, tri_index.ctypes.data_as(i64p), counts.ctypes.data_as(i64p)))
    packed = nodes[:counts[0]].copy()
    # flat reference layout: one entry per packed child (inner or leaf) + the root
    mins, maxs, left, right, start, count = [], [], [], [], [], []

    def new_node(lo, hi):
        mins.append(lo)
        maxs.append(hi)
        left.append(-1), right.append(-1), start.append(0), count.append(0)
        return len(mins) - 1

    rec = packed
    boxes = lambda r, c: (np.array([r[f"c{c}x"][0], r[f"c{c}y"][0], r[f"c{c}z"][0]], np.float64),  # noqa: E731
                          np.array([r[f"c{c}x"][1], r[f"c{c}y"][1], r[f"c{c}z"][1]], np.float64))
    r0 = rec[0]
    lo0, hi0 = boxes(r0, 0)
    lo1, hi1 = boxes(r0, 1)
    if lo1[0] > hi1[0]:          # single-leaf tree: child 1 is the empty box
        root = new_node(lo0, hi0)
        start[root], count[root] = _decode_leaf(r0["ref"][0])
    else:
        root = new_node(np.minimum(lo0, lo1), np.maximum(hi0, hi1))
        stack = [(0, root)]
        while stack:
            p, flat = stack.pop()
            kids = []
            for c in (0, 1):
                lo, hi = boxes(rec[p], c)
                k = new_node(lo, hi)
                ref = int(rec[p]["ref"][c])
                if ref >= 0:
                    stack.append((ref, k))
                else:
                    start[k], count[k] = _decode_leaf(ref)
                kids.append(k)
            left[flat], right[flat] = kids
    tris_f64 = verts[faces[tri_index]]
    return BVH(node_min=np.array(mins), node_max=np.array(maxs), left=np.array(left, np.int32),
               right=np.array(right, np.int32), start=np.array(start, np.int32), count=np.array(count, np.int32),
               tri_v0=tris_f64[:, 0].copy(), tri_v1=tris_f64[:, 1].copy(), tri_v2=tris_f64[:, 2].copy(),
               tri_index=tri_index, packed_nodes=packed, packed_tris=tris)


def validate_bvh(bvh: BVH, mesh=None) -> None:
    """Structural invariants (bvh.py:220-260); raises AssertionError on violation."""
    n = bvh.num_nodes
    seen = np.zeros(bvh.num_triangles, dtype=bool)
    inner = bvh.left >= 0
    assert np.all(bvh.node_min <= bvh.node_max + 1e-12), "inverted bounds"
    for i in np.nonzero(inner)[0]:
        l, r = int(bvh.left[i]), int(bvh.right[i])
        assert 0 <= l < n and 0 <= r < n, f"node {i} child out of range"
        assert bvh.count[i] == 0, f"inner node {i} holds triangles"
        for c in (l, r):
            assert np.all(bvh.node_min[i] <= bvh.node_min[c] + 1e-9) and \
                np.all(bvh.node_max[c] <= bvh.node_max[i] + 1e-9), f"child {c} escapes parent {i}"
    for i in np.nonzero(~inner)[0]:
        s, c = int(bvh.start[i]), int(bvh.count[i])
        assert c >= 1, f"leaf {i} is empty"
        assert 0 <= s and s + c <= bvh.num_triangles, f"leaf {i} range out of bounds"
        assert not seen[s:s + c].any(), f"leaf {i} overlaps another leaf"
        seen[s:s + c] = True
        corners = np.concatenate([bvh.tri_v0[s:s + c], bvh.tri_v1[s:s + c], bvh.tri_v2[s:s + c]])
        assert np.all(corners >= bvh.node_min[i] - 1e-9) and np.all(corners <= bvh.node_max[i] + 1e-9), \
            f"a triangle escapes leaf {i}"
    assert seen.all(), "some triangles belong to no leaf"
    assert len(np.unique(bvh.tri_index)) == bvh.num_triangles, "triangle permutation is not a bijection"
    if mesh is not None:
        tris = mesh.triangles()
        assert bvh.num_triangles == len(tris), "triangle count differs from mesh"
        src = tris[bvh.tri_index]
        assert (np.array_equal(src[:, 0], bvh.tri_v0) and np.array_equal(src[:, 1], bvh.tri_v1)
                and np.array_equal(src[:, 2], bvh.tri_v2)), "permuted triangle data does not match the mesh"


def query_bvh(bvh: BVH, origin, direction, t_max: float = np.inf):
    """Closest hit (t, face) of rays against the tree, on the GPU (bvh.py:189-217).

    One ray (shape (3,)) returns ``(t, face)`` as Python numbers; (R, 3) batches
    return arrays. Miss: ``(inf, -1)``. Hits count for 1e-6 < t <= t_max.
    Numpy/CPU inputs are computed on the current CUDA device; CUDA tensors
    stay on their device.
    """
    single = np.ndim(origin) == 1 if not isinstance(origin, torch.Tensor) else origin.dim() == 1
    on_cuda = isinstance(origin, torch.Tensor) and origin.is_cuda
    dev = origin.device if on_cuda else torch.device("cuda", torch.cuda.current_device())
    o = torch.as_tensor(origin, dtype=torch.float32, device=dev).reshape(-1, 3).contiguous()
    d = torch.as_tensor(direction, dtype=torch.float32, device=dev).reshape(-1, 3).contiguous()
    if o.shape != d.shape:
        raise ValueError(f"origin {tuple(o.shape)} and direction {tuple(d.shape)} differ")
    if not t_max >= 0:
        raise ValueError("t_max must be >= 0")
    nodes, tris = bvh.device_records(dev)
    n = o.shape[0]
    t = torch.empty(n, dtype=torch.float32, device=dev)
    face = torch.empty(n, dtype=torch.int32, device=dev)
    _native.check(_native.lib().mdrt_query_rays(
        ctypes.c_void_p(nodes.data_ptr()), ctypes.c_void_p(tris.data_ptr()), ctypes.c_void_p(o.data_ptr()),
        ctypes.c_void_p(d.data_ptr()), n, float(t_max), ctypes.c_void_p(t.data_ptr()),
        ctypes.c_void_p(face.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    if on_cuda:
        return (t[0], face[0]) if single else (t, face)
    tn, fn = t.cpu().numpy().astype(np.float64), face.cpu().numpy().astype(np.int64)
    return (float(tn[0]), int(fn[0])) if single else (tn, fn)
