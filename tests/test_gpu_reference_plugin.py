"""The drop-in, end to end inside the reference: INTEGRATION.md section 1 applied to the
reference package itself (pip-installed unmodified into baseline/_ref).

The reference's backend registry (multidepth/kernels/__init__.py:53-60) gets the
"cuda" entry the integration guide describes, and the reference's own
``render(scene, backend="cuda")`` (scene.py:332-348: its camera_world_poses, its
ray-grid cache, its FlatGeometry, its freshly allocated numpy ``out``) drives this
repo's CUDA backend. The result is compared with the same reference call on its
numpy brute-force backend (numpy_backend.py:31-111), on parented, randomised cameras.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture()
def ref(monkeypatch):
    if not os.path.isdir(os.path.join(REF, "multidepth")):
        pytest.skip("reference not installed in baseline/_ref (build() installs it)")
    monkeypatch.syspath_prepend(REF)
    monkeypatch.setenv("NUMBA_CACHE_DIR", "/tmp/mdrt_numba_cache")
    import multidepth
    from multidepth import kernels as mk
    from paper_2602_03002_b200.kernels import cuda_backend
    original = mk.get_render_fn

    def get_render_fn(backend=None):        # the two-line registry change of INTEGRATION.md section 1
        if backend is not None and backend.strip().lower() == "cuda":
            return "cuda", cuda_backend.render_batch
        return original(backend)

    monkeypatch.setattr(mk, "BACKENDS", tuple(mk.BACKENDS) + ("cuda",))
    monkeypatch.setattr(mk, "get_render_fn", get_render_fn)
    yield multidepth
    for name in [m for m in sys.modules if m == "multidepth" or m.startswith("multidepth.")]:
        del sys.modules[name]


def test_reference_render_drives_the_cuda_backend(ref):
    f32 = lambda x: np.asarray(x, np.float64).astype(np.float32).astype(np.float64)  # noqa: E731
    rng = np.random.default_rng(11)
    links = [ref.make_box(size=(0.3, 0.2, 0.4)), ref.make_icosphere(0.15, subdivisions=2)]
    bodies = [(f"l{i}", ref.TriMesh(f32(m.vertices), m.faces, frame="body-local")) for i, m in enumerate(links)]
    xs = np.linspace(-3, 3, 25)
    gx, gy = np.meshgrid(xs, xs)
    a = (np.arange(24)[:, None] * 25 + np.arange(24)[None, :]).ravel()
    faces = np.concatenate([np.column_stack([a, a + 1, a + 26]), np.column_stack([a, a + 26, a + 25])])
    terrain = ref.TriMesh(f32(np.column_stack([gx.ravel(), gy.ravel(), 0.15 * np.sin(1.3 * gx.ravel())])), faces)
    mount = ref.look_at_pose([0.1, 0.0, 0.3], [1.0, 0.0, -0.4])
    cams = [ref.CameraModel(width=24, height=16, hfov_deg=90.0, vfov_deg=60.0, d_max=6.0, mount=mount,
                            parent_body=0, name="front"),
            ref.CameraModel(width=24, height=16, hfov_deg=90.0, vfov_deg=60.0, d_max=5.0,
                            mount=ref.look_at_pose([-0.1, 0.0, 0.3], [-1.0, 0.2, -0.5]), parent_body=0, name="back")]
    n = 3
    scene = ref.Scene(num_envs=n, bodies=bodies, cameras=cams, terrain=terrain)
    pos = f32(np.column_stack([rng.uniform(-1, 1, n), rng.uniform(-1, 1, n), np.full(n, 0.9)]))
    pos = np.stack([pos, pos + np.array([0.5, 0.1, -0.2])], axis=1)
    rot = rng.normal(size=(n, 2, 4))
    rot = f32(rot / np.linalg.norm(rot, axis=-1, keepdims=True))
    scene.set_body_poses(pos, rot)
    off = ref.sample_camera_offsets(ref.CameraRandomization(seed=4), n, 2)
    scene.set_camera_randomization(f32(off[0]), f32(off[1] / np.linalg.norm(off[1], axis=-1, keepdims=True)),
                                   f32(off[2]))
    got = ref.render(scene, backend="cuda").data
    want = ref.render(scene, backend="numpy").data
    assert isinstance(got, np.ndarray) and got.dtype == np.float32 and got.shape == want.shape
    dmax = np.array([6.0, 5.0], np.float32).reshape(1, 2, 1, 1)
    flips = (got < dmax) != (want < dmax)
    diff = np.abs(got.astype(np.float64) - want)
    assert flips.sum() <= 1 and (diff[~flips] > 1e-4).sum() <= 1, (flips.sum(), (diff > 1e-4).sum())
    assert (want < dmax).mean() > 0.3                       # the scene is mostly hits
