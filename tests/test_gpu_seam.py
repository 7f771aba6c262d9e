"""The reference's backend seam driven with the arguments the LIVE reference passes.

tests/golden/seam_capture.npz holds one recorded call of the numba
``render_batch`` made by ``multidepth.render`` (kernels/__init__.py:53-60,
scene.py:332-348): the real FlatGeometry (median-split forest, leaf-ordered
triangles, scene.py:49-147), f64 body/camera poses of parented cameras with
per-env camera randomisation, the (N,C,H,W,3) FOV-randomised ray grids, d_max,
and the output the reference wrote. The same call is replayed through
``get_render_fn("cuda")`` (the drop-in) into a fresh numpy ``out``.
"""

import os
import types

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _capture():
    z = np.load(os.path.join(GOLDEN, "seam_capture.npz"))
    flat = types.SimpleNamespace(**{k[5:]: z[k] for k in z.files if k.startswith("flat_")})
    args = {k: z[k] for k in z.files if not k.startswith("flat_")}
    return flat, args


def _check(got, ref, d_max):
    dmax = np.asarray(d_max, np.float32).reshape(1, -1, 1, 1)
    diff = np.abs(got.astype(np.float64) - ref)
    flips = (got < dmax) != (ref < dmax)
    assert flips.sum() <= 1e-4 * got.size + 1, f"{flips.sum()} hit/miss flips"
    assert ((diff > 1e-4) & ~flips).sum() <= 1e-4 * got.size + 1
    return diff


def test_seam_replays_live_reference_call(pkg):
    from paper_2602_03002_b200 import kernels
    flat, a = _capture()
    name, render_batch = kernels.get_render_fn("cuda")
    assert name == "cuda"
    out = np.empty(a["out"].shape, np.float32)          # fresh, as scene.render allocates it
    render_batch(flat, a["body_pos"], a["body_rot"], a["cam_pos"], a["cam_rot"], a["ray_dirs"], a["ray_scale"],
                 a["d_max"], bool(a["early"]), out, 4)
    diff = _check(out, a["out"], a["d_max"])
    assert diff[(a["out"] < 10.0)].max() < 1e-4
    # misses are exactly float32(d_max)
    miss = a["out"] >= np.float32(a["d_max"][0])
    assert np.array_equal(out[miss], a["out"][miss])


def test_seam_ray_grid_cache_tracks_the_callers_arrays(pkg):
    """Repeated calls with the same grid arrays reuse the device copy; a different
    array, or the same array changed in place, is uploaded again."""
    from paper_2602_03002_b200 import kernels
    from paper_2602_03002_b200.kernels import cuda_backend as cb
    flat, a = _capture()
    _, render_batch = kernels.get_render_fn("cuda")
    dirs, scale = a["ray_dirs"].copy(), a["ray_scale"].copy()

    def call(d, s):
        out = np.empty(a["out"].shape, np.float32)
        render_batch(flat, a["body_pos"], a["body_rot"], a["cam_pos"], a["cam_rot"], d, s, a["d_max"],
                     bool(a["early"]), out)
        return out

    first = call(dirs, scale)
    cached = {id(t) for _, _, t in cb._grid_cache[0]}
    second = call(dirs, scale)
    assert {id(t) for _, _, t in cb._grid_cache[0]} == cached      # no re-upload
    assert np.array_equal(first, second)
    # in-place change of the caller's grid: all rays of env 0 flipped upwards -> different image
    dirs[0, :, :, :, 1] *= -1.0
    third = call(dirs, scale)
    assert not np.array_equal(third[0], first[0])
    assert np.array_equal(third[1:], first[1:])
    # a brand-new array with the original values gives the original image again
    fourth = call(a["ray_dirs"].copy(), scale)
    assert np.array_equal(fourth, first)
