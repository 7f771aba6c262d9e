"""Lifetime, ownership and stream-ordering rules of the GPU path:

* a CapturedStep keeps every buffer its graph reads by pointer alive, refuses
  to replay after the scene replaced one of them, and hands the context's single
  device step state to a newer CapturedStep;
* re-randomising cameras writes the scene's buffers in place, so a captured
  graph sees the new offsets;
* renders of one scene on different streams are ordered by the context
  (mdrt_render / mdrt_order_begin/end), so they never share scratch concurrently;
* the fused block minimum refuses a negative side-mask fill.
"""

import gc
import os

import numpy as np
import pytest
import torch

import casefile
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _scene(pkg):
    case = casefile.load(os.path.join(GOLDEN, "render_cfg2_slice.npz"))
    return case, casefile.build_scene(case, pkg)


def test_captured_step_keeps_outputs_alive(pkg):
    from paper_2602_03002_b200.pipeline import CapturedStep
    case, scene = _scene(pkg)
    n, c, h, w = scene.frame_shape
    ds = torch.empty((n, c, h // 4, w // 4), device="cuda")
    cap = CapturedStep(scene, sensor=pkg.SensorConfig(seed=1), ds_out=ds, downsample_factor=4)
    ptr = ds.data_ptr()
    del ds
    gc.collect()
    torch.cuda.empty_cache()
    junk = [torch.full((n, c, h // 4, w // 4), 7.0, device="cuda") for _ in range(4)]   # would reuse freed memory
    cap.replay()
    torch.cuda.synchronize()
    assert cap.ds_out.data_ptr() == ptr
    assert all(bool((j == 7.0).all()) for j in junk)     # nobody else's memory was written
    ref = pkg.downsample_min(cap.out, 4)
    assert torch.equal(cap.ds_out, ref)


def test_captured_step_sees_in_place_rerandomisation(pkg):
    from paper_2602_03002_b200.pipeline import CapturedStep
    case, s_graph = _scene(pkg)
    _, s_eager = _scene(pkg)
    n, c = s_graph.num_envs, s_graph.num_cameras
    off = pkg.sample_camera_offsets(pkg.CameraRandomization(seed=2), n, c)
    s_graph.set_camera_randomization(*off)
    cap = CapturedStep(s_graph)
    for episode in range(3):
        off = pkg.sample_camera_offsets(pkg.CameraRandomization(seed=2), n, c, episode=episode)
        s_graph.set_camera_randomization(*off)           # same buffers, new values
        s_eager.set_camera_randomization(*off)
        got = cap.replay()
        ref = pkg.render(s_eager).data
        assert torch.equal(got, ref), f"episode {episode}"


def test_captured_step_refuses_stale_pointers_and_lost_state(pkg):
    from paper_2602_03002_b200.pipeline import CapturedStep
    case, scene = _scene(pkg)
    cap = CapturedStep(scene)
    cap.replay()
    scene.set_camera_randomization(*pkg.sample_camera_offsets(pkg.CameraRandomization(seed=1),
                                                                scene.num_envs, scene.num_cameras))
    with pytest.raises(RuntimeError, match="replaced after capture"):
        cap.replay()
    cap2 = CapturedStep(scene)
    cap2.replay()
    scene.clear_camera_randomization()
    with pytest.raises(RuntimeError):
        cap2.replay()
    cap3 = CapturedStep(scene)
    cap4 = CapturedStep(scene)                           # takes over the device step state
    with pytest.raises(RuntimeError, match="no longer owns"):
        cap3.replay()
    cap4.replay()
    cap4.close()
    with pytest.raises(RuntimeError):
        cap4.replay()


def test_renders_on_two_streams_are_ordered(pkg):
    """Renders of one scene issued on two streams with no user synchronisation (same
    poses, different sensor seeds) equal the serial renders: the context makes each
    call wait for the previous call on the other stream before it rewrites the
    shared per-step scratch (view/link records, tile counters)."""
    case, scene = _scene(pkg)
    want = [pkg.render_pipeline(scene, sensor=pkg.SensorConfig(seed=k), step=k).clone() for k in range(8)]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for st in streams:
        st.wait_stream(torch.cuda.current_stream())
    outs = [torch.empty(scene.frame_shape, device="cuda") for _ in range(8)]
    for k in range(8):
        with torch.cuda.stream(streams[k % 2]):
            pkg.render_pipeline(scene, sensor=pkg.SensorConfig(seed=k), step=k, out=outs[k])
    torch.cuda.synchronize()
    for k in range(8):
        assert torch.equal(outs[k], want[k]), f"call {k}"


def test_fused_downsample_rejects_negative_rsm_fill(pkg):
    case, scene = _scene(pkg)
    n, c, h, w = scene.frame_shape
    ds = torch.empty((n, c, h // 4, w // 4), device="cuda")
    rsm = pkg.RsmConfig(seed=5, fill_low=-1.0)
    modes = np.ones((n, c), np.int32)
    with pytest.raises(ValueError, match="rsm_fill_low"):
        pkg.render_pipeline(scene, rsm=rsm, rsm_modes=modes, ds_out=ds, downsample_factor=4)
