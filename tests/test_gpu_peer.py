"""Fused frame gather over peer memory (PeerFrameSink).

Two processes share one GPU: rank 0 owns the (N_total, C, H, W) buffers, rank 1
maps them through CUDA IPC, and each rank's render epilogue stores its env
block straight into rank 0's buffer. Neither rank's kernels wait on the other
(ordering is a host barrier over gloo), so one GPU is a faithful stand-in for
the data path; on a multi-GPU box the same mapping goes over NVLink. Rank 0
checks the gathered batch bitwise against a single-process render of all envs.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import casefile
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sub(case, lo, hi):
    sub = dict(case)
    sub["body_pos"], sub["body_rot"] = case["body_pos"][lo:hi], case["body_rot"][lo:hi]
    sub["num_envs"] = np.array(hi - lo)
    return sub


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2602_03002_b200 as md
        from paper_2602_03002_b200 import distributed as pd
        case = casefile.load(os.path.join(GOLDEN, "render_cfg2_slice.npz"))
        total = int(case["num_envs"])
        start, n = pd.env_slice(total, rank, world)
        scene = casefile.build_scene(_sub(case, start, start + n), md)
        scene.env_offset = start
        sink = pd.PeerFrameSink(scene.frame_shape[1:], total, start, n, dst=0, slots=2)
        cfg = md.SensorConfig(seed=9)
        got = []
        for step in (4, 5):
            obs = md.render_pipeline(scene, sensor=cfg, step=step, out=sink.local(step))
            assert obs.data_ptr() == sink.local(step).data_ptr()
            sink.publish()
            if rank == 0:
                got.append(sink.full(step).cpu().numpy().copy())
        sink.close()
        q.put((rank, got))
        dist.destroy_process_group()
    except Exception as exc:  # surface worker failures to the parent
        import traceback
        q.put((rank, "error: " + repr(exc) + "\n" + traceback.format_exc()))


def test_peer_sink_two_processes_one_gpu(pkg):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=300)
        res[r[0]] = r[1]
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    case = casefile.load(os.path.join(GOLDEN, "render_cfg2_slice.npz"))
    full = casefile.build_scene(case, pkg)
    cfg = pkg.SensorConfig(seed=9)
    for k, step in enumerate((4, 5)):
        ref = pkg.render_pipeline(full, sensor=cfg, step=step).cpu().numpy()
        assert np.array_equal(res[0][k], ref)


def test_peer_sink_single_rank(pkg):
    """World size 1: the sink is a local double buffer; render writes into it in place."""
    from paper_2602_03002_b200 import distributed as pd
    case = casefile.load(os.path.join(GOLDEN, "render_cfg2_slice.npz"))
    scene = casefile.build_scene(case, pkg)
    n = scene.num_envs
    sink = pd.PeerFrameSink(scene.frame_shape[1:], n, 0, n)
    assert sink.slots == 2 and sink.local(0).device == scene.device
    out = pkg.render_pipeline(scene, sensor=pkg.SensorConfig(seed=1), step=2, out=sink.local(0))
    ref = pkg.render_pipeline(scene, sensor=pkg.SensorConfig(seed=1), step=2)
    assert torch.equal(sink.full(0), ref) and out.data_ptr() == sink.full(0).data_ptr()
    sink.close()
