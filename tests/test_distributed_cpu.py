"""World-size-2 gloo tests of the multi-GPU host logic (runs on CPU).

Covers the N>1 path of bench.py / INTEGRATION.md section 3: contiguous env
slices, per-rank slices of the globally keyed per-env draws (latencies,
camera offsets, sensor noise) and the optional frame gather.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_03002_b200 import distributed as pd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_env_slice_partitions():
    for total in (1, 7, 4096, 32768, 1001):
        for world in (1, 2, 3, 8):
            if world > total:
                continue
            spans = [pd.env_slice(total, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (s0, c0), (s1, _) in zip(spans, spans[1:]):
                assert s0 + c0 == s1
            assert sum(c for _, c in spans) == total
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        pd.env_slice(10, 2, 2)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import oracle as orc
        import paper_2602_03002_b200 as md
        total = 10
        start, n = pd.env_slice(total, rank, world)
        # globally keyed per-env draws, sliced per rank, equal the single-process draws
        lat = md.sample_latencies(md.SensorConfig(seed=3), total)[start:start + n]
        off = [np.asarray(a)[start:start + n] for a in md.sample_camera_offsets(md.CameraRandomization(seed=2),
                                                                                total, 2)]
        # sensor noise on this rank's slice with its global env offset (oracle = reference algorithm)
        depth = np.full((n, 2, 4, 6), 2.5, np.float32)
        noisy = orc.apply_noise_dropout(depth, noise_scale=0.1, dropout_p=0.2, seed=5, d_max=[8.0, 9.0],
                                        step=3, env_offset=start)
        t = torch.from_numpy(noisy)
        full_all = pd.gather_frames(t, dst=None)
        full_dst = pd.gather_frames(t, dst=0)
        # uneven slices (11 envs over 2 ranks: 6 + 5) gather in rank order too
        s2, n2 = pd.env_slice(11, rank, world)
        u = torch.arange(s2 * 6, (s2 + n2) * 6, dtype=torch.float32).reshape(n2, 1, 2, 3)
        ua = pd.gather_frames(u, dst=None)
        ud = pd.gather_frames(u, dst=0, sizes=[pd.env_slice(11, r, world)[1] for r in range(world)])
        uneven = (ua.numpy(), None if ud is None else ud.numpy())
        q.put((rank, lat, off, full_all.numpy(), None if full_dst is None else full_dst.numpy(), uneven))
        dist.destroy_process_group()
    except Exception as exc:  # surface worker failures to the parent
        q.put((rank, "error", repr(exc), None, None, None))


def test_two_rank_gloo_slices_and_gather():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r][1], str), res[r][2]
    import paper_2602_03002_b200 as md
    from oracle import oracle as orc
    lat_full = md.sample_latencies(md.SensorConfig(seed=3), 10)
    off_full = md.sample_camera_offsets(md.CameraRandomization(seed=2), 10, 2)
    assert np.array_equal(np.concatenate([res[0][1], res[1][1]]), lat_full)
    for k in range(3):
        assert np.array_equal(np.concatenate([res[0][2][k], res[1][2][k]]), np.asarray(off_full[k]))
    ref = orc.apply_noise_dropout(np.full((10, 2, 4, 6), 2.5, np.float32), noise_scale=0.1, dropout_p=0.2,
                                  seed=5, d_max=[8.0, 9.0], step=3)
    for r in range(world):
        assert np.array_equal(res[r][3], ref)          # all_gather on every rank
    assert np.array_equal(res[0][4], ref)              # gather to rank 0
    assert res[1][4] is None
    full11 = np.arange(11 * 6, dtype=np.float32).reshape(11, 1, 2, 3)
    for r in range(world):
        assert np.array_equal(res[r][5][0], full11)   # uneven all_gather (padded blocks, sliced)
    assert np.array_equal(res[0][5][1], full11)        # uneven gather to rank 0
    assert res[1][5][1] is None


def test_peer_block_offsets_and_pointer_views():
    """Host logic of the fused peer-memory gather: block offsets and raw-pointer tensor views."""
    spans = [pd.env_slice(4096, r, 8) for r in range(8)]
    per_env = 2 * 48 * 64
    offs = [pd.peer_block_offsets(4096, s, c, per_env) for s, c in spans]
    assert offs[0] == (0, 4 * 512 * per_env)
    for (o0, l0), (o1, _) in zip(offs, offs[1:]):
        assert o0 + l0 == o1
    with pytest.raises(ValueError):
        pd.peer_block_offsets(10, 8, 3, per_env)
    buf = np.arange(10 * 6, dtype=np.float32)
    keep = []
    off, _ = pd.peer_block_offsets(10, 4, 3, 6)
    view = pd.wrap_pointer(buf.ctypes.data + off, (3, 2, 3), torch.device("cpu"), keep)
    assert view.shape == (3, 2, 3) and view.is_contiguous()
    assert np.array_equal(view.numpy().ravel(), buf[24:42])
    view.fill_(-1.0)
    assert np.all(buf[24:42] == -1.0) and buf[23] == 23.0 and buf[42] == 42.0


def test_numa_helpers_cpu():
    """cpulist parsing, and the NUMA binder degrades to 'unknown node, all CPUs' without a GPU."""
    assert pd._cpulist("0-3,8,10-11\n") == {0, 1, 2, 3, 8, 10, 11}
    assert pd._cpulist("") == set()
    before = os.sched_getaffinity(0)
    info = pd.bind_to_gpu_numa(torch.device("cuda", 0)) if not torch.cuda.is_available() else None
    if info is not None:
        assert info["node"] is None and info["cpus"] == len(before)
        assert os.sched_getaffinity(0) == before
