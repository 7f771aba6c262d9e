"""Multi-GPU readiness on the B200.

* NCCL paths (>= 2 visible GPUs, skipped otherwise): gather_frames to a rank and
  to all ranks with even and uneven env slices, and PeerFrameSink whose publish()
  is a stream-ordered NCCL all_reduce, each checked bitwise against a
  single-process render of all envs.
* bench.py's launcher: `--gpus 2` re-launches itself under torch.distributed.run;
  on a one-GPU box it fails loudly, and with MDRT_BENCH_SHARE_GPU=1 it runs two
  ranks on the one GPU (gloo; a control-flow check: kernels of the two ranks
  never wait on each other) and rank 0 prints n_gpus 2.
* a small single-GPU bench run carries the roofline / parity / cpu_baseline objects.
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import casefile
from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu
two_gpus = pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs for NCCL")


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


def _nccl_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        import paper_2602_03002_b200 as md
        from paper_2602_03002_b200 import distributed as pd
        case = casefile.load(os.path.join(GOLDEN, "render_cfg2_slice.npz"))
        cfg = md.SensorConfig(seed=9)
        out = {}
        for total in (int(case["num_envs"]), int(case["num_envs"]) - 1):     # even, then uneven slices
            start, n = pd.env_slice(total, rank, world)
            scene = casefile.build_scene(_sub(case, start, start + n), md, device=dev)
            scene.env_offset = start
            obs = md.render_pipeline(scene, sensor=cfg, step=4)
            full_all = pd.gather_frames(obs, dst=None)
            full_dst = pd.gather_frames(obs, dst=0)
            out[total] = (full_all.cpu().numpy(), None if full_dst is None else full_dst.cpu().numpy())
            # fused path: every rank's epilogue stores into rank 0's buffer over peer memory
            sink = pd.PeerFrameSink(scene.frame_shape[1:], total, start, n, dst=0, slots=2, device=dev)
            for step in (4, 5):
                md.render_pipeline(scene, sensor=cfg, step=step, out=sink.local(step))
                sink.publish()
                if rank == 0:
                    out[(total, step)] = sink.full(step).cpu().numpy().copy()
            sink.close()
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as exc:  # surface worker failures to the parent
        import traceback
        q.put((rank, "error: " + repr(exc) + "\n" + traceback.format_exc()))


@two_gpus
def test_nccl_gather_and_peer_sink(pkg):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_nccl_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=600)
        res[r[0]] = r[1]
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    case = casefile.load(os.path.join(GOLDEN, "render_cfg2_slice.npz"))
    cfg = pkg.SensorConfig(seed=9)
    for total in (int(case["num_envs"]), int(case["num_envs"]) - 1):
        scene = casefile.build_scene(_sub(case, 0, total), pkg)
        ref = {s: pkg.render_pipeline(scene, sensor=cfg, step=s).cpu().numpy() for s in (4, 5)}
        for r in range(world):
            assert np.array_equal(res[r][total][0], ref[4])      # NCCL all_gather (padded when uneven)
        assert np.array_equal(res[0][total][1], ref[4])          # NCCL P2P gather to rank 0
        assert res[1][total][1] is None
        for s in (4, 5):
            assert np.array_equal(res[0][(total, s)], ref[s])    # fused peer stores, NCCL publish


def _bench(args, env_extra=None, timeout=900):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK",
                                                               "MDRT_BENCH_SHARE_GPU")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=env, timeout=timeout, cwd=ROOT)


def _line(res):
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    return lines[0]


@pytest.mark.skipif(torch.cuda.device_count() >= 2, reason="checks the failure on a one-GPU box")
def test_bench_two_gpus_fails_loudly_on_one_gpu():
    res = _bench(["--gpus", "2", "--steps", "3", "--warmup", "3", "--envs", "64"])
    assert res.returncode != 0 and "needs 2 visible GPUs" in res.stderr


def test_bench_two_ranks_share_mode():
    small = ["--steps", "3", "--warmup", "3", "--envs", "64", "--no-cpu-baseline", "--parity-envs", "8"]
    d = _line(_bench(["--gpus", "2", *small], {"MDRT_BENCH_SHARE_GPU": "1"}))
    assert d["n_gpus"] == 2 and "share_gpu" in d
    assert d["config"]["global_envs"] == 128 and d["config"]["envs_per_gpu"] == 64
    assert d["parity"]["flips_within_1e-4"] or d["parity"]["hit_miss_flips"]["total"] <= 1


def test_bench_single_gpu_line():
    d = _line(_bench(["--steps", "3", "--warmup", "3", "--envs", "256", "--cpu-seconds", "2", "--parity-envs", "64"]))
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] == 9
    r = d["roofline"]
    assert r["bound"] == "l2" and r["peak"] == r["l2_probe_gbs"] and 0 < r["frac"] < 1.5
    p = d["parity"]
    assert p["pixels"] == 64 * 2 * 64 * 48
    assert p["in_band_over_1e-4"] <= 2 and p["hit_miss_flips"]["total"] <= 2
    s = p["sensor"]
    assert s["noisy_mismatch_where_clean_equal"] == 0
    assert s["dropout_rate_rel_diff"] < 0.01 and s["residual_std_rel_diff"] < 0.01
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


@pytest.mark.parametrize("cfg", ["cfg3", "paper"])
def test_bench_parity_other_configs(cfg):
    """The in-run oracle parity of the bench on the stepping-stone (4 cameras, raised arms)
    and paper (240x135 + fused 5x5 min-pool) workloads: the north star's criteria."""
    d = _line(_bench(["--config", cfg, "--steps", "3", "--warmup", "3", "--envs", "64", "--no-cpu-baseline",
                      "--parity-envs", "32"]))
    p = d["parity"]
    assert p["flips_within_1e-4"] and p["over_1e-4_frac"] <= 1e-4
    s = p["sensor"]
    assert s["noisy_mismatch_where_clean_equal"] == 0
    assert s["dropout_rate_rel_diff"] < 0.01 and s["residual_std_rel_diff"] < 0.01
    assert d["roofline"]["bound"] == "l2"
