"""Benchmark: depth rays/s of the multi-depth pipeline on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

One *step* = one pass of the hot path over one batch: for every env slice of
this rank, camera poses from link poses (prologue), a ray per (env, cam,
pixel) through the G1-proxy link BVHs (link frames) and the terrain BVH, the
sensor model (noise, dropout, clamp) and the latency ring write + delayed
read -- i.e. ``render_pipeline`` (render -> apply_noise_dropout ->
FrameBuffer.push -> fetch_delayed_batch of the reference).

Default workload = config 2 of BASELINE.json: 4096 envs x 2 cams x 64x48 per
GPU (weak scaling; 8 GPUs = config 4's 32768 envs), 259,200-triangle
slope/stairs tile field, 30-link G1 proxy, full noise/dropout/latency.

``value``: rays/s with inputs resident in HBM (per-step device pose update +
pipeline), CUDA-event timed per step with an L2 flush (256 MiB write) between
steps. ``e2e``: the same through the public API with host buffers: pinned
host poses -> H2D, pipeline, D2H of the observation, every step.
``--impl reference``: the CPU restatement of the reference path
(oracle/oracle.c, OpenMP on all host cores) on a bounded env sample.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "depth rays/sec at 4096 envs x 2 cams, 1/2/4/8 B200; % of L2/HBM BW roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2", choices=["cfg2", "cfg3", "cfg5", "cfg5_1m", "paper"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--envs", type=int, default=None, help="envs per GPU (default: config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--pose-sets", type=int, default=8)
    ap.add_argument("--gather", action="store_true",
                    help="N>1: also time the step + gather of all observations to rank 0 "
                         "(NCCL, and the fused peer-memory store path)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32)


def cfg_envs(name):
    return {"cfg2": 4096, "cfg3": 4096, "cfg5": 4096, "cfg5_1m": 4096, "paper": 1024}[name]


def workload_desc(name):
    return {
        "cfg2": "4096 envs x 2 cams (front+back) 64x48 per GPU, 3x3 slope/stairs tiles (259,200 tris, the reference "
                "generate_terrain meshes), 30-link G1 proxy (8,060 tris), full noise/dropout/latency",
        "cfg3": "4096 envs x 4 cams 64x48, stepping stones 25cm/60cm (8,750 tris, the reference generate_terrain "
                "mesh), arms raised, full sensor",
        "cfg5": "4096 envs x 2 cams 160x120, 1300x1300-node rolling terrain (3,373,802 tris, BVH ~270 MB > 2x L2), "
                "full sensor",
        "cfg5_1m": "4096 envs x 2 cams 160x120, 708x708-node rolling terrain (999,698 tris), full sensor",
        "paper": "1024 envs x 2 cams 240x135 (paper native res) on the cfg2 tiles, full sensor + latency, "
                 "fused 5x5 block-min to the 48x27 policy input",
    }[name]


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampler during the timed region)
# ---------------------------------------------------------------------------
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, gpu_index: int):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.fh, stderr=subprocess.DEVNULL)
            # nvidia-smi takes a few hundred ms to start: wait for its first sample so
            # short timed regions are still covered
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 3.0 and os.path.getsize(self.path) == 0:
                time.sleep(0.02)
        except Exception:
            self.proc = None

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        time.sleep(0.06)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                bits = int(parts[2], 16)
            except ValueError:
                continue
            for b, nm in REASON_BITS.items():
                if bits & b and nm != "gpu_idle":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the oracle restatement on host cores
# ---------------------------------------------------------------------------

def build_oracle_workload(name, n_sample, world_envs):
    from oracle import oracle as orc
    from paper_2602_03002_b200 import synth, sensor
    w = synth.config(name, world_envs)
    bodies = [(f32(m.vertices).astype(np.float64), m.faces) for _, m in w.bodies]
    terrain = (f32(w.terrain.mesh.vertices).astype(np.float64), w.terrain.mesh.faces)
    cams = [dict(width=c.width, height=c.height, hfov_deg=c.hfov_deg, vfov_deg=c.vfov_deg, d_max=c.d_max,
                 mount_pos=c.mount.translation, mount_rot=c.mount.rotation, parent=c.parent_body)
            for c in w.cameras]
    sc = orc.OracleScene(bodies, terrain, cams)
    return orc, w, sc


def run_cpu_sample(orc, w, sc, n_sample, step, threads, buf_state, delays, cfg):
    """render + apply_noise_dropout + FrameBuffer push/fetch on n_sample envs (oracle port)."""
    sl = slice(0, n_sample)
    bp, bq = w.poses(step, sl)
    bp, bq = f32(bp).astype(np.float64), f32(bq).astype(np.float64)
    t0 = time.perf_counter()
    depth = sc.render(bp, bq, threads=threads)
    buf_state[2].append(time.perf_counter() - t0)
    dmax = np.array([c["d_max"] for c in sc.cameras])
    noisy = orc.apply_noise_dropout(depth, noise_scale=cfg.noise_scale, dropout_p=cfg.dropout_p, seed=cfg.seed,
                                    d_max=dmax, step=step, threads=threads)
    times, frames = buf_state[0], buf_state[1]
    times.append(step * 0.02)
    frames.append(noisy)
    if len(times) > 8:
        times.pop(0)
        frames.pop(0)
    idx = orc.frame_select(np.array(times), step * 0.02, delays[:n_sample])
    obs = np.stack([frames[k][e] for e, k in enumerate(idx)])
    return obs


def cpu_measure(name, steps, warmup, seconds_target, threads):
    """Returns (rays_per_s, sample_desc, per-step list)."""
    from paper_2602_03002_b200 import sensor
    cfg = sensor.SensorConfig(noise_scale=0.1, dropout_p=0.05, seed=0)
    probe_n = 16
    orc, w, sc = build_oracle_workload(name, probe_n, cfg_envs(name))
    delays = sensor.sample_latencies(sensor.SensorConfig(max_delay=0.1, seed=3), w.num_envs)
    rays_per_env = len(w.cameras) * w.cameras[0].width * w.cameras[0].height
    # size the sample so each step costs ~seconds_target / steps
    state = ([], [], [])
    t0 = time.perf_counter()
    run_cpu_sample(orc, w, sc, probe_n, 0, threads, state, delays, cfg)
    per_env = (time.perf_counter() - t0) / probe_n
    n_sample = int(max(8, min(w.num_envs, seconds_target / max(steps, 1) / max(per_env, 1e-6))))
    state = ([], [], [])
    for s in range(warmup):
        run_cpu_sample(orc, w, sc, n_sample, s, threads, state, delays, cfg)
    state[2].clear()
    times = []
    for s in range(steps):
        t0 = time.perf_counter()
        run_cpu_sample(orc, w, sc, n_sample, warmup + s, threads, state, delays, cfg)
        times.append(time.perf_counter() - t0)
    rays = n_sample * rays_per_env
    value = rays * len(times) / sum(times)
    desc = (f"{n_sample} of {w.num_envs} envs x {len(w.cameras)} cams x {w.cameras[0].width}x"
            f"{w.cameras[0].height} per step (render + noise/dropout + latency), {len(times)} steps")
    split = {"render_plus_sensor_mean": value, "render_plus_sensor_best": rays / min(times),
             "render_only_mean": rays * len(state[2]) / sum(state[2]), "render_only_best": rays / min(state[2])}
    return value, desc, times, split


def cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as orc
    threads = orc.max_threads()
    value, desc, _, split = cpu_measure(args.config, args.steps, args.warmup, args.cpu_seconds * 3, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(args.config), "impl_detail": "oracle/oracle.c (C restatement of "
                   "multidepth numba_backend._render_kernel + sensor + FrameBuffer), OpenMP"},
        "cpu_baseline": {"value": value, "unit": "rays/s", "cores": threads, "kind": "port", "sample": desc,
                         "cpu": cpu_info(), "split": split},
        "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    import torch
    import torch.distributed as dist
    import paper_2602_03002_b200 as md
    from paper_2602_03002_b200 import _native, synth
    from paper_2602_03002_b200 import distributed as pdist

    rank, world, local = dist_env()
    if world != args.gpus:
        args.gpus = world if world > 1 else args.gpus
    # MDRT_BENCH_SHARE_GPU=1 (control-flow check only, never a measurement): ranks share
    # the visible GPUs round-robin and talk over gloo, so the N>1 code path can be
    # exercised on a one-GPU box; kernels of different ranks never wait on each other.
    share = os.environ.get("MDRT_BENCH_SHARE_GPU") == "1"
    gpu = local % torch.cuda.device_count() if share else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    n = args.envs or cfg_envs(args.config)
    total_envs = n * world
    w = synth.config(args.config, total_envs)
    env0, n_rank = pdist.env_slice(total_envs, rank, world)
    assert n_rank == n
    bodies = [(nm, md.TriMesh(f32(m.vertices).astype(np.float64), m.faces, frame="body-local"))
              for nm, m in w.bodies]
    terrain = md.TriMesh(f32(w.terrain.mesh.vertices).astype(np.float64), w.terrain.mesh.faces)
    t_build = time.perf_counter()
    scene = md.Scene(n, bodies=bodies, cameras=w.cameras, terrain=terrain, device=dev, env_offset=env0)
    t_build = time.perf_counter() - t_build
    C, H, W = scene.num_cameras, scene.height, scene.width
    rays_per_step = n * C * H * W

    # camera randomisation + latency per env (global counters, sliced to this rank)
    off = md.sample_camera_offsets(md.CameraRandomization(seed=3), total_envs, C)
    scene.set_camera_randomization(*(np.asarray(a)[env0:env0 + n] for a in off))
    sens = md.SensorConfig(noise_scale=0.1, dropout_p=0.05, max_delay=0.1, seed=0)
    delays_np = md.sample_latencies(md.SensorConfig(max_delay=0.1, seed=3), total_envs)[env0:env0 + n]
    delays = torch.from_numpy(np.ascontiguousarray(delays_np)).to(dev)
    dt = 0.02

    # per-step link poses: P distinct sets (host FK once), device-resident and pinned-host copies
    P = args.pose_sets
    pose_host = []
    for s in range(P):
        p, q = w.poses(s, slice(env0, env0 + n))
        pose_host.append((torch.from_numpy(f32(p)).pin_memory(), torch.from_numpy(f32(q)).pin_memory()))
    pose_dev = [(p.to(dev), q.to(dev)) for p, q in pose_host]

    buf = md.FrameBuffer(capacity=8)
    out = torch.empty(scene.frame_shape, dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    step_id = [0]

    # paper pipeline: the policy consumes the fused 5x5 block minimum of the observation
    ds = None
    if args.config == "paper":
        ds = torch.empty((n, C, H // 5, W // 5), dtype=torch.float32, device=dev)

    def step(poses):
        s = step_id[0]
        scene.set_body_poses(poses[0], poses[1], validate=False)
        md.render_pipeline(scene, sensor=sens, step=s, frame_buffer=buf, timestamp=s * dt, delays=delays,
                           out=out, ds_out=ds)
        step_id[0] += 1

    # ---- per-ray work counts (untimed, MDRT_COUNT) ----
    ctr = torch.zeros(4, dtype=torch.int64, device=dev)
    scene.set_body_poses(*pose_dev[0], validate=False)
    md.render(scene, counters=ctr)
    torch.cuda.synchronize()
    nodes_per_ray, tris_per_ray, link_nodes_per_ray, link_traces_per_ray = (x / rays_per_step for x in ctr.tolist())

    for i in range(args.warmup):
        step(pose_dev[i % P])
    torch.cuda.synchronize()

    # ---- timed: device-resident inputs ----
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    wall0 = time.perf_counter()
    for i in range(args.steps):
        flush.fill_(float(i))
        starts[i].record(stream)
        step(pose_dev[i % P])
        ends[i].record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)

    # ---- same step replayed as a captured CUDA graph (device step state) ----
    from paper_2602_03002_b200.pipeline import CapturedStep
    cap = CapturedStep(scene, sensor=sens, frame_buffer=buf, delays=delays, dt=dt, first_step=step_id[0], out=out,
                       ds_out=ds)
    for i in range(args.warmup):
        scene.body_positions.copy_(pose_dev[i % P][0])
        scene.body_rotations.copy_(pose_dev[i % P][1])
        cap.replay()
    gstart = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    gend = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.fill_(float(i))
        gstart[i].record(stream)
        scene.body_positions.copy_(pose_dev[i % P][0])
        scene.body_rotations.copy_(pose_dev[i % P][1])
        cap.replay()
        gend[i].record(stream)
    torch.cuda.synchronize()
    graph_ms = sum(s.elapsed_time(e) for s, e in zip(gstart, gend))
    step_id[0] = cap.next_step

    # ---- render-kernel-only timing (roofline of the dominant kernel) ----
    kstart = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kend = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    pstart = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    pend = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    from paper_2602_03002_b200.pipeline import _pipeline_args
    for i in range(args.steps):
        s = step_id[0]
        scene.set_body_poses(*pose_dev[i % P], validate=False)
        # the benchmarked step's own arguments (sensor + latency ring + fused downsample), launched
        # as two phases so the render kernel is timed alone
        a, keep = _pipeline_args(scene, out, sensor=sens, step=s, frame_buffer=buf, timestamp=s * dt,
                                 delays=delays, early_termination=True, clean_out=None, counters=None, rsm=None,
                                 rsm_modes=None, ds_out=ds, downsample_factor=5, host_ds_out=None)
        flags = a.flags
        a.flags = flags | _native.PHASE_PROLOGUE
        flush.fill_(float(i))                      # L2 flushed before the step, as in the timed loop
        pstart[i].record(stream)
        scene._launch(a)
        pend[i].record(stream)
        a.flags = flags | _native.PHASE_TRACE
        kstart[i].record(stream)
        scene._launch(a)
        kend[i].record(stream)
        step_id[0] += 1
    torch.cuda.synchronize()
    kernel_ms = statistics.mean(s.elapsed_time(e) for s, e in zip(kstart, kend))
    prologue_ms = statistics.mean(s.elapsed_time(e) for s, e in zip(pstart, pend))

    # ---- L2 read bandwidth probe (roofline denominator for L2-resident traversal) ----
    l2_gbs = None
    try:
        import ctypes
        pb = torch.empty(32 * 1024 * 1024 // 4, dtype=torch.float32, device=dev).fill_(1.0)
        sink = torch.empty(8192, dtype=torch.float32, device=dev)
        L = _native.lib()
        L.mdrt_probe_read(ctypes.c_void_p(pb.data_ptr()), pb.numel() * 4, 4, ctypes.c_void_p(sink.data_ptr()),
                          ctypes.c_void_p(stream.cuda_stream))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        iters = 50
        _native.check(L.mdrt_probe_read(ctypes.c_void_p(pb.data_ptr()), pb.numel() * 4, iters,
                                        ctypes.c_void_p(sink.data_ptr()), ctypes.c_void_p(stream.cuda_stream)))
        e1.record(stream)
        torch.cuda.synchronize()
        l2_gbs = pb.numel() * 4 * iters / (e0.elapsed_time(e1) * 1e-3) / 1e9
    except Exception as exc:  # probe is diagnostic only
        print(f"l2 probe failed: {exc}", file=sys.stderr)

    # ---- e2e: public API with host buffers (H2D poses, D2H observation) ----
    # Every step: pinned host poses -> device (async H2D on the compute stream), fused
    # pipeline, observation -> pinned host (scene copy stream, overlapping the next
    # step's kernels; two output buffers alternate). The L2 flush stays inside the
    # timed region here. Timed with events around the whole loop (the copy stream
    # joins before the end event).
    outs = [out, torch.empty_like(out)]
    # the step's result delivered to the host: the observation, or for the paper pipeline
    # the 48x27 block minimum the policy reads (sensor.py:85-100)
    deliver = [ds, torch.empty_like(ds)] if ds is not None else outs
    host_obs = [torch.empty(tuple(deliver[0].shape), dtype=torch.float32).pin_memory() for _ in range(2)]

    def e2e_step(i):
        kw = (dict(ds_out=deliver[i % 2], host_ds_out=host_obs[i % 2]) if ds is not None
              else dict(host_out=host_obs[i % 2]))
        md.render_pipeline(scene, sensor=sens, step=step_id[0], frame_buffer=buf, timestamp=step_id[0] * dt,
                           delays=delays, out=outs[i % 2], **kw)
        step_id[0] += 1

    for i in range(2):   # warm the copy path
        scene.set_body_poses(*pose_host[i % P], validate=False)
        e2e_step(i)
    scene.host_sync()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_wall0 = time.perf_counter()
    for i in range(args.steps):
        flush.fill_(float(i))
        hp, hq = pose_host[i % P]
        scene.set_body_poses(hp, hq, validate=False)        # pinned host -> device
        e2e_step(i)
    # host wall time of the loop: the host runs at most two steps ahead (staging and
    # output double buffers), so this includes waits on the GPU, not just API cost
    e2e_host_ms = (time.perf_counter() - e2e_wall0) * 1e3
    stream.wait_event(scene._last_copy)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    h2d = pose_host[0][0].numel() * 4 + pose_host[0][1].numel() * 4
    d2h = host_obs[0].numel() * 4
    # PCIe reference: one observation-sized pinned D2H copy alone (the e2e floor)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    for i in range(5):
        host_obs[i % 2].copy_(deliver[0], non_blocking=True)
    c1.record(stream)
    torch.cuda.synchronize()
    d2h_gbs = 5 * d2h / (c0.elapsed_time(c1) * 1e-3) / 1e9

    # ---- the reference's own plugin seam: render_batch with host numpy buffers ----
    # Called as multidepth.scene.render calls its backend (numba_backend.py:222-234):
    # f64 numpy poses / camera poses / ray grids in, a freshly allocated numpy out
    # written in place; wall clock per call (render only: the seam has no sensor stage).
    seam = None
    try:
        from paper_2602_03002_b200 import kernels as mdk

        class _Flat:   # the FlatGeometry fields the CUDA backend reads (scene.py:49-78)
            pass

        flat = _Flat()
        tl = [m.triangles() for _, m in bodies]
        flat.tri_v0, flat.tri_v1, flat.tri_v2 = (np.concatenate([t[:, k] for t in tl]) for k in range(3))
        flat.body_tri_offsets = np.cumsum([0] + [len(t) for t in tl])
        flat.body_root = np.zeros(len(tl), np.int32)
        gt = terrain.triangles()
        flat.g_tri_v0, flat.g_tri_v1, flat.g_tri_v2 = gt[:, 0], gt[:, 1], gt[:, 2]
        _, render_batch = mdk.get_render_fn("cuda")
        dmax_c = np.array([c.d_max for c in w.cameras])
        seam_in = []
        for i in range(2):
            hp = pose_host[i][0].numpy().astype(np.float64)
            hq = pose_host[i][1].numpy().astype(np.float64)
            scene.set_body_poses(hp, hq, validate=False)
            cp_, cq_ = scene.camera_world_poses()
            seam_in.append((hp, hq, cp_, cq_))
        grids = scene.ray_grids()
        seam_t = []
        for i in range(6):
            hp, hq, cp_, cq_ = seam_in[i % 2]
            seam_out = np.empty(scene.frame_shape, np.float32)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            render_batch(flat, hp, hq, cp_, cq_, grids[0], grids[1], dmax_c, True, seam_out, None)
            torch.cuda.synchronize()
            seam_t.append(time.perf_counter() - t0)
        seam_ms = 1e3 * float(np.mean(seam_t[2:]))
        seam = {"value": rays_per_step / (seam_ms * 1e-3), "unit": "rays/s", "ms_per_call": seam_ms,
                "how": "kernels.get_render_fn('cuda') render_batch with f64 numpy inputs and a fresh numpy out "
                       "(the reference's backend seam, render only), wall clock per call, this rank"}
    except Exception as exc:   # diagnostic only
        print(f"seam measurement failed: {exc}", file=sys.stderr)

    # ---- optional: step + NCCL gather of every rank's observation to rank 0 ----
    gather_ms = p2p_ms = 0.0
    if args.gather and world > 1:
        dist.barrier()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for i in range(args.steps):
            scene.set_body_poses(*pose_dev[i % P], validate=False)
            obs = md.render_pipeline(scene, sensor=sens, step=step_id[0], frame_buffer=buf,
                                     timestamp=step_id[0] * dt, delays=delays, out=out)
            pdist.gather_frames(obs, dst=0)
            step_id[0] += 1
        g1.record(stream)
        torch.cuda.synchronize()
        gather_ms = g0.elapsed_time(g1)
        # fused gather: the render epilogue stores straight into rank 0's buffers over peer memory
        start_env = rank * scene.num_envs
        sink = pdist.PeerFrameSink(scene.frame_shape[1:], world * scene.num_envs, start_env, scene.num_envs,
                                   dst=0, slots=2, device=dev)
        dist.barrier()
        torch.cuda.synchronize()
        g0.record(stream)
        for i in range(args.steps):
            scene.set_body_poses(*pose_dev[i % P], validate=False)
            md.render_pipeline(scene, sensor=sens, step=step_id[0], frame_buffer=buf,
                               timestamp=step_id[0] * dt, delays=delays, out=sink.local(i))
            sink.publish()
            step_id[0] += 1
        g1.record(stream)
        torch.cuda.synchronize()
        p2p_ms = g0.elapsed_time(g1)
        sink.close()

    # max over ranks
    tt = torch.tensor([total_ms, e2e_ms, kernel_ms, gather_ms, graph_ms, p2p_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    total_ms, e2e_ms, kernel_ms, gather_ms, graph_ms, p2p_ms = tt.tolist()

    if rank == 0:
        all_rays = rays_per_step * world * args.steps
        value = all_rays / (total_ms * 1e-3)
        e2e_value = all_rays / (e2e_ms * 1e-3)
        # algorithmic bytes of one render-kernel launch (this rank's slice)
        # a node visit reads 56 of the 64 B record (boxes + child refs; the pad is not fetched)
        node_b = scene.geometry_stats["node_record_size"] - 8
        tri_b = scene.geometry_stats["tri_record_size"]
        tw = int(os.environ.get("MDRT_TILE_W", "0")) or (4 if W <= 96 else 8)   # render_tile_width
        warps = n * C * math.ceil(W / tw) * math.ceil(H / (32 // tw))
        lag_frac = float(np.mean(delays_np >= dt))    # envs reading an older ring slot
        io_b = 4 + 4 + 4 * lag_frac                   # ring write + obs write + delayed read
        bytes_per_ray = nodes_per_ray * node_b + tris_per_ray * tri_b + io_b
        launch_bytes = rays_per_step * bytes_per_ray + warps * 128
        achieved = launch_bytes / (kernel_ms * 1e-3) / 1e9
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        traffic = None
        ncu_units = None
        tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
        if os.path.exists(tpath):
            tj = json.load(open(tpath))
            traffic = tj.get("dram_bytes_per_launch")
            if "l1_lsu_data_pipe_pct" in tj:
                ncu_units = {"l1_lsu_data_pipe": tj["l1_lsu_data_pipe_pct"] / 100.0,
                             "issue_active": tj["issue_active_pct"] / 100.0,
                             "l2_throughput": tj["l2_throughput_pct"] / 100.0, "source": tj.get("source")}
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            from oracle import oracle as orc
            th = orc.max_threads()
            cv, cdesc, _, split = cpu_measure(args.config, 3, 1, args.cpu_seconds, th)
            cpu = {"value": cv, "unit": "rays/s", "cores": th, "kind": "port", "sample": cdesc, "cpu": cpu_info(),
                   "split": split}
        line = {
            "metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_desc(args.config), "envs_per_gpu": n, "cams": C,
                       "resolution": f"{W}x{H}", "global_envs": total_envs,
                       "parallelism": f"env-slice x{world} (replicated BVHs, no collective in the step)",
                       "l2": "flushed between timed steps (256 MiB write, untimed)",
                       "terrain_tris": scene.geometry_stats["terrain_triangles"],
                       "body_tris": scene.geometry_stats["body_triangles"],
                       "bvh_bytes": scene.geometry_stats["node_bytes"] + scene.geometry_stats["tri_bytes"],
                       "build_s": round(t_build, 3)},
            "frames_per_s": value / (H * W),
            "steps_per_s": 1e3 / (total_ms / args.steps),
            "per_ray": {"node_fetches": nodes_per_ray, "tri_tests": tris_per_ray, "bytes": bytes_per_ray,
                        "link_node_fetches": link_nodes_per_ray, "link_traversals": link_traces_per_ray,
                        "node_record_b": node_b + 8, "node_fetch_b": node_b, "tri_record_b": tri_b, "io_b": io_b},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic,
                         "kernel": "render_kernel (K1+K2+K3 fused)", "kernel_ms": kernel_ms,
                         "prologue_ms": prologue_ms,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback",
                         "l2_probe_gbs": l2_gbs,
                         "l2_frac": (achieved / l2_gbs) if l2_gbs else None,
                         "unit_utilisation_ncu": ncu_units,
                         "note": "algorithmic bytes = node/triangle records fetched per ray (counted on the device "
                                 "BVH) + I/O; the BVH is L2/L1-resident by design, so DRAM traffic per launch "
                                 "(traffic, ncu) is ~1% of them and achieved exceeds the HBM copy peak; lanes "
                                 "share node fetches, so achieved also approaches the L2 probe (l2_frac) while ncu "
                                 "shows L2 at ~23%: the binding unit is the L1's LSU data pipe "
                                 "(unit_utilisation_ncu, from the committed ncu capture of this config)"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "rays/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms / args.steps, "d2h_alone_gbs": d2h_gbs,
                    "host_loop_ms_per_step": e2e_host_ms / args.steps,
                    "d2h_floor_ms": d2h / (d2h_gbs * 1e9) * 1e3,
                    "delivered": "48x27 block-min observation (policy input)" if ds is not None
                                 else "full observation (N,C,H,W) f32",
                    "how": "pinned-host poses H2D (upload stream) + fused pipeline + result D2H (copy stream, "
                           "double-buffered) every step, L2 flush inside the timed loop, events around the whole loop"},
            "gpu_launches": 2 * args.steps,
            "graph": {"value": all_rays / (graph_ms * 1e-3), "unit": "rays/s", "ms_per_step": graph_ms / args.steps,
                      "how": "CapturedStep replay (advance+prologue+render CUDA graph, device step state), "
                             "device pose copy + L2 flush between steps as for value"},
            "e2e_seam": seam,
            "gather": ({"value": all_rays / (gather_ms * 1e-3), "unit": "rays/s",
                        "how": "step + NCCL P2P gather of all observations to rank 0, no L2 flush",
                        "fused_p2p": {"value": all_rays / (p2p_ms * 1e-3), "unit": "rays/s",
                                      "how": "PeerFrameSink: render epilogue stores into rank 0's IPC-mapped "
                                             "buffers over NVLink + 1-element NCCL all_reduce per step"}}
                       if gather_ms > 0 else None),
            "clocks": clk,
            "wall_s_timed": wall,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
