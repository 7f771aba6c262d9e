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
steps, max over ranks. ``e2e``: the same through the public API with host
buffers: pinned host poses -> H2D, pipeline, D2H of the observation, every
step. ``parity``: the benchmarked step re-rendered for a sample of envs and
compared with the CPU oracle in the same run. ``--impl reference``: the
reference itself (``multidepth`` installed in baseline/_ref, numba backend,
all host cores) on the same config; the C restatement (oracle/oracle.c) when
the reference cannot be imported.

``--gpus N`` without torchrun re-launches itself under
``torch.distributed.run`` with N ranks (one per GPU, NCCL) and fails when
fewer than N GPUs are visible; ``MDRT_BENCH_SHARE_GPU=1`` runs the ranks on the
visible GPUs round-robin over gloo (a control-flow check, never a measurement).
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
    ap.add_argument("--ref-impl", default="auto", choices=["auto", "live", "port"],
                    help="--impl reference: the installed reference (live), the C port, or live if importable")
    ap.add_argument("--ref-budget-s", type=float, default=240.0,
                    help="--impl reference: wall-clock budget of the timed + warm-up steps")
    ap.add_argument("--parity-envs", type=int, default=256, help="envs of the in-run oracle parity check")
    ap.add_argument("--morton-envs", action="store_true",
                    help="experiment: number the envs along a Morton curve of their root position "
                         "(spatially coherent view order)")
    return ap.parse_args()


def fail(msg: str, code: int = 2) -> int:
    print(f"bench.py: {msg}", file=sys.stderr, flush=True)
    return code


def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args) -> int:
    """--gpus N>1 started as a plain process: re-launch under torch.distributed.run
    with N ranks (one process per GPU, as the driver does)."""
    import torch
    share = os.environ.get("MDRT_BENCH_SHARE_GPU") == "1"
    have = torch.cuda.device_count()
    if have == 0:
        return fail("no CUDA device visible")
    if have < args.gpus and not share:
        return fail(f"--gpus {args.gpus} needs {args.gpus} visible GPUs, found {have} (MDRT_BENCH_SHARE_GPU=1 "
                    "runs the ranks round-robin on the visible GPUs over gloo: a control-flow check, never a "
                    "measurement)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32)


def config_dict(name, n_per_gpu, world, w):
    """The workload description both arms print (identical for the same run shape)."""
    c0 = w.cameras[0]
    return {"workload": workload_desc(name), "envs_per_gpu": n_per_gpu, "cams": len(w.cameras),
            "resolution": f"{c0.width}x{c0.height}", "global_envs": n_per_gpu * world,
            "parallelism": f"env-slice x{world} (replicated BVHs, no collective in the step)",
            "l2": "flushed between timed steps (256 MiB write, untimed)",
            "terrain_tris": int(w.terrain.mesh.num_faces),
            "body_tris": int(sum(m.num_faces for _, m in w.bodies)),
            "sensor": "noise 0.1, dropout 0.05, latency U[0, 0.1] s at dt 0.02 (ring 8), camera randomisation "
                      "(CameraRandomization(seed=3))",
            "pose_sets": "8 per-step link pose sets (synth.Workload.poses), cycled"}


def morton_order(w):
    """Renumber a workload's envs along a Z-order curve of their root x/y (experiment)."""
    xy = w.roots[:, :2]
    q = ((xy - xy.min(0)) / np.maximum(np.ptp(xy, 0), 1e-9) * 65535).astype(np.uint64)

    def spread(v):
        v = v & 0xFFFF
        v = (v | (v << 8)) & 0x00FF00FF
        v = (v | (v << 4)) & 0x0F0F0F0F
        v = (v | (v << 2)) & 0x33333333
        return (v | (v << 1)) & 0x55555555
    order = np.argsort(spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1)), kind="stable")
    w.roots, w.yaws = w.roots[order], w.yaws[order]


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
# reference arm / cpu baseline
# ---------------------------------------------------------------------------

class CpuWorkload:
    """The benchmark workload prepared for the CPU oracle (C restatement of the
    reference path, oracle/oracle.c): f32-rounded meshes, poses and camera
    randomisation exactly as the GPU arm uploads them."""

    def __init__(self, name, total_envs):
        from oracle import oracle as orc
        from paper_2602_03002_b200 import synth
        import paper_2602_03002_b200 as md
        self.orc = orc
        self.w = w = synth.config(name, total_envs)
        bodies = [(f32(m.vertices).astype(np.float64), m.faces) for _, m in w.bodies]
        terrain = (f32(w.terrain.mesh.vertices).astype(np.float64), w.terrain.mesh.faces)
        self.cams = [dict(width=c.width, height=c.height, hfov_deg=c.hfov_deg, vfov_deg=c.vfov_deg, d_max=c.d_max,
                          mount_pos=c.mount.translation, mount_rot=c.mount.rotation, parent=c.parent_body)
                     for c in w.cameras]
        self.sc = orc.OracleScene(bodies, terrain, self.cams)
        C = len(w.cameras)
        # camera randomisation of every global env, as the GPU arm sets it (float32 on the device)
        self.off = [f32(a).astype(np.float64) for a in md.sample_camera_offsets(md.CameraRandomization(seed=3),
                                                                                total_envs, C)]
        self.delays = md.sample_latencies(md.SensorConfig(max_delay=0.1, seed=3), total_envs)
        self.dmax = np.array([c["d_max"] for c in self.cams])
        self._grids = {}

    def grids(self, e0, n):
        key = (e0, n)
        if key not in self._grids:
            self._grids = {key: self.orc.ray_grids(self.cams, n, self.off[2][e0:e0 + n])}
        return self._grids[key]

    def render(self, step, e0, n, threads):
        bp, bq = self.w.poses(step, slice(e0, e0 + n))
        o = self.off
        return self.sc.render(f32(bp).astype(np.float64), f32(bq).astype(np.float64), rand_pos=o[0][e0:e0 + n],
                              rand_rot=o[1][e0:e0 + n], grids=self.grids(e0, n), threads=threads)


def run_cpu_sample(cw, n_sample, step, threads, buf_state, cfg):
    """render + apply_noise_dropout + FrameBuffer push/fetch on n_sample envs (oracle port)."""
    orc = cw.orc
    t0 = time.perf_counter()
    depth = cw.render(step, 0, n_sample, threads)
    buf_state[2].append(time.perf_counter() - t0)
    noisy = orc.apply_noise_dropout(depth, noise_scale=cfg.noise_scale, dropout_p=cfg.dropout_p, seed=cfg.seed,
                                    d_max=cw.dmax, step=step, threads=threads)
    times, frames = buf_state[0], buf_state[1]
    times.append(step * 0.02)
    frames.append(noisy)
    if len(times) > 8:
        times.pop(0)
        frames.pop(0)
    idx = orc.frame_select(np.array(times), step * 0.02, cw.delays[:n_sample])
    obs = np.stack([frames[k][e] for e, k in enumerate(idx)])
    return obs


def cpu_measure(cw, steps, warmup, seconds_target, threads):
    """The port on a bounded env sample. Returns (rays_per_s, sample_desc, per-step list, split)."""
    from paper_2602_03002_b200 import sensor
    cfg = sensor.SensorConfig(noise_scale=0.1, dropout_p=0.05, seed=0)
    w = cw.w
    probe_n = 16
    rays_per_env = len(w.cameras) * w.cameras[0].width * w.cameras[0].height
    # size the sample so each step costs ~seconds_target / steps
    state = ([], [], [])
    run_cpu_sample(cw, probe_n, 0, threads, state, cfg)          # builds the probe's ray grids
    t0 = time.perf_counter()
    run_cpu_sample(cw, probe_n, 1, threads, state, cfg)
    per_env = (time.perf_counter() - t0) / probe_n
    n_sample = int(max(8, min(w.num_envs, seconds_target / max(steps, 1) / max(per_env, 1e-6))))
    state = ([], [], [])
    for s in range(warmup):
        run_cpu_sample(cw, n_sample, s, threads, state, cfg)
    state[2].clear()
    times = []
    for s in range(steps):
        t0 = time.perf_counter()
        run_cpu_sample(cw, n_sample, warmup + s, threads, state, cfg)
        times.append(time.perf_counter() - t0)
    rays = n_sample * rays_per_env
    value = rays * len(times) / sum(times)
    desc = (f"{n_sample} of {w.num_envs} envs x {len(w.cameras)} cams x {w.cameras[0].width}x"
            f"{w.cameras[0].height} per step (render with per-env camera randomisation + noise/dropout + latency), "
            f"{len(times)} steps")
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


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def load_live_reference():
    """The reference package installed in baseline/_ref (pip --target), or (None, why)."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "multidepth")):
        return None, "baseline/_ref/multidepth not installed"
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "mdrt_numba_cache"))
    os.environ.setdefault("NUMBA_NUM_THREADS", str(host_cores()))
    sys.path.insert(0, path)
    try:
        import multidepth
        from multidepth.kernels import numba_backend  # noqa: F401  (numba must import)
    except Exception as exc:   # no numba on this host, broken install, ...
        sys.path.remove(path)
        return None, f"import failed: {exc!r}"[:200]
    if not os.path.abspath(multidepth.__file__).startswith(os.path.abspath(path)):
        return None, f"multidepth resolved outside baseline/_ref: {multidepth.__file__}"
    return multidepth, None


def live_reference_measure(ref, name, total_envs, steps, warmup, budget_s):
    """The reference's own CPU path through its public API, per step:
    render(scene, backend="numba", threads=all cores) (scene.py:332-348, incl. its
    camera_world_poses and ray-grid cache) -> apply_noise_dropout (sensor.py:55-82)
    -> FrameBuffer.push + fetch_delayed_batch (sensor.py:122-150), on the GPU arm's
    workload (same f32-rounded meshes, poses, camera randomisation, latencies)."""
    from paper_2602_03002_b200 import synth
    import paper_2602_03002_b200 as md
    threads = host_cores()
    w = synth.config(name, total_envs)
    f64 = lambda x: f32(x).astype(np.float64)  # noqa: E731
    bodies = [(nm, ref.TriMesh(f64(m.vertices), m.faces, frame="body-local")) for nm, m in w.bodies]
    cams = [ref.CameraModel(width=c.width, height=c.height, hfov_deg=c.hfov_deg, vfov_deg=c.vfov_deg, d_max=c.d_max,
                            mount=ref.RigidPose(c.mount.translation, c.mount.rotation), parent_body=c.parent_body,
                            name=c.name) for c in w.cameras]
    terrain = ref.TriMesh(f64(w.terrain.mesh.vertices), w.terrain.mesh.faces)
    C = len(cams)
    off = [f64(a) for a in md.sample_camera_offsets(md.CameraRandomization(seed=3), total_envs, C)]
    cfg = ref.SensorConfig(noise_scale=0.1, dropout_p=0.05, max_delay=0.1, seed=0)
    delays_all = ref.sample_latencies(ref.SensorConfig(max_delay=0.1, seed=3), total_envs)
    P = 8
    pose_sets = [tuple(f64(a) for a in w.poses(s)) for s in range(P)]
    rays_per_env = C * cams[0].width * cams[0].height

    def make(n):
        sc = ref.Scene(num_envs=n, bodies=bodies, cameras=cams, terrain=terrain)
        sc.set_camera_randomization(off[0][:n], off[1][:n], off[2][:n])
        return sc

    def one_step(sc, n, buf, k):
        bp, bq = pose_sets[k % P]
        sc.set_body_poses(bp[:n], bq[:n])
        t0 = time.perf_counter()
        frame = ref.render(sc, backend="numba", threads=threads, timestamp=k * 0.02)
        t1 = time.perf_counter()
        noisy = ref.apply_noise_dropout(frame.data, cfg, d_max=sc.d_max_per_camera, step=k)
        buf.push(ref.DepthFrame(noisy, k * 0.02))
        buf.fetch_delayed_batch(k * 0.02, delays_all[:n])
        return t1 - t0, time.perf_counter() - t0

    n = total_envs
    t_build = time.perf_counter()
    sc = make(n)
    t_build = time.perf_counter() - t_build
    buf = ref.FrameBuffer(capacity=8)
    _, t_first = one_step(sc, n, buf, 0)     # numba JIT (cached on disk afterwards) + ray-grid cache
    # the reference at full size may not fit the budget (it is ~1000x slower than the GPU arm):
    # then every timed step renders a contiguous sample of the envs
    per_step = t_first
    if n > 64:
        _, per_step = one_step(sc, n, buf, 1)
    if (steps + max(warmup - 2, 0)) * per_step > budget_s:
        n = int(max(64, min(n, n * budget_s / ((steps + max(warmup - 2, 0)) * per_step))))
        sc = make(n)
        buf = ref.FrameBuffer(capacity=8)
    for k in range(2, 2 + max(warmup - 2, 0)):
        one_step(sc, n, buf, k)
    render_t, total_t = [], []
    for k in range(steps):
        r, t = one_step(sc, n, buf, warmup + k)
        render_t.append(r)
        total_t.append(t)
    rays = n * rays_per_env
    value = rays * len(total_t) / sum(total_t)
    desc = (f"{n} of {total_envs} envs x {C} cams x {cams[0].width}x{cams[0].height} per step "
            f"({'the full workload' if n == total_envs else 'a contiguous env sample sized to the time budget'}): "
            f"multidepth.render(backend='numba', threads={threads}) + apply_noise_dropout + FrameBuffer "
            f"push/fetch_delayed_batch, {len(total_t)} timed steps after {warmup}")
    split = {"render_plus_sensor_mean": value, "render_plus_sensor_best": rays / min(total_t),
             "render_only_mean": rays * len(render_t) / sum(render_t), "render_only_best": rays / min(render_t),
             "first_step_s": t_first, "scene_build_s": t_build}
    return value, desc, split, threads, n


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2602_03002_b200 import synth
    n = args.envs or cfg_envs(args.config)
    total = n * world if world > 1 else n * args.gpus
    # the reference renders at most one GPU's env count per step (a bounded sample at N > 1)
    ref_envs = min(total, n)
    wdesc = synth.config(args.config, ref_envs)
    config = config_dict(args.config, n, max(world, args.gpus), wdesc)
    ref, why = (None, "--ref-impl port") if args.ref_impl == "port" else load_live_reference()
    if ref is None and args.ref_impl == "live":
        return fail(f"--ref-impl live: {why}")
    if ref is not None:
        value, desc, split, threads, n_used = live_reference_measure(ref, args.config, ref_envs, args.steps,
                                                                     args.warmup, args.ref_budget_s)
        kind = "reference"
        detail = (f"multidepth {getattr(ref, '__version__', '')} (the reference package, pip-installed unmodified "
                  f"into baseline/_ref) through its public API, numba backend, {threads} threads")
    else:
        from oracle import oracle as orc
        threads = orc.max_threads()
        cw = CpuWorkload(args.config, ref_envs)
        value, desc, _, split = cpu_measure(cw, args.steps, args.warmup, args.cpu_seconds * 3, threads)
        kind = "port"
        detail = (f"oracle/oracle.c (C restatement of multidepth numba_backend._render_kernel + sensor + "
                  f"FrameBuffer), OpenMP; live reference unavailable: {why}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": max(world, args.gpus),
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
        "impl_detail": detail,
        "cpu_baseline": {"value": value, "unit": "rays/s", "cores": threads, "kind": kind, "sample": desc,
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
    launched = "WORLD_SIZE" in os.environ
    rank, world, local = dist_env()
    if launched and world != args.gpus:
        return fail(f"--gpus {args.gpus} but the launcher started WORLD_SIZE={world} ranks")
    if args.impl == "reference":
        return reference_arm(args)
    if args.gpus > 1 and not launched:
        return self_launch(args)
    return ours(args)


def ours(args):
    import torch
    import torch.distributed as dist
    import paper_2602_03002_b200 as md
    from paper_2602_03002_b200 import _native, synth
    from paper_2602_03002_b200 import distributed as pdist

    rank, world, local = dist_env()
    # MDRT_BENCH_SHARE_GPU=1 (control-flow check only, never a measurement): ranks share
    # the visible GPUs round-robin and talk over gloo, so the N>1 code path can be
    # exercised on a one-GPU box; kernels of different ranks never wait on each other.
    share = os.environ.get("MDRT_BENCH_SHARE_GPU") == "1"
    have = torch.cuda.device_count()
    if have == 0:
        return fail("no CUDA device visible")
    if world > have and not share:
        return fail(f"{world} ranks but only {have} visible GPUs (MDRT_BENCH_SHARE_GPU=1 for a control-flow run)")
    gpu = local % have if share else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    # pin this rank's threads (and so its pinned host buffers) to its GPU's NUMA node
    all_cpus = os.sched_getaffinity(0)
    numa = pdist.bind_to_gpu_numa(dev) if not share else {"node": None, "cpus": len(all_cpus)}

    n = args.envs or cfg_envs(args.config)
    total_envs = n * world
    w = synth.config(args.config, total_envs)
    if args.morton_envs:
        morton_order(w)
    env0, n_rank = pdist.env_slice(total_envs, rank, world)
    assert n_rank == n
    config = config_dict(args.config, n, world, w)
    bodies = [(nm, md.TriMesh(f32(m.vertices).astype(np.float64), m.faces, frame="body-local"))
              for nm, m in w.bodies]
    terrain = md.TriMesh(f32(w.terrain.mesh.vertices).astype(np.float64), w.terrain.mesh.faces)
    t_build = time.perf_counter()
    scene = md.Scene(n, bodies=bodies, cameras=w.cameras, terrain=terrain, device=dev, env_offset=env0)
    t_build = time.perf_counter() - t_build
    if os.environ.get("MDRT_NO_TILE_ENTRY") == "1":      # A/B: terrain traversal from the root
        scene.debug_flags |= _native.NO_TILE_ENTRY
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
    # Algorithmic work: a single-ray closest-hit traversal from each tree's
    # root, counted on the device BVH with the tile entries off; `issued` counts what the
    # render kernel fetches per ray when each tile's rays start at its entry record (the
    # shared top-level fetches are made once per tile by entry_kernel instead).
    ctr = torch.zeros(4, dtype=torch.int64, device=dev)
    scene.set_body_poses(*pose_dev[0], validate=False)
    flags0 = scene.debug_flags
    scene.debug_flags = flags0 | _native.NO_TILE_ENTRY
    md.render(scene, counters=ctr)
    scene.debug_flags = flags0
    ctr_issued = torch.zeros(4, dtype=torch.int64, device=dev)
    md.render(scene, counters=ctr_issued)
    torch.cuda.synchronize()
    nodes_per_ray, tris_per_ray, link_nodes_per_ray, link_traces_per_ray = (x / rays_per_step for x in ctr.tolist())
    nodes_issued_per_ray = ctr_issued[0].item() / rays_per_step

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
        sink = torch.empty(8192, dtype=torch.float32, device=dev)
        L = _native.lib()
        for mib in (32, 64):                          # both L2-resident (126 MB); best of 3 each
            pb = torch.empty(mib * 1024 * 1024 // 4, dtype=torch.float32, device=dev).fill_(1.0)
            L.mdrt_probe_read(ctypes.c_void_p(pb.data_ptr()), pb.numel() * 4, 4, ctypes.c_void_p(sink.data_ptr()),
                              ctypes.c_void_p(stream.cuda_stream))
            iters = 50
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                _native.check(L.mdrt_probe_read(ctypes.c_void_p(pb.data_ptr()), pb.numel() * 4, iters,
                                                ctypes.c_void_p(sink.data_ptr()), ctypes.c_void_p(stream.cuda_stream)))
                e1.record(stream)
                torch.cuda.synchronize()
                g = pb.numel() * 4 * iters / (e0.elapsed_time(e1) * 1e-3) / 1e9
                l2_gbs = max(l2_gbs or 0.0, g)
            del pb
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
    # clocks sampled from the first timed loop through the e2e loop (value, graph,
    # kernel-only and e2e timed regions; a 20-step value loop alone is ~40 ms)
    clk = clocks.stop()
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
            pdist.gather_frames(obs, dst=0, sizes=[n] * world)     # equal slices: no size exchange
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

    # ---- rank 0: CPU baseline (oracle port, all host cores) + in-run parity ----
    cpu = parity = None
    if rank == 0 and not (args.no_cpu_baseline and args.parity_envs <= 0):
        os.sched_setaffinity(0, all_cpus)        # the CPU baseline uses every host core
        from oracle import oracle as orc
        th = orc.max_threads()
        cw = CpuWorkload(args.config, total_envs)
        if not args.no_cpu_baseline:
            cv, cdesc, _, split = cpu_measure(cw, 3, 1, args.cpu_seconds, th)
            cpu = {"value": cv, "unit": "rays/s", "cores": th, "kind": "port", "sample": cdesc, "cpu": cpu_info(),
                   "split": split}
        if args.parity_envs > 0:
            parity = parity_check(md, cw, scene, sens, env0, min(n, args.parity_envs), step_id[0] + 1000, th)

    # max over ranks
    tt = torch.tensor([total_ms, e2e_ms, kernel_ms, gather_ms, graph_ms, p2p_ms], dtype=torch.float64,
                      device="cpu" if share else dev)
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
        achieved_alg = launch_bytes / (kernel_ms * 1e-3) / 1e9
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        tj = {}
        tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
        if os.path.exists(tpath) and n == cfg_envs(args.config):   # captured at the config's own env count
            tj = json.load(open(tpath))
        traffic = tj.get("dram_bytes_per_launch")
        ncu_units = None
        if "l1_lsu_data_pipe_pct" in tj:
            ncu_units = {"l1_lsu_data_pipe": tj["l1_lsu_data_pipe_pct"] / 100.0,
                         "issue_active": tj["issue_active_pct"] / 100.0,
                         "l2_throughput": tj["l2_throughput_pct"] / 100.0, "source": tj.get("source")}
            if tj.get("ncu_duration_ms"):
                # actual traffic of the captured launch: L2 -> L1 reads and DRAM
                dur = tj["ncu_duration_ms"] * 1e-3
                if tj.get("l2_to_l1_read_bytes_per_launch"):
                    ncu_units["l2_to_l1_read_gbs"] = tj["l2_to_l1_read_bytes_per_launch"] / dur / 1e9
                if tj.get("dram_bytes_per_launch"):
                    ncu_units["dram_gbs"] = tj["dram_bytes_per_launch"] / dur / 1e9
        bvh_bytes = scene.geometry_stats["node_bytes"] + scene.geometry_stats["tri_bytes"]
        l2_size = torch.cuda.get_device_properties(dev).L2_cache_size
        if bvh_bytes <= l2_size and l2_gbs:
            # L2-resident BVH: the traversal is bounded by on-chip delivery of
            # node/triangle records; denominator = the L2 read bandwidth probed in this run
            req = tj.get("l1_requested_sectors_per_launch")
            roof = {"bound": "l2", "achieved": achieved_alg, "peak": l2_gbs, "unit": "GB/s",
                    "frac": achieved_alg / l2_gbs, "traffic": traffic,
                    "peak_source": L2_PROBE_HOW,
                    "achieved_how": "algorithmic bytes per launch (node 56 B x node fetches + triangle 48 B x tests "
                                    "per ray of a single-ray traversal from the tree roots, counted on the device "
                                    "BVH, + I/O) / render-kernel event time",
                    "frac_requested": (req * 32 / (kernel_ms * 1e-3) / 1e9 / l2_gbs) if req else None,
                    "frac_requested_how": "L1-requested sectors per launch (ncu l1tex__t_sectors, global loads + "
                                          "texture, lanes of a request deduplicated) x 32 B / kernel time / L2 "
                                          "probe; cannot exceed 1 through lane sharing (profiles/traffic_*.json)",
                    "hbm_frac": (traffic / (kernel_ms * 1e-3) / 1e9 / hbm_peak) if traffic else None}
        else:
            # BVH larger than L2 (config 5): DRAM traffic of the launch (ncu) over its event time
            ach = traffic / (kernel_ms * 1e-3) / 1e9 if traffic else None
            roof = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                    "frac": (ach / hbm_peak) if ach else None, "traffic": traffic,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
                    "achieved_how": "ncu dram__bytes_read+write per launch (profiles/traffic_*.json) / render-kernel "
                                    "event time",
                    "algorithmic_gbs": achieved_alg,
                    "l2_frac_algorithmic": (achieved_alg / l2_gbs) if l2_gbs else None}
        roof.update({"kernel": "render_kernel (K1+K2+K3 fused)", "kernel_ms": kernel_ms, "prologue_ms": prologue_ms,
                     "l2_probe_gbs": l2_gbs, "hbm_peak_gbs": hbm_peak, "bvh_bytes": bvh_bytes, "l2_bytes": l2_size,
                     "unit_utilisation_ncu": ncu_units,
                     "note": "lanes of a warp share node records through L1, so algorithmic bytes can exceed what "
                             "L2 serves; ncu shows the binding unit is the L1's LSU data pipe (bytes delivered per "
                             "lane) jointly with issue (unit_utilisation_ncu, committed capture of this config)"})
        line = {
            "metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config,
            "geometry": {"terrain_tris_built": scene.geometry_stats["terrain_triangles"],
                         "body_tris_built": scene.geometry_stats["body_triangles"], "bvh_bytes": bvh_bytes,
                         "build_s": round(t_build, 3)},
            "frames_per_s": value / (H * W),
            "steps_per_s": 1e3 / (total_ms / args.steps),
            "per_ray": {"node_fetches": nodes_per_ray, "node_fetches_issued": nodes_issued_per_ray,
                        "tri_tests": tris_per_ray, "bytes": bytes_per_ray,
                        "link_node_fetches": link_nodes_per_ray, "link_traversals": link_traces_per_ray,
                        "node_record_b": node_b + 8, "node_fetch_b": node_b, "tri_record_b": tri_b, "io_b": io_b},
            "roofline": roof,
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": {"value": e2e_value, "unit": "rays/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms / args.steps, "d2h_alone_gbs": d2h_gbs,
                    "host_loop_ms_per_step": e2e_host_ms / args.steps,
                    "d2h_floor_ms": d2h / (d2h_gbs * 1e9) * 1e3,
                    # the e2e leg's own ceiling: the step's result crossing PCIe at the measured
                    # pinned D2H rate (the device step overlaps it)
                    "pcie_ceiling_rays_per_s": rays_per_step * world / (d2h / (d2h_gbs * 1e9)),
                    "frac_of_pcie_ceiling": e2e_value / (rays_per_step * world / (d2h / (d2h_gbs * 1e9))),
                    "delivered": "48x27 block-min observation (policy input)" if ds is not None
                                 else "full observation (N,C,H,W) f32",
                    "how": "pinned-host poses H2D (upload stream) + fused pipeline + result D2H (copy stream, "
                           "double-buffered) every step, L2 flush inside the timed loop, events around the whole loop"},
            # prologue + per-tile entry kernel + render kernel per step
            "gpu_launches": (2 if (scene.debug_flags & _native.NO_TILE_ENTRY or
                                   scene.geometry_stats["terrain_triangles"] < 65536) else 3) * args.steps,
            "graph": {"value": all_rays / (graph_ms * 1e-3), "unit": "rays/s", "ms_per_step": graph_ms / args.steps,
                      "how": "CapturedStep replay (advance+prologue+render CUDA graph, device step state), "
                             "device pose copy + L2 flush between steps as for value"},
            "e2e_seam": seam,
            "gather": ({"value": all_rays / (gather_ms * 1e-3), "unit": "rays/s",
                        "how": "step + NCCL P2P gather of all observations to rank 0, no L2 flush",
                        "fused_p2p": {"value": all_rays / (p2p_ms * 1e-3), "unit": "rays/s",
                                      "how": "PeerFrameSink: render epilogue stores into rank 0's IPC-mapped "
                                             "buffers over NVLink (8-wide tiles, 32 B row stores) + 1-element NCCL "
                                             "all_reduce per step"}}
                       if gather_ms > 0 else None),
            "numa": numa,
            "clocks": clk,
            "wall_s_timed": wall,
        }
        if share and world > 1:
            line["share_gpu"] = "MDRT_BENCH_SHARE_GPU=1: ranks shared the visible GPUs; control-flow run, not a " \
                                "measurement"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


L2_PROBE_HOW = ("L2 read bandwidth measured in this run: mdrt_probe_read over 32 and 64 MiB buffers "
                "(L2-resident), 32 B ld.global.cg loads (bypass L1), 4 blocks of 256 threads per SM (the fastest "
                "shape of the tools/micro/l2_probe_sweep.cu sweep), max of 2 sizes x best of 3 x 50 passes, CUDA events")


def parity_check(md, cw, scene, sens, env0, n_par, step, threads):
    """The benchmarked step re-rendered for envs [0, n_par) of this rank and compared with
    the CPU oracle on identical inputs (the reference bench's cross-implementation check,
    multidepth bench.py:137-151). Clean depth: max |diff|, pixels beyond 1e-4 m, hit/miss
    flips split by cause (flips the oracle reproduces with the GPU's 1e-5 barycentric
    margin vs the rest, grazing fp32/f64 disagreements). Sensor: dropout rate and
    residual statistics of both sides, noisy values compared bit for bit where the clean
    depth agrees."""
    import torch
    orc = cw.orc
    w = cw.w
    bp, bq = w.poses(step, slice(env0, env0 + scene.num_envs))
    scene.set_body_poses(f32(bp), f32(bq), validate=False)
    clean = torch.empty(scene.frame_shape, dtype=torch.float32, device=scene.device)
    obs = torch.empty_like(clean)
    md.render_pipeline(scene, sensor=sens, step=step, out=obs, clean_out=clean)
    g_clean = clean[:n_par].cpu().numpy()
    g_obs = obs[:n_par].cpu().numpy()
    o_clean = cw.render(step, env0, n_par, threads)
    orc.set_bary_eps(1e-5)
    try:
        o_eps = cw.render(step, env0, n_par, threads)
    finally:
        orc.set_bary_eps(0.0)
    o_obs = orc.apply_noise_dropout(o_clean, noise_scale=sens.noise_scale, dropout_p=sens.dropout_p, seed=sens.seed,
                                    d_max=cw.dmax, step=step, env_offset=env0, threads=threads)
    dmax = np.asarray(cw.dmax, np.float32).reshape(1, -1, 1, 1)
    g_hit, o_hit, e_hit = g_clean < dmax, o_clean < dmax, o_eps < dmax
    flips = g_hit != o_hit
    bary = flips & (e_hit == g_hit)
    diff = np.abs(g_clean.astype(np.float64) - o_clean)
    both = g_hit & o_hit
    band = (diff > 1e-4) & both                    # both hit, different depth (e.g. another surface)
    band_bary = band & (np.abs(g_clean.astype(np.float64) - o_eps) <= 1e-4)
    px = g_clean.size

    def sensor_stats(c, o):
        # pixels whose noisy value cannot reach d_max (6 sigma): dropped <=> obs == d_max
        sel = c < dmax / (1.0 + 6.0 * sens.noise_scale)
        drop = (o == dmax) & sel
        keep = sel & ~drop
        r = (o[keep].astype(np.float64) / c[keep] - 1.0) / sens.noise_scale
        return {"dropout_rate": float(drop.sum() / max(sel.sum(), 1)), "residual_mean": float(r.mean()),
                "residual_std": float(r.std()), "pixels": int(sel.sum())}
    gs, os_ = sensor_stats(g_clean, g_obs), sensor_stats(o_clean, o_obs)
    same = g_clean == o_clean
    return {
        "sample": f"envs [{env0}, {env0 + n_par}) x {scene.num_cameras} cams x {scene.width}x{scene.height} of the "
                  f"benchmarked scene at step {step} (poses, camera randomisation, sensor counters as in the timed "
                  f"loop) vs oracle/oracle.c (f64, the reference algorithm)",
        "pixels": int(px),
        "max_abs_diff_m": float(diff.max()),
        "max_abs_diff_hits_m": float(diff[both].max()) if both.any() else 0.0,
        "over_1e-4_m": int((diff > 1e-4).sum()),
        "over_1e-4_frac": float((diff > 1e-4).sum() / px),
        "in_band_over_1e-4": int(band.sum()),
        "in_band_over_1e-4_bary_margin": int(band_bary.sum()),
        "hit_miss_flips": {"total": int(flips.sum()), "bary_margin": int(bary.sum()),
                           "grazing": int((flips & ~bary).sum()), "frac": float(flips.sum() / px),
                           "how": "bary_margin = the oracle also flips with the GPU kernel's 1e-5 barycentric "
                                  "watertightness margin (silhouette edges); grazing = the rest (fp32 vs f64)"},
        "flips_within_1e-4": bool(flips.sum() <= 1e-4 * px),
        "sensor": {"gpu": gs, "oracle": os_,
                   "dropout_rate_rel_diff": abs(gs["dropout_rate"] - os_["dropout_rate"]) / max(os_["dropout_rate"],
                                                                                                1e-12),
                   "residual_std_rel_diff": abs(gs["residual_std"] - os_["residual_std"]) / max(os_["residual_std"],
                                                                                                1e-12),
                   "residual_mean_abs_diff": abs(gs["residual_mean"] - os_["residual_mean"]),
                   "noisy_mismatch_where_clean_equal": int(((g_obs != o_obs) & same).sum()),
                   "clean_equal_pixels": int(same.sum())},
    }


if __name__ == "__main__":
    sys.exit(main())
