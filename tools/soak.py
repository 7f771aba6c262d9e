"""Soak: 3200 e2e-style steps (pinned pose upload, fused pipeline, async host delivery);
checks that device memory and host RSS stay flat.

    python tools/soak.py
"""
import os, sys, resource, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2602_03002_b200 as md
from paper_2602_03002_b200 import synth
w = synth.config("cfg2", 1024)
scene = md.Scene(w.num_envs, bodies=w.bodies, cameras=w.cameras, terrain=w.terrain.mesh)
buf = md.FrameBuffer(capacity=8)
delays = md.sample_latencies(md.SensorConfig(max_delay=0.1, seed=3), w.num_envs)
poses = [tuple(torch.from_numpy(np.asarray(x, np.float32)).pin_memory() for x in w.poses(s)) for s in range(4)]
host = [torch.empty(scene.frame_shape).pin_memory() for _ in range(2)]
outs = [torch.empty(scene.frame_shape, device="cuda") for _ in range(2)]
def run(k0, n):
    for k in range(k0, k0 + n):
        scene.set_body_poses(*poses[k % 4], validate=False)
        md.render_pipeline(scene, sensor=md.SensorConfig(), step=k, frame_buffer=buf, timestamp=0.02 * k,
                           delays=delays, out=outs[k % 2], host_out=host[k % 2])
    scene.host_sync(); torch.cuda.synchronize()
run(0, 200)
m0, r0 = torch.cuda.memory_allocated(), resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
run(200, 3000)
m1, r1 = torch.cuda.memory_allocated(), resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
print("cuda alloc MB", m0 / 2**20, "->", m1 / 2**20, "; max RSS MB", r0 / 1024, "->", r1 / 1024)
assert m1 <= m0 + 1e6 and r1 <= r0 + 200 * 1024
print("soak ok")

# CUDA-graph replays with per-episode camera re-randomisation (written in place into the
# scene's buffers) and a replay stream that alternates: memory must stay flat too
from paper_2602_03002_b200.pipeline import CapturedStep  # noqa: E402
scene.set_camera_randomization(*md.sample_camera_offsets(md.CameraRandomization(seed=1), w.num_envs, 2))
cap = CapturedStep(scene, sensor=md.SensorConfig(), frame_buffer=md.FrameBuffer(capacity=8), delays=delays, dt=0.02)
side = torch.cuda.Stream()


def replays(n):
    for k in range(n):
        if k % 100 == 0:
            scene.set_camera_randomization(*md.sample_camera_offsets(md.CameraRandomization(seed=1), w.num_envs, 2,
                                                                     episode=k // 100))
        scene.body_positions.copy_(poses[k % 4][0], non_blocking=True)
        if k % 2:
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                cap.replay()
            torch.cuda.current_stream().wait_stream(side)
        else:
            cap.replay()
    torch.cuda.synchronize()


replays(200)
m0, r0 = torch.cuda.memory_allocated(), resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
replays(3000)
m1, r1 = torch.cuda.memory_allocated(), resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
print("graph replays: cuda alloc MB", m0 / 2**20, "->", m1 / 2**20, "; max RSS MB", r0 / 1024, "->", r1 / 1024)
assert m1 <= m0 + 1e6 and r1 <= r0 + 200 * 1024
print("graph soak ok")
