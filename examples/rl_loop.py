"""A distillation-style RL loop on the B200 renderer (drop-in usage example).

The simulator's link states live on the GPU as an (N, L, 13) tensor
(position, xyzw quaternion, linear and angular velocity); the renderer reads
them in place (``Scene.bind_link_states``) and the whole depth step -- camera
poses, link culling, traversal, noise/dropout, latency ring, 5x5 block-min
downsample -- is one CUDA-graph replay (``CapturedStep``). The policy input
(48x27 per camera) is delivered to pinned host memory on a side stream.

    python examples/rl_loop.py [--envs 1024] [--steps 200]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_03002_b200 as md  # noqa: E402
from paper_2602_03002_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()

    # scene: synthetic G1 proxy (30 links) on slope/stairs tiles, two torso cameras at 240x135
    w = synth.config("paper", a.envs)
    scene = md.Scene(w.num_envs, bodies=w.bodies, cameras=w.cameras, terrain=w.terrain.mesh)
    n, links = scene.num_envs, scene.num_bodies + 3        # the simulator has a few extra links
    link_map = np.arange(scene.num_bodies) + 3

    # the "simulator" state tensor, written in place every physics step
    pos, rot = (torch.as_tensor(x, dtype=torch.float32, device="cuda") for x in w.poses(0))
    states = torch.zeros((n, links, 13), device="cuda")
    states[:, link_map, 0:3] = pos
    states[:, link_map, 3:7] = rot[..., [1, 2, 3, 0]]        # wxyz -> xyzw
    scene.bind_link_states(states, link_map, pos_offset=0, rot_offset=3, quat_order="xyzw")
    scene.set_camera_randomization(*md.sample_camera_offsets(md.CameraRandomization(seed=1), n,
                                                             scene.num_cameras))

    sensor = md.SensorConfig(noise_scale=0.1, dropout_p=0.05, seed=0)
    buf = md.FrameBuffer(capacity=8)
    delays = md.sample_latencies(md.SensorConfig(max_delay=0.1, seed=3), n)
    obs = torch.empty((n, scene.num_cameras, scene.height // 5, scene.width // 5), device="cuda")
    step = md.CapturedStep(scene, sensor=sensor, frame_buffer=buf, delays=delays, dt=0.02, ds_out=obs)
    host = [torch.empty(tuple(obs.shape)).pin_memory() for _ in range(2)]
    copy = torch.cuda.Stream()
    done = [torch.cuda.Event() for _ in range(2)]

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(a.steps):
        states[:, link_map, 0:2] += 0.002 * torch.randn((n, scene.num_bodies, 2), device="cuda")  # "physics"
        step.replay()                                  # depth step: one graph launch, no host arguments
        copy.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(copy):
            done[k % 2].synchronize()                  # host buffer k % 2 consumed two steps ago
            host[k % 2].copy_(obs, non_blocking=True)
            done[k % 2].record(copy)
        # ... the policy would read host[(k - 1) % 2] here ...
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    rays = n * scene.num_cameras * scene.height * scene.width * a.steps
    print(f"{a.steps} steps x {n} envs x {scene.num_cameras} cams {scene.width}x{scene.height}: "
          f"{rays / dt:.3g} rays/s wall clock, obs {tuple(obs.shape)}, "
          f"mean policy depth {host[(a.steps - 1) % 2].mean():.3f} m")


if __name__ == "__main__":
    main()
