"""Minimal driver for ncu: build a workload scene and run a few fused pipeline steps.

    python tools/profile_step.py [--config cfg2] [--steps 3]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_03002_b200 as md  # noqa: E402
from paper_2602_03002_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--envs", type=int, default=None)
    a = ap.parse_args()
    w = synth.config(a.config, a.envs)
    n = w.num_envs
    f32 = lambda x: np.asarray(x, np.float64).astype(np.float32).astype(np.float64)  # noqa: E731
    bodies = [(nm, md.TriMesh(f32(m.vertices), m.faces, frame="body-local")) for nm, m in w.bodies]
    scene = md.Scene(n, bodies=bodies, cameras=w.cameras,
                     terrain=md.TriMesh(f32(w.terrain.mesh.vertices), w.terrain.mesh.faces))
    scene.set_camera_randomization(*md.sample_camera_offsets(md.CameraRandomization(seed=3), n, len(w.cameras)))
    delays = torch.from_numpy(md.sample_latencies(md.SensorConfig(seed=3), n)).cuda()
    sens = md.SensorConfig()
    buf = md.FrameBuffer(capacity=8)
    out = torch.empty(scene.frame_shape, device="cuda")
    for s in range(a.steps):
        p, q = w.poses(s)
        scene.set_body_poses(p, q, validate=False)
        md.render_pipeline(scene, sensor=sens, step=s, frame_buffer=buf, timestamp=0.02 * s, delays=delays, out=out)
    torch.cuda.synchronize()
    print("ok", float(out.mean()))


if __name__ == "__main__":
    main()
