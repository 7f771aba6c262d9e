"""Where does a bench step's time go outside the render kernel? Times, per step
with CUDA events: (a) the bench step (pose copy + prologue + render) after an
L2 flush, (b) the same without the flush, (c) prologue only, (d) render only
(records from the last prologue), each after a flush.

    python tools/step_split.py [--config cfg2] [--steps 100]
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_03002_b200 as md  # noqa: E402
from paper_2602_03002_b200 import _native, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--steps", type=int, default=100)
    a = ap.parse_args()
    w = synth.config(a.config)
    n = w.num_envs
    f32 = lambda x: np.asarray(x, np.float64).astype(np.float32)  # noqa: E731
    bodies = [(nm, md.TriMesh(f32(m.vertices).astype(np.float64), m.faces, frame="body-local")) for nm, m in w.bodies]
    scene = md.Scene(n, bodies=bodies, cameras=w.cameras,
                     terrain=md.TriMesh(f32(w.terrain.mesh.vertices).astype(np.float64), w.terrain.mesh.faces))
    scene.set_camera_randomization(*md.sample_camera_offsets(md.CameraRandomization(seed=3), n, len(w.cameras)))
    delays = torch.from_numpy(md.sample_latencies(md.SensorConfig(max_delay=0.1, seed=3), n)).cuda()
    sens = md.SensorConfig(max_delay=0.1)
    buf = md.FrameBuffer(capacity=8)
    poses = [tuple(torch.from_numpy(f32(x)).cuda() for x in w.poses(s)) for s in range(4)]
    out = torch.empty(scene.frame_shape, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    k = [0]

    def full(i):
        scene.set_body_poses(*poses[i % 4], validate=False)
        md.render_pipeline(scene, sensor=sens, step=k[0], frame_buffer=buf, timestamp=k[0] * 0.02, delays=delays,
                           out=out)
        k[0] += 1

    def phase(flag):
        def run(i):
            a_ = scene._step_args(out, True)
            a_.flags |= flag
            scene._launch(a_)
        return run

    res = {}
    for name, fn, fl in (("step_flush", full, True), ("step_noflush", full, False),
                         ("prologue_flush", phase(_native.PHASE_PROLOGUE), True),
                         ("render_flush", phase(_native.PHASE_TRACE), True),
                         ("render_noflush", phase(_native.PHASE_TRACE), False)):
        for i in range(3):
            fn(i)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        for i in range(a.steps):
            if fl:
                flush.fill_(float(i))
            ev[i][0].record()
            fn(i)
            ev[i][1].record()
        torch.cuda.synchronize()
        res[name] = statistics.mean(s.elapsed_time(e) for s, e in ev)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
