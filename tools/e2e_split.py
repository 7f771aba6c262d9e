"""Attribute the end-to-end step time: the e2e loop of bench.py with the L2
flush, the pinned pose upload and the observation download toggled.

    python tools/e2e_split.py [--config cfg2] [--steps 100]
"""
import argparse
import itertools
import json
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
    poses_h = [tuple(torch.from_numpy(f32(x)).pin_memory() for x in w.poses(s)) for s in range(4)]
    poses_d = [tuple(x.cuda() for x in p) for p in poses_h]
    outs = [torch.empty(scene.frame_shape, device="cuda") for _ in range(2)]
    host = [torch.empty(scene.frame_shape).pin_memory() for _ in range(2)]
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    stream = torch.cuda.current_stream()
    k = [0]
    res = {}
    for fl, h2d, d2h in itertools.product((0, 1), (0, 1), (0, 1)):
        def run(steps):
            for i in range(steps):
                if fl:
                    flush.fill_(float(i))
                p = (poses_h if h2d else poses_d)[i % 4]
                scene.set_body_poses(*p, validate=False)
                md.render_pipeline(scene, sensor=sens, step=k[0], frame_buffer=buf, timestamp=k[0] * 0.02,
                                   delays=delays, out=outs[i % 2], host_out=host[i % 2] if d2h else None)
                k[0] += 1
        run(4)
        scene.host_sync()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run(a.steps)
        if d2h:
            stream.wait_event(scene._last_copy)
        e1.record(stream)
        torch.cuda.synchronize()
        res[f"flush{fl}_h2d{h2d}_d2h{d2h}"] = e0.elapsed_time(e1) / a.steps
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
