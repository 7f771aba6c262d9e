"""Where does the render step's time go? Times the fused pipeline with the
sensor epilogue / latency ring switched on and off (CUDA events, same poses).

    python tools/phase_split.py [--config cfg2] [--reps 30]
"""
import argparse
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
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    w = synth.config(a.config)
    n = w.num_envs
    f32 = lambda x: np.asarray(x, np.float64).astype(np.float32).astype(np.float64)  # noqa: E731
    bodies = [(nm, md.TriMesh(f32(m.vertices), m.faces, frame="body-local")) for nm, m in w.bodies]
    scene = md.Scene(n, bodies=bodies, cameras=w.cameras,
                     terrain=md.TriMesh(f32(w.terrain.mesh.vertices), w.terrain.mesh.faces))
    scene.set_camera_randomization(*md.sample_camera_offsets(md.CameraRandomization(seed=3), n, len(w.cameras)))
    delays = torch.from_numpy(md.sample_latencies(md.SensorConfig(seed=3), n)).cuda()
    p, q = w.poses(0)
    scene.set_body_poses(p, q, validate=False)
    out = torch.empty(scene.frame_shape, device="cuda")
    variants = {
        "full": dict(sensor=md.SensorConfig(), latency=True),
        "sensor_only": dict(sensor=md.SensorConfig(), latency=False),
        "noise_off_dropout_on": dict(sensor=md.SensorConfig(noise_scale=0.0), latency=False),
        "render_only": dict(sensor=None, latency=False),
    }
    res = {}
    for name, v in variants.items():
        buf = md.FrameBuffer(capacity=8) if v["latency"] else None
        kw = dict(frame_buffer=buf, delays=delays) if buf is not None else {}
        for s in range(3):
            md.render_pipeline(scene, sensor=v["sensor"], step=s, timestamp=0.02 * s, out=out, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in range(a.reps):
            md.render_pipeline(scene, sensor=v["sensor"], step=3 + s, timestamp=0.02 * (3 + s), out=out, **kw)
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / a.reps
    rays = scene.num_envs * scene.num_cameras * scene.width * scene.height
    print(json.dumps({k: {"ms": v, "rays_per_s": rays / (v * 1e-3)} for k, v in res.items()}))


if __name__ == "__main__":
    main()
