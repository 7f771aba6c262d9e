"""Where a seam call's time goes: cProfile over render_batch calls made as the
reference's render() makes them (config-2 workload with per-env FOV
randomisation: (N,C,H,W,3) f64 ray grids, fresh numpy out per call).

    python tools/seam_profile.py [--calls 8]
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_03002_b200 as md  # noqa: E402
from paper_2602_03002_b200 import kernels, synth  # noqa: E402
from paper_2602_03002_b200.scene import _FlatTris  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=8)
    ap.add_argument("--quiet", action="store_true")
    a = ap.parse_args()
    w = synth.config("cfg2")
    n, cams = w.num_envs, w.cameras
    scene = md.Scene(n, bodies=w.bodies, cameras=cams, terrain=w.terrain.mesh)
    scene.set_camera_randomization(*md.sample_camera_offsets(md.CameraRandomization(seed=3), n, len(cams)))
    flat = _FlatTris([m.triangles() for _, m in w.bodies], w.terrain.mesh.triangles())
    _, render_batch = kernels.get_render_fn("cuda")
    dmax = np.array([c.d_max for c in cams])
    grids = scene.ray_grids()
    args = []
    for k in range(2):
        bp, bq = w.poses(k)
        scene.set_body_poses(bp, bq)
        args.append((bp, bq) + scene.camera_world_poses())

    def calls(m):
        ts = []
        for k in range(m):
            bp, bq, cp, cq = args[k % 2]
            out = np.empty(scene.frame_shape, np.float32)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            render_batch(flat, bp, bq, cp, cq, grids[0], grids[1], dmax, True, out, None)
            ts.append(time.perf_counter() - t0)
        return ts

    calls(3)
    pr = cProfile.Profile()
    pr.enable()
    ts = calls(a.calls)
    pr.disable()
    tag = f"mode={os.environ.get('MDRT_SEAM_MODE', 'stage')} touch={os.environ.get('MDRT_SEAM_TOUCH', '1')}"
    print(tag, "ms per call: median", round(1e3 * float(np.median(ts)), 2), "mean", round(1e3 * float(np.mean(ts)), 2), "min", round(1e3 * min(ts), 2))
    if not a.quiet:
        pstats.Stats(pr).sort_stats("cumulative").print_stats(25)


if __name__ == "__main__":
    main()
