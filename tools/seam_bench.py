"""Throughput through the reference's own plugin seam: ``render_batch`` called
exactly as ``multidepth.scene.render`` calls its backend (numba_backend.py:
222-234): f64 numpy poses, camera poses and ray grids in, a fresh numpy
(N,C,H,W) float32 ``out`` written in place (wall clock per call, host buffers).

    python tools/seam_bench.py [--config cfg2] [--calls 20]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_03002_b200 as md  # noqa: E402
from paper_2602_03002_b200 import kernels, synth  # noqa: E402


class Flat:
    """The FlatGeometry fields the CUDA backend reads (scene.py:49-78)."""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--calls", type=int, default=20)
    a = ap.parse_args()
    w = synth.config(a.config)
    n, cams = w.num_envs, w.cameras
    flat = Flat()
    tris = [m.triangles() for _, m in w.bodies]
    flat.tri_v0, flat.tri_v1, flat.tri_v2 = (np.concatenate([t[:, k] for t in tris]) for k in range(3))
    flat.body_tri_offsets = np.cumsum([0] + [len(t) for t in tris])
    flat.body_root = np.zeros(len(tris), np.int32)
    g = w.terrain.mesh.triangles()
    flat.g_tri_v0, flat.g_tri_v1, flat.g_tri_v2 = g[:, 0], g[:, 1], g[:, 2]
    scene = md.Scene(n, bodies=w.bodies, cameras=cams, terrain=w.terrain.mesh)   # host mirrors of the poses
    _, render_batch = kernels.get_render_fn("cuda")
    dmax = np.array([c.d_max for c in cams])
    grids = scene.ray_grids()
    res = []
    for k in range(a.calls + 2):
        bp, bq = w.poses(k)
        scene.set_body_poses(bp, bq)
        cp, cq = scene.camera_world_poses()
        out = np.empty(scene.frame_shape, np.float32)            # scene.py:344-347 allocates per call
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        render_batch(flat, bp, bq, cp, cq, grids[0], grids[1], dmax, True, out, None)
        torch.cuda.synchronize()
        res.append(time.perf_counter() - t0)
    t = np.mean(res[2:])
    rays = n * len(cams) * cams[0].width * cams[0].height
    print(json.dumps({"config": a.config, "ms_per_call": t * 1e3, "rays_per_s": rays / t,
                      "how": "render_batch(flat, f64 numpy inputs, fresh numpy out) wall clock per call"}))


if __name__ == "__main__":
    main()
