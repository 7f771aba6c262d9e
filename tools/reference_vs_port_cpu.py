"""CPU speed of the live reference (numba backend) vs the C oracle port on the
same sample of the config-2 workload, in THIS container (the reference does
not exist on GPU boxes). Shows that bench.py's reference arm (the port) is not
slower than the reference it stands in for.

    python tools/reference_vs_port_cpu.py [--envs 128] > profiles/r01_reference_vs_port_cpu.json
"""
import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=128)
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    a = ap.parse_args()
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "numba_cache_cmp"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, a.ref)
    import multidepth as ref
    from oracle import oracle as orc
    from paper_2602_03002_b200 import synth
    threads = os.cpu_count()
    w = synth.config("cfg2", a.envs)
    f32 = lambda x: np.asarray(x, np.float64).astype(np.float32).astype(np.float64)  # noqa: E731
    bodies = [(nm, ref.TriMesh(f32(m.vertices), m.faces, frame="body-local")) for nm, m in w.bodies]
    cams = [ref.CameraModel(width=c.width, height=c.height, hfov_deg=c.hfov_deg, vfov_deg=c.vfov_deg,
                            d_max=c.d_max, mount=ref.RigidPose(c.mount.translation, c.mount.rotation),
                            parent_body=c.parent_body) for c in w.cameras]
    scene = ref.Scene(num_envs=w.num_envs, bodies=bodies, cameras=cams,
                      terrain=ref.TriMesh(f32(w.terrain.mesh.vertices), w.terrain.mesh.faces))
    bp, bq = w.poses(0)
    scene.set_body_poses(f32(bp), f32(bq))
    rays = w.num_envs * len(cams) * cams[0].width * cams[0].height
    ref.render(scene, backend="numba", threads=threads)          # JIT warm-up
    t = []
    for _ in range(3):
        t0 = time.perf_counter()
        ref.render(scene, backend="numba", threads=threads)
        t.append(time.perf_counter() - t0)
    ref_render = rays / min(t)
    ocams = [dict(width=c.width, height=c.height, hfov_deg=c.hfov_deg, vfov_deg=c.vfov_deg, d_max=c.d_max,
                  mount_pos=c.mount.translation, mount_rot=c.mount.rotation, parent=c.parent_body) for c in w.cameras]
    osc = orc.OracleScene([(f32(m.vertices), m.faces) for _, m in w.bodies],
                          (f32(w.terrain.mesh.vertices), w.terrain.mesh.faces), ocams)
    osc.render(f32(bp), f32(bq), threads=threads)
    t = []
    for _ in range(3):
        t0 = time.perf_counter()
        osc.render(f32(bp), f32(bq), threads=threads)
        t.append(time.perf_counter() - t0)
    port_render = rays / min(t)
    print(json.dumps({"workload": f"config 2 sample: {w.num_envs} envs x {len(cams)} cams x 64x48, render only",
                      "threads": threads, "reference_numba_rays_per_s": ref_render,
                      "oracle_port_rays_per_s": port_render, "port_over_reference": port_render / ref_render,
                      "how": "best of 3 after warm-up, this container's CPU; tools/reference_vs_port_cpu.py"}, indent=1))


if __name__ == "__main__":
    main()
