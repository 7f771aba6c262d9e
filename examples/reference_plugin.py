"""INTEGRATION.md section 1, end to end: the reference package (`multidepth`, installed
unmodified into baseline/_ref by `__graft_entry__.build()`) renders through this repo's
CUDA backend after the two-line registry change, then through its own numba backend.

    python examples/reference_plugin.py [--envs 256]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/mdrt_numba_cache")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=256)
    a = ap.parse_args()
    import multidepth as ref
    from multidepth import kernels as mk
    from paper_2602_03002_b200.kernels import cuda_backend
    from paper_2602_03002_b200 import synth

    # the registry change a maintainer adds (multidepth/kernels/__init__.py:53-60)
    original = mk.get_render_fn
    mk.BACKENDS = tuple(mk.BACKENDS) + ("cuda",)
    mk.get_render_fn = lambda backend=None: (("cuda", cuda_backend.render_batch)
                                             if backend == "cuda" else original(backend))

    w = synth.config("cfg2", a.envs)
    f64 = lambda x: np.asarray(x, np.float64).astype(np.float32).astype(np.float64)  # noqa: E731
    bodies = [(nm, ref.TriMesh(f64(m.vertices), m.faces, frame="body-local")) for nm, m in w.bodies]
    cams = [ref.CameraModel(width=c.width, height=c.height, hfov_deg=c.hfov_deg, vfov_deg=c.vfov_deg, d_max=c.d_max,
                            mount=ref.RigidPose(c.mount.translation, c.mount.rotation), parent_body=c.parent_body)
            for c in w.cameras]
    scene = ref.Scene(num_envs=a.envs, bodies=bodies, cameras=cams,
                      terrain=ref.TriMesh(f64(w.terrain.mesh.vertices), w.terrain.mesh.faces))
    bp, bq = w.poses(0)
    scene.set_body_poses(f64(bp), f64(bq))
    rays = a.envs * len(cams) * cams[0].width * cams[0].height
    for backend in ("cuda", "numba"):
        ref.render(scene, backend=backend)                       # warm-up (context build / JIT)
        t0 = time.perf_counter()
        frame = ref.render(scene, backend=backend)
        dt = time.perf_counter() - t0
        print(f"multidepth.render(backend={backend!r}): {dt * 1e3:.1f} ms, {rays / dt:.3g} rays/s "
              f"(includes the reference's own host-side camera poses and ray grids)")
        if backend == "cuda":
            cuda_depth = frame.data
    diff = np.abs(cuda_depth.astype(np.float64) - frame.data)
    print(f"cuda vs numba: max |diff| {diff.max():.2e} m, pixels beyond 1e-4 m: {(diff > 1e-4).sum()} of {diff.size}")


if __name__ == "__main__":
    main()
