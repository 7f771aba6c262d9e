"""CPU estimate of how many top-of-tree node visits a per-tile (or per-view)
frustum entry node saves per ray (design study for the tile-entry pre-pass).

For each tile of a view, descend the packed terrain BVH from the root while
exactly one child box overlaps the tile's ray frustum (apex = camera, base at
camera z = d_max); the depth reached is the number of node fetches every ray of
the tile skips.

    python tools/entry_depth_sim.py --config cfg2 --views 128
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def frustum(o, R, u0, u1, v0, v1, far):
    """world points: apex + 4 base corners; inward side-plane normals (world)."""
    corners_c = np.array([[u0, v0, 1.0], [u1, v0, 1.0], [u1, v1, 1.0], [u0, v1, 1.0]])
    base = o + (corners_c * far) @ R.T
    pts = np.vstack([o, base])
    dirs = corners_c @ R.T
    planes = []
    for k in range(4):
        n = np.cross(dirs[k], dirs[(k + 1) % 4])
        if np.dot(n, dirs[(k + 2) % 4]) < 0:
            n = -n
        planes.append(n / np.linalg.norm(n))
    fwd = R[:, 2]
    return pts.min(0), pts.max(0), planes, fwd


def overlaps(lo, hi, flo, fhi, planes, fwd, o, far, eps=0.01):
    if np.any(lo > fhi + eps) or np.any(hi < flo - eps):
        return False
    c, h = 0.5 * (lo + hi), 0.5 * (hi - lo)
    for n in planes:
        if np.dot(n, c - o) + np.dot(np.abs(n), h) < -eps:
            return False
    if np.dot(fwd, c - o) - np.dot(np.abs(fwd), h) > far + eps:
        return False
    return True


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--views", type=int, default=64)
    ap.add_argument("--tw", type=int, default=0)
    ap.add_argument("--hint", type=float, default=0.0,
                    help="> 0: far plane = min(d_max, hint * tile max depth + 0.05) from an oracle render")
    a = ap.parse_args()
    import paper_2602_03002_b200 as md
    from paper_2602_03002_b200 import synth, bvh as mbvh
    from oracle import oracle as orc
    w = synth.config(a.config, 4096 if a.config != "paper" else 1024)
    t = w.terrain.mesh
    f32 = lambda x: np.asarray(x, np.float64).astype(np.float32).astype(np.float64)  # noqa: E731
    tree = mbvh.build_bvh(md.TriMesh(f32(t.vertices), t.faces))
    nodes = tree.packed_nodes
    print("terrain nodes", len(nodes))
    C = len(w.cameras)
    n_env = max(1, a.views // C)
    bp, bq = w.poses(0, slice(0, n_env))
    cams = [dict(width=c.width, height=c.height, hfov_deg=c.hfov_deg, vfov_deg=c.vfov_deg, d_max=c.d_max,
                 mount_pos=c.mount.translation, mount_rot=c.mount.rotation, parent=c.parent_body) for c in w.cameras]
    cp, cq = orc.camera_world_poses(cams, bp, bq)
    W, H = w.cameras[0].width, w.cameras[0].height
    depth = None
    if a.hint > 0:
        bodies = [(f32(m.vertices), m.faces) for _, m in w.bodies]
        sc = orc.OracleScene(bodies, (f32(t.vertices), t.faces), cams)
        depth = sc.render(bp, bq, threads=0)
    tw = a.tw or (4 if W <= 96 else 8)
    th = 32 // tw
    depths_tile, depths_view = [], []
    for e in range(n_env):
        for c in range(C):
            cam = w.cameras[c]
            fx = (W / 2) / np.tan(np.radians(cam.hfov_deg) / 2)
            fy = (H / 2) / np.tan(np.radians(cam.vfov_deg) / 2)
            R = orc.quat_to_mat(cq[e, c]) if hasattr(orc, "quat_to_mat") else None
            if R is None:
                q = cq[e, c]
                wq, x, y, z = q
                R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - wq * z), 2 * (x * z + wq * y)],
                              [2 * (x * y + wq * z), 1 - 2 * (x * x + z * z), 2 * (y * z - wq * x)],
                              [2 * (x * z - wq * y), 2 * (y * z + wq * x), 1 - 2 * (x * x + y * y)]])
            o = cp[e, c]
            far = cam.d_max

            def descend(u0, u1, v0, v1, far=far):
                flo, fhi, planes, fwd = frustum(o, R, u0, u1, v0, v1, far)
                ref, d = 0, 0
                while ref >= 0:
                    r = nodes[ref]
                    hits = []
                    for k in (0, 1):
                        lo = np.array([r[f"c{k}x"][0], r[f"c{k}y"][0], r[f"c{k}z"][0]], np.float64)
                        hi = np.array([r[f"c{k}x"][1], r[f"c{k}y"][1], r[f"c{k}z"][1]], np.float64)
                        if lo[0] <= hi[0] and overlaps(lo, hi, flo, fhi, planes, fwd, o, far):
                            hits.append(k)
                    if len(hits) != 1:
                        break
                    ref = int(r["ref"][hits[0]])
                    d += 1
                return d

            u = lambda x: (x + 0.5 - W / 2) / fx  # noqa: E731
            v = lambda y: (y + 0.5 - H / 2) / fy  # noqa: E731
            depths_view.append(descend(u(0), u(W - 1), v(0), v(H - 1)))
            for ty in range(0, H, th):
                for tx in range(0, W, tw):
                    fr = far
                    if depth is not None:
                        blk = depth[e, c, ty:ty + th, tx:tx + tw]
                        fr = min(far, a.hint * float(blk.max()) + 0.05)
                    depths_tile.append(descend(u(tx), u(min(tx + tw, W) - 1), v(ty), v(min(ty + th, H) - 1), fr))
    dt, dv = np.array(depths_tile), np.array(depths_view)
    print(f"{a.config}: tile {tw}x{th}: entry depth mean {dt.mean():.2f} (p10 {np.percentile(dt, 10):.0f}, "
          f"p50 {np.median(dt):.0f}, p90 {np.percentile(dt, 90):.0f}); per-view mean {dv.mean():.2f}")


if __name__ == "__main__":
    main()
