"""Serialised render cases shared by the golden generator and the parity tests.

A case is a flat dict of numpy arrays (stored as .npz):

  body{i}_v (V,3) f64, body{i}_f (F,3) i64, num_bodies ()
  terrain_v, terrain_f (optional)
  cam_w, cam_h (), cam_hfov/cam_vfov/cam_dmax (C,), cam_parent (C,) (-1 = world mount),
  cam_mpos (C,3), cam_mrot (C,4) (RigidPose rotations, already unit)
  body_pos (N,B,3), body_rot (N,B,4) -- float32-representable values
  rand_pos (N,C,3), rand_rot (N,C,4), rand_fov (N,C) (optional)
  early () bool
  out (N,C,H,W) f32 -- the reference renderer's output on exactly these inputs
"""

from __future__ import annotations

import numpy as np


def bodies(case):
    return [(case[f"body{i}_v"], case[f"body{i}_f"]) for i in range(int(case["num_bodies"]))]


def terrain(case):
    return (case["terrain_v"], case["terrain_f"]) if "terrain_v" in case else None


def cameras_dicts(case):
    out = []
    for c in range(len(case["cam_hfov"])):
        p = int(case["cam_parent"][c])
        out.append(dict(width=int(case["cam_w"]), height=int(case["cam_h"]),
                        hfov_deg=float(case["cam_hfov"][c]), vfov_deg=float(case["cam_vfov"][c]),
                        d_max=float(case["cam_dmax"][c]), mount_pos=case["cam_mpos"][c],
                        mount_rot=case["cam_mrot"][c], parent=None if p < 0 else p))
    return out


def rand(case):
    if "rand_pos" in case:
        return case["rand_pos"], case["rand_rot"], case["rand_fov"]
    return None


def load(path) -> dict:
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def build_scene(case, pkg, device=None):
    """Construct the package Scene (GPU) for a case. ``pkg`` is paper_2602_03002_b200."""
    meshes = [(f"b{i}", pkg.TriMesh(v, f, frame="body-local")) for i, (v, f) in enumerate(bodies(case))]
    t = terrain(case)
    cams = []
    for d in cameras_dicts(case):
        mount = pkg.RigidPose(d["mount_pos"], d["mount_rot"])
        cams.append(pkg.CameraModel(width=d["width"], height=d["height"], hfov_deg=d["hfov_deg"],
                                    vfov_deg=d["vfov_deg"], d_max=d["d_max"], mount=mount,
                                    parent_body=d["parent"]))
    n = case["body_pos"].shape[0] if int(case["num_bodies"]) else int(case.get("num_envs", 1))
    scene = pkg.Scene(n, bodies=meshes, cameras=cams,
                      terrain=None if t is None else pkg.TriMesh(*t), device=device)
    if int(case["num_bodies"]):
        scene.set_body_poses(case["body_pos"], case["body_rot"])
    r = rand(case)
    if r is not None:
        scene.set_camera_randomization(*r)
    return scene
