"""ICP known-answer cases of SPEC.md:354-356 (track_depth examples), shared by
the oracle tests (tests/test_oracle_icp.py) and the B200 tests
(tests/test_gpu_icp.py).

  (a) init = GT pose, plane + sphere scene -> converged pose within
      1e-4 rad / 0.1 mm of GT  [TRIVIAL: zero-residual fixed point];
  (b) init = GT perturbed by 2 deg + 2 cm, sphere-in-room -> recovered within
      0.2 deg / 2 mm  [DERIVED];
  (c) flat featureless plane, pure in-plane translation offset -> Hessian
      near-singular along the sliding directions; the summary reflects the
      low det (and SPEC.md:352: the init pose is returned).
"""
from __future__ import annotations

import numpy as np

from helpers import AFF, INTR_C1, MAP_C1, PARAMS_C1

ITERS = (6, 10, 20)  # bench.py (finest first; SPEC.md:391 20/10/6 coarse -> fine)
DIST = (0.01, 0.02, 0.04)


def pose_err(a, b):
    """(rotation angle rad, camera-centre distance m) between two world->camera poses."""
    Ra, Rb = a[:, :3].astype(np.float64), b[:, :3].astype(np.float64)
    dR = Ra @ Rb.T
    w = np.array([dR[2, 1] - dR[1, 2], dR[0, 2] - dR[2, 0], dR[1, 0] - dR[0, 1]]) / 2
    ang = float(np.arcsin(min(1.0, np.linalg.norm(w))))
    ca = -Ra.T @ a[:, 3].astype(np.float64)
    cb = -Rb.T @ b[:, 3].astype(np.float64)
    return ang, float(np.linalg.norm(ca - cb))


def rot(axis, ang):
    axis = np.asarray(axis, np.float64)
    axis = axis / np.linalg.norm(axis)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + np.sin(ang) * K + (1 - np.cos(ang)) * K @ K


def perturb(pose34, axis, deg, trans):
    """GT pose perturbed by a rotation of `deg` about `axis` and a translation
    `trans` (m), both in the camera frame: P * T_wc."""
    P = np.eye(4)
    P[:3, :3] = rot(axis, np.deg2rad(deg))
    P[:3, 3] = trans
    G = np.vstack([pose34, [0, 0, 0, 1]]).astype(np.float64)
    return (P @ G)[:3].astype(np.float32)


def f32_inverse(pose34):
    """pose.hpp:33-36 in float with Eigen's order (the tracker's T_cw seed)."""
    R = pose34[:, :3].astype(np.float32)
    t = pose34[:, 3].astype(np.float32)
    Rt = R.T.copy()
    ti = np.empty(3, np.float32)
    for r in range(3):
        ti[r] = -(Rt[r, 0] * t[0] + (Rt[r, 1] * t[1] + Rt[r, 2] * t[2]))
    return Rt, ti


def zero_residual_maps(depth, intr, pose34, normals_cam):
    """Render maps that coincide with the frame itself: V(x, y) = the
    tracker's own p_w of pixel (x, y) at the GT pose (backproject then T_cw,
    float ops in the tracker's order), N = the view normals rotated to the
    world.  At init = GT every associated residual is exactly 0."""
    h, w = depth.shape
    R, t = f32_inverse(pose34)
    ys, xs = np.mgrid[0:h, 0:w].astype(np.float32)
    fx, fy = np.float32(intr["fx"]), np.float32(intr["fy"])
    cx, cy = np.float32(intr["cx"]), np.float32(intr["cy"])
    z = depth.astype(np.float32)
    X = (xs - cx) / fx * z
    Y = (ys - cy) / fy * z
    P = np.stack([X, Y, z], -1)
    pw = np.empty_like(P)
    for r in range(3):
        pw[..., r] = (R[r, 0] * P[..., 0] + (R[r, 1] * P[..., 1] + R[r, 2] * P[..., 2])) + t[r]
    valid = (z > 0) & (normals_cam[..., 3] > 0)
    pts = np.zeros((h, w, 4), np.float32)
    nrm = np.zeros((h, w, 4), np.float32)
    pts[..., :3] = pw
    pts[..., 3] = np.where(valid, 1.0, -1.0)
    nc = normals_cam[..., :3].astype(np.float32)
    for r in range(3):
        nrm[..., r] = R[r, 0] * nc[..., 0] + (R[r, 1] * nc[..., 1] + R[r, 2] * nc[..., 2])
    nrm[..., 3] = np.where(valid, 1.0, -1.0)
    return pts, nrm


def frames(F, scene, poses, idx):
    intr = F.Intrinsics(**INTR_C1)
    return [F.synth_render(scene, poses[i], intr)[0] for i in idx]


def oracle_model_maps(rfo, raws, poses, render_pose):
    """An oracle map integrated from `raws` at `poses` (GT), rendered at
    render_pose: (points, normals)."""
    o = rfo.OracleEngine(*MAP_C1)
    for raw, p in zip(raws, poses):
        d = rfo.build_view(raw, INTR_C1, AFF, 1)[0]
        o.allocate(d, INTR_C1, p, PARAMS_C1)
        o.integrate(d, INTR_C1, p, PARAMS_C1)
    o.render_ranges(render_pose, INTR_C1, PARAMS_C1)
    _, pts, nrm, _ = o.render_icp(render_pose, INTR_C1, PARAMS_C1)
    return pts, nrm


def plane_pose():
    """Camera at the origin looking down +z at the checker wall (plane z = 1 m,
    synth.cpp:130-134)."""
    p = np.zeros((3, 4), np.float32)
    p[:3, :3] = np.eye(3, dtype=np.float32)
    return p
