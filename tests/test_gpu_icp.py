"""ICP depth tracker on the B200 vs the restated CPU oracle (oracle/rfo.c).

Per-pixel work is bit-identical; the 29 sums are accumulated in a different
(fixed, tree) order in double, so sums are compared to 1e-9 relative and the
tracked pose to the north-star tolerance 1e-5 rad / 1e-5 m."""
import numpy as np
import pytest

from helpers import AFF, INTR_C1, MAP_C1, PARAMS_C1, GpuEngine
from oracle import rfo

pytestmark = pytest.mark.gpu

ITERS = (6, 10, 20)
DIST = (0.01, 0.02, 0.04)


def _frame(F, poses, f, intr):
    raw, _, _ = F.synth_render(0, poses[f], intr)
    return raw


def _setup(n_render=0):
    import torch  # noqa: F401
    from paper_1708_00783_b200 import fusion as F
    intr = F.Intrinsics(**INTR_C1)
    params = F.SceneParams(**PARAMS_C1)
    poses = F.orbit_trajectory(frames=100)
    g = GpuEngine(*MAP_C1)
    o = rfo.OracleEngine(*MAP_C1)
    raw0 = _frame(F, poses, n_render, intr)
    d0 = rfo.build_view(raw0, INTR_C1, AFF, 1)[0]
    for e in (g, o):
        e.allocate(d0, INTR_C1, poses[n_render], PARAMS_C1)
        e.integrate(d0, INTR_C1, poses[n_render], PARAMS_C1)
        e.render_ranges(poses[n_render], INTR_C1, PARAMS_C1)
    _, gp, gn, _ = g.render_icp(poses[n_render], INTR_C1, PARAMS_C1)
    _, op, on, _ = o.render_icp(poses[n_render], INTR_C1, PARAMS_C1)
    assert np.array_equal(gp.view(np.uint32), op.view(np.uint32))
    return F, intr, params, poses, g, op, on


def rot_err(a, b):
    R = a[:, :3] @ b[:, :3].T
    return float(np.arccos(np.clip((np.trace(R) - 1) / 2, -1, 1)))


@pytest.mark.parametrize("level", [0, 1, 2])
def test_icp_reduce_matches_oracle(level):
    F, intr, params, poses, g, op, on = _setup()
    raw1 = _frame(F, poses, 1, intr)
    calib = F.RgbdCalib(intrinsics_rgb=intr, intrinsics_d=intr, depth_affine=F.DepthAffine(*AFF))
    view = F.build_view(raw1, None, calib, levels=3)
    c2w = np.linalg.inv(np.vstack([poses[0], [0, 0, 0, 1]]).astype(np.float64))[:3].astype(np.float32)
    sums = F.icp_reduce(g.map, view.pyramid[level].depth, level, intr, g.state, c2w, DIST[level])
    lv = rfo.build_view(raw1, INTR_C1, AFF, 3)
    il = intr.atLevel(level)
    ref = rfo.icp_reduce(lv[level], [il.fx, il.fy, il.cx, il.cy], op, on, INTR_C1, poses[0], INTR_C1, c2w,
                         DIST[level])
    assert sums[28] == ref[28] and sums[28] > 1000
    np.testing.assert_allclose(sums, ref, rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("frame", [1, 2])
def test_icp_track_matches_oracle_and_gt(frame):
    F, intr, params, poses, g, op, on = _setup()
    raw = _frame(F, poses, frame, intr)
    calib = F.RgbdCalib(intrinsics_rgb=intr, intrinsics_d=intr, depth_affine=F.DepthAffine(*AFF))
    view = F.build_view(raw, None, calib, levels=3)
    pose_g, summ = F.track_depth(g.map, view, g.state, poses[0], iters=ITERS, dist=DIST)
    lv = rfo.build_view(raw, INTR_C1, AFF, 3)
    pose_o, st = rfo.icp_track(lv, INTR_C1, op, on, poses[0], INTR_C1, poses[0], ITERS, 10, DIST)
    assert summ.ok and st[7] == 1
    assert summ.iterations == int(st[0])
    assert rot_err(pose_g, pose_o) < 1e-5
    assert np.abs(pose_g[:, 3] - pose_o[:, 3]).max() < 1e-5
    # and it actually tracks: within 2 mm / 1e-3 rad of ground truth
    assert np.abs(pose_g[:, 3] - poses[frame][:, 3]).max() < 2e-3
    assert rot_err(pose_g, poses[frame]) < 1e-3


def test_icp_degenerate_empty_depth_keeps_pose():
    F, intr, params, poses, g, op, on = _setup()
    raw = np.zeros((480, 640), np.uint16)
    calib = F.RgbdCalib(intrinsics_rgb=intr, intrinsics_d=intr, depth_affine=F.DepthAffine(*AFF))
    view = F.build_view(raw, None, calib, levels=3)
    pose_g, summ = F.track_depth(g.map, view, g.state, poses[0], iters=ITERS, dist=DIST)
    assert not summ.ok and summ.iterations == 0
    assert np.abs(pose_g - poses[0]).max() < 1e-6


def test_pipeline_with_zero_tracker_iterations_keeps_pose():
    """iters = (0, 0, 0): the tracker launch runs no iteration (and so no
    grid barrier of its own); the frame still renders at, and hands on, the
    seed pose."""
    from paper_1708_00783_b200 import fusion as F
    intr = F.Intrinsics(320, 240, 262.5, 262.5, 159.5, 119.5)
    poses = F.orbit_trajectory(frames=100)
    m = F.VoxelBlockMap(F.VoxelBlockMapConfig(1 << 16, 1 << 14, 1 << 16))
    p = F.Pipeline(m, intr, F.SceneParams(), iters=(0, 0, 0))
    for f in range(4):
        p.process(F.synth_render(0, poses[f], intr)[0], poses[0] if f == 0 else None)
        st, pose, icp = p.result()
        assert icp[0] == 0  # no iteration
        assert np.abs(pose - poses[0]).max() < 1e-6
        assert st.visibleCount > 0
