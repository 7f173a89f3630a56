"""ICP depth tracker on the B200 vs the CPU oracle (oracle/rfo.c:rfo_icp_track)
and SPEC.md's known answers for track_depth.

The tracker's sums are fixed-point integers (order-independent), and the
solve / SE(3) update run the oracle's IEEE operation sequence, so everything
is compared BIT-exact: the 31 sums, the tracked pose, the 12-value
TrackerIterationSummary."""
import numpy as np
import pytest

import icp_cases as K
from helpers import AFF, INTR_C1, MAP_C1, PARAMS_C1, GpuEngine
from oracle import rfo

pytestmark = pytest.mark.gpu

ITERS, DIST = K.ITERS, K.DIST


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


def _view(F, intr, raw):
    calib = F.RgbdCalib(intrinsics_rgb=intr, intrinsics_d=intr, depth_affine=F.DepthAffine(*AFF))
    return F.build_view(raw, None, calib, levels=3)


def _state_from_maps(F, intr, pts, nrm, pose):
    """A RenderState holding given (host) points / normals rendered at `pose`."""
    import torch
    rs = F.RenderState()
    rs.resize(intr)
    rs.points.copy_(torch.from_numpy(np.ascontiguousarray(pts, np.float32)))
    rs.normals.copy_(torch.from_numpy(np.ascontiguousarray(nrm, np.float32)))
    rs.pose = np.asarray(pose, np.float32).copy()
    rs.hasRaycast = True
    return rs


def _track_both(F, intr, raw, pts, nrm, render_pose, init, iters=ITERS, map_=None):
    """GPU track_depth and the oracle on the same inputs: both results, asserted identical."""
    view = _view(F, intr, raw)
    rs = _state_from_maps(F, intr, pts, nrm, render_pose)
    m = map_ or F.VoxelBlockMap(F.VoxelBlockMapConfig(1 << 10, 1 << 8, 1 << 8))
    pose_g, summ = F.track_depth(m, view, rs, init, iters=iters, dist=DIST)
    lv = rfo.build_view(raw, INTR_C1, AFF, 3)
    pose_o, st = rfo.icp_track(lv, INTR_C1, pts, nrm, render_pose, INTR_C1, init, iters, 10, DIST)
    assert np.array_equal(pose_g.view(np.uint32), pose_o.view(np.uint32)), "tracked pose differs from the oracle"
    assert summ == F.TrackerIterationSummary.from_stats(st), f"summary {summ} vs {st}"
    return pose_g, summ


@pytest.mark.parametrize("level", [0, 1, 2])
def test_icp_reduce_matches_oracle_exactly(level):
    F, intr, params, poses, g, op, on = _setup()
    raw1 = _frame(F, poses, 1, intr)
    view = _view(F, intr, raw1)
    c2w = np.linalg.inv(np.vstack([poses[0], [0, 0, 0, 1]]).astype(np.float64))[:3].astype(np.float32)
    fixed_g = F.icp_reduce(g.map, view.pyramid[level].depth, level, intr, g.state, c2w, DIST[level], fixed=True)
    sums_g = F.icp_reduce(g.map, view.pyramid[level].depth, level, intr, g.state, c2w, DIST[level])
    lv = rfo.build_view(raw1, INTR_C1, AFF, 3)
    il = intr.atLevel(level)
    args = (lv[level], [il.fx, il.fy, il.cx, il.cy], op, on, INTR_C1, poses[0], INTR_C1, c2w, DIST[level])
    fixed_o = rfo.icp_reduce(*args, fixed=True)
    assert np.array_equal(fixed_g, fixed_o)
    assert np.array_equal(sums_g, rfo.icp_reduce(*args))
    assert fixed_g[28] > 1000 and fixed_g[30] == (lv[level] > 0).sum()


@pytest.mark.parametrize("frame", [1, 2, 5])
def test_icp_track_matches_oracle_and_gt(frame):
    F, intr, params, poses, g, op, on = _setup()
    raw = _frame(F, poses, frame, intr)
    pose_g, summ = _track_both(F, intr, raw, op, on, poses[0], poses[0], map_=g.map)
    assert summ.ok and summ.converged
    # and it actually tracks: within 2 mm / 1e-3 rad of ground truth
    ang, dc = K.pose_err(pose_g, poses[frame])
    assert ang < 1e-3 and dc < 2e-3


def test_zero_residual_fixed_point():
    """SPEC.md:354 (a): maps equal to the frame itself, init = GT -> one
    zero step, converged at GT."""
    from paper_1708_00783_b200 import fusion as F
    intr = F.Intrinsics(**INTR_C1)
    poses = F.orbit_trajectory(frames=100)
    raw = _frame(F, poses, 10, intr)
    lv = rfo.build_view(raw, INTR_C1, AFF, 3)
    pts, nrm = K.zero_residual_maps(lv[0], INTR_C1, poses[10], rfo.compute_normals(lv[0], INTR_C1))
    pose, summ = _track_both(F, intr, raw, pts, nrm, poses[10], poses[10], iters=(6, 0, 0))
    assert summ.ok and summ.converged and summ.iterations == 1 and summ.residual_sum == 0.0
    ang, dc = K.pose_err(pose, poses[10])
    assert ang < 1e-6 and dc < 1e-6


@pytest.mark.parametrize("axis,trans", [([1, 0, 0], [0, 0.02, 0]), ([0, 0, 1], [0.02, 0, 0]),
                                        ([1, 1, 0], [0, 0.0142, 0.0142])])
def test_recovers_2deg_2cm_perturbation(axis, trans):
    """SPEC.md:355 (b): GT + 2 deg + 2 cm -> within 0.2 deg / 2 mm."""
    from paper_1708_00783_b200 import fusion as F
    rfo.set_threads()
    intr = F.Intrinsics(**INTR_C1)
    poses = F.orbit_trajectory(frames=100)
    f = 10
    raws = K.frames(F, 0, poses, range(f + 1))
    pts, nrm = K.oracle_model_maps(rfo, raws[:f], poses[:f], poses[f - 1])
    init = K.perturb(poses[f], axis, 2.0, trans)
    pose, summ = _track_both(F, intr, raws[f], pts, nrm, poses[f - 1], init)
    ang, dc = K.pose_err(pose, poses[f])
    assert summ.ok and np.rad2deg(ang) < 0.2 and dc < 2e-3


def test_plane_degenerate_returns_init():
    """SPEC.md:356 (c) + :352: exact plane, in-plane offset -> degenerate,
    init pose returned, hessian_det < 1e-12."""
    from paper_1708_00783_b200 import fusion as F
    intr = F.Intrinsics(**INTR_C1)
    gt = K.plane_pose()
    raw = K.frames(F, 2, [gt], [0])[0]
    lv = rfo.build_view(raw, INTR_C1, AFF, 3)
    pts, nrm = K.zero_residual_maps(lv[0], INTR_C1, gt, rfo.compute_normals(lv[0], INTR_C1))
    init = gt.copy()
    init[0, 3] += 0.02
    pose, summ = _track_both(F, intr, raw, pts, nrm, gt, init)
    assert not summ.ok and not summ.converged and summ.iterations == 0
    assert summ.hessian_det < 1e-12 and summ.count > 10_000
    assert np.array_equal(pose, init)


def test_icp_degenerate_empty_depth_keeps_pose():
    F, intr, params, poses, g, op, on = _setup()
    raw = np.zeros((480, 640), np.uint16)
    view = _view(F, intr, raw)
    pose_g, summ = F.track_depth(g.map, view, g.state, poses[0], iters=ITERS, dist=DIST)
    assert not summ.ok and summ.iterations == 0 and summ.valid == 0 and summ.inlier_fraction == 0.0
    assert np.array_equal(pose_g, poses[0])


def test_icp_rejects_gates_outside_fixed_point_range():
    F, intr, params, poses, g, op, on = _setup()
    view = _view(F, intr, _frame(F, poses, 1, intr))
    with pytest.raises(Exception, match="gates"):
        F.track_depth(g.map, view, g.state, poses[0], iters=ITERS, dist=(0.01, 0.02, 3.0))


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
