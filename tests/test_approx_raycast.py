"""Approximate raycast (useApproximateRaycast):
forward_project (proj/src/raycast.cpp:141-188) + render_maps(missingOnly)
(proj/include/rf/raycast.hpp:200-202).  The oracle is pinned to the
reference build; the B200 kernels are compared with the oracle bit-exactly."""
import numpy as np
import pytest

from helpers import AFF, PARAMS_C1, small_intr
from oracle import ref, rfo

CFG = (1 << 14, 1 << 12, 1 << 14)


def _fuse(E, intr, poses, frames, render):
    for f in frames:
        raw, _, _ = render(0, poses[f], intr)
        d = rfo.build_view(raw, intr, AFF, 1)[0]
        E.allocate(d, intr, poses[f], PARAMS_C1)
        E.integrate(d, intr, poses[f], PARAMS_C1)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_oracle_forward_project_pinned_to_reference():
    intr = small_intr(160, 120)
    poses = ref.orbit_poses([0, 0.15, 1.4], 1.4, 100, 0.5)
    A, B = ref.RefEngine(*CFG), rfo.OracleEngine(*CFG)
    for E in (A, B):
        _fuse(E, intr, poses, (0, 3), ref.render)
        E.render_ranges(poses[3], intr, PARAMS_C1)
    A.render_icp(poses[3], intr, PARAMS_C1)
    rc, pts, nrm = [x.copy() for x in B.render_icp(poses[3], intr, PARAMS_C1)[:3]]
    for new in (5, 9):  # small and larger motion
        ma = A.forward_project(poses[new], intr, 0.005)
        mb = rfo.forward_project(True, rc, pts, nrm, poses[new], intr, 0.005)
        assert np.array_equal(ma, mb) and 0 < len(ma) < 160 * 120
        for E in (A, B):
            E.render_ranges(poses[new], intr, PARAMS_C1)
        xa = A.render_icp_missing(poses[new], intr, PARAMS_C1, ma)
        B.render_icp_list(poses[new], intr, PARAMS_C1, mb, rc, pts, nrm)
        for a, b in zip(xa, (rc, pts, nrm)):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_oracle_forward_project_without_raycast_marks_everything():
    intr = small_intr(32, 24)
    z = np.zeros((24, 32, 4), np.float32)
    m = rfo.forward_project(False, z.copy(), z.copy(), z.copy(), np.eye(3, 4, dtype=np.float32), intr, 0.005)
    assert len(m) == 32 * 24 and m[0].tolist() == [0, 0] and m[-1].tolist() == [31, 23]


@pytest.mark.gpu
def test_gpu_forward_project_and_missing_render_match_oracle():
    from helpers import GpuEngine
    from paper_1708_00783_b200 import fusion as F
    intr = small_intr(320, 240)
    poses = F.orbit_trajectory(frames=100)
    g, o = GpuEngine(*CFG), rfo.OracleEngine(*CFG)
    render = lambda s, p, i: F.synth_render(s, p, F.Intrinsics(**i))  # noqa: E731
    for E in (g, o):
        _fuse(E, intr, poses, (0, 3), render)
        E.render_ranges(poses[3], intr, PARAMS_C1)
    g.render_icp(poses[3], intr, PARAMS_C1)
    rc, pts, nrm = [x.copy() for x in o.render_icp(poses[3], intr, PARAMS_C1)[:3]]
    Fi = F.Intrinsics(**intr)
    # no previous raycast: every pixel is missing
    fresh = F.RenderState()
    assert len(F.forward_project(fresh, poses[3], Fi, 0.005, g.map)) == 320 * 240
    for new in (5, 9):
        miss = F.forward_project(g.state, poses[new], Fi, 0.005, g.map)
        mo = rfo.forward_project(True, rc, pts, nrm, poses[new], intr, 0.005)
        assert np.array_equal(miss.xy(), mo)
        for name, a, b in (("raycast", g.state.raycastResult, rc), ("points", g.state.points, pts),
                           ("normals", g.state.normals, nrm)):
            assert np.array_equal(a.cpu().numpy().view(np.uint32), b.view(np.uint32)), name
        g.render_ranges(poses[new], intr, PARAMS_C1)
        o.render_ranges(poses[new], intr, PARAMS_C1)
        F.render_maps(g.map, poses[new], Fi, F.SceneParams(**PARAMS_C1), F.RenderMode.kIcpMaps, g.state,
                      missingOnly=miss)
        o.render_icp_list(poses[new], intr, PARAMS_C1, mo, rc, pts, nrm)
        for name, a, b in (("raycast", g.state.raycastResult, rc), ("points", g.state.points, pts),
                           ("normals", g.state.normals, nrm)):
            assert np.array_equal(a.cpu().numpy().view(np.uint32), b.view(np.uint32)), name
