"""Edge cases on the GPU vs the oracle:
* ragged image sizes — 173x131 and 97x61, multiples of none of the kernels'
  tiles (16x16 range tiles, 16x8 ray tiles, 32x8 bilateral / stage-1 tiles,
  2x2 pyramid with odd sizes) — through allocation, integration, expected
  ranges, the ICP maps, colour / grey rendering, the full ViewBuilder and
  marching cubes, bit-exact;
* block coordinates beyond the int16 entry layout fail loudly (RFG_ERANGE)
  instead of aliasing;
* the graph-replayed pipeline on a ragged size equals the step-by-step calls.
"""
import numpy as np
import pytest

from helpers import AFF, GpuEngine
from oracle import rfo
from test_gpu_parity import compare_state, run_sequence

pytestmark = pytest.mark.gpu


def _intr(w, h):
    s = w / 640.0
    return dict(width=w, height=h, fx=525.0 * s, fy=525.0 * s, cx=w / 2 - 0.31, cy=h / 2 - 0.77)


def _seq(intr, n, step, rgb=False):
    from paper_1708_00783_b200 import fusion as F
    fi = F.Intrinsics(**intr)
    poses = F.orbit_trajectory(frames=100)
    out = []
    for k in range(n):
        raw, _, col = F.synth_render(0, poses[step * k], fi, rgb=True)
        out.append((poses[step * k], rfo.build_view(raw, intr, AFF, 1)[0], col))
    return out


@pytest.mark.parametrize("wh", [(173, 131), (97, 61)])
def test_ragged_sizes_full_chain_bit_exact(wh):
    from paper_1708_00783_b200 import fusion as F
    intr = _intr(*wh)
    params = F.SceneParams(voxelSize=0.008).as_dict()
    cfg = (1 << 13, 1 << 12, 1 << 13)
    g, o = GpuEngine(*cfg, colour=True), rfo.OracleEngine(*cfg)
    seq = _seq(intr, 5, 9)
    run_sequence(g, o, seq, intr, params, render=True, colour=True)
    pose = seq[-1][0]
    for mode in (1, 2):
        rc, _, nm, col = g.render_maps(mode, pose, intr, params)
        orc, _, onm, _ = o.render_icp(pose, intr, params)
        assert np.array_equal(rc.view(np.uint32), orc.view(np.uint32))
        assert np.array_equal(col, o.render_colour(mode, pose, intr, orc, onm))
    vs = params["voxelSize"]
    mg = F.extract_mesh(g.map, vs)
    vo, to = o.extract_mesh(vs)
    assert np.array_equal(mg.vertices.view(np.uint32), vo.view(np.uint32)) and np.array_equal(mg.triangles, to)
    # full ViewBuilder on the ragged frame (odd pyramid sizes)
    raw, _, col = F.synth_render(0, pose, F.Intrinsics(**intr), rgb=True)
    rng = np.random.default_rng(1)
    noisy = np.clip(raw.astype(np.int64) + rng.integers(-30, 31, raw.shape), 0, 65535).astype(np.uint16)
    noisy[raw == 0] = 0
    cal = F.RgbdCalib(intrinsics_rgb=F.Intrinsics(**intr), intrinsics_d=F.Intrinsics(**intr),
                      depth_affine=F.DepthAffine(*AFF))
    v = F.build_view(noisy, col, cal, F.ViewBuildOptions(bilateral=True, levels=3))
    ov = rfo.build_view_full(noisy, intr, AFF, levels=3, bilateral=True, rgb=col)
    for lv, od, oi in zip(v.pyramid, ov["depth"], ov["intensity"]):
        assert lv.depth.shape == od.shape
        assert np.array_equal(lv.depth.cpu().numpy().view(np.uint32), od.view(np.uint32))
        assert np.array_equal(lv.intensity.cpu().numpy().view(np.uint32), oi.view(np.uint32))
    assert np.array_equal(v.normals.cpu().numpy().view(np.uint32), ov["normals"].view(np.uint32))


def test_block_coordinates_beyond_int16_fail_loudly():
    """16-B entries store int16 block coordinates (1.3 km at 5 mm); a segment
    beyond that raises RFG_ERANGE rather than aliasing another block."""
    from paper_1708_00783_b200 import _lib
    intr = _intr(64, 48)
    g = GpuEngine(1 << 10, 1 << 8, 1 << 10)
    pose = np.eye(3, 4, dtype=np.float32)
    pose[0, 3] = -2000.0  # world x = +2 km in front of the camera's x axis
    d = np.full((48, 64), 1.0, np.float32)
    with pytest.raises(_lib.RfgError) as ei:
        g.allocate(d, intr, pose, dict(voxelSize=0.005, mu=0.02, maxW=100, viewFrustum_min=0.2,
                                       viewFrustum_max=6.0, stopIntegratingAtMaxW=False))
    assert ei.value.code == _lib.RFG_ERANGE


def test_pipeline_ragged_graph_equals_step_calls():
    import torch
    from paper_1708_00783_b200 import fusion as F
    intr = _intr(173, 131)
    fi = F.Intrinsics(**intr)
    params = F.SceneParams(voxelSize=0.008)
    cfg = F.VoxelBlockMapConfig(1 << 13, 1 << 12, 1 << 13)
    poses = F.orbit_trajectory(frames=100)
    raws = [F.synth_render(0, poses[4 * f], fi)[0] for f in range(6)]
    # graph-replayed pipeline at known poses (no tracking)
    m1 = F.VoxelBlockMap(cfg)
    p = F.Pipeline(m1, fi, params, levels=1, track=False, use_graph=True)
    for f, r in enumerate(raws):
        p.process(torch.from_numpy(r.view(np.int16)).cuda(), poses[4 * f])
    p.result()
    # the same frames through the stage calls
    g, o = GpuEngine(cfg.bucketCount, cfg.excessCount, cfg.blockCapacity), rfo.OracleEngine(
        cfg.bucketCount, cfg.excessCount, cfg.blockCapacity)
    for f, r in enumerate(raws):
        d = rfo.build_view(r, intr, AFF, 1)[0]
        for e in (g, o):
            e.allocate(d, intr, poses[4 * f], params.as_dict())
            e.integrate(d, intr, poses[4 * f], params.as_dict())
    compare_state(g, o)
    e1 = m1.entries()
    assert np.array_equal(e1, g.entries())
    ptrs = e1[e1[:, 4] >= 0, 4]
    assert np.array_equal(m1.blocks(ptrs), g.blocks(ptrs))


def test_pipeline_pinned_host_frames_equal_device_frames():
    """rfg_pipeline_process_host reads a pinned host frame in place (the
    graph's view node is pointed at its device alias), a pageable frame is
    copied in: both, with tracking on, give the device-frame pipeline's map,
    pose and tracker summary bit for bit."""
    import torch
    from paper_1708_00783_b200 import fusion as F
    fi = F.Intrinsics(**_intr(160, 120))
    params = F.SceneParams(voxelSize=0.01)
    cfg = F.VoxelBlockMapConfig(1 << 13, 1 << 12, 1 << 13)
    poses = F.orbit_trajectory(frames=100)
    raws = [F.synth_render(0, poses[2 * f], fi)[0] for f in range(8)]
    outs = []
    for mode in ("device", "pinned", "pageable"):
        m = F.VoxelBlockMap(cfg)
        p = F.Pipeline(m, fi, params, levels=2, track=True, use_graph=True)
        res = []
        for f, r in enumerate(raws):
            t = torch.from_numpy(r.view(np.int16))
            src = t.cuda() if mode == "device" else (t.pin_memory().numpy().view(np.uint16) if mode == "pinned" else r)
            p.process(src, poses[0] if f == 0 else None)
            st, pose, icp = p.result()
            res.append((np.asarray(pose).copy(), np.asarray(icp).copy(), str(st)))
        outs.append((res, m.entries()))
    for res, ent in outs[1:]:
        assert np.array_equal(ent, outs[0][1])
        for (pa, ia, sa), (pb, ib, sb) in zip(res, outs[0][0]):
            assert np.array_equal(pa, pb) and np.array_equal(ia, ib) and sa == sb


@pytest.mark.parametrize("other", [(160, 120), (1408, 1024)])
def test_pipeline_recaptures_after_range_scratch_reallocation(other):
    """a map-level render at another image size
    reallocates the map's expected-range scratch, which a pipeline's captured
    frame graph holds; the pipeline must re-capture instead of replaying the
    freed scratch.  The interrupted pipeline matches an uninterrupted one
    bit for bit.  At 1408x1024 the per-tile counters (5,632 tiles) no longer
    fit the map's in-allocation tile scratch and get an allocation of their
    own; back at 320x240 they return to the scratch."""
    import torch
    from paper_1708_00783_b200 import fusion as F
    intr = F.Intrinsics(320, 240, 262.5, 262.5, 159.5, 119.5)
    s = other[0] / 640.0
    small = F.Intrinsics(other[0], other[1], 525.0 * s, 525.0 * s, other[0] / 2 - 0.5, other[1] / 2 - 0.5)
    params = F.SceneParams()
    poses = F.orbit_trajectory(frames=100)
    cfg = F.VoxelBlockMapConfig(1 << 16, 1 << 14, 1 << 16)
    m1, m2 = F.VoxelBlockMap(cfg), F.VoxelBlockMap(cfg)
    p1, p2 = F.Pipeline(m1, intr, params), F.Pipeline(m2, intr, params)
    for f in range(8):
        raw = torch.from_numpy(F.synth_render(0, poses[f], intr)[0].view(np.int16)).cuda()
        if f in (3, 5):  # another size on the pipeline's map, between frames
            rs = F.RenderState()
            F.render_expected_ranges(m1, poses[f], small, params, rs)
            torch.cuda.synchronize()
        p1.process(raw, poses[0] if f == 0 else None)
        p2.process(raw, poses[0] if f == 0 else None)
        s1, q1, i1 = p1.result()
        s2, q2, i2 = p2.result()
        assert np.array_equal(q1, q2) and np.array_equal(i1, i2) and s1 == s2, f"frame {f}"
        for a, b in zip(p1.maps(), p2.maps()):
            assert torch.equal(a.view(torch.int32), b.view(torch.int32)), f"frame {f}: maps differ"


def test_limits_are_rejected_not_truncated():
    """Configurations outside the B200 path's limits fail loudly (the
    reference would run them): mu / voxelSize >= 80 (the 64-cell request-key
    ordinal) and images of >= 2^25 pixels (the 25-bit pixel key)."""
    from paper_1708_00783_b200 import fusion as F
    m = F.VoxelBlockMap(F.VoxelBlockMapConfig(1 << 12, 1 << 10, 1 << 12))
    intr = F.Intrinsics(160, 120, 131.25, 131.25, 79.5, 59.5)
    with pytest.raises(Exception):
        F.Pipeline(m, intr, F.SceneParams(voxelSize=0.001, mu=0.1))
    with pytest.raises(Exception, match="25-bit"):
        F.Pipeline(m, F.Intrinsics(8192, 4096, 4000.0, 4000.0, 4095.5, 2047.5), F.SceneParams())


def test_icp_world_point_out_of_fixed_point_range_fails_loudly():
    """The tracker's fixed-point sums hold world points within +-128 m; a
    frame 200 m from the origin returns RFG_ERANGE instead of wrong sums."""
    import icp_cases as K
    from test_gpu_icp import _track_both  # noqa: F401  (same setup helpers)
    from paper_1708_00783_b200 import fusion as F
    from test_gpu_icp import _state_from_maps, _view
    from helpers import INTR_C1
    intr = F.Intrinsics(**INTR_C1)
    gt = K.plane_pose()
    raw = K.frames(F, 2, [gt], [0])[0]
    lv = rfo.build_view(raw, INTR_C1, AFF, 3)
    far = gt.copy()
    far[0, 3] -= 200.0  # camera (and the wall it sees) 200 m along x
    pts, nrm = K.zero_residual_maps(lv[0], INTR_C1, far, rfo.compute_normals(lv[0], INTR_C1))
    rs = _state_from_maps(F, intr, pts, nrm, far)
    m = F.VoxelBlockMap(F.VoxelBlockMapConfig(1 << 10, 1 << 8, 1 << 8))
    with pytest.raises(Exception, match="fixed-point range"):
        F.track_depth(m, _view(F, intr, raw), rs, far, iters=(6, 0, 0))
    with pytest.raises(ValueError):
        rfo.icp_track(lv, INTR_C1, pts, nrm, far, INTR_C1, far, (6, 0, 0), 10, K.DIST)
