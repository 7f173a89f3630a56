"""BASELINE.json configs[2] (C3): ITMVoxel_s_rgb colour fusion, 640x480 depth +
RGB, 4 mm voxels, through the frame pipeline (the colour packing kernel and
k_integrate_rgbd inside the captured graph) against the CPU oracle, bit for
bit: AllocationStats, the ICP maps every frame, and at checkpoints the whole
hash table and every resident VoxelSRgb block (sdf, w_depth, clr, w_color)
(P/src/fusion.cpp:38-70 colour update, gated at :257).

Plus the map-level colour path with NON-identity extrinsics and a different
colour camera (the general projection of update_voxel_colour,
fusion.cpp:48-52) and with stopIntegratingAtMaxW."""
import numpy as np
import pytest

from helpers import AFF, INTR_C1, PARAMS_C1, GpuEngine, small_intr
from oracle import rfo

pytestmark = pytest.mark.gpu

PARAMS_C3 = dict(PARAMS_C1, voxelSize=0.004)
MAP_C3 = (0x40000, 0x20000, 0x40000)
N_SEQ = 300           # the C3 orbit length
FRAMES = range(0, N_SEQ, 12)  # 25 frames spread over the whole orbit
CHECKPOINTS = (0, 12, 144, 288)


def u32(a):
    return np.ascontiguousarray(a).view(np.uint32)


def _compare_blocks(m, o, f):
    eg, eo = m.entries(), o.entries()
    assert np.array_equal(eg, eo), f"frame {f}: hash entries differ"
    ptrs = eo[eo[:, 4] >= 0, 4]
    bg, bo = m.blocks(ptrs), o.blocks(ptrs)
    if not np.array_equal(bg, bo):
        bad = np.argwhere((bg != bo).any(axis=2))
        raise AssertionError(f"frame {f}: VoxelSRgb differs in {len(bad)} voxels, first {bad[:5].tolist()}")
    colour_w = bo[..., 6]
    return int((colour_w > 0).sum())


@pytest.mark.parametrize("host", [False, True])
def test_c3_colour_pipeline_matches_oracle(host):
    import torch
    from paper_1708_00783_b200 import fusion as F
    rfo.set_threads()
    intr = F.Intrinsics(**INTR_C1)
    params = F.SceneParams(**PARAMS_C3)
    poses = F.orbit_trajectory(frames=N_SEQ)
    m = F.VoxelBlockMap(F.VoxelBlockMapConfig(*MAP_C3), colour=True)
    pipe = F.Pipeline(m, intr, params, F.DepthAffine(*AFF), levels=3, track=False, colour=True, use_graph=True)
    o = rfo.OracleEngine(*MAP_C3)
    coloured = 0
    frames = list(FRAMES) if not host else list(FRAMES)[:8]
    for f in frames:
        raw, _, rgb = F.synth_render(F.SCENE_SPHERE_IN_ROOM, poses[f], intr, rgb=True)
        if host:
            rp = torch.from_numpy(raw.view(np.int16)).pin_memory()
            cp = torch.from_numpy(rgb).pin_memory()
            pipe.process(rp.numpy().view(np.uint16), poses[f], rgb=cp.numpy())
        else:
            pipe.process(torch.from_numpy(raw.view(np.int16)).cuda(), poses[f],
                         rgb=torch.from_numpy(rgb).cuda())
        st_g, pose_g, _ = pipe.result()
        assert np.array_equal(pose_g, poses[f])
        d = rfo.build_view(raw, INTR_C1, AFF, 1)[0]
        st_o, _ = o.allocate(d, INTR_C1, poses[f], PARAMS_C3)
        assert np.array_equal(st_g.as_array(), st_o), f"frame {f}: AllocationStats {st_g} vs {st_o}"
        o.integrate(d, INTR_C1, poses[f], PARAMS_C3, rgb=rgb, intr_rgb=INTR_C1)
        o.render_ranges(poses[f], INTR_C1, PARAMS_C3)
        rc_o, pts_o, nrm_o, _ = o.render_icp(poses[f], INTR_C1, PARAMS_C3)
        _, rc_g, pts_g, nrm_g = (t.cpu().numpy() for t in pipe.maps())
        assert np.array_equal(u32(pts_g), u32(pts_o)), f"frame {f}: points differ"
        assert np.array_equal(u32(nrm_g), u32(nrm_o)), f"frame {f}: normals differ"
        if f in CHECKPOINTS or f == frames[-1]:
            coloured = _compare_blocks(m, o, f)
    assert coloured > 1_000_000  # the colour planes were really written


def test_c3_tracked_colour_pipeline_matches_oracle():
    """Colour fusion with the tracker on (C2 + C3): the oracle runs its own
    tracked chain; poses and colour voxels bit-exact."""
    import torch
    from paper_1708_00783_b200 import fusion as F
    rfo.set_threads()
    intr = F.Intrinsics(**INTR_C1)
    params = F.SceneParams(**PARAMS_C3)
    poses = F.orbit_trajectory(frames=100)
    m = F.VoxelBlockMap(F.VoxelBlockMapConfig(*MAP_C3), colour=True)
    pipe = F.Pipeline(m, intr, params, F.DepthAffine(*AFF), levels=3, track=True, colour=True)
    o = rfo.OracleEngine(*MAP_C3)
    prev = None
    for f in range(12):
        raw, _, rgb = F.synth_render(F.SCENE_SPHERE_IN_ROOM, poses[f], intr, rgb=True)
        pipe.process(torch.from_numpy(raw.view(np.int16)).cuda(), poses[0] if f == 0 else None,
                     rgb=torch.from_numpy(rgb).cuda())
        _, pose_g, _ = pipe.result()
        lv = rfo.build_view(raw, INTR_C1, AFF, 3)
        pose_o = poses[0]
        if prev is not None:
            pose_o, st = rfo.icp_track(lv, INTR_C1, prev[0], prev[1], prev[2], INTR_C1, prev[2])
            assert st[7] == 1
        assert np.array_equal(u32(pose_g), u32(pose_o)), f"frame {f}: pose differs"
        o.allocate(lv[0], INTR_C1, pose_o, PARAMS_C3)
        o.integrate(lv[0], INTR_C1, pose_o, PARAMS_C3, rgb=rgb, intr_rgb=INTR_C1)
        o.render_ranges(pose_o, INTR_C1, PARAMS_C3)
        _, pts_o, nrm_o, _ = o.render_icp(pose_o, INTR_C1, PARAMS_C3)
        prev = (pts_o, nrm_o, pose_o.copy())
    _compare_blocks(m, o, 11)


def _extr(deg, t):
    c, s = np.cos(np.deg2rad(deg)), np.sin(np.deg2rad(deg))
    e = np.zeros((3, 4), np.float32)
    e[:3, :3] = np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]], np.float32)
    e[:, 3] = t
    return e


@pytest.mark.parametrize("extr,intr_rgb", [
    (_extr(3.0, [0.025, -0.004, 0.002]), small_intr(320, 240)),          # rotated + shifted colour camera
    (np.eye(3, 4, dtype=np.float32), dict(small_intr(320, 240), fx=300.0, cx=150.25)),  # other intrinsics
])
def test_colour_general_camera_matches_oracle(extr, intr_rgb):
    from paper_1708_00783_b200 import fusion as F
    intr = small_intr(320, 240)
    poses = F.orbit_trajectory(frames=20)
    g = GpuEngine(1 << 16, 1 << 14, 1 << 16, colour=True)
    o = rfo.OracleEngine(1 << 16, 1 << 14, 1 << 16)
    i = F.Intrinsics(**intr)
    ir = F.Intrinsics(**intr_rgb)
    for k in range(0, 20, 4):
        raw, _, _ = F.synth_render(0, poses[k], i)
        _, _, rgb = F.synth_render(0, poses[k], ir, rgb=True)  # colour image of the colour camera's size
        d = rfo.build_view(raw, intr, AFF, 1)[0]
        for e in (g, o):
            e.allocate(d, intr, poses[k], PARAMS_C3)
            e.integrate(d, intr, poses[k], PARAMS_C3, rgb=rgb, intr_rgb=intr_rgb, extr34=extr)
    n = _compare_blocks(g, o, "last")
    assert n > 10_000


def test_colour_stop_at_max_w_matches_oracle():
    from paper_1708_00783_b200 import fusion as F
    intr = small_intr(160, 120)
    params = dict(PARAMS_C3, maxW=3, stopIntegratingAtMaxW=True)
    pose = F.orbit_trajectory(frames=10)[2]
    raw, _, rgb = F.synth_render(0, pose, F.Intrinsics(**intr), rgb=True)
    d = rfo.build_view(raw, intr, AFF, 1)[0]
    g = GpuEngine(1 << 14, 1 << 12, 1 << 14, colour=True)
    o = rfo.OracleEngine(1 << 14, 1 << 12, 1 << 14)
    for _ in range(5):
        for e in (g, o):
            e.allocate(d, intr, pose, params)
            e.integrate(d, intr, pose, params, rgb=rgb, intr_rgb=intr)
    _compare_blocks(g, o, "last")
