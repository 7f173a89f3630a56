"""Colour / grey render modes (§8(f)4, raycast.hpp:157-207,
raycast.cpp:129-139) on the GPU vs the oracle, bit-exact, on a colour-fused
sequence (C3 style: RGB integration, 4 mm voxels) and a depth-only map;
plus the missing-only (approximate raycast) form.  The oracle's colour pass
(oracle/rfo.c:rfo_render_colour) is pinned to the reference build in
tests/test_oracle_render_modes.py."""
import numpy as np
import pytest

from helpers import AFF, GpuEngine, small_intr
from oracle import rfo

pytestmark = pytest.mark.gpu


def _run(colour, vs=0.004, frames=4):
    from paper_1708_00783_b200 import fusion as F
    intr = small_intr(160, 120)
    fi = F.Intrinsics(**intr)
    pd = F.SceneParams(voxelSize=vs).as_dict()
    poses = F.orbit_trajectory(frames=100)
    cfg = (0x8000, 0x4000, 0x8000)
    g, o = GpuEngine(*cfg, colour=colour), rfo.OracleEngine(*cfg)
    for f in range(frames):
        raw, _, col = F.synth_render(0, poses[5 * f], fi, rgb=True)
        d = rfo.build_view(raw, intr, AFF, 1)[0]
        for e in (g, o):
            e.allocate(d, intr, poses[5 * f], pd)
            if colour:
                e.integrate(d, intr, poses[5 * f], pd, rgb=col, intr_rgb=intr)
            else:
                e.integrate(d, intr, poses[5 * f], pd)
            e.render_ranges(poses[5 * f], intr, pd)
    return g, o, intr, pd, poses[5 * (frames - 1)]


@pytest.mark.parametrize("colour", [True, False])
def test_colour_and_grey_modes_bit_exact(colour):
    g, o, intr, pd, pose = _run(colour)
    for mode in (1, 2):
        rc, pts, nrm, col = g.render_maps(mode, pose, intr, pd)
        orc, opt, onm, _ = o.render_icp(pose, intr, pd)
        assert np.array_equal(rc.view(np.uint32), orc.view(np.uint32))
        assert np.array_equal(nrm.view(np.uint32), onm.view(np.uint32))
        ocol = o.render_colour(mode, pose, intr, orc, onm)
        assert np.array_equal(col, ocol)
        lit = (col > 0).any(axis=2).sum()
        assert lit > (5000 if (mode == 2 or colour) else -1)
        if not colour and mode == 1:
            assert lit == 0  # depth-only map: no colour (an un-coloured VoxelSRgb map renders black)


def test_colour_mode_missing_only():
    """render_maps(kColour, missingOnly): only the listed pixels are
    rewritten."""
    import torch
    from paper_1708_00783_b200 import fusion as F
    g, o, intr, pd, pose = _run(True)
    fi = F.Intrinsics(**intr)
    F.render_maps(g.map, pose, fi, F.SceneParams(**pd), F.RenderMode.kColour, g.state)
    base = g.state.colour.clone()
    n = intr["width"] * intr["height"]
    rng = np.random.default_rng(0)
    pick = np.sort(rng.choice(n, n // 5, replace=False)).astype(np.int32)
    g.state.colour.fill_(7)
    miss = F.MissingPixels(n, intr["width"])
    miss.index[: len(pick)] = torch.as_tensor(pick, device="cuda")
    miss.count.fill_(len(pick))
    F.render_maps(g.map, pose, fi, F.SceneParams(**pd), F.RenderMode.kColour, g.state, missingOnly=miss)
    got = g.state.colour.cpu().numpy().reshape(-1, 3)
    want = np.full_like(got, 7)
    want[pick] = base.cpu().numpy().reshape(-1, 3)[pick]
    assert np.array_equal(got, want)
