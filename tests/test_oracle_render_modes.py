"""The oracle's colour / grey render modes (oracle/rfo.c:rfo_render_colour)
pinned bit-for-bit to the reference build's render_maps(kColour / kGrey)
(oracle/_ref; raycast.cpp:129-139, raycast.hpp:157-207)."""
import numpy as np
import pytest

from helpers import AFF, small_intr
from oracle import ref, rfo

pytestmark = pytest.mark.skipif(not ref.available(), reason="reference build (oracle/_ref) not available")


@pytest.mark.parametrize("colour", [True, False])
def test_render_modes_oracle_pinned_to_reference(colour):
    from paper_1708_00783_b200 import fusion as F
    intr = small_intr(96, 72)
    fi = F.Intrinsics(**intr)
    pd = F.SceneParams(voxelSize=0.008).as_dict()
    poses = F.orbit_trajectory(frames=100)
    cfg = (0x4000, 0x2000, 0x4000)
    R, O = ref.RefEngine(*cfg), rfo.OracleEngine(*cfg)
    for f in range(3):
        raw, _, col = F.synth_render(0, poses[6 * f], fi, rgb=True)
        d = rfo.build_view(raw, intr, AFF, 1)[0]
        for e in (R, O):
            e.allocate(d, intr, poses[6 * f], pd)
            if colour:
                e.integrate(d, intr, poses[6 * f], pd, rgb=col, intr_rgb=intr)
            else:
                e.integrate(d, intr, poses[6 * f], pd)
            e.render_ranges(poses[6 * f], intr, pd)
    pose = poses[12]
    for mode in (1, 2):
        rc, pts, nrm, rcol = R.render_maps(mode, pose, intr, pd)
        orc, opt, onm, _ = O.render_icp(pose, intr, pd)
        assert np.array_equal(rc.view(np.uint32), orc.view(np.uint32))
        ocol = O.render_colour(mode, pose, intr, orc, onm)
        assert np.array_equal(rcol, ocol)
        assert (rcol > 0).any(axis=2).sum() > (1000 if (mode == 2 or colour) else -1)
