"""Swapping engine on the GPU (rfg_swap.cu) vs the oracle's restatement of
SPEC.md:407-465 (oracle/rfo.c:rfo_swap_*), bit-exact every frame of a
revisiting trajectory: entries, visible list + types (incl. kBoundary and
kVisibleSwapped), free stack, resident VBA, host-store flags, invisible-frame
ages and the stored blocks — with a transfer capacity small enough that
demand is deferred across frames and one large enough that it is not; plus
the reference hooks (reserveBlockForEntry / releaseBlock) and colour maps."""
import numpy as np
import pytest

from helpers import AFF, GpuEngine, small_intr
from oracle import rfo
from test_oracle_swapping import CFG, ORDER, _frames, _params, _same_state

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cap,chunked", [(37, False), (100000, False), (37, True)])
def test_swapping_engine_bit_exact_vs_oracle(cap, chunked, monkeypatch):
    if chunked:  # host tier grown in 64-slot pinned chunks instead of pinned up front
        monkeypatch.setenv("RFG_SWAP_PIN_UPFRONT", "0")
        monkeypatch.setenv("RFG_SWAP_CHUNK_SLOTS", "64")
    intr, pd = small_intr(), _params()
    g, o = GpuEngine(*CFG), rfo.OracleEngine(*CFG)
    for e in (g, o):
        e.set_fusion_options(True, 8.0)
        e.swap_create(cap)
    moved = 0
    for pose, d in _frames(intr, ORDER + ORDER[1:]):
        for e in (g, o):
            e.allocate(d, intr, pose, pd)
        ni = (g.swap_in(), o.swap_in())
        assert ni[0] == ni[1]
        for e in (g, o):
            e.integrate(d, intr, pose, pd)
        no = (g.swap_out(), o.swap_out())
        assert no[0] == no[1]
        moved += ni[0] + no[0]
        _same_state(g, o)
        hg, ag = g.swap_stored()
        ho, ao = o.swap_stored()
        assert np.array_equal(hg, ho) and np.array_equal(ag, ao)
    assert moved > 200
    for i in np.nonzero(ho)[0][::17]:
        assert np.array_equal(g.swap_host_block(int(i)), o.swap_host_block(int(i)))


def test_reserve_release_hooks_bit_exact():
    intr, pd = small_intr(), _params()
    g, o = GpuEngine(*CFG), rfo.OracleEngine(*CFG)
    fr = _frames(intr, [0, 30, 60])
    for k, (pose, d) in enumerate(fr):
        for e in (g, o):
            e.allocate(d, intr, pose, pd)
            e.integrate(d, intr, pose, pd)
        if k == 0:
            ent = o.entries()
            for idx in np.nonzero(ent[:, 4] >= 0)[0][::5][:60]:
                for e in (g, o):
                    e.release_block(int(idx))
        if k == 1:
            ent = o.entries()
            for idx in np.nonzero(ent[:, 4] == -1)[0][:30]:
                assert g.reserve_block(int(idx)) == o.reserve_block(int(idx)) == 1
        _same_state(g, o)


def test_swapping_colour_map():
    """Colour planes travel with the depth planes."""
    from paper_1708_00783_b200 import fusion as F
    intr, pd = small_intr(), _params()
    fi = F.Intrinsics(**intr)
    poses = F.orbit_trajectory(frames=100)
    g, o = GpuEngine(*CFG, colour=True), rfo.OracleEngine(*CFG)
    for e in (g, o):
        e.set_fusion_options(True, 8.0)
        e.swap_create(50)
    for f in [0, 30, 60, 90, 60, 30, 0]:
        raw, _, col = F.synth_render(0, poses[f], fi, rgb=True)
        d = rfo.build_view(raw, intr, AFF, 1)[0]
        for e in (g, o):
            e.allocate(d, intr, poses[f], pd)
        assert g.swap_in() == o.swap_in()
        for e in (g, o):
            e.integrate(d, intr, poses[f], pd, rgb=col, intr_rgb=intr)
        assert g.swap_out() == o.swap_out()
        _same_state(g, o)


def test_swapping_equivalence_on_the_gpu():
    """SPEC.md:444-446 (the swapping engine's external anchor) on the B200
    path itself: a GPU map fused with swapping enabled ends with the same
    hash structure and, for every block, the same sdf / w_depth as a GPU map
    fused without swapping (host-tier copy for blocks still swapped out);
    allocated + free = capacity after every frame.  (Margin 0, as the oracle
    test: kBoundary blocks are integrated only with swapping.)"""
    intr, pd = small_intr(), _params()
    frames = _frames(intr)
    a, b = GpuEngine(*CFG), GpuEngine(*CFG)
    for pose, d in frames:
        a.allocate(d, intr, pose, pd)
        a.integrate(d, intr, pose, pd)
    b.set_fusion_options(True, 0.0)
    b.swap_create(100000)
    swapped = 0
    for pose, d in frames:
        b.allocate(d, intr, pose, pd)
        swapped += b.swap_in()
        b.integrate(d, intr, pose, pd)
        swapped += b.swap_out()
        ent = b.entries()
        assert (ent[:, 4] >= 0).sum() + b.free_counts()[0] == CFG[2]
    assert swapped > 100
    ea, eb = a.entries(), b.entries()
    assert np.array_equal(ea[:, :4], eb[:, :4])  # same hash structure
    has, _ = b.swap_stored()
    resident_a = np.nonzero(ea[:, 4] >= 0)[0]
    assert has[resident_a].sum() > 0  # some blocks end the run on the host tier
    want = a.blocks(ea[resident_a, 4])
    for k, i in enumerate(resident_a):
        got = b.blocks(np.array([eb[i, 4]]))[0] if eb[i, 4] >= 0 else b.swap_host_block(int(i))
        assert np.array_equal(want[k][:, :3], got[:, :3]), i  # sdf + w_depth
