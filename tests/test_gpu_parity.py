"""B200 kernels vs the C restatement oracle (oracle/rfo.c, itself pinned to
the reference build) on the same synthetic frames.  Integer / quantised state
must be bit-exact; the raycast maps are compared bit-exactly too (tolerance
1e-4 m is the contract; the mismatch count is asserted 0)."""
import numpy as np
import pytest

from helpers import (AFF, INTR_C1, MAP_C1, PARAMS_C1, GpuEngine, canonical_blocks, same_bits, small_intr)
from oracle import rfo

pytestmark = pytest.mark.gpu


def frames(scene, intr, n, poses=None):
    from paper_1708_00783_b200 import fusion as F
    i = F.Intrinsics(**intr)
    if poses is None:
        poses = F.orbit_trajectory(frames=n)
    out = []
    for k in range(n):
        raw, dep, col = F.synth_render(scene, poses[k], i, rgb=True)
        d = rfo.build_view(raw, intr, AFF, 1)[0]
        out.append((poses[k], d, col))
    return out


def compare_state(g, o, check_vba=True):
    eg, eo = g.entries(), o.entries()
    assert np.array_equal(eg, eo), "hash entries differ"
    vg, tg = g.visible()
    vo, to = o.visible()
    assert np.array_equal(vg, vo), "visible list differs"
    assert np.array_equal(tg, to), "visibility types differ"
    assert g.free_counts() == o.free_counts()
    if check_vba:
        ptrs = eo[eo[:, 4] >= 0, 4]
        bg, bo = g.blocks(ptrs), o.blocks(ptrs)
        if not np.array_equal(bg, bo):
            bad = np.argwhere((bg != bo).any(axis=2))
            raise AssertionError(f"VBA differs in {len(bad)} voxels, first {bad[:5].tolist()}")


def run_sequence(gpu, orc, seq, intr, params, render=True, colour=False, check_every=1):
    for k, (pose, d, col) in enumerate(seq):
        sg, _ = gpu.allocate(d, intr, pose, params)
        so, _ = orc.allocate(d, intr, pose, params)
        assert np.array_equal(sg, so), f"frame {k}: stats {sg} vs {so}"
        rgb = col if colour else None
        gpu.integrate(d, intr, pose, params, rgb=rgb, intr_rgb=intr if colour else None)
        orc.integrate(d, intr, pose, params, rgb=rgb, intr_rgb=intr if colour else None)
        if k % check_every == 0 or k == len(seq) - 1:
            compare_state(gpu, orc)
        if render:
            rg, _ = gpu.render_ranges(pose, intr, params)
            ro, _ = orc.render_ranges(pose, intr, params)
            assert same_bits(rg, ro), f"frame {k}: expected ranges differ"
            mg = gpu.render_icp(pose, intr, params)
            mo = orc.render_icp(pose, intr, params)
            for name, a, b in zip(("raycast", "points", "normals"), mg[:3], mo[:3]):
                diff = ~(a.view(np.uint32) == b.view(np.uint32)).all(axis=-1)
                assert diff.sum() == 0, f"frame {k}: {name} differs at {diff.sum()} px"


def test_c1_sequence_bit_exact():
    """C1 (640x480, 5 mm, 0x40000 buckets), first 6 frames of the orbit."""
    seq = frames(0, INTR_C1, 6)
    run_sequence(GpuEngine(*MAP_C1), rfo.OracleEngine(*MAP_C1), seq, INTR_C1, PARAMS_C1)


def test_small_image_many_frames():
    intr = small_intr(160, 120)
    seq = frames(0, intr, 24)
    run_sequence(GpuEngine(1 << 14, 1 << 12, 1 << 14), rfo.OracleEngine(1 << 14, 1 << 12, 1 << 14), seq, intr,
                 PARAMS_C1)


def test_collisions_tiny_bucket_table():
    """Few buckets => long excess chains and many intra-frame collisions."""
    intr = small_intr(160, 120)
    seq = frames(0, intr, 6)
    run_sequence(GpuEngine(64, 4096, 8192), rfo.OracleEngine(64, 4096, 8192), seq, intr, PARAMS_C1)


def test_exhaustion_block_and_excess():
    """VBA / excess stacks run out mid-frame: failures must match exactly."""
    intr = small_intr(160, 120)
    seq = frames(0, intr, 3)
    run_sequence(GpuEngine(256, 40, 300), rfo.OracleEngine(256, 40, 300), seq, intr, PARAMS_C1)


def test_empty_and_invalid_depth():
    intr = small_intr(64, 48)
    g, o = GpuEngine(1 << 10, 1 << 8, 1 << 10), rfo.OracleEngine(1 << 10, 1 << 8, 1 << 10)
    pose = np.eye(3, 4, dtype=np.float32)
    empty = np.full((48, 64), -1.0, np.float32)
    st, _ = g.allocate(empty, intr, pose, PARAMS_C1)
    assert st.tolist() == [0, 0, 0, 0]
    out_of_range = np.full((48, 64), 7.0, np.float32)  # beyond viewFrustum_max
    st, _ = g.allocate(out_of_range, intr, pose, PARAMS_C1)
    assert st.tolist() == [0, 0, 0, 0]
    one = empty.copy()
    one[24, 32] = 1.0  # single valid pixel
    sg, _ = g.allocate(one, intr, pose, PARAMS_C1)
    so, _ = o.allocate(one, intr, pose, PARAMS_C1)
    assert np.array_equal(sg, so) and 1 <= sg[1] <= 3
    compare_state(g, o)


def test_colour_fusion_c3_like():
    """ITMVoxel_s_rgb colour fusion (C3: 4 mm voxels, RGB)."""
    intr = small_intr(320, 240)
    params = dict(PARAMS_C1, voxelSize=0.004)
    seq = frames(0, intr, 4)
    run_sequence(GpuEngine(1 << 16, 1 << 14, 1 << 16, colour=True), rfo.OracleEngine(1 << 16, 1 << 14, 1 << 16),
                 seq, intr, params, render=True, colour=True)


def test_stop_integrating_at_max_w():
    intr = small_intr(80, 60)
    params = dict(PARAMS_C1, maxW=3, stopIntegratingAtMaxW=True)
    seq = frames(0, intr, 1) * 5  # same frame 5x => weights saturate
    run_sequence(GpuEngine(1 << 12, 1 << 10, 1 << 12), rfo.OracleEngine(1 << 12, 1 << 10, 1 << 12), seq, intr,
                 params, render=False)


def test_shard_filter_matches_per_shard_oracle():
    intr = small_intr(160, 120)
    seq = frames(0, intr, 3)
    for rank in range(2):
        g, o = GpuEngine(1 << 14, 1 << 12, 1 << 14), rfo.OracleEngine(1 << 14, 1 << 12, 1 << 14)
        g.set_shard(rank, 2, 2)
        o.set_shard(rank, 2, 2)
        run_sequence(g, o, seq, intr, PARAMS_C1, render=True)
