"""The benchmarked C2 frame graph, tracking on, over the whole 100-frame orbit,
against the CPU oracle's own tracked run (BASELINE.json configs[1];
SPEC.md:348-356; P/src/fusion.cpp:144-263; P/include/rf/raycast.hpp:157-207).

This drives EXACTLY bench.py's timed path: `Pipeline(use_graph=True,
track=True, levels=3)` at 640x480, 5 mm, 0x40000 buckets, raw u16 frames on
the device — the captured graph k_view_pyramid -> k_icp_track ->
allocation -> k_integrate_depth -> k_range_bin -> k_raycast_tiles.

Contract for a tracked sequence: the oracle runs its OWN
tracked chain — it tracks each frame against its own previous render from
its own previous pose — and every frame of the two runs is compared BIT for
bit.  This holds because every stage is bit-exact: the tracker's sums are
fixed-point integers (order-independent), its solve runs the oracle's IEEE
sequence, and allocation / integration / ranges / raycast are bit-exact
given the pose.  Per frame: the depth pyramid, the tracked pose and the
12-value tracker summary, AllocationStats, the visible list + visibility
bytes, the expected ranges, raycastResult / points / normals; at
checkpoints the whole hash table, the free stacks and every resident voxel
block.  The north-star tolerance (1e-5 rad / 1e-5 m per frame) is therefore
met with zero error.
"""
import numpy as np
import pytest

from helpers import AFF, INTR_C1, MAP_C1, PARAMS_C1
from oracle import rfo

pytestmark = pytest.mark.gpu

ITERS = (6, 10, 20)  # bench.py ICP_ITERS (finest first)
DIST = (0.01, 0.02, 0.04)
N_FRAMES = 100
CHECKPOINTS = (0, 1, 10, 50, 99)


def u32(a):
    return np.ascontiguousarray(a).view(np.uint32)


def test_tracked_c2_sequence_matches_oracle():
    import torch
    from paper_1708_00783_b200 import fusion as F

    rfo.set_threads()  # the oracle's per-pixel raycast on every host core (results do not depend on it)
    intr = F.Intrinsics(**INTR_C1)
    params = F.SceneParams(**PARAMS_C1)
    poses = F.orbit_trajectory(frames=N_FRAMES)
    raws = np.stack([F.synth_render(F.SCENE_SPHERE_IN_ROOM, poses[f], intr)[0] for f in range(N_FRAMES)])
    raw_dev = torch.from_numpy(raws.view(np.int16)).cuda()

    m = F.VoxelBlockMap(F.VoxelBlockMapConfig(*MAP_C1))
    pipe = F.Pipeline(m, intr, params, F.DepthAffine(*AFF), levels=3, track=True, iters=ITERS, dist=DIST,
                      use_graph=True)
    o = rfo.OracleEngine(*MAP_C1)

    prev = None  # the oracle's (points, normals, pose) of frame f-1
    gt_err, iters = [], []
    for f in range(N_FRAMES):
        pipe.process(raw_dev[f], poses[0] if f == 0 else None)
        st_g, pose_g, icp_g = pipe.result()
        lv = rfo.build_view(raws[f], INTR_C1, AFF, 3)
        for lg, lo in zip(pipe.depth_levels(), lv):
            assert np.array_equal(u32(lg.cpu().numpy()), u32(lo)), f"frame {f}: depth pyramid differs"

        # the oracle's own tracked chain
        if prev is None:
            pose_o = poses[0].copy()
        else:
            pose_o, st_o = rfo.icp_track(lv, INTR_C1, prev[0], prev[1], prev[2], INTR_C1, prev[2], ITERS, 10, DIST)
            assert np.array_equal(u32(pose_g), u32(pose_o)), \
                f"frame {f}: tracked pose differs (max {np.abs(pose_g - pose_o).max():.2e})"
            assert np.array_equal(icp_g, st_o), f"frame {f}: tracker summary {icp_g} vs {st_o}"
            assert st_o[7] == 1, f"frame {f}: tracking failed"
            gt_err.append(float(np.abs(pose_o[:, 3] - poses[f][:, 3]).max()))
            iters.append(st_o[0])

        st_o, _ = o.allocate(lv[0], INTR_C1, pose_o, PARAMS_C1)
        assert np.array_equal(st_g.as_array(), st_o), f"frame {f}: AllocationStats {st_g} vs {st_o}"
        o.integrate(lv[0], INTR_C1, pose_o, PARAMS_C1)
        rng_o, _ = o.render_ranges(pose_o, INTR_C1, PARAMS_C1)
        rc_o, pts_o, nrm_o, _ = o.render_icp(pose_o, INTR_C1, PARAMS_C1)
        rng_g, rc_g, pts_g, nrm_g = (t.cpu().numpy() for t in pipe.maps())
        assert np.array_equal(u32(rng_g), u32(rng_o)), f"frame {f}: expected ranges differ"
        assert np.array_equal(u32(rc_g), u32(rc_o)), f"frame {f}: raycastResult differs"
        assert np.array_equal(u32(pts_g), u32(pts_o)), f"frame {f}: points differ"
        assert np.array_equal(u32(nrm_g), u32(nrm_o)), f"frame {f}: normals differ"
        assert (pts_g[..., 3] > 0).sum() > 100_000, f"frame {f}: render nearly empty"
        lg, tg = m.visible()
        lo, to = o.visible()
        assert np.array_equal(lg, lo) and np.array_equal(tg, to), f"frame {f}: visible list differs"
        if f in CHECKPOINTS:
            eg, eo = m.entries(), o.entries()
            assert np.array_equal(eg, eo), f"frame {f}: hash entries differ"
            ptrs = eo[eo[:, 4] >= 0, 4]
            bg = m.blocks(ptrs)
            assert np.array_equal(bg, o.blocks(ptrs)), f"frame {f}: voxel blocks differ"
            assert tuple(m.free_counts()) == tuple(o.free_counts()), f"frame {f}: free stacks differ"
            if f == N_FRAMES - 1:  # voxels seen in every frame have reached maxW (fusion.cpp:26-31)
                assert int(bg[..., 2].max()) == PARAMS_C1["maxW"]
        prev = (pts_o, nrm_o, pose_o.copy())

    # and the run tracks the ground truth (frame-to-model, no loop closure)
    assert max(gt_err) < 0.006 and float(np.mean(gt_err)) < 0.003
    print(f"tracked C2 x{N_FRAMES}: bit-exact; {np.mean(iters):.1f} iterations/frame; vs ground truth mean "
          f"{np.mean(gt_err) * 1e3:.2f} mm, max {max(gt_err) * 1e3:.2f} mm")
