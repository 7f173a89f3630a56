"""Config C5 (BASELINE.json configs[4]) at full resolution on one GPU: the C4
multi-room scene (640x480, 2 mm, 2^21 buckets) with the voxel-hash space
sharded over G ranks, each rank's frame graph run in turn on the one device.

* Per-shard parity (SURVEY §8(e) caveat 1: the parity oracle for a shard is
  the CPU oracle run with the same owner()/halo filter): for every rank the
  hash table, every resident voxel, the expected ranges and the ICP maps of
  the rank's pipeline are bit-identical to the oracle's shard
  (P/src/fusion.cpp:168-176 collisions resolved inside the shard).
* Composition: the device nearest-hit kernels (rfg_compose_keys /
  rfg_compose_select, the NCCL path's arithmetic) applied to the G renders
  and reduced as the collectives would (MIN over the keys, SUM over the
  maps) give exactly the per-pixel nearest hit of the oracle shards' renders
  (P/include/rf/raycast.hpp:142-147 halo reads inside each shard).
* Each shard holds a strict part of the monolithic map, and the shards
  together cover every block the monolithic map allocates.
(tests/test_gpu_shard_multi.py runs the same path across real GPUs when a box
has more than one; tests/test_shard_gloo.py covers the collectives on CPU.)"""
import numpy as np
import pytest

from helpers import AFF

pytestmark = pytest.mark.gpu

INTR = dict(width=640, height=480, fx=525.0, fy=525.0, cx=319.5, cy=239.5)
PARAMS = dict(voxelSize=0.002, mu=0.02, maxW=100, viewFrustum_min=0.2, viewFrustum_max=6.0,
              stopIntegratingAtMaxW=False)
GPU_CFG = (1 << 21, 1 << 19, 1 << 20)
ORACLE_CFG = (1 << 21, 1 << 19, 1 << 19)  # host RAM: 2^19 blocks x 4 KiB; no allocation fails at these frames
FRAMES = (0, 3, 6)
TILE_SHIFT = 3


def u32(a):
    return np.ascontiguousarray(a).view(np.uint32)


def _render_shard(F, rfo, rank, world, frames, poses):
    """GPU pipeline (shard filter on, known poses) and oracle shard over the
    frames; asserts bit-exactness; returns the last frame's maps and the
    shard's allocated block set."""
    import torch
    intr = F.Intrinsics(**INTR)
    params = F.SceneParams(**PARAMS)
    m = F.VoxelBlockMap(F.VoxelBlockMapConfig(*GPU_CFG))
    if world > 1:
        m.set_shard(rank, world, TILE_SHIFT)
    pipe = F.Pipeline(m, intr, params, F.DepthAffine(*AFF), levels=1, track=False)
    o = rfo.OracleEngine(*ORACLE_CFG)
    if world > 1:
        o.set_shard(rank, world, TILE_SHIFT)
    for f in frames:
        raw, _, _ = F.synth_render(F.SCENE_MULTI_ROOM, poses[f], intr)
        pipe.process(torch.from_numpy(raw.view(np.int16)).cuda(), poses[f])
        st_g, _, _ = pipe.result()
        d = rfo.build_view(raw, INTR, AFF, 1)[0]
        st_o, _ = o.allocate(d, INTR, poses[f], PARAMS)
        assert np.array_equal(st_g.as_array(), st_o), f"rank {rank}/{world} frame {f}: {st_g} vs {st_o}"
        assert st_o[2] == 0
        o.integrate(d, INTR, poses[f], PARAMS)
    eg, eo = m.entries(), o.entries()
    # pointers differ (capacity 2^20 vs 2^19: the free stacks pop from their
    # backs), positions and chains do not
    assert np.array_equal(eg[:, :4], eo[:, :4]), f"rank {rank}/{world}: hash entries differ"
    ag, ao = eg[:, 4] >= 0, eo[:, 4] >= 0
    assert np.array_equal(ag, ao)
    assert np.array_equal(m.blocks(eg[ag, 4]), o.blocks(eo[ao, 4])), f"rank {rank}/{world}: voxels differ"
    rng_o, _ = o.render_ranges(poses[frames[-1]], INTR, PARAMS)
    rc_o, pts_o, nrm_o, _ = o.render_icp(poses[frames[-1]], INTR, PARAMS)
    rng_g, rc_g, pts_g, nrm_g = (t.clone() for t in pipe.maps())
    assert np.array_equal(u32(rng_g.cpu().numpy()), u32(rng_o)), f"rank {rank}/{world}: ranges differ"
    for a, b, name in ((rc_g, rc_o, "raycast"), (pts_g, pts_o, "points"), (nrm_g, nrm_o, "normals")):
        assert np.array_equal(u32(a.cpu().numpy()), u32(b)), f"rank {rank}/{world}: {name} differ"
    blocks = {tuple(p) for p in eo[ao, :3].tolist()}
    del pipe, m
    torch.cuda.empty_cache()
    return (rc_g, pts_g, nrm_g), (rc_o, pts_o, nrm_o), blocks


@pytest.mark.parametrize("world", [2, 4])
def test_c5_per_shard_parity_and_composition(world):
    import torch
    from oracle import rfo
    from paper_1708_00783_b200 import fusion as F
    from paper_1708_00783_b200.shard import Composer
    rfo.set_threads()
    poses = F.multiroom_trajectory(100)
    pose = poses[FRAMES[-1]]
    gpu_maps, oracle_maps, shard_blocks = [], [], []
    for rank in range(world):
        g, o, b = _render_shard(F, rfo, rank, world, FRAMES, poses)
        gpu_maps.append(g)
        oracle_maps.append(o)
        shard_blocks.append(b)
    # the collectives' arithmetic on one device: keys per rank -> MIN ->
    # select per rank -> SUM
    keys = [Composer(r, world)._keys_gpu(gpu_maps[r][1], pose) for r in range(world)]
    kmin = torch.stack(keys).min(dim=0).values
    acc = None
    for r in range(world):
        rc, pts, nrm = (t.clone() for t in gpu_maps[r])
        Composer(r, world)._select_gpu(kmin, rc, pts, nrm)
        s = torch.stack([rc, pts, nrm])
        acc = s if acc is None else acc + s
    torch.cuda.synchronize()
    composed = [a.cpu().numpy() for a in acc]
    # the nearest hit of the oracle shards (camera z in the reference's order)
    P = pose.astype(np.float32)
    zs = []
    for rc, pts, nrm in oracle_maps:
        z = (P[2, 0] * pts[..., 0] + (P[2, 1] * pts[..., 1] + P[2, 2] * pts[..., 2])) + P[2, 3]
        zs.append(np.where(pts[..., 3] > 0, np.maximum(z, np.float32(0)), np.inf))
    zs = np.stack(zs)
    win = np.argmin(zs, axis=0)  # ties -> lowest rank, as the (z bits << 32 | rank) key
    hit = np.isfinite(zs.min(axis=0))
    assert hit.mean() > 0.5
    for k in range(3):
        exp = np.stack([om[k] for om in oracle_maps])
        exp = np.take_along_axis(exp, win[None, ..., None], 0)[0]
        assert np.array_equal(u32(composed[k][hit]), u32(exp[hit])), f"composed map {k} differs"
        assert (composed[k][~hit][:, 3] == -1.0).all()
    # strict parts of the monolithic map that cover it
    mono_blocks = _render_shard(F, rfo, 0, 1, FRAMES, poses)[2]
    union = set().union(*shard_blocks)
    assert all(len(b) < len(mono_blocks) for b in shard_blocks)
    assert mono_blocks <= union
