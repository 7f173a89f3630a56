"""The multi-GPU path's device pieces on one GPU: the nearest-hit composition
kernels against their CPU restatement (tests/test_shard_gloo.py), and the
NCCL ShardedPipeline at world size 1 (composition = identity) against the
single-GPU pipeline.  (Only one GPU is available per run; the N > 1 exchange
is covered on CPU by tests/test_shard_gloo.py.)"""
import os
import socket

import numpy as np
import pytest
import torch

from test_shard_gloo import cpu_keys, cpu_select

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_compose_kernels_match_cpu_restatement():
    from paper_1708_00783_b200 import fusion as F
    from paper_1708_00783_b200.shard import Composer
    rng = np.random.default_rng(3)
    n = 5000
    pts = rng.normal(0, 1, size=(n, 4)).astype(np.float32)
    pts[:, 2] += 2.0
    pts[:, 3] = np.where(rng.random(n) < 0.8, 1.0, -1.0)
    pose = F.orbit_trajectory(frames=10)[4]
    for rank in (0, 1, 3):
        comp = Composer(rank, 4)
        kg = comp._keys_gpu(torch.from_numpy(pts).cuda(), pose).cpu().numpy()
        kc = cpu_keys(rank)(torch.from_numpy(pts), pose).numpy()
        assert np.array_equal(kg, kc)
        keymin = np.minimum(kc, np.roll(kc, 7) ^ 1)  # some pixels won by another rank
        maps = [torch.from_numpy(rng.normal(size=(n, 4)).astype(np.float32)) for _ in range(3)]
        gpu_maps = [m.cuda() for m in maps]
        comp._select_gpu(torch.from_numpy(keymin).cuda(), *gpu_maps)
        cpu_select(rank)(torch.from_numpy(keymin), *maps)
        for a, b in zip(gpu_maps, maps):
            assert np.array_equal(a.cpu().numpy(), b.numpy())


def test_sharded_pipeline_world1_equals_single_gpu_pipeline():
    import torch.distributed as dist
    from paper_1708_00783_b200 import fusion as F
    from paper_1708_00783_b200.shard import ShardedPipeline
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        intr = F.Intrinsics(320, 240, 262.5, 262.5, 159.5, 119.5)
        params = F.SceneParams()
        poses = F.orbit_trajectory(frames=100)
        raws = [F.synth_render(0, poses[f], intr)[0] for f in range(6)]
        cfg = F.VoxelBlockMapConfig(1 << 16, 1 << 14, 1 << 16)
        m1 = F.VoxelBlockMap(cfg)
        m1.set_shard(0, 1, 3)
        sp = ShardedPipeline(m1, intr, params, 0, 1)
        m2 = F.VoxelBlockMap(cfg)
        pp = F.Pipeline(m2, intr, params, use_graph=False)
        for f in range(6):
            sp.process(raws[f], poses[0] if f == 0 else None)
            pp.process(raws[f], poses[0] if f == 0 else None)
            s1, p1, _ = sp.result()
            s2, p2, _ = pp.result()
            assert np.abs(p1 - p2).max() < 1e-5
        assert np.array_equal(m1.entries(), m2.entries())
        assert np.array_equal(m1.visibleList(), m2.visibleList())
        # composed (world 1) maps == a direct render of the unsharded map
        rs = F.RenderState()
        F.render_expected_ranges(m2, p1, intr, params, rs)
        F.render_maps(m2, p1, intr, params, F.RenderMode.kIcpMaps, rs)
        sr, sp_pts, sn = sp.maps()
        for a, b in ((sp_pts, rs.points), (sn, rs.normals), (sr, rs.raycastResult)):
            assert torch.equal(a, b)
        assert (rs.points[..., 3] > 0).float().mean().item() > 0.8
    finally:
        dist.destroy_process_group()
