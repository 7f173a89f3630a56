"""The sharded pipeline across real GPUs (NCCL over NVLink): one process per
GPU runs ShardedPipeline (the device-resident frame graph + the nearest-hit
composition) on the same frames.  Skipped unless at least two GPUs are
visible — the round's GPU runs have one, where tests/test_gpu_shard.py (NCCL
world of one) and tests/test_shard_gloo.py (world size 2 on CPU) cover the
path.  Checks: every rank ends each frame with the identical pose and
identical composed maps; the composed maps are the per-pixel nearest hit of
the ranks' own renders; each rank allocated a strict subset of the blocks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

W, H = 320, 240


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1708_00783_b200 import fusion as F
    from paper_1708_00783_b200.shard import ShardedPipeline

    intr = F.Intrinsics(W, H, 262.5, 262.5, 159.5, 119.5)
    poses = F.orbit_trajectory(frames=100)
    m = F.VoxelBlockMap(F.VoxelBlockMapConfig(1 << 16, 1 << 14, 1 << 16), device=rank)
    m.set_shard(rank, world, 3)
    sp = ShardedPipeline(m, intr, F.SceneParams(), rank, world)
    pose_log = []
    for f in range(6):
        sp.process(F.synth_render(0, poses[f], intr)[0], poses[0] if f == 0 else None)
        _, pose, _ = sp.result()
        pose_log.append(pose)
    # the last frame's own (uncomposed) render, for the nearest-hit check:
    # render this rank's shard at the final pose
    rs = F.RenderState()
    F.render_expected_ranges(m, pose_log[-1], intr, F.SceneParams(), rs)
    F.render_maps(m, pose_log[-1], intr, F.SceneParams(), F.RenderMode.kIcpMaps, rs)
    own = rs.points.clone()
    gathered = [torch.zeros_like(own) for _ in range(world)]
    dist.all_gather(gathered, own)
    rc, pts, nrm = (t.cpu().numpy() for t in sp.maps())
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), poses=np.stack(pose_log), rc=rc, pts=pts, nrm=nrm,
             g_pts=np.stack([g.cpu().numpy() for g in gathered]),
             n_alloc=int((m.entries()[:, 4] >= 0).sum()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (NCCL across devices)")
def test_sharded_pipeline_two_gpus(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r = [np.load(tmp_path / f"rank{k}.npz") for k in range(world)]
    # replicated tracking on identical composed maps: identical poses and maps
    assert np.array_equal(r[0]["poses"], r[1]["poses"])
    for k in ("rc", "pts", "nrm"):
        assert np.array_equal(r[0][k], r[1][k])
    # the composed points are the per-pixel nearest hit of the shard renders
    from paper_1708_00783_b200 import fusion as F
    pose = r[0]["poses"][-1].astype(np.float32)
    g = r[0]["g_pts"]
    z = (pose[2, 0] * g[..., 0] + (pose[2, 1] * g[..., 1] + pose[2, 2] * g[..., 2])) + pose[2, 3]
    z = np.where(g[..., 3] > 0, z, np.inf)
    win = np.argmin(z, axis=0)
    hit = np.isfinite(z.min(axis=0))
    exp = np.take_along_axis(g, win[None, ..., None], 0)[0]
    assert hit.mean() > 0.8
    assert np.array_equal(r[0]["pts"][hit], exp[hit])
    # each shard is a strict part of the map
    assert 0 < r[0]["n_alloc"] and 0 < r[1]["n_alloc"]
    del F
