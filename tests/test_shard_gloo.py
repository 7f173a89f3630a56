"""World-size-2 test of the multi-GPU path's host logic on CPU (gloo).

Each rank fuses the same frames into its spatial shard (the per-shard oracle:
oracle/rfo.c with the same owner/halo filter as k_alloc_stage1), renders it,
and the shards are composed with paper_1708_00783_b200.shard.Composer — the
same collective sequence the NCCL path runs — with CPU stand-ins for the two
composition kernels.  Checks: (1) the composition equals the per-pixel
nearest hit of the gathered per-rank renders, exactly; (2) the composed
render agrees with the monolithic (unsharded) render."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

INTR = dict(width=96, height=72, fx=78.75, fy=78.75, cx=47.5, cy=35.5)
PARAMS = dict(voxelSize=0.005, mu=0.02, maxW=100, viewFrustum_min=0.2, viewFrustum_max=6.0,
              stopIntegratingAtMaxW=False)
AFF = (1.0 / 5000.0, 0.0)
CFG = (1 << 15, 1 << 13, 1 << 15)  # roomy: no allocation failures in the monolithic map


def cpu_keys(rank):
    def keys(points: torch.Tensor, pose):
        p = points.numpy().reshape(-1, 4)
        R = np.asarray(pose, np.float32).reshape(3, 4)
        # z row of pose_apply in the reference's (Eigen) order, float32
        z = (R[2, 0] * p[:, 0] + (R[2, 1] * p[:, 1] + R[2, 2] * p[:, 2])) + R[2, 3]
        bits = np.maximum(z, np.float32(0)).astype(np.float32).view(np.uint32).astype(np.int64)
        k = (bits << 32) | rank
        k[p[:, 3] <= 0] = np.iinfo(np.int64).max
        return torch.from_numpy(k)
    return keys


def cpu_select(rank):
    def select(keymin, raycast, points, normals):
        k = keymin.numpy()
        nobody = k == np.iinfo(np.int64).max
        mine = ~nobody & ((k & 0xffffffff) == rank)
        inval = np.zeros(4, np.float32)
        for t in (raycast, points, normals):
            a = t.view(-1, 4).numpy()
            a[~mine] = inval
            if rank == 0:
                a[nobody, 3] = -1.0
    return select


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import rfo
    from paper_1708_00783_b200 import fusion as F
    from paper_1708_00783_b200.shard import Composer

    poses = F.orbit_trajectory(frames=100)
    E = rfo.OracleEngine(*CFG)
    E.set_shard(rank, world, 2)
    comp = Composer(rank, world, keys_fn=cpu_keys(rank), select_fn=cpu_select(rank))
    for f in (0, 4, 8):
        raw, _, _ = F.synth_render(0, poses[f], F.Intrinsics(**INTR))
        d = rfo.build_view(raw, INTR, AFF, 1)[0]
        E.allocate(d, INTR, poses[f], PARAMS)
        E.integrate(d, INTR, poses[f], PARAMS)
        E.render_ranges(poses[f], INTR, PARAMS)
    rc, pts, nrm, _ = E.render_icp(poses[8], INTR, PARAMS)
    mine = [torch.from_numpy(a.copy()) for a in (rc, pts, nrm)]
    # gather the un-composed per-rank renders for the exact check
    gathered = [[torch.zeros_like(t) for _ in range(world)] for t in mine]
    for t, g in zip(mine, gathered):
        dist.all_gather(g, t)
    comp.compose(poses[8], *mine)
    n_alloc = int((E.entries()[:, 4] >= 0).sum())
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), rc=mine[0].numpy(), pts=mine[1].numpy(),
             nrm=mine[2].numpy(), g_pts=np.stack([g.numpy() for g in gathered[1]]),
             g_nrm=np.stack([g.numpy() for g in gathered[2]]), g_rc=np.stack([g.numpy() for g in gathered[0]]),
             n_alloc=n_alloc)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_nearest_hit_composition(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r = [np.load(tmp_path / f"rank{k}.npz") for k in range(world)]
    # every rank ends with the same composed maps
    for k in ("rc", "pts", "nrm"):
        assert np.array_equal(r[0][k], r[1][k])
    # each shard holds a strict subset of the blocks
    from oracle import rfo
    from paper_1708_00783_b200 import fusion as F
    # (1) composition == per-pixel nearest hit of the per-rank renders
    pose = F.orbit_trajectory(frames=100)[8]
    g_pts, g_nrm, g_rc = r[0]["g_pts"], r[0]["g_nrm"], r[0]["g_rc"]
    R = pose.astype(np.float32)
    z = (R[2, 0] * g_pts[..., 0] + (R[2, 1] * g_pts[..., 1] + R[2, 2] * g_pts[..., 2])) + R[2, 3]
    z = np.where(g_pts[..., 3] > 0, z, np.inf)
    win = np.argmin(z, axis=0)  # ties -> lower rank, like the key's rank bits
    hit = np.isfinite(z.min(axis=0))
    exp_pts = np.take_along_axis(g_pts, win[None, ..., None], 0)[0]
    exp_nrm = np.take_along_axis(g_nrm, win[None, ..., None], 0)[0]
    assert np.array_equal(r[0]["pts"][hit], exp_pts[hit])
    assert np.array_equal(r[0]["nrm"][hit], exp_nrm[hit])
    assert (r[0]["pts"][~hit] == np.array([0, 0, 0, -1], np.float32)).all()
    # (2) against the monolithic render
    mono = rfo.OracleEngine(*CFG)
    poses = F.orbit_trajectory(frames=100)
    for f in (0, 4, 8):
        raw, _, _ = F.synth_render(0, poses[f], F.Intrinsics(**INTR))
        d = rfo.build_view(raw, INTR, AFF, 1)[0]
        mono.allocate(d, INTR, poses[f], PARAMS)
        mono.integrate(d, INTR, poses[f], PARAMS)
        mono.render_ranges(poses[f], INTR, PARAMS)
    _, mpts, _, _ = mono.render_icp(poses[8], INTR, PARAMS)
    n_mono = int((mono.entries()[:, 4] >= 0).sum())
    assert max(r[0]["n_alloc"], r[1]["n_alloc"]) < n_mono <= r[0]["n_alloc"] + r[1]["n_alloc"]
    both = (mpts[..., 3] > 0) & (r[0]["pts"][..., 3] > 0)
    agree = ((mpts[..., 3] > 0) == (r[0]["pts"][..., 3] > 0)).mean()
    assert agree > 0.99, agree
    err = np.linalg.norm(mpts[both][:, :3] - r[0]["pts"][both][:, :3], axis=1)
    assert np.median(err) < 1e-4 and np.percentile(err, 99) < 5e-3
