#!/usr/bin/env python
"""ICP stage device time (CUDA events inside the profiled pipeline) for
different per-level iteration caps, frames 5..14 of the C2 orbit."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1708_00783_b200 import fusion as F  # noqa: E402

intr = F.Intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
params = F.SceneParams()
poses = F.orbit_trajectory(frames=100)
raws = [torch.from_numpy(F.synth_render(0, poses[f], intr)[0].view(np.int16)).cuda() for f in range(15)]
for iters in [(6, 10, 20), (0, 0, 20), (0, 10, 0), (6, 0, 0), (1, 1, 1)]:
    m = F.VoxelBlockMap(F.VoxelBlockMapConfig(0x40000, 0x20000, 0x40000))
    p = F.Pipeline(m, intr, params, iters=iters, use_graph=False, profile=True)
    icp, its = [], []
    for f in range(15):
        p.process(raws[f], poses[0] if f == 0 else None)
        st = p.stage_times()
        _, _, s = p.result()
        if f >= 5:
            icp.append(st["icp"])
            its.append(s[0])
    us = 1e3 * np.mean(icp)
    print(f"iters {iters}: icp {us:.1f} us/frame, {np.mean(its):.1f} iterations, {us / max(np.mean(its), 1):.2f} us/iter")
    del p, m
