#!/usr/bin/env python
"""Per-level ICP iteration counts of the C2 pipeline over the 100-frame orbit
(stats[4..6] of each frame), to see where the tracker spends its iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1708_00783_b200 import fusion as F  # noqa: E402

intr = F.Intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
poses = F.orbit_trajectory(frames=100)
dist = tuple(float(x) for x in sys.argv[1].split(",")) if len(sys.argv) > 1 else (0.01, 0.02, 0.04)
m = F.VoxelBlockMap(F.VoxelBlockMapConfig(0x40000, 0x20000, 0x40000))
p = F.Pipeline(m, intr, F.SceneParams(), use_graph=False, dist=dist)
rows = []
for f in range(100):
    raw = torch.from_numpy(F.synth_render(0, poses[f], intr)[0].view(np.int16)).cuda()
    p.process(raw, poses[0] if f == 0 else None)
    st, pose, icp = p.result()
    err = np.abs(pose - poses[f]).max()
    rows.append((f, int(icp[4]), int(icp[5]), int(icp[6]), int(icp[0]), icp[3], err))
a = np.array([r[1:4] for r in rows[1:]])
errs = np.array([r[6] for r in rows])
print("dist", dist, "mean iterations per level (0 fine .. 2 coarse):", a.mean(0).round(2), " coarse cap hits:",
      (a[:, 2] >= 20).sum(), " max |pose-gt| %.2e  mean %.2e" % (errs.max(), errs.mean()))
if len(sys.argv) > 2:
    sys.exit(0)
for r in rows[1::10]:
    print("frame %3d  it l0 %2d l1 %2d l2 %2d  total %2d  converged %.0f  |pose - gt| %.2e" % r)
