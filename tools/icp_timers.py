#!/usr/bin/env python
"""Per-phase device time of the ICP level kernel (CTA 0 %globaltimer stamps,
rfg_icp_timers) over frames 5..94 of the C2 graph pipeline."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1708_00783_b200 import fusion as F  # noqa: E402
from paper_1708_00783_b200._lib import check, lib  # noqa: E402

intr = F.Intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
params = F.SceneParams()
poses = F.orbit_trajectory(frames=100)
raws = torch.from_numpy(np.stack([F.synth_render(0, poses[f], intr)[0] for f in range(100)]).view(np.int16)).cuda()
m = F.VoxelBlockMap(F.VoxelBlockMapConfig(0x40000, 0x20000, 0x40000))
p = F.Pipeline(m, intr, params)
t = (C.c_uint64 * 8)()
for f in range(95):
    p.process(raws[f], poses[0] if f == 0 else None)
    if f == 4:
        p.result()
        check(lib().rfg_icp_timers(m.handle, t, 1))
p.result()
check(lib().rfg_icp_timers(m.handle, t, 0))
it = max(int(t[4]), 1)
names = ["associate+block reduce", "grid barrier", "final sum", "solve"]
print(f"iterations {it} over 90 frames ({it / 90:.1f}/frame)")
for k, nm in enumerate(names):
    print(f"  {nm:24s} {t[k] / it / 1e3:7.2f} us/iteration   {t[k] / 90 / 1e3:7.1f} us/frame")
for lv in range(3):
    print(f"  level {lv} iterations total   {t[5 + lv] / 90 / 1e3:7.1f} us/frame")
