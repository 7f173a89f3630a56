#!/usr/bin/env python
"""Ray-march statistics of the C2 frames (needs a RFG_RC_STATS or RFG_RC_TIMING build,
with RFG_RC_SPLIT for the timing slots of k_raycast_icp:
RFG_LIB_PATH=.variants/stats/librfg.so)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1708_00783_b200 import _lib  # noqa: E402
from paper_1708_00783_b200 import fusion as F  # noqa: E402

intr = F.Intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
poses = F.orbit_trajectory(frames=100)
m = F.VoxelBlockMap(F.VoxelBlockMapConfig(0x40000, 0x20000, 0x40000))
p = F.Pipeline(m, intr, F.SceneParams(), use_graph=False, profile=True)
L = _lib.lib()
buf = (C.c_ulonglong * 32)()
acc = np.zeros(32, np.float64)
timing = []
for f in range(40):
    raw = torch.from_numpy(F.synth_render(0, poses[f], intr)[0].view(np.int16)).cuda()
    torch.cuda.synchronize()
    L.rfg_debug_rc_stats(buf, 1)
    p.process(raw, poses[0] if f == 0 else None)
    torch.cuda.synchronize()
    L.rfg_debug_rc_stats(buf, 0)
    if f >= 30:
        acc += np.array(list(buf), np.float64)
        timing.append((buf[7] / 1e3, (buf[25] - buf[24]) / 1e3, buf[26] / max(buf[27], 1) / 1e3))
s = acc
nf = 10
tm = np.array(timing)
if s[0] == 0:  # RFG_RC_TIMING build (slots 7, 24-27: kernel span and ray durations)
    print(f"k_raycast_icp per frame: span {tm[:, 1].mean():.1f} us, longest ray {tm[:, 0].mean():.1f} us "
          f"(max {tm[:, 0].max():.1f}), mean ray {tm[:, 2].mean():.2f} us")
    sys.exit(0)
print(f"per frame: rays {s[0]/nf:.0f} steps {s[1]/nf:.0f} coarse {s[2]/nf:.0f} invalid-fine {s[3]/nf:.0f} "
      f"nearest {s[4]/nf:.0f} trilinear {s[5]/nf:.0f} lookups {s[6]/nf:.0f}  max steps (last frame) {buf[31]}")
if s[24]:
    print(f"rays >= 64 steps: {s[24]/nf:.0f}/frame, their steps: {s[25]/s[24]:.1f}/ray = coarse {s[26]/s[24]:.1f} + "
          f"invalid-fine {s[27]/s[24]:.1f} + one-voxel {s[28]/s[24]:.1f} + longer {s[29]/s[24]:.1f} (+ the hit/miss step)")
print("steps/ray histogram (log2 buckets):", {f"<{2**b}": int(s[8 + b] // nf) for b in range(16) if s[8 + b]})
