#!/usr/bin/env python
"""Per-stage device times of the C2 pipeline (profile mode: CUDA events
around each stage, L2 flushed before every frame), mean over frames 5..34.
RFG_LIB_PATH=<variant .so> compares kernel variants."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1708_00783_b200 import _lib  # noqa: E402
from paper_1708_00783_b200 import fusion as F  # noqa: E402

intr = F.Intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
params = F.SceneParams()
poses = F.orbit_trajectory(frames=100)
raws = torch.from_numpy(np.stack([F.synth_render(0, poses[f], intr)[0] for f in range(35)]).view(np.int16)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
m = F.VoxelBlockMap(F.VoxelBlockMapConfig(0x40000, 0x20000, 0x40000))
p = F.Pipeline(m, intr, params, use_graph=False, profile=True)
acc = {}
for f in range(35):
    flush.fill_(f & 0xFF)
    torch.cuda.synchronize()
    p.process(raws[f], poses[0] if f == 0 else None)
    st = p.stage_times()
    if f >= 5:
        for k, v in st.items():
            acc.setdefault(k, []).append(v * 1e3)
name = os.path.basename(os.path.dirname(_lib.LIB_PATH)) if os.environ.get("RFG_LIB_PATH") else "default"
print(f"{name:12s} " + "  ".join(f"{k} {np.mean(v):6.1f}" for k, v in acc.items()) + "  (us)")
