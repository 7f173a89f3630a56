#!/usr/bin/env python
"""Sub-phases of the tracker's evaluation per level (needs the RFG_ICP_SUB
build: RFG_LIB_PATH=.variants_rc/icpsub/librfg.so), frames 5..94 of the C2
graph pipeline, L2 flushed before every frame as in bench.py: CTA 0's
fill / associate+gather+accumulate / warp reduce / wait for its warps / CTA
sum + atomics, the slowest CTA's evaluation, and the per-iteration phases of
rfg_icp_timers (barrier, read, solve)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1708_00783_b200 import fusion as F  # noqa: E402
from paper_1708_00783_b200._lib import check, lib  # noqa: E402

intr = F.Intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
poses = F.orbit_trajectory(frames=100)
raws = torch.from_numpy(np.stack([F.synth_render(0, poses[f], intr)[0] for f in range(100)]).view(np.int16)).cuda()
m = F.VoxelBlockMap(F.VoxelBlockMapConfig(0x40000, 0x20000, 0x40000))
p = F.Pipeline(m, intr, F.SceneParams())
L = lib()
L.rfg_debug_icp_sub.argtypes = [C.c_void_p, C.c_int]
sub = np.zeros((3, 8), np.uint64)
t = (C.c_uint64 * 8)()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for f in range(95):
    flush.fill_(f & 0xFF)
    p.process(raws[f], poses[0] if f == 0 else None)
    if f == 4:
        p.result()
        check(L.rfg_icp_timers(m.handle, t, 1))
        L.rfg_debug_icp_sub(sub.ctypes.data, 1)
p.result()
check(L.rfg_icp_timers(m.handle, t, 0))
L.rfg_debug_icp_sub(sub.ctypes.data, 0)
it = max(int(t[4]), 1)
print(f"iterations {it} over 90 frames ({it / 90:.1f}/frame); per iteration: barrier {t[1] / it / 1e3:.2f} us, "
      f"read {t[2] / it / 1e3:.2f} us, solve {t[3] / it / 1e3:.2f} us")
names = ["fill", "assoc+gather+acc", "warp reduce", "wait CTA warps", "CTA sum+atomics", "slowest CTA eval"]
for lv in range(3):
    n = max(int(sub[lv, 7]), 1)
    print(f"level {lv}: {n / 90:.1f} it/frame; " + ", ".join(f"{nm} {sub[lv, k] / n / 1e3:.2f}" for k, nm in enumerate(names))
          + " us/iteration")
