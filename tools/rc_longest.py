#!/usr/bin/env python
"""The longest march of each C2 frame and what it did (needs the RFG_RC_TIMING
build of k_raycast_tiles: RFG_LIB_PATH=.variants/rctiming/librfg.so).

Per frame: the kernel span, the longest ray's duration / steps / hash lookups
/ bucket-entry loads / nearest loads / trilinear reads and when it started,
the max step count over all rays, and the mean ray duration."""
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
p = F.Pipeline(m, intr, F.SceneParams(), levels=3, track=True, use_graph=True)
L = _lib.lib()
L.rfg_debug_rc_warps.argtypes = [C.c_void_p, C.c_int]
NW = 1 << 14
rec = np.zeros((NW, 16), np.uint64)
raws = [torch.from_numpy(F.synth_render(0, poses[f], intr)[0].view(np.int16)).cuda() for f in range(100)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rows = []
segs = []
for f in range(100):
    if not os.environ.get("RC_NOFLUSH"):
        flush.fill_(f & 0xFF)
    torch.cuda.synchronize()
    L.rfg_debug_rc_warps(None, 1)
    p.process(raws[f], poses[0] if f == 0 else None)
    torch.cuda.synchronize()
    L.rfg_debug_rc_warps(rec.ctypes.data, 0)
    r = rec[rec[:, 0] > 0].astype(np.int64)
    k0 = r[:, 10].min()
    span = (r[:, 2].max() - k0) / 1e3
    w = int(np.argmax(r[:, 0]))
    lw = r[w]
    # warps whose end is within 10 % of the kernel end: the tail
    tail = (r[:, 2] - k0) > 0.9 * (r[:, 2].max() - k0)
    rows.append((f, span, lw[0] / 1e3, (lw[1] - k0) / 1e3, *[int(v) for v in lw[3:8]], int(r[:, 8].max()),
                 r[:, 9].sum() / (len(r) * 32) / 1e3, int(tail.sum()), (lw[1] - lw[10]) / 1e3))
    seg = [(lw[12 + k] - lw[11 + k]) / 16.0 if lw[12 + k] else 0.0 for k in range(2)]
    segs.append([(lw[11] - k0) / 1e3] + seg + [lw[14] / max(lw[15], 1) if lw[15] else 0.0])
print("frame span_us longest_us start_us steps lookups chain_loads nearest trilinear | max_steps mean_ray_us "
      "tail_warps its_range_us ns/step")
for r in rows[5:]:
    print(f"{r[0]:3d} {r[1]:7.1f} {r[2]:7.1f} {r[3]:6.1f} {r[4]:5d} {r[5]:5d} {r[6]:5d} {r[7]:5d} {r[8]:5d} | "
          f"{r[9]:5d} {r[10]:6.2f} {r[11]:5d} {r[12]:6.2f} {r[2] * 1e3 / max(r[4], 1):6.0f}")
a = np.array([r[1:] for r in rows[5:]], np.float64)
print(f"mean over frames 5..99: span {a[:, 0].mean():.1f} us, longest ray {a[:, 1].mean():.1f} us starting at "
      f"{a[:, 2].mean():.1f} us, its steps {a[:, 3].mean():.0f} (max steps of any ray {a[:, 8].mean():.0f}), "
      f"{a[:, 1].mean() * 1e3 / a[:, 3].mean():.0f} ns/step; lookups {a[:, 4].mean():.0f}, chain loads "
      f"{a[:, 5].mean():.0f}, nearest {a[:, 6].mean():.0f}, trilinear {a[:, 7].mean():.0f}; mean ray "
      f"{a[:, 9].mean():.2f} us; warps in the last 10 % {a[:, 10].mean():.0f}")
sg = np.array(segs[5:], np.float64)
print("longest ray: march starts at %.1f us; ns per step over steps 0-15 / 16-31: %s" %
      (sg[:, 0].mean(), " / ".join(f"{v:.0f}" for v in sg[:, 1:3].mean(axis=0))))
if sg[:, 3].any():  # RFG_RC_REMARCH build: the same ray marched again right after, its blocks warm
    print("  marched again with its blocks warm: %.0f ns per step" % sg[:, 3][sg[:, 3] > 0].mean())
