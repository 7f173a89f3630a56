#!/usr/bin/env python
"""Device timeline of the end-to-end frame path (bench.py's e2e leg: host
u16 frame -> Pipeline.process -> Pipeline.result, L2 flushed before each
frame): per frame, the device span from the frame's first activity (H2D copy
or view kernel) to its last kernel, the view kernel, the H2D copy, the
result kernel and the idle gaps between them (torch.profiler CUDA activity
records)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1708_00783_b200 import fusion as F  # noqa: E402

intr = F.Intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
poses = F.orbit_trajectory(frames=100)
raws = torch.from_numpy(np.stack([F.synth_render(0, poses[f], intr)[0] for f in range(100)]).view(np.int16)).pin_memory()
views = [raws[f].numpy().view(np.uint16) for f in range(100)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
m = F.VoxelBlockMap(F.VoxelBlockMapConfig(0x40000, 0x20000, 0x40000))
p = F.Pipeline(m, intr, F.SceneParams())
N0, N1 = 10, 40
host = []
for f in range(N0):
    p.process(views[f], poses[0] if f == 0 else None)
    p.result()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for f in range(N0, N1):
        flush.fill_(f & 0xFF)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p.process(views[f])
        t1 = time.perf_counter()
        p.result()
        t2 = time.perf_counter()
        host.append((t1 - t0, t2 - t0))
ev = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        ev.append((e.time_range.start, e.time_range.end, e.name))
ev.sort()
# frames: split at the flush kernels (at::...FillFunctor)
frames, cur = [], None
for s, t, n in ev:
    if "fill" in n.lower() and "rfg" not in n:
        if cur:
            frames.append(cur)
        cur = []
        continue
    if cur is not None:
        cur.append((s, t, n))
if cur:
    frames.append(cur)
rows = []
for fr in frames:
    if not fr:
        continue
    span = fr[-1][1] - fr[0][0]
    busy = sum(t - s for s, t, _ in fr)
    view = sum(t - s for s, t, n in fr if "view" in n)
    cpy = sum(t - s for s, t, n in fr if "emcpy" in n or "HtoD" in n)
    res = sum(t - s for s, t, n in fr if "frame_result" in n)
    rows.append((span, busy, view, cpy, res))
a = np.array(rows, np.float64)
h = np.array(host) * 1e6
print(f"{len(a)} frames: e2e host {h[:, 1].mean():.1f} us (process() returns after {h[:, 0].mean():.1f} us); device "
      f"span {a[:, 0].mean():.1f} us, busy {a[:, 1].mean():.1f} us, idle gaps {a[:, 0].mean() - a[:, 1].mean():.1f} us; "
      f"view kernel {a[:, 2].mean():.1f} us, H2D copy {a[:, 3].mean():.1f} us, result kernel {a[:, 4].mean():.1f} us")
print("activities of the last frame:", [(n.split('(')[0][:30], round(t - s, 1)) for s, t, n in frames[-1]][:12])
