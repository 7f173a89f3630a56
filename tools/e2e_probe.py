#!/usr/bin/env python
"""Where the end-to-end frame time goes (host API vs device): C2 frames
through Pipeline.process(host u16) + Pipeline.result(), L2 flushed before
each frame (as bench.py's e2e leg)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1708_00783_b200 import fusion as F  # noqa: E402

intr = F.Intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
poses = F.orbit_trajectory(frames=100)
raws = torch.from_numpy(np.stack([F.synth_render(0, poses[f], intr)[0] for f in range(100)]).view(np.int16)).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
m = F.VoxelBlockMap(F.VoxelBlockMapConfig(0x40000, 0x20000, 0x40000))
p = F.Pipeline(m, intr, F.SceneParams())
s = torch.cuda.ExternalStream(p.stream)
tp, tr, tt, dev = [], [], [], []
for f in range(100):
    flush.fill_(f & 0xFF)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host = raws[f].numpy().view(np.uint16)
    t0 = time.perf_counter()
    a.record(s)
    p.process(host, poses[0] if f == 0 else None)
    b.record(s)
    t1 = time.perf_counter()
    p.result()
    t2 = time.perf_counter()
    if f >= 5:
        tp.append(t1 - t0)
        tr.append(t2 - t1)
        tt.append(t2 - t0)
        dev.append(a.elapsed_time(b) / 1e3)
us = lambda v: 1e6 * float(np.mean(v))  # noqa: E731
print(f"e2e {us(tt):.1f} us/frame ({1e6 / us(tt):.0f} frames/s): process() host {us(tp):.1f} us, "
      f"result() host {us(tr):.1f} us; device H2D + graph {us(dev):.1f} us")
