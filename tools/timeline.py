#!/usr/bin/env python
"""Device timeline of the graph-replayed C2 frame (CUPTI kernel activity via
torch.profiler): per-kernel start/end inside each frame, the idle gaps
between consecutive kernels, and the frame span.  Frames 5..24 of the orbit,
L2 flushed before each frame (the flush kernel is excluded from the span).

    python tools/timeline.py [--no-graph] [--json out.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1708_00783_b200 import fusion as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--no-graph", action="store_true")
ap.add_argument("--frames", type=int, default=25)
ap.add_argument("--json", default=None)
args = ap.parse_args()

intr = F.Intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
params = F.SceneParams()
poses = F.orbit_trajectory(frames=100)
raws = torch.from_numpy(np.stack([F.synth_render(0, poses[f], intr)[0] for f in range(args.frames)]).view(np.int16)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
m = F.VoxelBlockMap(F.VoxelBlockMapConfig(0x40000, 0x20000, 0x40000))
p = F.Pipeline(m, intr, params, use_graph=not args.no_graph)
s = torch.cuda.ExternalStream(p.stream)
for f in range(5):
    p.process(raws[f], poses[0] if f == 0 else None)
torch.cuda.synchronize()
pairs = []
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for f in range(5, args.frames):
        flush.fill_(f & 0xFF)
        s.wait_stream(torch.cuda.current_stream())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            p.process(raws[f])
            b.record(s)
        pairs.append((a, b))
        torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
ev_us = float(np.mean([a.elapsed_time(b) * 1e3 for a, b in pairs]))

evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = sorted([(e.time_range.start, e.time_range.end, e.name) for e in evs])
# split into frames at the flush kernels
frames, cur = [], None
for st, en, name in kern:
    if "FillFunctor" in name or "elementwise" in name:
        if cur:
            frames.append(cur)
        cur = []
        continue
    if cur is not None:
        cur.append((st, en, name.split("(")[0].replace("void ", "")))
if cur:
    frames.append(cur)
frames = [fr for fr in frames if fr]
per_kernel = {}
gaps = {}
spans, busy = [], []
for fr in frames:
    spans.append(fr[-1][1] - fr[0][0])
    busy.append(sum(en - st for st, en, _ in fr))
    for i, (st, en, name) in enumerate(fr):
        per_kernel.setdefault((i, name), []).append(en - st)
        if i > 0:
            gaps.setdefault((i, name), []).append(st - fr[i - 1][1])
print(f"event-timed frame {ev_us:.1f} us")
print(f"frames {len(frames)}  kernels/frame {np.mean([len(f) for f in frames]):.1f}  "
      f"span {np.mean(spans):.1f} us  busy {np.mean(busy):.1f} us  idle {np.mean(spans) - np.mean(busy):.1f} us")
print(f"{'#':>3} {'kernel':40s} {'dur us':>8} {'gap before':>10}")
rows = []
for (i, name), d in sorted(per_kernel.items()):
    g = np.mean(gaps.get((i, name), [0.0]))
    rows.append({"i": i, "kernel": name, "us": float(np.mean(d)), "gap_before_us": float(g)})
    print(f"{i:3d} {name[:40]:40s} {np.mean(d):8.2f} {g:10.2f}")
if args.json:
    with open(args.json, "w") as fh:
        json.dump({"graph": not args.no_graph, "span_us": float(np.mean(spans)), "busy_us": float(np.mean(busy)), "event_us": ev_us,
                   "kernels": rows}, fh, indent=1)
