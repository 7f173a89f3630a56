#!/usr/bin/env python
"""Graph-mode frame time of the C2 pipeline under variants (tracking on/off,
L2 flush on/off, ICP caps).  CUDA events around each frame on the pipeline
stream; frames 5..94 of the orbit."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1708_00783_b200 import fusion as F  # noqa: E402

intr = F.Intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
params = F.SceneParams()
poses = F.orbit_trajectory(frames=100)
raws = torch.from_numpy(np.stack([F.synth_render(0, poses[f], intr)[0] for f in range(100)]).view(np.int16)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def run(track=True, do_flush=True, iters=(6, 10, 20), graph=True):
    m = F.VoxelBlockMap(F.VoxelBlockMapConfig(0x40000, 0x20000, 0x40000))
    p = F.Pipeline(m, intr, params, track=track, iters=iters, use_graph=graph)
    s = torch.cuda.ExternalStream(p.stream)
    ms = []
    for f in range(95):
        if do_flush:
            flush.fill_(f & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.wait_stream(torch.cuda.current_stream())
        a.record(s)
        p.process(raws[f], poses[0] if f == 0 else None)
        b.record(s)
        torch.cuda.current_stream().wait_stream(s)
        if f >= 5:
            ms.append((a, b))
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) * 1e3 for a, b in ms]
    del p, m
    return np.mean(t), np.median(t)


for name, kw in [("graph, track, flush", {}), ("graph, track, no flush", dict(do_flush=False)),
                 ("graph, no track, flush", dict(track=False)), ("graph, no track, no flush", dict(track=False, do_flush=False)),
                 ("graph, icp (1,1,1), no flush", dict(iters=(1, 1, 1), do_flush=False)),
                 ("graph, icp (0,0,20), no flush", dict(iters=(0, 0, 20), do_flush=False)),
                 ("no graph, track, no flush", dict(graph=False, do_flush=False))]:
    mean, med = run(**kw)
    print(f"{name:34s} mean {mean:7.1f} us  median {med:7.1f} us")
