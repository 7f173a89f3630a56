#!/usr/bin/env python
"""Device frame rate of every BASELINE.json config on one B200 (bench.py
measures configs[1] = C2; this tool reports the others beside it).  Frames
are pre-staged in HBM, L2 flushed before every timed frame, CUDA events on
the work's stream around each frame; frames W..N-1 timed.

  C1  640x480, 5 mm, 0x40000 buckets, depth-only, known poses (no tracker):
      the frame graph with the ground-truth pose per frame
  C2  C1 + the ICP tracker (3-level pyramid)                 (= bench.py)
  C3  ITMVoxel_s_rgb colour fusion, 640x480 depth + RGB, 4 mm voxels,
      known poses: the colour frame pipeline (view, RGB pack, allocate,
      RGB-D integrate, expected ranges, ICP-map raycast)
  C4  builder-defined multi-room scene, 2 mm voxels, 2^21 buckets, 2^22
      blocks (8 GiB depth plane), known poses: the frame graph

  python tools/configs_bench.py [--frames N] [--json out.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1708_00783_b200 import fusion as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=60)
ap.add_argument("--warmup", type=int, default=5)
ap.add_argument("--json", default=None)
args = ap.parse_args()

INTR = F.Intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(step, stream, n):
    """Mean device ms of step(f) over frames warmup..n-1 (L2 flushed before each)."""
    ms = []
    for f in range(n):
        flush.fill_(f & 0xFF)
        stream.wait_stream(torch.cuda.current_stream())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            step(f)
            b.record(stream)
        torch.cuda.current_stream().wait_stream(stream)
        if f >= args.warmup:
            ms.append((a, b))
    torch.cuda.synchronize()
    return float(np.mean([a.elapsed_time(b) for a, b in ms]))


def kernel_times(step, stream, frames):
    """Mean device duration (us) per kernel name over `frames` (CUPTI)."""
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for f in frames:
            flush.fill_(f & 0xFF)
            stream.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(stream):
                step(f)
            torch.cuda.current_stream().wait_stream(stream)
        torch.cuda.synchronize()
    acc = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA and "rfg::" in e.name:
            acc.setdefault(e.name.split("(")[0].replace("void ", ""), []).append(e.time_range.end - e.time_range.start)
    return {k: float(np.sum(v)) / len(frames) for k, v in acc.items()}


def pipeline_config(scene, poses, mapcfg, params, track, kernels=False):
    raws = torch.from_numpy(np.stack([F.synth_render(scene, poses[f], INTR)[0]
                                      for f in range(args.frames)]).view(np.int16)).cuda()
    m = F.VoxelBlockMap(F.VoxelBlockMapConfig(*mapcfg))
    p = F.Pipeline(m, INTR, params, track=track)
    s = torch.cuda.ExternalStream(p.stream)

    def step(f):
        p.process(raws[f], poses[f] if (not track or f == 0) else None)
    ms = timed(step, s, args.frames)
    st, _, icp = p.result()
    kt = None
    if kernels:  # the same frames again (a fresh map), kernel by kernel
        m.clear()
        p.reset()
        for f in range(args.warmup):
            step(f)
        kt = kernel_times(step, s, range(args.warmup, args.frames))
        st = p.result()[0]
    return ms, st, kt


out = {}
poses = F.orbit_trajectory(frames=100)
p5 = F.SceneParams(voxelSize=0.005, mu=0.02)
ms, st, _ = pipeline_config(0, poses, (0x40000, 0x20000, 0x40000), p5, track=False)
out["C1"] = {"ms": ms, "fps": 1e3 / ms, "visible_last": st.visibleCount}
ms, st, _ = pipeline_config(0, poses, (0x40000, 0x20000, 0x40000), p5, track=True)
out["C2"] = {"ms": ms, "fps": 1e3 / ms, "visible_last": st.visibleCount}

# C3: colour fusion through the colour frame pipeline (graph: view, RGB
# pack, allocate, RGB-D integrate, ranges, raycast), 300-frame orbit at 4 mm
p4 = F.SceneParams(voxelSize=0.004, mu=0.02)
poses3 = F.orbit_trajectory(frames=300)
n3 = min(300, args.frames)
frames = [F.synth_render(0, poses3[f], INTR, rgb=True) for f in range(n3)]
raws = torch.from_numpy(np.stack([r for r, _, _ in frames]).view(np.int16)).cuda()
rgbs = torch.from_numpy(np.stack([c for _, _, c in frames])).cuda()
mc = F.VoxelBlockMap(F.VoxelBlockMapConfig(0x40000, 0x20000, 0x40000), colour=True)
pc = F.Pipeline(mc, INTR, p4, track=False, colour=True)
sc = torch.cuda.ExternalStream(pc.stream)


def c3(f):
    pc.process(raws[f], poses3[f], rgb=rgbs[f])


ms = timed(c3, sc, n3)
out["C3"] = {"ms": ms, "fps": 1e3 / ms, "path": "colour frame pipeline (CUDA graph)",
             "visible_last": pc.result()[0].visibleCount}

# C4: multi-room, 2 mm, full capacity
mr = F.multiroom_trajectory(100)
p2 = F.SceneParams(voxelSize=0.002, mu=0.02)
ms, st, kt = pipeline_config(F.SCENE_MULTI_ROOM, mr, (1 << 21, 1 << 19, 1 << 22), p2, track=False, kernels=True)
out["C4"] = {"ms": ms, "fps": 1e3 / ms, "visible_last": st.visibleCount,
             "kernel_us": {k: round(v, 2) for k, v in sorted(kt.items(), key=lambda x: -x[1])}}
# integration roofline at C4: 2 x 2 KiB per visible block + the depth image
# (visible count of the last frame as the per-frame estimate)
ki = kt.get("rfg::k_integrate_depth")
if ki:
    byts = st.visibleCount * 2 * 512 * 4 + 640 * 480 * 4
    out["C4"]["integrate_GBps"] = byts / (ki * 1e-6) / 1e9

for k, v in out.items():
    print(f"{k}: {v['ms'] * 1e3:7.1f} us/frame  {v['fps']:8.1f} frames/s  " +
          "  ".join(f"{a}={b}" for a, b in v.items() if a not in ("ms", "fps")))
if args.json:
    with open(args.json, "w") as fh:
        json.dump(out, fh, indent=1)
