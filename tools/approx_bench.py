#!/usr/bin/env python
"""Parts of the approximate raycast (§8(f)1) at C1: forward_project alone,
the missing-only raycast alone, the full raycast — CUDA-graph replays, L2
flushed before each (tools/rows_bench.py:dev_time)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1708_00783_b200 import fusion as F  # noqa: E402
from tools.rows_bench import INTR, dev_time  # noqa: E402

params = F.SceneParams()
poses = F.orbit_trajectory(frames=100)
calib = F.RgbdCalib(intrinsics_rgb=INTR, intrinsics_d=INTR, depth_affine=F.DepthAffine(1 / 5000.0, 0.0))
m = F.VoxelBlockMap(F.VoxelBlockMapConfig(0x40000, 0x20000, 0x40000))
fe, st = F.FusionEngine(), F.RenderState()
for f in range(40):
    r, _, _ = F.synth_render(0, poses[f], INTR)
    v = F.build_view(r, None, calib, F.ViewBuildOptions(False, 1))
    fe.allocate_from_depth(m, v, poses[f], params)
    fe.integrate_frame(m, v, poses[f], params)
F.render_expected_ranges(m, poses[39], INTR, params, st)
F.render_maps(m, poses[39], INTR, params, F.RenderMode.kIcpMaps, st)
# the frame-40 render: expected ranges at the NEW pose, then either the full
# raycast or forward_project of the frame-39 maps + the missing-only raycast
# (the reference's order)
print("expected ranges       %.1f us" % dev_time(lambda: F.render_expected_ranges(m, poses[40], INTR, params, st)))
F.render_expected_ranges(m, poses[40], INTR, params, st)
print("full raycast          %.1f us" % dev_time(lambda: F.render_maps(m, poses[40], INTR, params, F.RenderMode.kIcpMaps, st)))
F.render_maps(m, poses[39], INTR, params, F.RenderMode.kIcpMaps, st)  # previous maps for forward projection
miss = F.forward_project(st, poses[40], INTR, params.voxelSize, m)
print("missing pixels", len(miss))
F.render_maps(m, poses[39], INTR, params, F.RenderMode.kIcpMaps, st)
print("forward_project       %.1f us" % dev_time(lambda: F.forward_project(st, poses[40], INTR, params.voxelSize, m)))
print("missing-only raycast  %.1f us" % dev_time(lambda: F.render_maps(m, poses[40], INTR, params, F.RenderMode.kIcpMaps, st, missingOnly=miss)))
