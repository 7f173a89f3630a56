#!/usr/bin/env python
"""Measurement of the SURVEY §8(f) rows beyond the per-frame hot path, at C1
size on one B200: device time per call (the call captured in a CUDA graph,
replays timed with CUDA events, L2 flushed before every replay, median of N), algorithmic bytes -> GB/s against the measured HBM
peak, and the reference CPU path on the same inputs (oracle/_ref, one core)
where it exists.  Prints one JSON object (profiles/r1b_rows.json).

Rows: (f)1 approximate raycast (forward_project + missing-only raycast vs the
full raycast), (f)2 full ViewBuilder (depth + bilateral + normals +
intensity + pyramids), (f)3 swapping (blocks out / in per second through the
transfer buffers), (f)4 marching cubes (extract_mesh) and the colour / grey
render modes."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1708_00783_b200 import fusion as F  # noqa: E402

INTR = F.Intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
AFF = (1.0 / 5000.0, 0.0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        for k in ("hbm_gbs", "hbm_copy_gbs", "hbm_GBs"):
            if k in d:
                return float(d[k])
    except Exception:
        pass
    return 6650.0


def dev_time(fn, reps=20, warm=3):
    """Device time of fn's kernels: fn is captured once into a CUDA graph
    (our ctypes launches go to torch's current stream, i.e. the capture
    stream) and the replays are timed with CUDA events, L2 flushed before
    each — no host launch gaps inside the measured interval."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warm):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def cpu_time(fn, reps=3):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    return float(np.median(ts))


def main():
    out = {"device": torch.cuda.get_device_name(0), "peak_gbs": peak_gbs(), "rows": {}}
    peak = out["peak_gbs"]
    try:
        from oracle import ref
        have_ref = ref.available()
    except Exception:
        have_ref = False
    poses = F.orbit_trajectory(frames=100)
    raw, _, col = F.synth_render(0, poses[20], INTR, rgb=True)
    rng = np.random.default_rng(0)
    noisy = np.clip(raw.astype(np.int64) + rng.integers(-40, 41, raw.shape), 0, 65535).astype(np.uint16)
    noisy[raw == 0] = 0
    calib = F.RgbdCalib(intrinsics_rgb=INTR, intrinsics_d=INTR, depth_affine=F.DepthAffine(*AFF))
    raw_d = torch.from_numpy(noisy.view(np.int16)).cuda()
    col_d = torch.from_numpy(col).cuda()
    n = INTR.width * INTR.height

    # ---- (f)2 ViewBuilder
    vb = {}
    for name, opts, rgb in (("depth+pyramid", F.ViewBuildOptions(False, 3), None),
                            ("+bilateral", F.ViewBuildOptions(True, 3), None),
                            ("+bilateral+normals+intensity", F.ViewBuildOptions(True, 3), col_d)):
        us = dev_time(lambda: F.build_view(raw_d, rgb, calib, opts))
        # bytes: raw 2 + depth 4 (+ bilateral 4 in + 4 out) + normals 16 (+ 20 in)
        # + rgb 3 + intensity 4 per px, pyramids 1.25x of level-0 outputs
        b = n * (2 + 4 + 16 + 20) + 0.25 * n * 4 * 1.25
        if opts.bilateral:
            b += n * 8
        if rgb is not None:
            b += n * (3 + 4) + 0.25 * n * 4 * 1.25
        vb[name] = {"us": round(us, 2), "alg_bytes": int(b), "gbs": round(b / (us * 1e-6) / 1e9, 1),
                    "frac_hbm": round(b / (us * 1e-6) / 1e9 / peak, 3)}
    if have_ref:
        intr_d = INTR.as_dict()
        for name, bil, rgb in (("+bilateral+normals+intensity", True, col),):
            vb[name]["cpu_ref_us"] = round(cpu_time(lambda: ref.build_view_full(noisy, intr_d, AFF, 3, bil, rgb)), 1)
    out["rows"]["f2_view_builder_640x480"] = vb

    # ---- fused C1 map for the rest (frames 0..39 at known poses)
    m = F.VoxelBlockMap(F.VoxelBlockMapConfig(0x40000, 0x20000, 0x40000), colour=True)
    fe = F.FusionEngine()
    params = F.SceneParams()
    st = F.RenderState()
    for f in range(0, 40):
        r, _, c = F.synth_render(0, poses[f], INTR, rgb=True)
        v = F.build_view(r, c, calib, F.ViewBuildOptions(False, 1))
        fe.allocate_from_depth(m, v, poses[f], params)
        fe.integrate_frame(m, v, poses[f], params)
    pose = poses[39]
    F.render_expected_ranges(m, pose, INTR, params, st)

    # ---- render modes / approximate raycast
    rm = {}
    for mode in (F.RenderMode.kIcpMaps, F.RenderMode.kColour, F.RenderMode.kGrey):
        rm[mode.name] = {"us": round(dev_time(lambda: F.render_maps(m, pose, INTR, params, mode, st)), 2)}
    out["rows"]["f4_render_modes_640x480"] = rm
    F.render_maps(m, pose, INTR, params, F.RenderMode.kIcpMaps, st)
    ap = {}

    # frame 40 rendered from scratch vs approximately (ranges at the new pose
    # first in both, as the reference orders it)
    def full():
        F.render_expected_ranges(m, poses[40], INTR, params, st)
        F.render_maps(m, poses[40], INTR, params, F.RenderMode.kIcpMaps, st)
    ap["full_ranges+raycast_us"] = round(dev_time(full), 2)
    F.render_maps(m, pose, INTR, params, F.RenderMode.kIcpMaps, st)  # frame-39 maps

    def approx():
        F.render_expected_ranges(m, poses[40], INTR, params, st)
        miss = F.forward_project(st, poses[40], INTR, params.voxelSize, m)
        F.render_maps(m, poses[40], INTR, params, F.RenderMode.kIcpMaps, st, missingOnly=miss)
        return miss
    ap["ranges+forward_project+missing_raycast_us"] = round(dev_time(approx), 2)
    F.render_maps(m, pose, INTR, params, F.RenderMode.kIcpMaps, st)
    ap["missing_pixels"] = len(approx())
    out["rows"]["f1_approximate_raycast_640x480"] = ap

    # ---- marching cubes
    mesh = F.extract_mesh(m, params.voxelSize)
    mc = {"triangles": int(len(mesh.triangles)), "vertices": int(len(mesh.vertices)),
          "allocated_blocks": int((m.entries()[:, 4] >= 0).sum())}
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        F.extract_mesh(m, params.voxelSize)
    mc["gpu_us_incl_readback"] = round((time.perf_counter() - t0) / reps * 1e6, 1)
    mc["triangles_per_s"] = round(mc["triangles"] / (mc["gpu_us_incl_readback"] * 1e-6), 0)
    out["rows"]["f4_marching_cubes_c1_40frames"] = mc

    # ---- swapping throughput: evict everything invisible, bring it back
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sw = F.SwappingEngine(m, capacity=4096)
    create_ms = (time.perf_counter() - t0) * 1e3
    far = poses[99]
    opts = F.FusionEngine.Options(True, 8.0)
    r, _, c = F.synth_render(0, far, INTR, rgb=True)
    vfar = F.build_view(r, c, calib, F.ViewBuildOptions(False, 1))
    rn, _, cn = F.synth_render(0, poses[0], INTR, rgb=True)
    vnear = F.build_view(rn, cn, calib, F.ViewBuildOptions(False, 1))
    outs, t_out = 0, 0.0
    for _ in range(3):
        fe.allocate_from_depth(m, vfar, far, params, opts)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        outs += sw.swap_out()
        torch.cuda.synchronize()
        t_out += time.perf_counter() - t0
    fe.allocate_from_depth(m, vnear, poses[0], params, opts)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ins = sw.swap_in()
    torch.cuda.synchronize()
    t_in = time.perf_counter() - t0
    blk = 2 * 2048  # depth + colour plane per block
    out["rows"]["f3_swapping"] = {
        "create_ms_incl_host_tier_pinning": round(create_ms, 1), "blocks_out": outs, "out_blocks_per_s": round(outs / t_out, 0) if t_out else None,
        "out_gbs": round(outs * blk / t_out / 1e9, 2) if t_out else None,
        "blocks_in": ins, "in_blocks_per_s": round(ins / t_in, 0) if t_in else None,
        "in_gbs": round(ins * blk / t_in / 1e9, 2) if t_in else None,
        "note": "host wall time per call until the device is idle: device-side selection, the selected indices back to the host, slot lookup, and the kernel copying the blocks to / from the pinned mapped host slots over PCIe"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
