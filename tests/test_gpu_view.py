"""Full ViewBuilder on the GPU (§8(f)2, rfg_view.cu) vs the CPU oracle
(oracle/rfo.c, pinned to the reference in tests/test_view_io.py), bit-exact:
depth conversion (host order and PGM16 big-endian payloads), bilateral
filter (including the reference's expf), normals, intensity, both pyramids;
the pipeline's PGM input path and its bilateral option."""
import os
import subprocess
import tempfile

import numpy as np
import pytest
import torch

from helpers import AFF, INTR_C1, small_intr
from oracle import rfo

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bits(a):
    if torch.is_tensor(a):
        a = a.cpu().numpy()
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def _noisy_frame(intr, seed, amp=40):
    from paper_1708_00783_b200 import fusion as F
    poses = F.orbit_trajectory(frames=100)
    raw, _, col = F.synth_render(0, poses[(7 * seed) % 100], F.Intrinsics(**intr), rgb=True)
    rng = np.random.default_rng(seed)
    noisy = np.clip(raw.astype(np.int64) + rng.integers(-amp, amp + 1, raw.shape), 0, 65535).astype(np.uint16)
    noisy[raw == 0] = 0
    noisy[rng.random(raw.shape) < 0.01] = 0
    return noisy, col


def _calib(intr):
    from paper_1708_00783_b200 import fusion as F
    i = F.Intrinsics(**intr)
    return F.RgbdCalib(intrinsics_rgb=i, intrinsics_d=i, depth_affine=F.DepthAffine(*AFF))


@pytest.mark.parametrize("bilateral", [False, True])
def test_build_view_full_bit_exact_vs_oracle(bilateral):
    from paper_1708_00783_b200 import fusion as F
    for intr, seeds in ((INTR_C1, (0, 1)), (small_intr(), (2, 3))):
        for seed in seeds:
            raw, col = _noisy_frame(intr, seed)
            v = F.build_view(raw, col, _calib(intr), F.ViewBuildOptions(bilateral=bilateral, levels=3))
            o = rfo.build_view_full(raw, intr, AFF, levels=3, bilateral=bilateral, rgb=col)
            for lv, od in zip(v.pyramid, o["depth"]):
                assert np.array_equal(_bits(lv.depth), _bits(od))
            for lv, oi in zip(v.pyramid, o["intensity"]):
                assert np.array_equal(_bits(lv.intensity), _bits(oi))
            assert np.array_equal(_bits(v.normals), _bits(o["normals"]))
            # the PGM16 payload path decodes the big-endian words on the GPU
            vb = F.build_view(raw.byteswap(), col, _calib(intr), F.ViewBuildOptions(bilateral=bilateral, levels=3),
                              big_endian=True)
            for a, b in zip(vb.pyramid, v.pyramid):
                assert np.array_equal(_bits(a.depth), _bits(b.depth))


def test_bilateral_filter_extremes_bit_exact():
    """Depth jumps of metres push exp() into glibc's underflow branches."""
    from paper_1708_00783_b200 import fusion as F
    rng = np.random.default_rng(11)
    d = rng.uniform(0.3, 6.0, (97, 131)).astype(np.float32)
    d[rng.random(d.shape) < 0.2] = -1.0
    for ss, rs in [(2.0, 0.002), (2.0, 0.05), (0.7, 0.5), (3.0, 1e-4)]:
        g = F.bilateral_filter(d, ss, rs)
        assert np.array_equal(_bits(g), _bits(rfo.bilateral_filter(d, ss, rs)))
    # constant image: identity (test_core.cpp:124-129)
    g = F.bilateral_filter(np.full((16, 16), 1.5, np.float32), 2.0, 0.01)
    assert np.allclose(g.cpu().numpy(), 1.5, rtol=1e-6)


def test_view_elements_known_answers():
    from paper_1708_00783_b200 import fusion as F
    # test_core.cpp:90-96
    it = F.rgb_to_intensity(np.full((4, 4, 3), 100, np.uint8)).cpu().numpy()
    assert abs(it[1, 1] - 100.0 / 255.0) <= 1e-6 * 100.0 / 255.0
    # test_core.cpp:155-160 and 131-141
    d = np.full((8, 8), -1.0, np.float32)
    d[4, 4] = 1.0
    assert F.compute_normals(d, F.Intrinsics(8, 8, 10.0, 10.0, 3.5, 3.5)).cpu().numpy()[4, 4, 3] < 0
    n = F.compute_normals(np.full((48, 64), 2.0, np.float32), F.Intrinsics(64, 48, 60.0, 60.0, 31.5, 23.5))
    n = n.cpu().numpy()[24, 32]
    assert n[3] > 0 and np.abs(n[:3] - [0, 0, -1]).max() < 1e-4
    img = np.random.default_rng(3).random((30, 42)).astype(np.float32)
    assert np.array_equal(_bits(F.downsample_intensity(img)), _bits(rfo.downsample_intensity(img)))


def test_expf_replica_matches_host_libm():
    """rfg_expf.cuh:expf_glibc == the host libm's expf for every float in
    [-110, 0], a sweep of (0, 89] and the special values."""
    src = os.path.join(ROOT, "tests", "cuda", "expf_glibc.cu")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "expf_glibc")
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                        "-fmad=false", "-std=c++17", src, "-o", exe], check=True)
        p = subprocess.run([exe], capture_output=True, text=True, timeout=600)
        assert p.returncode == 0 and "mismatches 0" in p.stdout, p.stdout + p.stderr


def test_pipeline_pgm_input_matches_host_input(tmp_path):
    """Pipeline.process_pgm (payload uploaded as stored, decoded in the view
    stage) reproduces the host-array path bit for bit."""
    from paper_1708_00783_b200 import fusion as F
    intr = F.Intrinsics(**INTR_C1)
    poses = F.orbit_trajectory(frames=100)
    raws = [F.synth_render(0, poses[f], intr)[0] for f in range(6)]
    for f, r in enumerate(raws):
        F.write_pgm16(r, str(tmp_path / f"{f:04d}.pgm"))
    res = []
    for mode in ("host", "pgm"):
        m = F.VoxelBlockMap(F.VoxelBlockMapConfig(0x40000, 0x20000, 0x40000))
        p = F.Pipeline(m, intr, F.SceneParams(), use_graph=True, raw_big_endian=(mode == "pgm"))
        for f in range(6):
            if mode == "pgm":
                p.process_pgm(str(tmp_path / f"{f:04d}.pgm"), poses[0] if f == 0 else None)
            else:
                p.process(raws[f], poses[0] if f == 0 else None)
        st, pose, icp = p.result()
        res.append((st, pose, icp, m.entries()))
        del p, m
    assert res[0][0] == res[1][0]
    assert np.array_equal(res[0][1], res[1][1]) and np.array_equal(res[0][2], res[1][2])
    assert np.array_equal(res[0][3], res[1][3])


def test_pipeline_bilateral_matches_oracle_fusion():
    """Pipeline(bilateral=True) at known poses: the integrated map equals the
    oracle fed with rfo.build_view_full(bilateral=True) depth."""
    from helpers import GpuEngine, canonical_blocks  # noqa: F401
    from paper_1708_00783_b200 import fusion as F
    intr = small_intr()
    fi = F.Intrinsics(**intr)
    params = F.SceneParams(voxelSize=0.01)
    poses = F.orbit_trajectory(frames=100)
    cfg = (0x4000, 0x2000, 0x4000)
    m = F.VoxelBlockMap(F.VoxelBlockMapConfig(*cfg))
    p = F.Pipeline(m, fi, params, levels=1, track=False, use_graph=False, bilateral=True)
    o = rfo.OracleEngine(*cfg)
    pd = params.as_dict()
    for f in range(4):
        raw, _ = _noisy_frame(intr, f)
        p.process(raw, poses[f])
        d = rfo.build_view_full(raw, intr, AFF, levels=1, bilateral=True)["depth"][0]
        o.allocate(d, intr, poses[f], pd)
        o.integrate(d, intr, poses[f], pd)
        rng = o.render_ranges(poses[f], intr, pd)  # noqa: F841 (keeps the oracle's per-frame order)
        o.render_icp(poses[f], intr, pd)
    p.result()
    eg, eo = m.entries(), o.entries()
    assert np.array_equal(eg, eo)
    ptrs = eo[eo[:, 4] >= 0, 4]
    assert np.array_equal(m.blocks(ptrs), o.blocks(ptrs))


def test_build_view_matches_reference_golden():
    """GPU ViewBuilder against the reference's own outputs
    (tests/golden/view_full.npz, generated by tests/golden/make_golden.py)."""
    from paper_1708_00783_b200 import fusion as F
    g = np.load(os.path.join(ROOT, "tests", "golden", "view_full.npz"))
    w, h, fx, fy, cx, cy = g["intr"]
    intr = dict(width=int(w), height=int(h), fx=float(fx), fy=float(fy), cx=float(cx), cy=float(cy))
    for k in range(2):
        for bil in (0, 1):
            v = F.build_view(g[f"raw{k}"], g[f"rgb{k}"], _calib(intr), F.ViewBuildOptions(bilateral=bool(bil), levels=3))
            for l in range(3):
                assert np.array_equal(_bits(v.pyramid[l].depth), _bits(g[f"depth{k}_{bil}_{l}"]))
                assert np.array_equal(_bits(v.pyramid[l].intensity), _bits(g[f"intensity{k}_{bil}_{l}"]))
            assert np.array_equal(_bits(v.normals), _bits(g[f"normals{k}_{bil}"]))
    assert np.array_equal(_bits(F.bilateral_filter(g["bil_in"], 2.0, 0.002)), _bits(g["bil_out"]))
