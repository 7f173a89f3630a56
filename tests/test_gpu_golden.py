"""B200 kernels against the golden fixtures produced by the reference itself
(tests/golden/make_golden.py), through the C ABI, plus the C++ adapter run."""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

from helpers import GpuEngine
from test_oracle_golden import AFF, GOLD, PARAMS, _state_digests, digest, run_small_sequence

pytestmark = pytest.mark.gpu


def test_small_sequence_matches_reference_golden_on_gpu():
    g = np.load(os.path.join(GOLD, "seq_small.npz"))
    run_small_sequence(GpuEngine, g)


def test_c1_full_frames_match_reference_golden_on_gpu():
    from oracle import rfo
    from paper_1708_00783_b200 import fusion as F
    gold = json.load(open(os.path.join(GOLD, "c1_frames.json")))
    intr = dict(width=640, height=480, fx=525.0, fy=525.0, cx=319.5, cy=239.5)
    poses = F.orbit_trajectory(frames=100)
    E = GpuEngine(0x40000, 0x20000, 0x40000)
    for g in gold:
        raw, _, _ = F.synth_render(0, poses[g["frame"]], F.Intrinsics(**intr))
        assert digest(raw) == g["raw"]
        d = rfo.build_view(raw, intr, AFF, 1)[0]
        st, _ = E.allocate(d, intr, poses[g["frame"]], PARAMS)
        assert st.tolist() == g["stats"]
        E.integrate(d, intr, poses[g["frame"]], PARAMS)
        rng, _ = E.render_ranges(poses[g["frame"]], intr, PARAMS)
        maps = E.render_icp(poses[g["frame"]], intr, PARAMS)
        got = _state_digests(E, rng, maps)
        for k in ("entries", "visible", "visibility", "vba", "ranges", "raycast", "points", "normals", "free"):
            assert got[k] == g[k], f"frame {g['frame']}: {k}"


def test_cpp_adapter_runs_on_gpu():
    from paper_1708_00783_b200 import _lib
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "adapter_test")
        subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(root, "include"),
                        os.path.join(root, "tests", "cpp", "adapter_test.cpp"), "-o", exe, _lib.LIB_PATH,
                        f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}"], check=True)
        p = subprocess.run([exe], capture_output=True, text=True, timeout=120)
        assert p.returncode == 0, p.stdout + p.stderr
        assert "GPU sequence ok" in p.stdout
