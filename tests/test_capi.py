"""The C ABI library (CPU-side checks, no GPU compute): it loads, exports every
symbol include/rfg.h declares, rejects invalid arguments like the reference,
fails loudly without a GPU, and its synthetic frame source is bit-identical to
the reference's."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "rfg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rfg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1708_00783_b200 import _lib
    L = C.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # and the Python binding table covers them all
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a():
    import subprocess
    from paper_1708_00783_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_non_power_of_two_bucket_count_rejected():
    from paper_1708_00783_b200 import fusion as F
    with pytest.raises(ValueError, match="power of two"):
        F.VoxelBlockMap(F.VoxelBlockMapConfig(1000, 16, 16))


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1708_00783_b200 import fusion as F
    from paper_1708_00783_b200._lib import RfgError
    with pytest.raises(RfgError, match="no CUDA device"):
        F.VoxelBlockMap(F.VoxelBlockMapConfig.small())


def test_build_view_argument_errors():
    from paper_1708_00783_b200 import fusion as F
    intr = F.Intrinsics(8, 8, 10.0, 10.0, 3.5, 3.5)
    calib = F.RgbdCalib(intrinsics_rgb=intr, intrinsics_d=intr)
    with pytest.raises(ValueError, match="does not match"):
        F.build_view(np.zeros((4, 4), np.uint16), None, calib)   # view.cpp:102-103 (test_core.cpp:118-122)
    with pytest.raises(ValueError, match="levels"):
        F.build_view(np.zeros((8, 8), np.uint16), None, calib, levels=0)


def test_intrinsics_at_level_and_params():
    from paper_1708_00783_b200 import fusion as F
    i = F.Intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
    l2 = i.atLevel(2)
    assert (l2.width, l2.height) == (160, 120) and l2.fx == 131.25 and l2.cx == np.float32(319.5 * 0.25)
    assert F.SceneParams().blockSizeMetres() == np.float32(0.005) * np.float32(8)
    assert F.VoxelBlockMapConfig.small() == F.VoxelBlockMapConfig(1 << 14, 1 << 11, 1 << 13)


def test_synth_matches_reference():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    from paper_1708_00783_b200 import fusion as F
    intr = F.Intrinsics(160, 120, 131.25, 131.25, 79.5, 59.5)
    poses = F.orbit_trajectory(frames=100)
    rp = ref.orbit_poses([0, 0.15, 1.4], 1.4, 100, 0.5)
    assert np.array_equal(poses.view(np.uint32), rp.view(np.uint32))
    for f in (0, 33, 99):
        a = F.synth_render(0, poses[f], intr, rgb=True)
        b = ref.render(0, rp[f], intr.as_dict(), rgb=True)
        for x, y in zip(a, b):
            assert np.array_equal(x.view(np.uint8), y.view(np.uint8))
    a = F.synth_render(2, poses[5], intr, rgb=True)   # checker wall (textured)
    b = ref.render(2, rp[5], intr.as_dict(), rgb=True)
    assert np.array_equal(a[2], b[2])


def test_cpp_adapter_compiles():
    """include/rfg.hpp (the C++ adapter with the reference's rf:: names)
    compiles against the C ABI and links against librfg.so."""
    import subprocess
    import tempfile
    from paper_1708_00783_b200 import _lib
    src = os.path.join(ROOT, "tests", "cpp", "adapter_test.cpp")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "adapter_test")
        p = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", exe,
                            _lib.LIB_PATH, f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}"],
                           capture_output=True, text=True)
        assert p.returncode == 0, p.stderr
