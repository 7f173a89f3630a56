"""Exhaustive exactness checks of arithmetic shortcuts in the kernels."""
import os
import subprocess
import tempfile

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_sdf_to_logical_fast_path_is_ieee_exact_for_all_int16():
    src = os.path.join(ROOT, "tests", "cuda", "div32767.cu")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "div32767")
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                        "-fmad=false", "-std=c++17", src, "-o", exe], check=True)
        p = subprocess.run([exe], capture_output=True, text=True, timeout=60)
        assert p.returncode == 0 and "mismatches 0" in p.stdout, p.stdout + p.stderr


def test_hoisted_division_and_lround_are_ieee_exact():
    """div_fast/div_rcp (projection, eta/mu, weight merge) and lround_haz
    (quantisation, nearest reads) against __fdiv_rn / lroundf."""
    src = os.path.join(ROOT, "tests", "cuda", "divfast.cu")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "divfast")
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                        "-fmad=false", "-std=c++17", src, "-o", exe], check=True)
        p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stdout + p.stderr
        assert "exhaustive mismatches 0  random mismatches 0  lround mismatches 0" in p.stdout, p.stdout


def test_alu_conversions_are_exact():
    """u23_to_float / s16_to_float / trunc_pos_to_int / lround_haz_alu (the
    integration kernel's conversions on the FMA/ALU pipes) against the
    hardware conversions, exhaustively."""
    src = os.path.join(ROOT, "tests", "cuda", "magic_cvt.cu")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "magic_cvt")
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                        "-fmad=false", "-std=c++17", src, "-o", exe], check=True)
        p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
        assert p.returncode == 0 and "magic conversions: mismatches 0" in p.stdout, p.stdout + p.stderr
