"""Full ViewBuilder oracle + Netpbm IO, on the CPU.

* the C restatement (oracle/rfo.c: rgb_to_intensity, bilateral_filter with
  the C library's expf, compute_normals, downsample_intensity, build_view
  with every option) pinned bit-for-bit to the reference build
  (oracle/_ref, view.cpp:8-143) on noisy synthetic frames;
* librfg's Netpbm readers / writers (rfg_io.cpp, host code — no GPU needed)
  against the reference's image_io.cpp: round trips (test_io.cpp:89-112),
  files crossing between the two implementations, header comments, the
  reference's error cases and ImageStream (test_io.cpp:114-132).
"""
import os

import numpy as np
import pytest

from helpers import AFF, small_intr
from oracle import ref, rfo

needs_ref = pytest.mark.skipif(not ref.available(), reason="reference build (oracle/_ref) not available")


def _noisy_frame(intr, seed=0, amp=40):
    from paper_1708_00783_b200 import fusion as F
    poses = F.orbit_trajectory(frames=5)
    raw, _, col = F.synth_render(0, poses[seed % 5], F.Intrinsics(**intr), rgb=True)
    rng = np.random.default_rng(seed)
    noisy = np.clip(raw.astype(np.int64) + rng.integers(-amp, amp + 1, raw.shape), 0, 65535).astype(np.uint16)
    noisy[raw == 0] = 0
    noisy[rng.random(raw.shape) < 0.01] = 0  # dropouts
    return noisy, col


def _bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@needs_ref
@pytest.mark.parametrize("bilateral", [False, True])
def test_build_view_oracle_pinned_to_reference(bilateral):
    intr = small_intr()
    for seed in range(3):
        raw, col = _noisy_frame(intr, seed)
        a = ref.build_view_full(raw, intr, AFF, levels=3, bilateral=bilateral, rgb=col)
        b = rfo.build_view_full(raw, intr, AFF, levels=3, bilateral=bilateral, rgb=col)
        for x, y in zip(a["depth"], b["depth"]):
            assert np.array_equal(_bits(x), _bits(y))
        for x, y in zip(a["intensity"], b["intensity"]):
            assert np.array_equal(_bits(x), _bits(y))
        assert np.array_equal(_bits(a["normals"]), _bits(b["normals"]))
        assert (a["normals"][..., 3] > 0).sum() > 1000


@needs_ref
def test_bilateral_oracle_edge_cases_pinned():
    rng = np.random.default_rng(5)
    # depth jumps of metres drive exp() into its underflow branches
    # (x < -103.97 -> 0, [-103.97, -103.28) -> 2^-149)
    d = rng.uniform(0.3, 6.0, (40, 52)).astype(np.float32)
    d[rng.random(d.shape) < 0.2] = -1.0
    for ss, rs in [(2.0, 0.002), (2.0, 0.05), (0.7, 0.5), (3.0, 1e-4)]:
        assert np.array_equal(_bits(ref.bilateral_filter(d, ss, rs)), _bits(rfo.bilateral_filter(d, ss, rs)))
    # arguments that land exactly in glibc expf's special ranges
    base = np.full((9, 9), 1.0, np.float32)
    for dr in (0.0, 0.0203, 0.02035, 0.0204, 0.05):
        e = base.copy()
        e[4, 4] = 1.0 + dr
        assert np.array_equal(_bits(ref.bilateral_filter(e, 2.0, 0.002)), _bits(rfo.bilateral_filter(e, 2.0, 0.002)))


def test_bilateral_identity_on_constant_depth():
    # test_core.cpp:124-129
    out = rfo.bilateral_filter(np.full((16, 16), 1.5, np.float32), 2.0, 0.01)
    assert np.allclose(out, 1.5, rtol=1e-6)


def test_view_known_answers():
    # test_core.cpp:90-96: grey intensity weights sum to one
    it = rfo.rgb_to_intensity(np.full((4, 4, 3), 100, np.uint8))
    assert abs(it[1, 1] - 100.0 / 255.0) <= 1e-6 * 100.0 / 255.0
    # test_core.cpp:155-160: isolated pixel has no normal
    d = np.full((8, 8), -1.0, np.float32)
    d[4, 4] = 1.0
    n = rfo.compute_normals(d, dict(width=8, height=8, fx=10.0, fy=10.0, cx=3.5, cy=3.5))
    assert n[4, 4, 3] < 0
    # fronto-parallel plane faces the camera (test_core.cpp:131-141)
    n = rfo.compute_normals(np.full((48, 64), 2.0, np.float32), dict(width=64, height=48, fx=60.0, fy=60.0,
                                                                      cx=31.5, cy=23.5))
    assert n[24, 32, 3] > 0 and np.abs(n[24, 32, :3] - [0, 0, -1]).max() < 1e-4


# ------------------------------------------------------------------ Netpbm IO
def _rfg():
    from paper_1708_00783_b200 import fusion as F
    return F


def test_pnm_round_trips_bit_exact(tmp_path):
    # test_io.cpp:89-112 (37 x 23 random images)
    F = _rfg()
    rng = np.random.default_rng(99)
    rgb = rng.integers(0, 256, (23, 37, 3), dtype=np.uint8)
    depth = rng.integers(0, 65536, (23, 37), dtype=np.uint16)
    F.write_ppm(rgb, str(tmp_path / "t.ppm"))
    F.write_pgm16(depth, str(tmp_path / "t.pgm"))
    assert np.array_equal(F.read_ppm(str(tmp_path / "t.ppm")), rgb)
    assert np.array_equal(F.read_pgm16(str(tmp_path / "t.pgm")), depth)
    # the payload reader returns the stored big-endian words
    assert np.array_equal(F.read_pgm16_payload(str(tmp_path / "t.pgm")), depth.byteswap())


@needs_ref
def test_pnm_files_cross_between_implementations(tmp_path):
    F = _rfg()
    rng = np.random.default_rng(7)
    rgb = rng.integers(0, 256, (31, 45, 3), dtype=np.uint8)
    depth = rng.integers(0, 65536, (31, 45), dtype=np.uint16)
    ref.write_ppm(rgb, str(tmp_path / "r.ppm"))
    ref.write_pgm16(depth, str(tmp_path / "r.pgm"))
    F.write_ppm(rgb, str(tmp_path / "g.ppm"))
    F.write_pgm16(depth, str(tmp_path / "g.pgm"))
    for ext in ("ppm", "pgm"):  # byte-identical files
        assert (tmp_path / f"r.{ext}").read_bytes() == (tmp_path / f"g.{ext}").read_bytes()
    assert np.array_equal(F.read_pgm16(str(tmp_path / "r.pgm")), ref.read_pgm16(str(tmp_path / "g.pgm")))
    assert np.array_equal(F.read_ppm(str(tmp_path / "r.ppm")), ref.read_ppm(str(tmp_path / "g.ppm")))


def _header_cases(tmp_path):
    px = np.arange(6, dtype=">u2").tobytes()
    return {
        "comments": (b"P5\n# a comment\n3 # width\n2\n65535\n" + px, True),
        "tabs": (b"P5\t3\t2\t65535\n" + px, True),
        "wrong magic": (b"P2\n3 2\n65535\n" + px, False),
        "wrong maxval": (b"P5\n3 2\n255\n" + px, False),
        "truncated": (b"P5\n3 2\n65535\n" + px[:-1], False),
        "empty": (b"", False),
        "non-numeric": (b"P5\nx 2\n65535\n" + px, False),
    }


@needs_ref
def test_pgm_header_grammar_and_errors_match_reference(tmp_path):
    F = _rfg()
    for name, (data, ok) in _header_cases(tmp_path).items():
        p = tmp_path / (name.replace(" ", "_") + ".pgm")
        p.write_bytes(data)
        r = ref.read_pgm16(str(p))
        assert (r is not None) == ok, name
        if ok:
            assert np.array_equal(F.read_pgm16(str(p)), r)
            assert np.array_equal(r.reshape(-1), np.arange(6))
        else:
            with pytest.raises(RuntimeError):
                F.read_pgm16(str(p))


def test_pnm_error_messages_are_the_references(tmp_path):
    F = _rfg()
    missing = str(tmp_path / "nope.pgm")
    with pytest.raises(RuntimeError, match="cannot open " + missing):
        F.read_pgm16(missing)
    p = tmp_path / "m.pgm"
    p.write_bytes(b"P6\n1 1\n255\nabc")
    with pytest.raises(RuntimeError, match=r"not a binary PGM \(P5\)"):
        F.read_pgm16(str(p))
    p.write_bytes(b"P5\n1 1\n255\nab")
    with pytest.raises(RuntimeError, match=r"unsupported PGM maxval \(want 65535\)"):
        F.read_pgm16(str(p))
    p.write_bytes(b"P5\n2 2\n65535\nab")
    with pytest.raises(RuntimeError, match="truncated PGM"):
        F.read_pgm16(str(p))
    q = tmp_path / "m.ppm"
    q.write_bytes(b"P6\n1 1\n65535\nabc")
    with pytest.raises(RuntimeError, match=r"unsupported PPM maxval \(want 255\)"):
        F.read_ppm(str(q))


def test_image_stream_stops_at_first_gap(tmp_path):
    # test_io.cpp:114-132
    F = _rfg()
    depth = np.full((4, 4), 1234, np.uint16)
    for i in (0, 1, 2, 4):  # frame 3 missing
        F.write_pgm16(depth, str(tmp_path / f"{i:04d}.pgm"))
    stream = F.ImageStream(os.path.join(str(tmp_path), "%04d"), 0)
    n = 0
    while (f := stream.next()) is not None:
        assert f.index == n and f.rgb is None and np.array_equal(f.depth, depth)
        n += 1
    assert n == 3 and stream.nextIndex() == 3


# ------------------------------------------------ golden fixtures (reference)
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "view_full.npz")


def _gold_intr(g):
    w, h, fx, fy, cx, cy = g["intr"]
    return dict(width=int(w), height=int(h), fx=float(fx), fy=float(fy), cx=float(cx), cy=float(cy))


def test_view_oracle_matches_reference_golden():
    g = np.load(GOLD)
    intr = _gold_intr(g)
    for k in range(2):
        for bil in (0, 1):
            v = rfo.build_view_full(g[f"raw{k}"], intr, AFF, levels=3, bilateral=bool(bil), rgb=g[f"rgb{k}"])
            for l in range(3):
                assert np.array_equal(_bits(v["depth"][l]), _bits(g[f"depth{k}_{bil}_{l}"]))
                assert np.array_equal(_bits(v["intensity"][l]), _bits(g[f"intensity{k}_{bil}_{l}"]))
            assert np.array_equal(_bits(v["normals"]), _bits(g[f"normals{k}_{bil}"]))
    assert np.array_equal(_bits(rfo.bilateral_filter(g["bil_in"], 2.0, 0.002)), _bits(g["bil_out"]))


def test_pnm_readers_match_reference_golden_files(tmp_path):
    F = _rfg()
    g = np.load(GOLD)
    (tmp_path / "a.pgm").write_bytes(g["pgm_bytes"].tobytes())
    (tmp_path / "a.ppm").write_bytes(g["ppm_bytes"].tobytes())
    assert np.array_equal(F.read_pgm16(str(tmp_path / "a.pgm")), g["pgm_img"])
    assert np.array_equal(F.read_ppm(str(tmp_path / "a.ppm")), g["ppm_img"])
    F.write_pgm16(g["pgm_img"], str(tmp_path / "b.pgm"))
    F.write_ppm(g["ppm_img"], str(tmp_path / "b.ppm"))
    assert (tmp_path / "b.pgm").read_bytes() == g["pgm_bytes"].tobytes()
    assert (tmp_path / "b.ppm").read_bytes() == g["ppm_bytes"].tobytes()
