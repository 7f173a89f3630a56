"""The C restatement oracle (oracle/rfo.c) against the golden fixtures the
reference itself produced (tests/golden/make_golden.py, oracle/_ref).
CPU only; runs without /root/reference."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import rfo

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PARAMS = dict(voxelSize=0.005, mu=0.02, maxW=100, viewFrustum_min=0.2, viewFrustum_max=6.0,
              stopIntegratingAtMaxW=False)
AFF = (1.0 / 5000.0, 0.0)


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def el():
    return np.load(os.path.join(GOLD, "elements.npz"))


def test_hash_index_known_answers(el):
    # proj/tests/unit/test_voxelmap.cpp:33-44 frozen values are rows 0 and 1
    assert el["hash_out"][0] == 0 and el["hash_out"][1] == 455773
    for p, m, h in zip(el["hash_pos"], el["hash_mask"], el["hash_out"]):
        assert rfo.hash_index(p, int(m)) == h


def test_traverse_blocks_matches_reference(el):
    o = 0
    for seg, n in zip(el["dda_segs"], el["dda_counts"]):
        cells = rfo.traverse_blocks(seg[0], seg[1], 512)
        assert len(cells) == n
        assert np.array_equal(cells, el["dda_cells"][o:o + n])
        o += n


def test_block_in_frustum_matches_reference(el):
    intr = dict(width=640, height=480, fx=525.0, fy=525.0, cx=319.5, cy=239.5)
    for b, pose, want in zip(el["fr_blocks"], el["fr_pose"], el["fr_out"]):
        assert rfo.block_in_frustum(b, pose, intr, PARAMS) == bool(want)
    assert 0 < el["fr_out"].sum() < len(el["fr_out"])  # both outcomes covered


def test_update_voxel_depth_matches_reference(el):
    import ctypes as C
    from oracle.ref import P, _f, _i, _u8
    wh = np.array([640, 480], np.int32)
    f4 = np.array([525.0, 525.0, 319.5, 239.5], np.float32)
    d = np.ascontiguousarray(el["vu_depth"])
    pose = np.ascontiguousarray(el["vu_pose"])
    for pt, vin, vout, eta in zip(el["vu_pts"], el["vu_in"], el["vu_out"], el["vu_eta"]):
        v = vin.copy()
        e = rfo.lib().rfo_update_voxel_depth(P(v, _u8), P(pt.copy(), _f), P(pose, _f), P(wh, _i), P(f4, _f),
                                             C.c_float(0.02), 100, P(d, _f), 0)
        assert np.array_equal(v, vout)
        assert np.float32(e).view(np.uint32) == np.float32(eta).view(np.uint32)
    # the cases cover untouched, updated and invalid voxels
    changed = (el["vu_in"] != el["vu_out"]).any(axis=1)
    assert 0 < changed.sum() < len(changed) and (el["vu_eta"] == -1).any()


def test_build_view_pyramid(el):
    intr = dict(width=640, height=480, fx=525.0, fy=525.0, cx=319.5, cy=239.5)
    lv = rfo.build_view(el["bv_raw"], intr, AFF, 3)
    for a, k in zip(lv, ("bv_l0", "bv_l1", "bv_l2")):
        assert np.array_equal(a.view(np.uint32), el[k].view(np.uint32))
    assert lv[1].shape == (240, 320) and lv[2].shape == (120, 160)  # test_core.cpp:98-116


def _state_digests(E, rng, maps):
    ent = E.entries()
    vis, types = E.visible()
    ptrs = ent[ent[:, 4] >= 0, 4]
    blocks = E.blocks(np.sort(ptrs))
    return {"entries": digest(ent), "visible": digest(vis), "visibility": digest(types), "vba": digest(blocks),
            "ranges": digest(rng), "raycast": digest(maps[0]), "points": digest(maps[1]),
            "normals": digest(maps[2]), "free": list(E.free_counts())}


def run_small_sequence(make_engine, g):
    intr = json.loads(str(g["intr"]))
    E = make_engine(*[int(x) for x in g["cfg"]])
    digs = json.loads(str(g["digests"]))
    for f in range(len(g["poses"])):
        d = rfo.build_view(g["raw"][f], intr, AFF, 1)[0]
        st, _ = E.allocate(d, intr, g["poses"][f], PARAMS)
        assert np.array_equal(np.asarray(st), g["stats"][f]), f"frame {f} stats"
        E.integrate(d, intr, g["poses"][f], PARAMS)
        rng, _ = E.render_ranges(g["poses"][f], intr, PARAMS)
        maps = E.render_icp(g["poses"][f], intr, PARAMS)
        got = _state_digests(E, rng, maps)
        for k, v in digs[f].items():
            assert got[k] == v, f"frame {f}: {k} differs from the reference"
    ent = E.entries()
    assert np.array_equal(ent, g["final_entries"])
    assert np.array_equal(E.blocks(g["final_ptrs"]), g["final_blocks"])
    return E


def test_small_sequence_matches_reference_golden():
    g = np.load(os.path.join(GOLD, "seq_small.npz"))
    # the fixture exercises collisions (dropped requests) and excess chains
    assert (g["stats"][:, 0] >= g["stats"][:, 1]).all()
    assert (g["final_entries"][:, 3] > 0).any()
    run_small_sequence(rfo.OracleEngine, g)


def test_c1_full_frames_match_reference_golden():
    """Full C1 configuration (640x480, 0x40000 buckets), frames 0-1."""
    from paper_1708_00783_b200 import fusion as F
    gold = json.load(open(os.path.join(GOLD, "c1_frames.json")))
    intr = dict(width=640, height=480, fx=525.0, fy=525.0, cx=319.5, cy=239.5)
    poses = F.orbit_trajectory(frames=100)
    E = rfo.OracleEngine(0x40000, 0x20000, 0x40000)
    for g in gold:
        raw, _, _ = F.synth_render(0, poses[g["frame"]], F.Intrinsics(**intr))
        assert digest(raw) == g["raw"], "synthetic frame differs from the reference's"
        d = rfo.build_view(raw, intr, AFF, 1)[0]
        st, _ = E.allocate(d, intr, poses[g["frame"]], PARAMS)
        assert st.tolist() == g["stats"]
        E.integrate(d, intr, poses[g["frame"]], PARAMS)
        rng, _ = E.render_ranges(poses[g["frame"]], intr, PARAMS)
        maps = E.render_icp(poses[g["frame"]], intr, PARAMS)
        got = _state_digests(E, rng, maps)
        for k in ("entries", "visible", "visibility", "vba", "ranges", "raycast", "points", "normals", "free"):
            assert got[k] == g[k], f"frame {g['frame']}: {k}"
