#!/usr/bin/env python
"""Generate the golden fixtures in tests/golden/ from the REFERENCE ITSELF
(oracle/_ref/librfref.so = /root/reference/proj sources compiled against the
Eigen/doctest shims, see oracle/Makefile).  Run in the build container:

    make -C oracle ref && python tests/golden/make_golden.py

Fixtures:
  elements.npz   known-answer vectors for hash_index, traverse_blocks,
                 block_in_frustum, update_voxel_depth, build_view pyramid
  seq_small.npz  a 96x72 sphere-in-room sequence (6 frames, small map with
                 collisions): raw depth, poses, per-frame AllocationStats and
                 SHA-256 digests of entries / visible list / visibility / VBA /
                 ranges / ICP maps, plus the full final-frame state
  c1_frames.json full C1 (640x480, 0x40000 buckets) frames 0-1: stats and
                 digests of the canonical state after each stage
  view_full.npz  the full ViewBuilder (view.cpp:8-143) on noisy 96x72 frames
                 with colour: depth / intensity pyramids and normals with the
                 bilateral filter off and on, bilateral_filter on extreme depth
                 jumps, and PGM16 / PPM files as written by the reference
                 (image_io.cpp)

`python tests/golden/make_golden.py view` regenerates view_full.npz only.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

PARAMS = dict(voxelSize=0.005, mu=0.02, maxW=100, viewFrustum_min=0.2, viewFrustum_max=6.0,
              stopIntegratingAtMaxW=False)
AFF = (1.0 / 5000.0, 0.0)


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def state_digests(E, rng, maps):
    ent = E.entries()
    vis, types = E.visible()
    ptrs = ent[ent[:, 4] >= 0, 4]
    blocks = E.blocks(np.sort(ptrs))
    return {"entries": digest(ent), "visible": digest(vis), "visibility": digest(types), "vba": digest(blocks),
            "ranges": digest(rng), "raycast": digest(maps[0]), "points": digest(maps[1]),
            "normals": digest(maps[2]), "free": list(E.free_counts())}


def small_intr(w, h):
    s = w / 640.0
    return dict(width=w, height=h, fx=525.0 * s, fy=525.0 * s, cx=w / 2 - 0.5, cy=h / 2 - 0.5)


def make_elements(rng):
    out = {}
    # hash_index: the reference's own known answers + random
    pos = np.concatenate([np.array([[0, 0, 0], [1, 0, 0], [1, 1, 1], [-1, 2, -3]], np.int32),
                          rng.integers(-5000, 5000, size=(200, 3)).astype(np.int32)])
    masks = np.array([0xFFFFF, 0xFFFFF, 0x3FFFF, 0x3FFFF] + [0x3FFFF] * 200, np.uint32)
    out["hash_pos"] = pos
    out["hash_mask"] = masks
    out["hash_out"] = np.array([ref.lib().rr_hash_index(ref.P(p.copy(), ref._i), int(m)) for p, m in zip(pos, masks)],
                               np.uint32)
    # traverse_blocks: random segments in block units (incl. axis-aligned, tiny,
    # boundary-aligned)
    segs = rng.normal(0, 3, size=(300, 2, 3)).astype(np.float32)
    segs[:40, 1] = segs[:40, 0] + rng.normal(0, 0.2, size=(40, 3)).astype(np.float32)
    segs[40:60, 1, 1:] = segs[40:60, 0, 1:]            # axis-aligned in x
    segs[60:80] = np.round(segs[60:80])                 # endpoints on cell boundaries
    cells, counts = [], []
    buf = np.zeros((512, 3), np.int32)
    for a, b in segs:
        n = ref.lib().rr_traverse_blocks(ref.P(a.copy(), ref._f), ref.P(b.copy(), ref._f), ref.P(buf, ref._i), 512)
        counts.append(n)
        cells.append(buf[:n].copy())
    out["dda_segs"] = segs
    out["dda_counts"] = np.array(counts, np.int32)
    out["dda_cells"] = np.concatenate(cells)
    # block_in_frustum
    intr = dict(width=640, height=480, fx=525.0, fy=525.0, cx=319.5, cy=239.5)
    poses = ref.orbit_poses([0, 0.15, 1.4], 1.4, 7, 0.5)
    blocks = rng.integers(-40, 80, size=(400, 3)).astype(np.int32)
    pidx = rng.integers(0, 7, size=400)
    wh = np.array([640, 480], np.int32)
    f4 = np.array([525.0, 525.0, 319.5, 239.5], np.float32)
    pv = ref.params_vec(PARAMS)
    out["fr_blocks"] = blocks
    out["fr_pose"] = poses[pidx]
    out["fr_out"] = np.array([ref.lib().rr_block_in_frustum(ref.P(b.copy(), ref._i), ref.P(poses[k].copy(), ref._f),
                                                            ref.P(wh, ref._i), ref.P(f4, ref._f), ref.P(pv, ref._f))
                              for b, k in zip(blocks, pidx)], np.int32)
    # update_voxel_depth on a synthetic frame
    raw, dep, _ = ref.render(0, poses[3], intr)
    d = ref.build_view(raw, intr, AFF, 1)[0]
    pts = (rng.normal(0, 0.4, size=(600, 3)) + np.array([0, 0.15, 1.4])).astype(np.float32)
    vox = rng.integers(0, 256, size=(600, 8)).astype(np.uint8)
    vox[:, 2] = rng.integers(0, 101, size=600)           # w_depth <= maxW
    vox[:200, :3] = [0xFF, 0x7F, 0]                       # fresh voxels
    vox_out = vox.copy()
    etas = []
    for i in range(600):
        etas.append(ref.lib().rr_update_voxel_depth(ref.P(vox_out[i], ref._u8), ref.P(pts[i].copy(), ref._f),
                                                    ref.P(poses[3].copy(), ref._f), ref.P(wh, ref._i),
                                                    ref.P(f4, ref._f), 0.02, 100, ref.P(d, ref._f), 0))
    out["vu_depth"] = d
    out["vu_pose"] = poses[3]
    out["vu_pts"] = pts
    out["vu_in"] = vox
    out["vu_out"] = vox_out
    out["vu_eta"] = np.array(etas, np.float32)
    # build_view pyramid (depth conversion + 2x2 valid means)
    raw2 = raw.copy()
    raw2[::7, ::5] = 0  # holes
    lv = ref.build_view(raw2, intr, AFF, 3)
    out["bv_raw"] = raw2
    out["bv_l0"], out["bv_l1"], out["bv_l2"] = lv
    return out


def make_small_sequence():
    intr = small_intr(96, 72)
    cfg = (256, 2048, 4096)  # few buckets => collisions, long chains
    poses = ref.orbit_poses([0, 0.15, 1.4], 1.4, 100, 0.5)[::8][:6]
    E = ref.RefEngine(*cfg)
    raws, stats, digs = [], [], []
    for f in range(len(poses)):
        raw, _, _ = ref.render(0, poses[f], intr)
        raws.append(raw)
        d = ref.build_view(raw, intr, AFF, 1)[0]
        st, _ = E.allocate(d, intr, poses[f], PARAMS)
        E.integrate(d, intr, poses[f], PARAMS)
        rng_img, _ = E.render_ranges(poses[f], intr, PARAMS)
        maps = E.render_icp(poses[f], intr, PARAMS)
        stats.append(st)
        digs.append(state_digests(E, rng_img, maps))
    ent = E.entries()
    ptrs = np.sort(ent[ent[:, 4] >= 0, 4])[:64]  # full voxels for 64 blocks; the digest covers all
    return {"intr": json.dumps(intr), "cfg": np.array(cfg, np.int64), "poses": poses, "raw": np.stack(raws),
            "stats": np.stack(stats), "digests": json.dumps(digs), "final_entries": ent,
            "final_ptrs": ptrs, "final_blocks": E.blocks(ptrs), "final_visible": E.visible()[0],
            "final_ranges": rng_img, "final_points": maps[1], "final_normals": maps[2]}


def make_c1():
    intr = dict(width=640, height=480, fx=525.0, fy=525.0, cx=319.5, cy=239.5)
    poses = ref.orbit_poses([0, 0.15, 1.4], 1.4, 100, 0.5)
    E = ref.RefEngine(0x40000, 0x20000, 0x40000)
    frames = []
    for f in range(2):
        raw, _, _ = ref.render(0, poses[f], intr)
        d = ref.build_view(raw, intr, AFF, 1)[0]
        st, _ = E.allocate(d, intr, poses[f], PARAMS)
        E.integrate(d, intr, poses[f], PARAMS)
        rng_img, _ = E.render_ranges(poses[f], intr, PARAMS)
        maps = E.render_icp(poses[f], intr, PARAMS)
        frames.append({"frame": f, "raw": digest(raw), "stats": st.tolist(), **state_digests(E, rng_img, maps)})
    return frames


def make_view_full():
    import tempfile
    out = {}
    intr = small_intr(96, 72)
    poses = ref.orbit_poses([0, 0.15, 1.4], 1.4, 5, 0.5)
    for k in range(2):
        raw, _, col = ref.render(0, poses[2 * k], intr, AFF, rgb=True)
        rng = np.random.default_rng(100 + k)
        noisy = np.clip(raw.astype(np.int64) + rng.integers(-40, 41, raw.shape), 0, 65535).astype(np.uint16)
        noisy[raw == 0] = 0
        noisy[rng.random(raw.shape) < 0.01] = 0
        out[f"raw{k}"], out[f"rgb{k}"] = noisy, col
        for bil in (0, 1):
            v = ref.build_view_full(noisy, intr, AFF, levels=3, bilateral=bool(bil), rgb=col)
            for l in range(3):
                out[f"depth{k}_{bil}_{l}"] = v["depth"][l]
                out[f"intensity{k}_{bil}_{l}"] = v["intensity"][l]
            out[f"normals{k}_{bil}"] = v["normals"]
    rng = np.random.default_rng(7)
    d = rng.uniform(0.3, 6.0, (40, 52)).astype(np.float32)
    d[rng.random(d.shape) < 0.2] = -1.0
    out["bil_in"] = d
    out["bil_out"] = ref.bilateral_filter(d, 2.0, 0.002)
    with tempfile.TemporaryDirectory() as t:
        img = rng.integers(0, 65536, (23, 37), dtype=np.uint16)
        rgb = rng.integers(0, 256, (23, 37, 3), dtype=np.uint8)
        ref.write_pgm16(img, os.path.join(t, "a.pgm"))
        ref.write_ppm(rgb, os.path.join(t, "a.ppm"))
        out["pgm_img"], out["ppm_img"] = img, rgb
        out["pgm_bytes"] = np.frombuffer(open(os.path.join(t, "a.pgm"), "rb").read(), np.uint8)
        out["ppm_bytes"] = np.frombuffer(open(os.path.join(t, "a.ppm"), "rb").read(), np.uint8)
    out["intr"] = np.array([intr["width"], intr["height"], intr["fx"], intr["fy"], intr["cx"], intr["cy"]],
                           np.float64)
    return out


def main():
    assert ref.available(), "build oracle/_ref first: make -C oracle ref"
    if len(sys.argv) > 1 and sys.argv[1] == "view":
        np.savez_compressed(os.path.join(HERE, "view_full.npz"), **make_view_full())
        return
    rng = np.random.default_rng(1708)
    np.savez_compressed(os.path.join(HERE, "elements.npz"), **make_elements(rng))
    np.savez_compressed(os.path.join(HERE, "seq_small.npz"), **make_small_sequence())
    with open(os.path.join(HERE, "c1_frames.json"), "w") as f:
        json.dump(make_c1(), f, indent=1)
    np.savez_compressed(os.path.join(HERE, "view_full.npz"), **make_view_full())
    for n in os.listdir(HERE):
        print(n, os.path.getsize(os.path.join(HERE, n)))


if __name__ == "__main__":
    main()
