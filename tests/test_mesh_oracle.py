"""Marching cubes (§8(f)4, meshing.cpp) on the CPU side:
* the triangulation table built by librfg's host code (rfg_mc_table, what the
  GPU kernels use), by the oracle (rfo.c) and by the reference itself
  (detail::marchingCubesTable) are identical;
* the oracle's extract_mesh equals the reference's — same vertices, same
  triangles, same order — on integrated sequences and analytic TSDF maps;
* the reference's own meshing cases (test_voxelmap.cpp:231-280): empty map /
  all-positive block give no triangles; an analytic sphere is accurate,
  closed and outward-oriented."""
import numpy as np
import pytest

from helpers import AFF, small_intr
from oracle import ref, rfo

needs_ref = pytest.mark.skipif(not ref.available(), reason="reference build (oracle/_ref) not available")


def test_product_table_equals_oracle_table():
    from paper_1708_00783_b200 import fusion as F
    t = F.marching_cubes_table()
    assert t == rfo.mc_table()
    assert max(len(x) for x in t) == 5 and len(t[0]) == 0 and len(t[255]) == 0


@needs_ref
def test_tables_equal_reference_table():
    assert rfo.mc_table() == ref.mc_table()


def _analytic_sphere(engine, vs=0.005, mu=0.02, radius=0.1, centre=(0.2, 0.2, 0.2)):
    """test_voxelmap.cpp:244-251 via tests/unit/oracles.hpp buildAnalyticTsdf."""
    c = np.asarray(centre, np.float64)
    bs = vs * 8
    lo = np.floor((c - (radius + 4 * mu)) / bs).astype(int)
    hi = np.ceil((c + (radius + 4 * mu)) / bs).astype(int)
    brad = 0.5 * bs * np.sqrt(3.0)
    g = np.stack(np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij"), -1)[..., ::-1]  # (z,y,x)->xyz
    for z in range(lo[2], hi[2] + 1):
        for y in range(lo[1], hi[1] + 1):
            for x in range(lo[0], hi[0] + 1):
                bc = (np.array([x, y, z]) + 0.5) * bs
                if abs(np.linalg.norm(bc - c) - radius) > mu + brad:
                    continue
                p = (np.array([x, y, z]) * 8 + g.reshape(-1, 3)) * vs  # lx fastest
                sd = np.clip((np.linalg.norm(p - c, axis=1) - radius) / mu, -1, 1)
                q = np.round(sd * 32767).astype(np.int16)
                assert engine.set_block([x, y, z], q, np.ones(512, np.uint8)) == 0


def _mesh_checks(v, t, centre=(0.2, 0.2, 0.2), radius=0.1, vs=0.005):
    assert len(t) > 100
    assert np.abs(np.linalg.norm(v - np.asarray(centre, np.float32), axis=1) - radius).max() <= 0.5 * vs
    e = np.sort(np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]]), axis=1)
    _, counts = np.unique(e, axis=0, return_counts=True)
    assert (counts == 2).all()  # closed
    a, b, c = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    n = np.cross(b - a, c - a)
    out = (a + b + c) / 3 - np.asarray(centre, np.float32)
    # outward, except zero-area triangles: vertices coincide where a corner's
    # sdf quantises to exactly 0 — the same case that makes the reference's
    # own orientation check (test_voxelmap.cpp:271-279) fail
    area = np.linalg.norm(n, axis=1)
    dots = (n * out).sum(1)
    assert (dots[area > 1e-12] > 0).all()
    assert (area <= 1e-12).mean() < 0.01


def test_oracle_mesh_edge_cases_and_analytic_sphere():
    o = rfo.OracleEngine(64, 32, 128)
    v, t = o.extract_mesh(0.005)
    assert len(v) == 0 and len(t) == 0
    o.set_block([0, 0, 0], np.full(512, int(round(0.75 * 32767)), np.int16), np.ones(512, np.uint8))
    v, t = o.extract_mesh(0.005)
    assert len(t) == 0
    s = rfo.OracleEngine(1 << 12, 1 << 10, 1 << 12)
    _analytic_sphere(s)
    _mesh_checks(*s.extract_mesh(0.005))


@needs_ref
def test_oracle_mesh_equals_reference_analytic_sphere():
    r, o = ref.RefEngine(1 << 12, 1 << 10, 1 << 12), rfo.OracleEngine(1 << 12, 1 << 10, 1 << 12)
    _analytic_sphere(r)
    _analytic_sphere(o)
    (vr, tr), (vo, to) = r.extract_mesh(0.005), o.extract_mesh(0.005)
    assert np.array_equal(vr.view(np.uint32), vo.view(np.uint32)) and np.array_equal(tr, to)


@needs_ref
def test_oracle_mesh_equals_reference_on_fused_sequence():
    from paper_1708_00783_b200 import fusion as F
    intr = small_intr()
    fi = F.Intrinsics(**intr)
    pd = F.SceneParams(voxelSize=0.01).as_dict()
    poses = F.orbit_trajectory(frames=100)
    cfg = (0x2000, 0x1000, 0x2000)
    r, o = ref.RefEngine(*cfg), rfo.OracleEngine(*cfg)
    for f in range(3):
        raw, _, _ = F.synth_render(0, poses[8 * f], fi)
        d = rfo.build_view(raw, intr, AFF, 1)[0]
        for e in (r, o):
            e.allocate(d, intr, poses[8 * f], pd)
            e.integrate(d, intr, poses[8 * f], pd)
    (vr, tr), (vo, to) = r.extract_mesh(0.01), o.extract_mesh(0.01)
    assert len(tr) > 10000
    assert np.array_equal(vr.view(np.uint32), vo.view(np.uint32)) and np.array_equal(tr, to)
