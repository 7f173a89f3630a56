"""GPU marching cubes (rfg_mesh.cu) vs the oracle (oracle/rfo.c, pinned to
the reference in tests/test_mesh_oracle.py): identical vertex and triangle
arrays — same order — on fused maps (small and full C1 resolution, several
frames), plus the empty map."""
import numpy as np
import pytest

from helpers import AFF, INTR_C1, MAP_C1, GpuEngine, small_intr
from oracle import rfo

pytestmark = pytest.mark.gpu


def _fuse(intr, pd, cfg, frames, step):
    from paper_1708_00783_b200 import fusion as F
    fi = F.Intrinsics(**intr)
    poses = F.orbit_trajectory(frames=100)
    g, o = GpuEngine(*cfg), rfo.OracleEngine(*cfg)
    for f in range(frames):
        raw, _, _ = F.synth_render(0, poses[step * f], fi)
        d = rfo.build_view(raw, intr, AFF, 1)[0]
        for e in (g, o):
            e.allocate(d, intr, poses[step * f], pd)
            e.integrate(d, intr, poses[step * f], pd)
    return g, o


@pytest.mark.parametrize("case", ["small", "c1"])
def test_mesh_bit_exact_and_in_reference_order(case):
    from paper_1708_00783_b200 import fusion as F
    if case == "small":
        intr, pd, cfg, frames, step = small_intr(), F.SceneParams(voxelSize=0.01).as_dict(), (0x4000, 0x2000, 0x4000), 4, 7
    else:
        intr, pd, cfg, frames, step = INTR_C1, F.SceneParams().as_dict(), MAP_C1, 3, 10
    g, o = _fuse(intr, pd, cfg, frames, step)
    vs = pd["voxelSize"]
    mg = F.extract_mesh(g.map, vs)
    vo, to = o.extract_mesh(vs)
    assert len(to) > 10000
    assert np.array_equal(mg.vertices.view(np.uint32), vo.view(np.uint32))
    assert np.array_equal(mg.triangles, to)
    # a second extraction reuses the buffers and gives the same mesh
    m2 = F.extract_mesh(g.map, vs)
    assert np.array_equal(m2.triangles, to)


def test_mesh_empty_map():
    from paper_1708_00783_b200 import fusion as F
    m = F.VoxelBlockMap(F.VoxelBlockMapConfig(64, 32, 128))
    mesh = F.extract_mesh(m, 0.005)
    assert mesh.vertices.shape == (0, 3) and mesh.triangles.shape == (0, 3)
