"""Shared test helpers: configs, frame sources and canonical comparisons."""
from __future__ import annotations

import numpy as np

INTR_C1 = dict(width=640, height=480, fx=525.0, fy=525.0, cx=319.5, cy=239.5)
PARAMS_C1 = dict(voxelSize=0.005, mu=0.02, maxW=100, viewFrustum_min=0.2, viewFrustum_max=6.0,
                 stopIntegratingAtMaxW=False)
MAP_C1 = (0x40000, 0x20000, 0x40000)
AFF = (1.0 / 5000.0, 0.0)


def small_intr(w=160, h=120):
    s = w / 640.0
    return dict(width=w, height=h, fx=525.0 * s, fy=525.0 * s, cx=w / 2 - 0.5, cy=h / 2 - 0.5)


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32) if a.dtype == np.float32 else a


def same_bits(a, b):
    return np.array_equal(bits(a), bits(b))


def canonical_blocks(engine, entries):
    """{pos: 512x8 voxel bytes} for every resident block (ptr >= 0)."""
    alloc = entries[entries[:, 4] >= 0]
    order = np.lexsort((alloc[:, 2], alloc[:, 1], alloc[:, 0]))
    alloc = alloc[order]
    vox = engine.blocks(alloc[:, 4])
    return alloc[:, :3], vox


class GpuEngine:
    """Adapter giving the B200 engine the same call shape as oracle.rfo.OracleEngine
    (host numpy in/out) so parity tests can drive both identically."""

    def __init__(self, buckets, excess, capacity, colour=False):
        from paper_1708_00783_b200 import fusion as F
        self.F = F
        self.map = F.VoxelBlockMap(F.VoxelBlockMapConfig(buckets, excess, capacity), colour=colour)
        self.fusion = F.FusionEngine()
        self.state = F.RenderState()
        self.capacity = capacity

    def _intr(self, d):
        return self.F.Intrinsics(**d)

    def _params(self, d):
        return self.F.SceneParams(**d)

    def _view(self, depth, intr, rgb=None, intr_rgb=None, extr34=None):
        F = self.F
        i = self._intr(intr)
        cal = F.RgbdCalib(intrinsics_rgb=self._intr(intr_rgb) if intr_rgb else i, intrinsics_d=i)
        if extr34 is not None:
            cal.extrinsics_d_to_rgb = np.asarray(extr34, np.float32).reshape(3, 4)
        return F.view_from_depth(depth, i, rgb=rgb, calib=cal)

    def set_shard(self, rank, world, tile_shift=3):
        self.map.set_shard(rank, world, tile_shift)

    opts = None

    def set_fusion_options(self, swapping_enabled, swap_margin_px=8.0):
        self.opts = self.F.FusionEngine.Options(bool(swapping_enabled), swap_margin_px)

    def allocate(self, depth, intr, pose34, params):
        st = self.fusion.allocate_from_depth(self.map, self._view(depth, intr), pose34, self._params(params),
                                             opts=self.opts)
        return st.as_array(), 0.0

    def reserve_block(self, idx):
        return 1 if self.map.reserveBlockForEntry(idx) else 0

    def release_block(self, idx):
        self.map.releaseBlock(idx)

    def swap_create(self, capacity):
        self.sw = self.F.SwappingEngine(self.map, capacity)

    def swap_in(self, max_w=100):
        return self.sw.swap_in(max_w)

    def swap_out(self):
        return self.sw.swap_out()

    def swap_stored(self):
        return self.sw.stored()

    def swap_host_block(self, idx):
        return self.sw.host_block(idx)

    def integrate(self, depth, intr, pose34, params, rgb=None, intr_rgb=None, extr34=None):
        self.fusion.integrate_frame(self.map, self._view(depth, intr, rgb, intr_rgb, extr34), pose34,
                                    self._params(params))
        return 0.0

    def render_ranges(self, pose34, intr, params):
        self.F.render_expected_ranges(self.map, pose34, self._intr(intr), self._params(params), self.state)
        return self.state.expectedRange.cpu().numpy(), 0.0

    def set_ranges(self, intr, rng):
        import torch
        self.state.resize(self._intr(intr))
        self.state.expectedRange.copy_(torch.as_tensor(np.ascontiguousarray(rng, np.float32)))

    def render_icp(self, pose34, intr, params):
        F = self.F
        F.render_maps(self.map, pose34, self._intr(intr), self._params(params), F.RenderMode.kIcpMaps, self.state)
        return (self.state.raycastResult.cpu().numpy(), self.state.points.cpu().numpy(),
                self.state.normals.cpu().numpy(), 0.0)

    def render_maps(self, mode, pose34, intr, params):
        """render_maps(mode): (raycast, points, normals, colour RGB8)."""
        F = self.F
        F.render_maps(self.map, pose34, self._intr(intr), self._params(params), F.RenderMode(mode), self.state)
        return (self.state.raycastResult.cpu().numpy(), self.state.points.cpu().numpy(),
                self.state.normals.cpu().numpy(), self.state.colour.cpu().numpy())

    def entries(self):
        return self.map.entries()

    def blocks(self, ptrs):
        return self.map.blocks(ptrs)

    def visible(self):
        return self.map.visible()

    def free_counts(self):
        return self.map.free_counts()
