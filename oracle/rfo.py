"""ctypes wrapper over oracle/_build/librfo.so (the C restatement oracle).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg, never by the product package.  The API mirrors
oracle/ref.py so tests can swap the reference build and the restatement.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .ref import P, _d, _f, _f4, _f32, _i, _u8, _u16, _view_full, _wh, params_vec

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "librfo.so")

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE, "rfo"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.rfo_hash_index.argtypes = [_i, C.c_uint32]
        L.rfo_hash_index.restype = C.c_uint32
        L.rfo_traverse_blocks.argtypes = [_f, _f, _i, C.c_int]
        L.rfo_block_in_frustum.argtypes = [_i, _f, _i, _f, _f]
        L.rfo_update_voxel_depth.argtypes = [_u8, _f, _f, _i, _f, C.c_float, C.c_int, _f, C.c_int]
        L.rfo_update_voxel_depth.restype = C.c_float
        L.rfo_create.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32]
        L.rfo_create.restype = vp
        L.rfo_destroy.argtypes = [vp]
        L.rfo_clear.argtypes = [vp]
        L.rfo_set_shard.argtypes = [vp, C.c_int, C.c_int, C.c_int]
        L.rfo_allocate.argtypes = [vp, _f, _i, _f, _f, _f, _i]
        L.rfo_integrate.argtypes = [vp, _f, _u8, _i, _f, _i, _f, _f, _f, _f]
        L.rfo_render_ranges.argtypes = [vp, _f, _i, _f, _f, _f]
        L.rfo_set_ranges.argtypes = [vp, _i, _f]
        L.rfo_render_icp.argtypes = [vp, _f, _i, _f, _f, _f, _f, _f]
        L.rfo_build_view.argtypes = [_u16, _i, C.c_float, C.c_float, C.c_int, _f]
        L.rfo_set_fusion_options.argtypes = [vp, C.c_int, C.c_float]
        L.rfo_reserve_block.argtypes = [vp, C.c_int]
        L.rfo_release_block.argtypes = [vp, C.c_int]
        L.rfo_swap_create.argtypes = [vp, C.c_int]
        L.rfo_swap_create.restype = vp
        L.rfo_swap_destroy.argtypes = [vp]
        L.rfo_swap_in.argtypes = [vp, vp, C.c_int]
        L.rfo_swap_out.argtypes = [vp, vp]
        L.rfo_swap_export.argtypes = [vp, C.c_size_t, _u8, _u8]
        L.rfo_swap_host_block.argtypes = [vp, C.c_int, _u8]
        L.rfo_mc_table.argtypes = [_i, _i]
        L.rfo_extract_mesh.argtypes = [vp, C.c_float, C.POINTER(C.POINTER(C.c_float)),
                                       C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_longlong),
                                       C.POINTER(C.c_longlong)]
        L.rfo_free.argtypes = [vp]
        L.rfo_set_block.argtypes = [vp, _i, C.POINTER(C.c_int16), _u8]
        L.rfo_render_colour.argtypes = [vp, C.c_int, _f, _i, _f, _f, _f, _i, C.c_int, _u8]
        L.rfo_build_view_full.argtypes = [_u16, _u8, _i, _f, C.c_float, C.c_float, C.c_int, C.c_int, _f, _f, _f]
        L.rfo_bilateral_filter.argtypes = [_f, C.c_int, C.c_int, C.c_float, C.c_float, _f]
        L.rfo_compute_normals.argtypes = [_f, C.c_int, C.c_int, _f, _f]
        L.rfo_rgb_to_intensity.argtypes = [_u8, C.c_int, C.c_int, _f]
        L.rfo_downsample_intensity.argtypes = [_f, C.c_int, C.c_int, _f]
        L.rfo_icp_track.argtypes = [_f, _i, _f, _f, _f, _f, _f, _f, _i, _f, _f, _d]
        L.rfo_icp_reduce.argtypes = [_f, C.c_int, C.c_int, _f, _f, _f, _i, _f, _f, _f, C.c_float,
                                     C.POINTER(C.c_int64), _d]
        L.rfo_solve6.argtypes = [_d, _d, _d]
        L.rfo_se3_coeffs.argtypes = [C.c_double, _d]
        L.rfo_forward_project.argtypes = [C.c_int, _f, _f, _f, _f, _i, _f, C.c_float, _i]
        L.rfo_render_icp_list.argtypes = [vp, _f, _i, _f, _f, _i, C.c_int, _f, _f, _f]
        L.rfo_set_threads.argtypes = [C.c_int]
        L.rfo_total_entries.argtypes = [vp]
        L.rfo_total_entries.restype = C.c_uint32
        L.rfo_export_entries.argtypes = [vp, _i]
        L.rfo_export_blocks.argtypes = [vp, _i, C.c_int, _u8]
        L.rfo_export_visible.argtypes = [vp, _i, _u8]
        L.rfo_free_counts.argtypes = [vp, _i, _i]
        _lib = L
    return _lib


def set_threads(n: int | None = None):
    """Threads for the oracle's per-pixel raycast (default 1; results do not
    depend on it).  None = every core of this host."""
    lib().rfo_set_threads(int(n if n else (os.cpu_count() or 1)))


def hash_index(pos, mask):
    p = np.ascontiguousarray(pos, np.int32)
    return lib().rfo_hash_index(P(p, _i), mask)


def traverse_blocks(a, b, max_cells=256):
    out = np.zeros((max_cells, 3), np.int32)
    a, b = _f32(a), _f32(b)
    n = lib().rfo_traverse_blocks(P(a, _f), P(b, _f), P(out, _i), max_cells)
    return out[:min(n, max_cells)].copy()


def block_in_frustum(pos, pose34, intr, params):
    p = np.ascontiguousarray(pos, np.int32)
    pose = _f32(pose34)
    pv = params_vec(params)
    wh, f4 = _wh(intr), _f4(intr)
    return bool(lib().rfo_block_in_frustum(P(p, _i), P(pose, _f), P(wh, _i), P(f4, _f), P(pv, _f)))


def build_view(raw, intr, aff=(1.0 / 5000.0, 0.0), levels=1):
    w, h = intr["width"], intr["height"]
    sizes = [(w >> l) * (h >> l) for l in range(levels)]
    out = np.zeros(sum(sizes), np.float32)
    raw = np.ascontiguousarray(raw, np.uint16)
    wh = _wh(intr)
    lib().rfo_build_view(P(raw, _u16), P(wh, _i), aff[0], aff[1], levels, P(out, _f))
    res, o = [], 0
    for l, s in enumerate(sizes):
        res.append(out[o:o + s].reshape(h >> l, w >> l))
        o += s
    return res


def mc_table():
    cnt = np.zeros(256, np.int32)
    tri = np.zeros(256 * 16 * 3, np.int32)
    lib().rfo_mc_table(P(cnt, _i), P(tri, _i))
    tri = tri.reshape(256, 16, 3)
    return [[tuple(int(x) for x in tri[m, k]) for k in range(cnt[m])] for m in range(256)]


def build_view_full(raw, intr, aff=(1.0 / 5000.0, 0.0), levels=3, bilateral=False, rgb=None):
    """rfo_build_view_full (view.cpp:100-143 with every option)."""
    L = lib()

    def fn(raw_p, rgb_p, wh_p, f4_p, s, o, b, lv, dep_p, it_p, n_p):
        return L.rfo_build_view_full(raw_p, rgb_p, wh_p, f4_p, s, o, b, lv, dep_p, it_p, n_p)
    return _view_full(fn, raw, rgb, intr, aff, levels, bilateral)


def bilateral_filter(depth, spatial_sigma, range_sigma):
    d = _f32(depth)
    out = np.zeros_like(d)
    lib().rfo_bilateral_filter(P(d, _f), d.shape[1], d.shape[0], spatial_sigma, range_sigma, P(out, _f))
    return out


def compute_normals(depth, intr):
    d = _f32(depth)
    out = np.zeros(d.shape + (4,), np.float32)
    lib().rfo_compute_normals(P(d, _f), d.shape[1], d.shape[0], P(_f4(intr), _f), P(out, _f))
    return out


def rgb_to_intensity(rgb):
    c = np.ascontiguousarray(rgb, np.uint8)
    out = np.zeros(c.shape[:2], np.float32)
    lib().rfo_rgb_to_intensity(P(c, _u8), c.shape[1], c.shape[0], P(out, _f))
    return out


def downsample_intensity(img):
    a = _f32(img)
    out = np.zeros((a.shape[0] // 2, a.shape[1] // 2), np.float32)
    lib().rfo_downsample_intensity(P(a, _f), a.shape[1], a.shape[0], P(out, _f))
    return out


ICP_STATS = ("iterations", "count", "residual_sum", "converged", "it_l0", "it_l1", "it_l2", "ok",
             "inlier_fraction", "hessian_det", "residual_mean", "valid")


def icp_track(levels_depth, intr, points, normals, render_pose34, render_intr, init_pose34,
              iters=(6, 10, 20), min_count=10, dist=(0.01, 0.02, 0.04)):
    """rfo_icp_track: (pose (3, 4) f32, stats (12,) f64 in ICP_STATS order)."""
    flat = np.ascontiguousarray(np.concatenate([d.reshape(-1) for d in levels_depth]), np.float32)
    wh, f4 = _wh(intr), _f4(intr)
    rf4 = _f4(render_intr)
    icp6 = np.array([len(levels_depth), iters[0], iters[1], iters[2], min_count, 0], np.int32)
    d3 = _f32(dist)
    out = np.zeros((3, 4), np.float32)
    stats = np.zeros(12, np.float64)
    pts, nrm = _f32(points), _f32(normals)
    rp, ip = _f32(render_pose34), _f32(init_pose34)
    rc = lib().rfo_icp_track(P(flat, _f), P(wh, _i), P(f4, _f), P(pts, _f), P(nrm, _f), P(rp, _f), P(rf4, _f),
                             P(ip, _f), P(icp6, _i), P(d3, _f), P(out, _f), P(stats, _d))
    if rc != 0:
        raise ValueError("icp_track: world point outside the fixed-point range (|p| >= 128 m)")
    return out, stats


def icp_reduce(depth_l, f4l, points, normals, intr, render_pose34, render_intr, cam_to_world34, dist,
               fixed=False):
    """One evaluation: the 31 sums decoded to float64 (fixed=False) or the raw
    int64 fixed-point sums (fixed=True)."""
    d = _f32(depth_l)
    lh, lw = d.shape
    f4l = _f32(f4l)
    out = np.zeros(31, np.float64)
    raw = np.zeros(31, np.int64)
    pts, nrm = _f32(points), _f32(normals)
    rp, c2w = _f32(render_pose34), _f32(cam_to_world34)
    wh, rf4 = _wh(intr), _f4(render_intr)
    lib().rfo_icp_reduce(P(d, _f), lw, lh, P(f4l, _f), P(pts, _f), P(nrm, _f), P(wh, _i), P(rp, _f), P(rf4, _f),
                         P(c2w, _f), dist, raw.ctypes.data_as(C.POINTER(C.c_int64)), P(out, _d))
    return raw if fixed else out


def se3_coeffs(th2):
    out = np.zeros(3, np.float64)
    lib().rfo_se3_coeffs(float(th2), P(out, _d))
    return out


def solve6(sums31):
    """rfo_solve6: (ok, delta (6,), det(H/n))."""
    s = np.ascontiguousarray(sums31, np.float64)
    x = np.zeros(6, np.float64)
    det = np.zeros(1, np.float64)
    rc = lib().rfo_solve6(P(s, _d), P(x, _d), P(det, _d))
    return rc == 0, x, float(det[0])


def forward_project(has_raycast, raycast, points, normals, pose34, intr, voxel_size):
    """forward_project (raycast.cpp:141-188) on caller-owned (H, W, 4) images,
    updated in place; returns the (N, 2) int32 missing (x, y) list."""
    out = np.zeros((intr["width"] * intr["height"], 2), np.int32)
    pose = _f32(pose34)
    wh, f4 = _wh(intr), _f4(intr)
    for a in (raycast, points, normals):
        assert a.dtype == np.float32 and a.flags.c_contiguous
    n = lib().rfo_forward_project(1 if has_raycast else 0, P(raycast, _f), P(points, _f), P(normals, _f),
                                  P(pose, _f), P(wh, _i), P(f4, _f), voxel_size, P(out, _i))
    return out[:n].copy()


class OracleEngine:
    """C restatement of VoxelBlockMap + FusionEngine + RenderState."""

    def __init__(self, buckets, excess, capacity):
        self.h = lib().rfo_create(buckets, excess, capacity)
        if not self.h:
            raise ValueError("bucketCount must be a power of two")
        self.capacity = capacity

    def __del__(self):
        if getattr(self, "sw", None):
            lib().rfo_swap_destroy(self.sw)
            self.sw = None
        if getattr(self, "h", None):
            lib().rfo_destroy(self.h)
            self.h = None

    def set_shard(self, rank, world, tile_shift=3):
        lib().rfo_set_shard(self.h, rank, world, tile_shift)

    def allocate(self, depth, intr, pose34, params):
        stats = np.zeros(4, np.int32)
        d, pose, pv = _f32(depth), _f32(pose34), params_vec(params)
        wh, f4 = _wh(intr), _f4(intr)
        lib().rfo_allocate(self.h, P(d, _f), P(wh, _i), P(f4, _f), P(pose, _f), P(pv, _f), P(stats, _i))
        return stats, 0.0

    def integrate(self, depth, intr, pose34, params, rgb=None, intr_rgb=None, extr34=None):
        d, pose, pv = _f32(depth), _f32(pose34), params_vec(params)
        wh, f4 = _wh(intr), _f4(intr)
        whr = _wh(intr_rgb) if intr_rgb else None
        f4r = _f4(intr_rgb) if intr_rgb else None
        ex = _f32(extr34) if extr34 is not None else None
        c = np.ascontiguousarray(rgb, np.uint8) if rgb is not None else None
        lib().rfo_integrate(self.h, P(d, _f), P(c, _u8), P(wh, _i), P(f4, _f), P(whr, _i), P(f4r, _f), P(ex, _f),
                            P(pose, _f), P(pv, _f))
        return 0.0

    def render_ranges(self, pose34, intr, params):
        rng = np.zeros((intr["height"], intr["width"], 2), np.float32)
        pose, pv = _f32(pose34), params_vec(params)
        wh, f4 = _wh(intr), _f4(intr)
        lib().rfo_render_ranges(self.h, P(pose, _f), P(wh, _i), P(f4, _f), P(pv, _f), P(rng, _f))
        return rng, 0.0

    def set_ranges(self, intr, rng):
        wh = _wh(intr)
        r = _f32(rng)
        lib().rfo_set_ranges(self.h, P(wh, _i), P(r, _f))

    def render_icp(self, pose34, intr, params):
        h, w = intr["height"], intr["width"]
        rc = np.zeros((h, w, 4), np.float32)
        pts = np.zeros((h, w, 4), np.float32)
        nrm = np.zeros((h, w, 4), np.float32)
        pose, pv = _f32(pose34), params_vec(params)
        wh, f4 = _wh(intr), _f4(intr)
        rc_ = lib().rfo_render_icp(self.h, P(pose, _f), P(wh, _i), P(f4, _f), P(pv, _f), P(rc, _f), P(pts, _f),
                                   P(nrm, _f))
        if rc_ != 0:
            raise RuntimeError("render_icp before render_ranges")
        return rc, pts, nrm, 0.0

    def set_fusion_options(self, swapping_enabled, swap_margin_px=8.0):
        lib().rfo_set_fusion_options(self.h, 1 if swapping_enabled else 0, swap_margin_px)

    def reserve_block(self, idx):
        return lib().rfo_reserve_block(self.h, idx)

    def release_block(self, idx):
        lib().rfo_release_block(self.h, idx)

    def swap_create(self, capacity):
        self.sw = lib().rfo_swap_create(self.h, capacity)

    def swap_in(self, max_w=100):
        return lib().rfo_swap_in(self.h, self.sw, max_w)

    def swap_out(self):
        return lib().rfo_swap_out(self.h, self.sw)

    def swap_stored(self):
        n = lib().rfo_total_entries(self.h)
        has, age = np.zeros(n, np.uint8), np.zeros(n, np.uint8)
        lib().rfo_swap_export(self.sw, n, P(has, _u8), P(age, _u8))
        return has, age

    def swap_host_block(self, idx):
        out = np.zeros((512, 8), np.uint8)
        lib().rfo_swap_host_block(self.sw, idx, P(out, _u8))
        return out

    def extract_mesh(self, voxel_size):
        """rfo_extract_mesh (meshing.cpp:144-217): (vertices (N,3) f32, triangles (M,3) u32)."""
        vp_, tp_ = C.POINTER(C.c_float)(), C.POINTER(C.c_uint32)()
        nv, nt = C.c_longlong(0), C.c_longlong(0)
        lib().rfo_extract_mesh(self.h, voxel_size, C.byref(vp_), C.byref(tp_), C.byref(nv), C.byref(nt))
        v = np.ctypeslib.as_array(vp_, shape=(max(nv.value, 1) * 3,))[: nv.value * 3].reshape(-1, 3).copy()
        t = np.ctypeslib.as_array(tp_, shape=(max(nt.value, 1) * 3,))[: nt.value * 3].reshape(-1, 3).copy()
        lib().rfo_free(C.cast(vp_, C.c_void_p))
        lib().rfo_free(C.cast(tp_, C.c_void_p))
        return v, t

    def set_block(self, pos3, sdf512, w512):
        p = np.ascontiguousarray(pos3, np.int32)
        sd = np.ascontiguousarray(sdf512, np.int16)
        w = np.ascontiguousarray(w512, np.uint8)
        return lib().rfo_set_block(self.h, P(p, _i), P(sd, C.POINTER(C.c_int16)), P(w, _u8))

    def render_colour(self, mode, pose34, intr, raycast, normals, missing=None, out=None):
        """The colour image of render_maps(kColour = 1 / kGrey = 2) from the
        maps of the same render (raycast.hpp:169,191-197); with `missing`
        (pixel indices) only those pixels are (re)written, in `out`."""
        h, w = intr["height"], intr["width"]
        col = out if out is not None else np.zeros((h, w, 3), np.uint8)
        ls = np.ascontiguousarray(missing, np.int32) if missing is not None else None
        lib().rfo_render_colour(self.h, mode, P(_f32(pose34), _f), P(_wh(intr), _i), P(_f4(intr), _f),
                                P(_f32(raycast), _f), P(_f32(normals), _f), P(ls, _i), 0 if ls is None else len(ls),
                                P(col, _u8))
        return col

    def render_icp_list(self, pose34, intr, params, missing, raycast, points, normals):
        """render_maps(kIcpMaps, missingOnly) on caller-owned images (in place)."""
        pose, pv = _f32(pose34), params_vec(params)
        wh, f4 = _wh(intr), _f4(intr)
        ms = np.ascontiguousarray(missing, np.int32)
        rc_ = lib().rfo_render_icp_list(self.h, P(pose, _f), P(wh, _i), P(f4, _f), P(pv, _f), P(ms, _i), len(ms),
                                        P(raycast, _f), P(points, _f), P(normals, _f))
        if rc_ != 0:
            raise RuntimeError("render_icp_list before render_ranges")

    def entries(self):
        n = lib().rfo_total_entries(self.h)
        out = np.zeros((n, 5), np.int32)
        lib().rfo_export_entries(self.h, P(out, _i))
        return out

    def blocks(self, ptrs):
        ptrs = np.ascontiguousarray(ptrs, np.int32)
        out = np.zeros((len(ptrs), 512, 8), np.uint8)
        if len(ptrs):
            lib().rfo_export_blocks(self.h, P(ptrs, _i), len(ptrs), P(out, _u8))
        return out

    def visible(self):
        n = lib().rfo_total_entries(self.h)
        lst = np.zeros(n, np.int32)
        types = np.zeros(n, np.uint8)
        k = lib().rfo_export_visible(self.h, P(lst, _i), P(types, _u8))
        return lst[:k].copy(), types

    def free_counts(self):
        nb, ne = C.c_int(0), C.c_int(0)
        lib().rfo_free_counts(self.h, C.byref(nb), C.byref(ne))
        return nb.value, ne.value
