"""ctypes wrapper over oracle/_ref/librfref.so — TEST INFRASTRUCTURE ONLY.

librfref.so is the UNMODIFIED reference library (/root/reference/proj/src)
compiled against oracle/shim/ plus oracle/ref_driver.cpp.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / reference arm may use it.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "librfref.so")

_f = C.POINTER(C.c_float)
_i = C.POINTER(C.c_int)
_u8 = C.POINTER(C.c_uint8)
_u16 = C.POINTER(C.c_uint16)
_d = C.POINTER(C.c_double)

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.rr_orbit_poses.argtypes = [_f, C.c_float, C.c_int, C.c_float, _f]
        L.rr_render.argtypes = [C.c_int, _f, _i, _f, C.c_float, C.c_float, C.c_int, _u16, _f, _u8]
        L.rr_scene_sdf.argtypes = [C.c_int, _f]
        L.rr_scene_sdf.restype = C.c_float
        L.rr_build_view.argtypes = [_u16, _i, _f, C.c_float, C.c_float, C.c_int, _f]
        L.rr_hash_index.argtypes = [_i, C.c_uint32]
        L.rr_hash_index.restype = C.c_uint32
        L.rr_traverse_blocks.argtypes = [_f, _f, _i, C.c_int]
        L.rr_block_in_frustum.argtypes = [_i, _f, _i, _f, _f]
        L.rr_update_voxel_depth.argtypes = [_u8, _f, _f, _i, _f, C.c_float, C.c_int, _f, C.c_int]
        L.rr_update_voxel_depth.restype = C.c_float
        L.rr_create.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32]
        L.rr_create.restype = C.c_void_p
        L.rr_destroy.argtypes = [C.c_void_p]
        L.rr_allocate.argtypes = [C.c_void_p, _f, _i, _f, _f, _f, _i, _d]
        L.rr_integrate.argtypes = [C.c_void_p, _f, _u8, _i, _f, _i, _f, _f, _f, _f, _d]
        L.rr_render_ranges.argtypes = [C.c_void_p, _f, _i, _f, _f, _f, _d]
        L.rr_render_icp.argtypes = [C.c_void_p, _f, _i, _f, _f, _f, _f, _f, _d]
        L.rr_set_ranges.argtypes = [C.c_void_p, _i, _f, _f]
        L.rr_forward_project.argtypes = [C.c_void_p, _f, _i, _f, C.c_float, _i]
        L.rr_render_icp_missing.argtypes = [C.c_void_p, _f, _i, _f, _f, _i, C.c_int, _f, _f, _f]
        L.rr_total_entries.argtypes = [C.c_void_p]
        L.rr_total_entries.restype = C.c_uint32
        L.rr_export_entries.argtypes = [C.c_void_p, _i]
        L.rr_export_blocks.argtypes = [C.c_void_p, _i, C.c_int, _u8]
        L.rr_export_visible.argtypes = [C.c_void_p, _i, _u8]
        L.rr_free_counts.argtypes = [C.c_void_p, _i, _i]
        L.rr_set_fusion_options.argtypes = [C.c_void_p, C.c_int, C.c_float]
        L.rr_reserve_block.argtypes = [C.c_void_p, C.c_int]
        L.rr_release_block.argtypes = [C.c_void_p, C.c_int]
        L.rr_extract_mesh.argtypes = [C.c_void_p, C.c_float, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]
        L.rr_mesh_copy.argtypes = [C.c_void_p, _f, C.POINTER(C.c_uint32)]
        L.rr_mc_table.argtypes = [_i, _i]
        L.rr_set_block.argtypes = [C.c_void_p, _i, C.POINTER(C.c_int16), _u8]
        L.rr_render_maps.argtypes = [C.c_void_p, C.c_int, _f, _i, _f, _f, _f, _f, _f, _u8]
        L.rr_build_view_full.argtypes = [_u16, _u8, _i, _f, C.c_float, C.c_float, C.c_int, C.c_int, _f, _f, _f]
        L.rr_bilateral_filter.argtypes = [_f, C.c_int, C.c_int, C.c_float, C.c_float, _f]
        L.rr_compute_normals.argtypes = [_f, _i, _f, _f]
        L.rr_read_pgm16.argtypes = [C.c_char_p, _u16, C.c_int, _i, _i]
        L.rr_read_ppm.argtypes = [C.c_char_p, _u8, C.c_int, _i, _i]
        L.rr_write_pgm16.argtypes = [C.c_char_p, _u16, C.c_int, C.c_int]
        L.rr_write_ppm.argtypes = [C.c_char_p, _u8, C.c_int, C.c_int]
        _lib = L
    return _lib


def P(a, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _wh(intr):
    return np.array([intr["width"], intr["height"]], dtype=np.int32)


def _f4(intr):
    return np.array([intr["fx"], intr["fy"], intr["cx"], intr["cy"]], dtype=np.float32)


def params_vec(p) -> np.ndarray:
    return np.array([p["voxelSize"], p["mu"], p["maxW"], p["viewFrustum_min"], p["viewFrustum_max"],
                     1.0 if p.get("stopIntegratingAtMaxW", False) else 0.0], dtype=np.float32)


def orbit_poses(target, distance, frames, max_angle=0.5) -> np.ndarray:
    out = np.zeros((frames, 3, 4), np.float32)
    t = _f32(target)
    lib().rr_orbit_poses(P(t, _f), distance, frames, max_angle, P(out, _f))
    return out


def render(scene_kind, pose34, intr, aff=(1.0 / 5000.0, 0.0), rgb=False):
    w, h = intr["width"], intr["height"]
    raw = np.zeros((h, w), np.uint16)
    dep = np.zeros((h, w), np.float32)
    col = np.zeros((h, w, 3), np.uint8) if rgb else None
    pose = _f32(pose34)
    wh, f4 = _wh(intr), _f4(intr)
    lib().rr_render(scene_kind, P(pose, _f), P(wh, _i), P(f4, _f), aff[0], aff[1], 1 if rgb else 0,
                    P(raw, _u16), P(dep, _f), P(col, _u8))
    return raw, dep, col


def build_view(raw, intr, aff=(1.0 / 5000.0, 0.0), levels=1):
    w, h = intr["width"], intr["height"]
    sizes = [(w >> l) * (h >> l) for l in range(levels)]
    out = np.zeros(sum(sizes), np.float32)
    raw = np.ascontiguousarray(raw, np.uint16)
    wh, f4 = _wh(intr), _f4(intr)
    lib().rr_build_view(P(raw, _u16), P(wh, _i), P(f4, _f), aff[0], aff[1], levels, P(out, _f))
    res, o = [], 0
    for l, s in enumerate(sizes):
        res.append(out[o:o + s].reshape(h >> l, w >> l))
        o += s
    return res


def _view_full(fn, raw, rgb, intr, aff, levels, bilateral):
    w, h = intr["width"], intr["height"]
    sizes = [(w >> l) * (h >> l) for l in range(levels)]
    dep = np.zeros(sum(sizes), np.float32)
    inten = np.zeros(sum(sizes), np.float32) if rgb is not None else None
    nrm = np.zeros((h, w, 4), np.float32)
    raw = np.ascontiguousarray(raw, np.uint16)
    rgb = np.ascontiguousarray(rgb, np.uint8) if rgb is not None else None
    wh, f4 = _wh(intr), _f4(intr)
    rc = fn(P(raw, _u16), P(rgb, _u8), P(wh, _i), P(f4, _f), aff[0], aff[1], 1 if bilateral else 0, levels,
            P(dep, _f), P(inten, _f), P(nrm, _f))
    assert rc == 0
    d, it, o = [], [], 0
    for l, s in enumerate(sizes):
        d.append(dep[o:o + s].reshape(h >> l, w >> l))
        if inten is not None:
            it.append(inten[o:o + s].reshape(h >> l, w >> l))
        o += s
    return {"depth": d, "intensity": it if inten is not None else None, "normals": nrm}


def build_view_full(raw, intr, aff=(1.0 / 5000.0, 0.0), levels=3, bilateral=False, rgb=None):
    """build_view with every option (view.cpp:100-143): depth / intensity
    pyramids and level-0 normals."""
    return _view_full(lib().rr_build_view_full, raw, rgb, intr, aff, levels, bilateral)


def bilateral_filter(depth, spatial_sigma, range_sigma):
    d = _f32(depth)
    out = np.zeros_like(d)
    lib().rr_bilateral_filter(P(d, _f), d.shape[1], d.shape[0], spatial_sigma, range_sigma, P(out, _f))
    return out


def compute_normals(depth, intr):
    d = _f32(depth)
    out = np.zeros(d.shape + (4,), np.float32)
    wh, f4 = _wh(intr), _f4(intr)
    lib().rr_compute_normals(P(d, _f), P(wh, _i), P(f4, _f), P(out, _f))
    return out


# The reference's Netpbm IO goes through iostreams, which crash in a process
# that has numpy's C extension loaded (its bundled C++ runtime interferes);
# these four calls therefore run the reference in a numpy-free subprocess.
_IO_SCRIPT = r"""
import ctypes as C, sys
L = C.CDLL(sys.argv[1])
op, path, blob = sys.argv[2], sys.argv[3].encode(), sys.argv[4]
if op in ("rpgm", "rppm"):
    cap = 1 << 22
    elem = 2 if op == "rpgm" else 3
    buf = (C.c_uint8 * (cap * elem))()
    w, h = C.c_int(0), C.c_int(0)
    fn = L.rr_read_pgm16 if op == "rpgm" else L.rr_read_ppm
    rc = fn(path, buf, cap if op == "rpgm" else cap * 3, C.byref(w), C.byref(h))
    with open(blob, "wb") as f:
        f.write(rc.to_bytes(4, "little", signed=True) + w.value.to_bytes(4, "little") + h.value.to_bytes(4, "little"))
        if rc == 0:
            f.write(bytes(buf)[: w.value * h.value * elem])
else:
    w, h = int(sys.argv[5]), int(sys.argv[6])
    data = open(blob, "rb").read()
    buf = (C.c_uint8 * len(data)).from_buffer_copy(data)
    fn = L.rr_write_pgm16 if op == "wpgm" else L.rr_write_ppm
    sys.exit(0 if fn(path, buf, w, h) == 0 else 3)
"""


def _io(op, path, blob, *extra):
    import subprocess
    import sys
    r = subprocess.run([sys.executable, "-c", _IO_SCRIPT, LIB_PATH, op, path, blob, *map(str, extra)],
                       capture_output=True, text=True)
    return r.returncode


def _read(op, path, elem):
    import tempfile
    with tempfile.NamedTemporaryFile(suffix=".bin") as t:
        rc = _io(op, path, t.name)
        if rc != 0:
            raise RuntimeError(f"reference IO helper failed ({rc})")
        b = open(t.name, "rb").read()
    code = int.from_bytes(b[0:4], "little", signed=True)
    w, h = int.from_bytes(b[4:8], "little"), int.from_bytes(b[8:12], "little")
    if code != 0:
        return None
    if elem == 2:
        return np.frombuffer(b[12:], np.uint16).reshape(h, w).copy()
    return np.frombuffer(b[12:], np.uint8).reshape(h, w, 3).copy()


def read_pgm16(path):
    """The reference's read_pgm16 (None on its exception)."""
    return _read("rpgm", path, 2)


def read_ppm(path):
    return _read("rppm", path, 3)


def _write(op, img, path, dtype):
    import tempfile
    a = np.ascontiguousarray(img, dtype)
    with tempfile.NamedTemporaryFile(suffix=".bin") as t:
        t.write(a.tobytes())
        t.flush()
        return 0 if _io(op, path, t.name, a.shape[1], a.shape[0]) == 0 else -1


def write_pgm16(img, path):
    return _write("wpgm", img, path, np.uint16)


def write_ppm(img, path):
    return _write("wppm", img, path, np.uint8)


def mc_table():
    """detail::marchingCubesTable(): list of lists of edge triples."""
    cnt = np.zeros(256, np.int32)
    tri = np.zeros(256 * 16 * 3, np.int32)
    lib().rr_mc_table(P(cnt, _i), P(tri, _i))
    tri = tri.reshape(256, 16, 3)
    return [[tuple(int(x) for x in tri[m, k]) for k in range(cnt[m])] for m in range(256)]


class RefEngine:
    """VoxelBlockMap + FusionEngine + RenderState of the reference."""

    def __init__(self, buckets, excess, capacity):
        self.h = lib().rr_create(buckets, excess, capacity)
        if not self.h:
            raise ValueError("reference rejected the map config")
        self.capacity = capacity

    def __del__(self):
        if getattr(self, "h", None):
            lib().rr_destroy(self.h)
            self.h = None

    def allocate(self, depth, intr, pose34, params):
        stats = np.zeros(4, np.int32)
        ms = C.c_double(0)
        d = _f32(depth)
        pose = _f32(pose34)
        pv = params_vec(params)
        wh, f4 = _wh(intr), _f4(intr)
        lib().rr_allocate(self.h, P(d, _f), P(wh, _i), P(f4, _f), P(pose, _f), P(pv, _f), P(stats, _i), C.byref(ms))
        return stats, ms.value

    def integrate(self, depth, intr, pose34, params, rgb=None, intr_rgb=None, extr34=None):
        ms = C.c_double(0)
        d = _f32(depth)
        pose = _f32(pose34)
        pv = params_vec(params)
        wh, f4 = _wh(intr), _f4(intr)
        whr = _wh(intr_rgb) if intr_rgb else None
        f4r = _f4(intr_rgb) if intr_rgb else None
        ex = _f32(extr34) if extr34 is not None else None
        c = np.ascontiguousarray(rgb, np.uint8) if rgb is not None else None
        lib().rr_integrate(self.h, P(d, _f), P(c, _u8), P(wh, _i), P(f4, _f), P(whr, _i), P(f4r, _f), P(ex, _f),
                           P(pose, _f), P(pv, _f), C.byref(ms))
        return ms.value

    def render_ranges(self, pose34, intr, params):
        rng = np.zeros((intr["height"], intr["width"], 2), np.float32)
        ms = C.c_double(0)
        pose = _f32(pose34)
        pv = params_vec(params)
        wh, f4 = _wh(intr), _f4(intr)
        lib().rr_render_ranges(self.h, P(pose, _f), P(wh, _i), P(f4, _f), P(pv, _f), P(rng, _f), C.byref(ms))
        return rng, ms.value

    def set_ranges(self, intr, rng):
        wh, f4 = _wh(intr), _f4(intr)
        r = _f32(rng)
        lib().rr_set_ranges(self.h, P(wh, _i), P(f4, _f), P(r, _f))

    def set_fusion_options(self, swapping_enabled, swap_margin_px=8.0):
        lib().rr_set_fusion_options(self.h, 1 if swapping_enabled else 0, swap_margin_px)

    def reserve_block(self, idx):
        return lib().rr_reserve_block(self.h, idx)

    def release_block(self, idx):
        lib().rr_release_block(self.h, idx)

    def extract_mesh(self, voxel_size):
        """extract_mesh (meshing.cpp:144-217): (vertices (N,3) f32, triangles (M,3) u32)."""
        nv, nt = C.c_longlong(0), C.c_longlong(0)
        lib().rr_extract_mesh(self.h, voxel_size, C.byref(nv), C.byref(nt))
        v = np.zeros((nv.value, 3), np.float32)
        t = np.zeros((nt.value, 3), np.uint32)
        lib().rr_mesh_copy(self.h, P(v, _f), P(t, C.POINTER(C.c_uint32)))
        return v, t

    def set_block(self, pos3, sdf512, w512):
        p = np.ascontiguousarray(pos3, np.int32)
        sd = np.ascontiguousarray(sdf512, np.int16)
        w = np.ascontiguousarray(w512, np.uint8)
        return lib().rr_set_block(self.h, P(p, _i), P(sd, C.POINTER(C.c_int16)), P(w, _u8))

    def render_maps(self, mode, pose34, intr, params):
        """render_maps with RenderMode 0 kIcpMaps / 1 kColour / 2 kGrey:
        (raycast, points, normals, colour RGB8)."""
        h, w = intr["height"], intr["width"]
        rc = np.zeros((h, w, 4), np.float32)
        pts = np.zeros((h, w, 4), np.float32)
        nrm = np.zeros((h, w, 4), np.float32)
        col = np.zeros((h, w, 3), np.uint8)
        pose, pv = _f32(pose34), params_vec(params)
        wh, f4 = _wh(intr), _f4(intr)
        lib().rr_render_maps(self.h, mode, P(pose, _f), P(wh, _i), P(f4, _f), P(pv, _f), P(rc, _f), P(pts, _f),
                             P(nrm, _f), P(col, _u8))
        return rc, pts, nrm, col

    def render_icp(self, pose34, intr, params):
        h, w = intr["height"], intr["width"]
        rc = np.zeros((h, w, 4), np.float32)
        pts = np.zeros((h, w, 4), np.float32)
        nrm = np.zeros((h, w, 4), np.float32)
        ms = C.c_double(0)
        pose = _f32(pose34)
        pv = params_vec(params)
        wh, f4 = _wh(intr), _f4(intr)
        lib().rr_render_icp(self.h, P(pose, _f), P(wh, _i), P(f4, _f), P(pv, _f), P(rc, _f), P(pts, _f),
                            P(nrm, _f), C.byref(ms))
        return rc, pts, nrm, ms.value

    def forward_project(self, pose34, intr, voxel_size):
        """forward_project (raycast.cpp:141-188): (N, 2) int32 missing (x, y)."""
        out = np.zeros((intr["width"] * intr["height"], 2), np.int32)
        pose = _f32(pose34)
        wh, f4 = _wh(intr), _f4(intr)
        n = lib().rr_forward_project(self.h, P(pose, _f), P(wh, _i), P(f4, _f), voxel_size, P(out, _i))
        return out[:n].copy()

    def render_icp_missing(self, pose34, intr, params, missing):
        h, w = intr["height"], intr["width"]
        rc = np.zeros((h, w, 4), np.float32)
        pts = np.zeros((h, w, 4), np.float32)
        nrm = np.zeros((h, w, 4), np.float32)
        pose, pv = _f32(pose34), params_vec(params)
        wh, f4 = _wh(intr), _f4(intr)
        ms = np.ascontiguousarray(missing, np.int32)
        lib().rr_render_icp_missing(self.h, P(pose, _f), P(wh, _i), P(f4, _f), P(pv, _f), P(ms, _i), len(ms),
                                    P(rc, _f), P(pts, _f), P(nrm, _f))
        return rc, pts, nrm

    def entries(self):
        n = lib().rr_total_entries(self.h)
        out = np.zeros((n, 5), np.int32)
        lib().rr_export_entries(self.h, P(out, _i))
        return out

    def blocks(self, ptrs):
        ptrs = np.ascontiguousarray(ptrs, np.int32)
        out = np.zeros((len(ptrs), 512, 8), np.uint8)
        if len(ptrs):
            lib().rr_export_blocks(self.h, P(ptrs, _i), len(ptrs), P(out, _u8))
        return out

    def visible(self):
        n = lib().rr_total_entries(self.h)
        lst = np.zeros(n, np.int32)
        types = np.zeros(n, np.uint8)
        k = lib().rr_export_visible(self.h, P(lst, _i), P(types, _u8))
        return lst[:k].copy(), types

    def free_counts(self):
        nb, ne = C.c_int(0), C.c_int(0)
        lib().rr_free_counts(self.h, C.byref(nb), C.byref(ne))
        return nb.value, ne.value
