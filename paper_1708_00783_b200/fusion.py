"""Host API mirroring the reference's engine interface (rf:: namespace of
/root/reference/proj) on top of the librfg.so C ABI.

Names, argument meaning and error behaviour follow the reference so parity
tests read like its own tests:

  VoxelBlockMapConfig / VoxelBlockMap      proj/include/rf/voxel_block_map.hpp:36-144
  SceneParams / AllocationStats            proj/include/rf/fusion.hpp:11-27
  FusionEngine.allocate_from_depth /
               integrate_frame             proj/include/rf/fusion.hpp:52-79
  RenderState / render_expected_ranges /
  render_maps(RenderMode.kIcpMaps)         proj/include/rf/raycast.hpp:15-129
  build_view (depth + pyramid)             proj/include/rf/view.hpp:38-39
  track_depth (ICP)                        SPEC.md:348-356 (absent in the reference)

Images live on the GPU as torch tensors (torch is the device-memory and
stream plumbing); every computation runs in librfg's sm_100a kernels.
Poses are (3, 4) float32 arrays [R | t], world -> camera.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import check, lib

_f = C.POINTER(C.c_float)
_d = C.POINTER(C.c_double)
_i = C.POINTER(C.c_int32)
_u8 = C.POINTER(C.c_uint8)
_u16 = C.POINTER(C.c_uint16)


def _fp(a: np.ndarray):
    return a.ctypes.data_as(_f)


def _pose(p) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(p, dtype=np.float32).reshape(3, 4))
    return a


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("device tensor expected (librfg has no CPU path)")
    if not t.is_contiguous():
        raise ValueError("contiguous tensor expected")
    return C.c_void_p(t.data_ptr())


def _stream_handle():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


# ---------------------------------------------------------------- config
@dataclass
class Intrinsics:
    """proj/include/rf/camera.hpp:13-47"""
    width: int = 0
    height: int = 0
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0

    def atLevel(self, level: int) -> "Intrinsics":
        s = float(np.ldexp(np.float32(1.0), -level))
        return Intrinsics(self.width >> level, self.height >> level, float(np.float32(self.fx) * np.float32(s)),
                          float(np.float32(self.fy) * np.float32(s)), float(np.float32(self.cx) * np.float32(s)),
                          float(np.float32(self.cy) * np.float32(s)))

    def c(self) -> _lib.Intrinsics_:
        return _lib.Intrinsics_(self.width, self.height, self.fx, self.fy, self.cx, self.cy)

    def as_dict(self):
        return dict(width=self.width, height=self.height, fx=self.fx, fy=self.fy, cx=self.cx, cy=self.cy)


@dataclass
class DepthAffine:
    """proj/include/rf/camera.hpp:50-62 (m = raw*scale + offset)"""
    scale: float = 1.0 / 1000.0
    offset: float = 0.0


@dataclass
class RgbdCalib:
    """proj/include/rf/camera.hpp:64-69"""
    intrinsics_rgb: Intrinsics = field(default_factory=Intrinsics)
    intrinsics_d: Intrinsics = field(default_factory=Intrinsics)
    extrinsics_d_to_rgb: np.ndarray = field(default_factory=lambda: np.eye(3, 4, dtype=np.float32))
    depth_affine: DepthAffine = field(default_factory=DepthAffine)


@dataclass
class SceneParams:
    """proj/include/rf/fusion.hpp:11-20"""
    voxelSize: float = 0.005
    mu: float = 0.02
    maxW: int = 100
    viewFrustum_min: float = 0.2
    viewFrustum_max: float = 6.0
    stopIntegratingAtMaxW: bool = False

    def blockSizeMetres(self) -> float:
        return float(np.float32(self.voxelSize) * np.float32(8))

    def c(self) -> _lib.SceneParams_:
        return _lib.SceneParams_(self.voxelSize, self.mu, self.maxW, self.viewFrustum_min, self.viewFrustum_max,
                                 1 if self.stopIntegratingAtMaxW else 0)

    def as_dict(self):
        return dict(voxelSize=self.voxelSize, mu=self.mu, maxW=self.maxW, viewFrustum_min=self.viewFrustum_min,
                    viewFrustum_max=self.viewFrustum_max, stopIntegratingAtMaxW=self.stopIntegratingAtMaxW)


@dataclass
class VoxelBlockMapConfig:
    """proj/include/rf/voxel_block_map.hpp:36-45"""
    bucketCount: int = 1 << 20
    excessCount: int = 1 << 17
    blockCapacity: int = 1 << 18

    @staticmethod
    def small() -> "VoxelBlockMapConfig":
        return VoxelBlockMapConfig(1 << 14, 1 << 11, 1 << 13)


@dataclass
class AllocationStats:
    """proj/include/rf/fusion.hpp:22-27"""
    requested: int = 0
    allocated: int = 0
    allocFailures: int = 0
    visibleCount: int = 0

    def as_array(self):
        return np.array([self.requested, self.allocated, self.allocFailures, self.visibleCount], np.int32)


class Visibility(enum.IntEnum):
    """proj/include/rf/voxel_block_map.hpp:29-34"""
    kInvisible = 0
    kVisible = 1
    kVisibleSwapped = 2
    kBoundary = 3


class RenderMode(enum.IntEnum):
    """proj/include/rf/raycast.hpp:28"""
    kIcpMaps = 0
    kColour = 1
    kGrey = 2


# ------------------------------------------------------------------ map
class VoxelBlockMap:
    """Device-resident hashed TSDF (ordered buckets + excess list over a voxel
    block array).  Raises ValueError for a non-power-of-two bucketCount, like
    the reference constructor (proj/src/voxel_block_map.cpp:9-13)."""

    def __init__(self, config: VoxelBlockMapConfig | None = None, device: int = 0, colour: bool = False):
        self._h = None
        cfg = config or VoxelBlockMapConfig.small()
        self._config = cfg
        self.device = device
        self.colour = colour
        c = _lib.MapConfig(cfg.bucketCount, cfg.excessCount, cfg.blockCapacity, 1 if colour else 0)
        h = C.c_void_p()
        rc = lib().rfg_map_create(C.byref(c), device, C.byref(h))
        if rc == _lib.RFG_EINVAL:
            raise ValueError(lib().rfg_last_error().decode())
        check(rc)
        self._h = h

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib._lib is not None:
                _lib._lib.rfg_map_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown: module globals may be gone
            pass

    @property
    def handle(self):
        return self._h

    def config(self) -> VoxelBlockMapConfig:
        return self._config

    def bucketCount(self) -> int:
        return self._config.bucketCount

    def totalEntries(self) -> int:
        return self._config.bucketCount + self._config.excessCount

    def hashMask(self) -> int:
        return self._config.bucketCount - 1

    def bind_stream(self):
        check(lib().rfg_map_set_stream(self._h, _stream_handle()))

    def clear(self):
        self.bind_stream()
        check(lib().rfg_map_clear(self._h))

    def set_shard(self, rank: int, world: int, tile_shift: int = 3):
        check(lib().rfg_map_set_shard(self._h, rank, world, tile_shift))

    def sync(self):
        check(lib().rfg_map_sync(self._h))

    # -- parity exports (host copies) --
    def reserveBlockForEntry(self, idx: int) -> bool:
        """voxel_block_map.cpp:107-116"""
        self.bind_stream()
        rc = lib().rfg_map_reserve_block(self._h, idx)
        if rc < 0:
            check(rc)
        return rc == 1

    def releaseBlock(self, idx: int) -> None:
        """voxel_block_map.cpp:118-123"""
        self.bind_stream()
        check(lib().rfg_map_release_block(self._h, idx))

    def entries(self) -> np.ndarray:
        """(totalEntries, 5) int32 {x, y, z, offset, ptr}"""
        out = np.zeros((self.totalEntries(), 5), np.int32)
        check(lib().rfg_export_entries(self._h, out.ctypes.data_as(_i)))
        return out

    def blocks(self, ptrs) -> np.ndarray:
        """(n, 512, 8) uint8 VoxelSRgb bytes of the given VBA blocks"""
        ptrs = np.ascontiguousarray(ptrs, np.int32)
        out = np.zeros((len(ptrs), 512, 8), np.uint8)
        check(lib().rfg_export_blocks(self._h, ptrs.ctypes.data_as(_i), len(ptrs), out.ctypes.data_as(_u8)))
        return out

    def visible(self):
        n = C.c_int32(0)
        lst = np.zeros(self.totalEntries(), np.int32)
        types = np.zeros(self.totalEntries(), np.uint8)
        check(lib().rfg_export_visible(self._h, lst.ctypes.data_as(_i), types.ctypes.data_as(_u8), C.byref(n)))
        return lst[:n.value].copy(), types

    def visibleList(self) -> np.ndarray:
        return self.visible()[0]

    def visibilityTypes(self) -> np.ndarray:
        return self.visible()[1]

    def free_counts(self):
        nb, ne = C.c_int32(0), C.c_int32(0)
        check(lib().rfg_free_counts(self._h, C.byref(nb), C.byref(ne)))
        return nb.value, ne.value

    def freeBlockCount(self) -> int:
        return self.free_counts()[0]

    def freeExcessCount(self) -> int:
        return self.free_counts()[1]

    def allocatedBlockCount(self) -> int:
        return self._config.blockCapacity - self.freeBlockCount()


# ------------------------------------------------------------------ view
@dataclass
class ViewBuildOptions:
    """proj/include/rf/view.hpp:12-15."""
    bilateral: bool = False
    levels: int = 3


@dataclass
class ViewLevel:
    depth: torch.Tensor
    intr: Intrinsics
    intensity: torch.Tensor | None = None


@dataclass
class View:
    """proj/include/rf/view.hpp:24-34 (device images)."""
    calib: RgbdCalib
    depth_m: torch.Tensor
    rgb: torch.Tensor | None = None
    pyramid: list = field(default_factory=list)
    intensity: torch.Tensor | None = None
    normals: torch.Tensor | None = None  # (H, W, 4) camera-frame unit normals, w < 0 invalid

    def hasColour(self) -> bool:
        return self.rgb is not None


def _u16_tensor(raw):
    t = torch.as_tensor(raw) if torch.is_tensor(raw) else None
    if t is None or (t.dtype != torch.uint16 and t.dtype != torch.int16):
        t = torch.as_tensor(np.ascontiguousarray(np.asarray(raw, dtype=np.uint16)).view(np.int16))
    return t


def _rgb_tensor(rgb):
    if rgb is None:
        return None
    return torch.as_tensor(np.ascontiguousarray(rgb, dtype=np.uint8)).cuda() if not torch.is_tensor(rgb) \
        else rgb.cuda().contiguous()


def build_view(raw_depth, rgb, calib: RgbdCalib, opts: ViewBuildOptions | int | None = None, *,
               levels: int | None = None, big_endian: bool = False) -> View:
    """build_view (proj/src/view.cpp:100-143) on the GPU with every option:
    depth conversion, optional bilateral filter, level-0 normals, intensity
    (when rgb is given) and the depth / intensity pyramids.  raw_depth:
    (H, W) uint16 (numpy or CUDA tensor; big_endian=True for a PGM16 payload,
    see read_pgm16_payload).  Raises ValueError on a size mismatch or
    levels < 1, like the reference (view.cpp:102-106)."""
    if isinstance(opts, int):  # build_view(raw, rgb, calib, levels)
        opts = ViewBuildOptions(levels=opts)
    opts = opts or ViewBuildOptions()
    if levels is not None:
        opts = ViewBuildOptions(bilateral=opts.bilateral, levels=levels)
    intr = calib.intrinsics_d
    raw = _u16_tensor(raw_depth)
    if tuple(raw.shape) != (intr.height, intr.width):
        raise ValueError("build_view: depth image size does not match calibration")
    if rgb is not None and tuple(rgb.shape[:2]) != (calib.intrinsics_rgb.height, calib.intrinsics_rgb.width):
        raise ValueError("build_view: rgb image size does not match calibration")
    if opts.levels < 1:
        raise ValueError("build_view: levels must be >= 1")
    raw = raw.cuda().contiguous()
    rgb_t = _rgb_tensor(rgb)
    # intensity is defined on the depth grid (view.cpp:126-141 pairs
    # pyramid[0].intensity with the depth intrinsics)
    inten = rgb_t is not None and (calib.intrinsics_rgb.width, calib.intrinsics_rgb.height) == (intr.width, intr.height)
    sizes = [(intr.width >> l) * (intr.height >> l) for l in range(opts.levels)]
    dev = raw.device
    buf = torch.empty(sum(sizes), dtype=torch.float32, device=dev)
    ibuf = torch.empty(sum(sizes), dtype=torch.float32, device=dev) if inten else None
    normals = torch.empty((intr.height, intr.width, 4), dtype=torch.float32, device=dev)
    scratch = torch.empty(intr.width * intr.height, dtype=torch.float32, device=dev) if opts.bilateral else None
    check(lib().rfg_build_view(_ptr(raw), _ptr(rgb_t) if inten else None, C.byref(intr.c()),
                               calib.depth_affine.scale, calib.depth_affine.offset, 1 if opts.bilateral else 0,
                               opts.levels, 1 if big_endian else 0, _ptr(buf), _ptr(ibuf) if inten else None,
                               _ptr(normals), _ptr(scratch) if scratch is not None else None, _stream_handle()))
    pyr, o = [], 0
    for l, s in enumerate(sizes):
        il = intr.atLevel(l)
        pyr.append(ViewLevel(buf[o:o + s].view(il.height, il.width), il,
                             ibuf[o:o + s].view(il.height, il.width) if inten else None))
        o += s
    return View(calib=calib, depth_m=pyr[0].depth, rgb=rgb_t, pyramid=pyr,
                intensity=pyr[0].intensity, normals=normals)


def bilateral_filter(depth_m, spatial_sigma: float, range_sigma: float) -> torch.Tensor:
    """bilateral_filter (view.cpp:18-44): 5x5 edge-preserving filter, bit-exact
    including the reference's std::exp (glibc expf, reproduced on the GPU)."""
    d = torch.as_tensor(depth_m, dtype=torch.float32).cuda().contiguous()
    out = torch.empty_like(d)
    check(lib().rfg_bilateral_filter(_ptr(d), d.shape[1], d.shape[0], spatial_sigma, range_sigma, _ptr(out),
                                     _stream_handle()))
    return out


def compute_normals(depth_m, intr: Intrinsics) -> torch.Tensor:
    """compute_normals (view.cpp:46-67): (H, W, 4), w < 0 invalid."""
    d = torch.as_tensor(depth_m, dtype=torch.float32).cuda().contiguous()
    out = torch.empty((d.shape[0], d.shape[1], 4), dtype=torch.float32, device=d.device)
    check(lib().rfg_compute_normals(_ptr(d), C.byref(intr.c()), _ptr(out), _stream_handle()))
    return out


def rgb_to_intensity(rgb) -> torch.Tensor:
    """rgb_to_intensity (view.cpp:8-16)."""
    r = _rgb_tensor(rgb)
    out = torch.empty(r.shape[:2], dtype=torch.float32, device=r.device)
    check(lib().rfg_rgb_to_intensity(_ptr(r), r.shape[1], r.shape[0], _ptr(out), _stream_handle()))
    return out


def downsample_intensity(img) -> torch.Tensor:
    """downsample_intensity (view.cpp:90-98)."""
    i = torch.as_tensor(img, dtype=torch.float32).cuda().contiguous()
    out = torch.empty((i.shape[0] // 2, i.shape[1] // 2), dtype=torch.float32, device=i.device)
    check(lib().rfg_downsample_intensity(_ptr(i), i.shape[1], i.shape[0], _ptr(out), _stream_handle()))
    return out


# ----------------------------------------------------------------- mesh
@dataclass
class Mesh:
    """proj/include/rf/meshing.hpp:12-15: vertices in metres, triangles as
    vertex-index triples (normals toward positive sdf)."""
    vertices: np.ndarray   # (N, 3) float32
    triangles: np.ndarray  # (M, 3) uint32


def extract_mesh(map: "VoxelBlockMap", voxelSize: float) -> Mesh:
    """extract_mesh (proj/src/meshing.cpp:144-217) on the GPU: marching cubes
    over the in-memory blocks, vertices and triangles in the reference's
    order."""
    nv, nt = C.c_int64(0), C.c_int64(0)
    map.bind_stream()
    check(lib().rfg_extract_mesh(map.handle, voxelSize, C.byref(nv), C.byref(nt)))
    v = np.empty((nv.value, 3), np.float32)
    t = np.empty((nt.value, 3), np.uint32)
    check(lib().rfg_mesh_copy(map.handle, v.ctypes.data_as(C.c_void_p) if nv.value else None,
                              t.ctypes.data_as(C.c_void_p) if nt.value else None))
    return Mesh(v, t)


def marching_cubes_table():
    """The 256-case triangulation (meshing.cpp:27-118): list of lists of
    edge triples."""
    cnt = np.zeros(256, np.int32)
    tri = np.zeros(256 * 16 * 3, np.int32)
    check(lib().rfg_mc_table(cnt.ctypes.data_as(C.POINTER(C.c_int32)), tri.ctypes.data_as(C.POINTER(C.c_int32))))
    tri = tri.reshape(256, 16, 3)
    return [[tuple(int(x) for x in tri[m, k]) for k in range(cnt[m])] for m in range(256)]


# ------------------------------------------------------------ image IO
def _pnm_read(fn, path, channels, dtype):
    w, h = C.c_int32(0), C.c_int32(0)
    rc = fn(path.encode(), None, 0, C.byref(w), C.byref(h))
    if rc == _lib.RFG_EINVAL:
        raise RuntimeError(lib().rfg_last_error().decode())
    shape = (h.value, w.value) + ((channels,) if channels > 1 else ())
    out = np.empty(shape, dtype=dtype)
    check(fn(path.encode(), out.ctypes.data_as(C.c_void_p), w.value * h.value, C.byref(w), C.byref(h)))
    return out


def read_pgm16(path: str) -> np.ndarray:
    """read_pgm16 (image_io.cpp:96-113): (H, W) uint16, host order.  Raises
    RuntimeError with the reference's message on a bad file."""
    return _pnm_read(lib().rfg_read_pgm16, path, 1, np.uint16)


def read_pgm16_payload(path: str) -> np.ndarray:
    """The PGM16 pixel bytes as stored (big-endian u16), for the GPU decode
    (build_view(..., big_endian=True), Pipeline.process_pgm)."""
    return _pnm_read(lib().rfg_read_pgm16_payload, path, 1, np.uint16)


def read_ppm(path: str) -> np.ndarray:
    """read_ppm (image_io.cpp:53-64): (H, W, 3) uint8."""
    return _pnm_read(lib().rfg_read_ppm, path, 3, np.uint8)


def write_pgm16(img, path: str) -> None:
    a = np.ascontiguousarray(img, dtype=np.uint16)
    check(lib().rfg_write_pgm16(path.encode(), a.ctypes.data_as(C.c_void_p), a.shape[1], a.shape[0]))


def write_ppm(img, path: str) -> None:
    a = np.ascontiguousarray(img, dtype=np.uint8)
    check(lib().rfg_write_ppm(path.encode(), a.ctypes.data_as(C.c_void_p), a.shape[1], a.shape[0]))


@dataclass
class RawFrame:
    depth: np.ndarray
    rgb: np.ndarray | None
    index: int


class ImageStream:
    """ImageStream (image_io.hpp:26-38): frame i is <pattern % i>.pgm (depth,
    required) and <pattern % i>.ppm (colour, optional); the stream ends at the
    first missing depth file."""

    def __init__(self, pattern_no_ext: str, start_index: int = 0):
        self._pattern = pattern_no_ext
        self._index = start_index

    def next(self) -> RawFrame | None:
        import os
        base = self._pattern % self._index
        if not os.path.exists(base + ".pgm"):
            return None
        f = RawFrame(read_pgm16(base + ".pgm"), read_ppm(base + ".ppm") if os.path.exists(base + ".ppm") else None,
                     self._index)
        self._index += 1
        return f

    def nextIndex(self) -> int:
        return self._index


def view_from_depth(depth_m, intr: Intrinsics, rgb=None, calib: RgbdCalib | None = None) -> View:
    """A View around an existing metres depth image (float32, device or host)."""
    d = torch.as_tensor(np.ascontiguousarray(depth_m, np.float32)) if not torch.is_tensor(depth_m) else depth_m
    d = d.cuda().contiguous()
    cal = calib or RgbdCalib(intrinsics_rgb=intr, intrinsics_d=intr)
    rgb_t = None
    if rgb is not None:
        rgb_t = torch.as_tensor(np.ascontiguousarray(rgb, np.uint8)).cuda() if not torch.is_tensor(rgb) \
            else rgb.cuda().contiguous()
    return View(calib=cal, depth_m=d, rgb=rgb_t, pyramid=[ViewLevel(d, intr)])


# --------------------------------------------------------------- fusion
class FusionEngine:
    """proj/include/rf/fusion.hpp:52-79 — per-frame allocation + integration."""

    @dataclass
    class Options:
        """FusionEngine::Options (fusion.hpp:54-57)."""
        swappingEnabled: bool = False
        swapMarginPx: float = 8.0

    def allocate_from_depth(self, map: VoxelBlockMap, view: View, pose, params: SceneParams,
                            opts: "FusionEngine.Options | None" = None, sync: bool = True) -> AllocationStats | None:
        p = _pose(pose)
        map.bind_stream()
        st = _lib.AllocStats_()
        intr = view.calib.intrinsics_d.c()
        o = _lib.FusionOptions_(1 if opts.swappingEnabled else 0, opts.swapMarginPx) if opts else None
        check(lib().rfg_allocate_from_depth_ex(map.handle, _ptr(view.depth_m), C.byref(intr), _fp(p),
                                               C.byref(params.c()), C.byref(o) if o is not None else None,
                                               C.byref(st) if sync else None))
        if not sync:
            return None
        return AllocationStats(st.requested, st.allocated, st.allocFailures, st.visibleCount)

    def integrate_frame(self, map: VoxelBlockMap, view: View, pose, params: SceneParams):
        p = _pose(pose)
        map.bind_stream()
        intr_d = view.calib.intrinsics_d.c()
        intr_rgb = view.calib.intrinsics_rgb.c()
        extr = _pose(view.calib.extrinsics_d_to_rgb)
        use_colour = view.hasColour() and map.colour
        check(lib().rfg_integrate(map.handle, _ptr(view.depth_m), _ptr(view.rgb) if use_colour else None,
                                  C.byref(intr_d), C.byref(intr_rgb), _fp(extr), _fp(p), C.byref(params.c())))


class SwappingEngine:
    """The swapping engine (rfg_swap.cu): host voxel store +
    transfer buffers of `capacity` blocks per frame and direction.  Per frame:
    allocate_from_depth(opts=Options(swappingEnabled=True)) -> swap_in() ->
    integrate / render -> swap_out()."""

    def __init__(self, map: VoxelBlockMap, capacity: int = 512):
        self.map = map
        self._h = C.c_void_p()
        map.bind_stream()
        check(lib().rfg_swap_create(map.handle, capacity, C.byref(self._h)))

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib._lib is not None:
                _lib._lib.rfg_swap_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def swap_in(self, maxW: int = 100) -> int:
        n = C.c_int(0)
        check(lib().rfg_swap_in(self._h, maxW, C.byref(n)))
        return n.value

    def swap_out(self) -> int:
        n = C.c_int(0)
        check(lib().rfg_swap_out(self._h, C.byref(n)))
        return n.value

    def stored(self):
        """(has, age): per-entry host-data flags and invisible-frame ages."""
        n = self.map.totalEntries()
        has, age = np.zeros(n, np.uint8), np.zeros(n, np.uint8)
        check(lib().rfg_swap_export(self._h, has.ctypes.data_as(C.POINTER(C.c_uint8)),
                                    age.ctypes.data_as(C.POINTER(C.c_uint8))))
        return has, age

    def host_block(self, idx: int) -> np.ndarray:
        out = np.zeros((512, 8), np.uint8)
        check(lib().rfg_swap_host_block(self._h, idx, out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out


# -------------------------------------------------------------- raycast
class RenderState:
    """proj/include/rf/raycast.hpp:15-26 (device images)."""

    def __init__(self):
        self.expectedRange = None
        self.raycastResult = None
        self.points = None
        self.normals = None
        self.colour = None  # (H, W, 3) uint8 (colour / grey modes)
        self.pose = np.eye(3, 4, dtype=np.float32)
        self.intr = Intrinsics()
        self.hasRaycast = False

    def resize(self, intr: Intrinsics):
        if self.points is not None and self.intr.width == intr.width and self.intr.height == intr.height:
            return
        h, w = intr.height, intr.width
        self.expectedRange = torch.empty((h, w, 2), dtype=torch.float32, device="cuda")
        self.expectedRange[..., 0] = float(np.finfo(np.float32).max)
        self.expectedRange[..., 1] = -1.0
        inv = torch.tensor([0.0, 0.0, 0.0, -1.0], device="cuda")
        self.raycastResult = inv.repeat(h, w, 1).contiguous()
        self.points = inv.repeat(h, w, 1).contiguous()
        self.normals = inv.repeat(h, w, 1).contiguous()
        self.colour = torch.zeros((h, w, 3), dtype=torch.uint8, device="cuda")
        self.intr = intr
        self.hasRaycast = False


def render_expected_ranges(map: VoxelBlockMap, pose, intr: Intrinsics, params: SceneParams, state: RenderState):
    """proj/src/raycast.cpp:86-127"""
    state.resize(intr)
    p = _pose(pose)
    map.bind_stream()
    check(lib().rfg_render_expected_ranges(map.handle, _fp(p), C.byref(intr.c()), C.byref(params.c()),
                                           _ptr(state.expectedRange)))


class MissingPixels:
    """Device list of row-major linear pixel indices (forward_project output)."""

    def __init__(self, capacity: int, width: int):
        self.index = torch.empty(max(capacity, 1), dtype=torch.int32, device="cuda")
        self.count = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.width = width

    def __len__(self):
        return int(self.count.item())

    def xy(self) -> np.ndarray:
        """(N, 2) int32 (x, y), the reference's std::vector<Vector2i> order."""
        idx = self.index[:len(self)].cpu().numpy()
        return np.stack([idx % self.width, idx // self.width], axis=1).astype(np.int32)


def render_maps(map: VoxelBlockMap, pose, intr: Intrinsics, params: SceneParams, mode: RenderMode,
                state: RenderState, missingOnly: MissingPixels | None = None):
    """proj/src/raycast.cpp:129-139 with every RenderMode (kIcpMaps, kColour,
    kGrey -> state.colour).  missingOnly restricts the work to the listed
    pixels (raycast.hpp:200-202)."""
    if state.expectedRange is None:
        raise RuntimeError("render_maps needs render_expected_ranges first")
    state.resize(intr)
    p = _pose(pose)
    map.bind_stream()
    col = _ptr(state.colour) if mode != RenderMode.kIcpMaps else None
    if missingOnly is None:
        check(lib().rfg_render_maps(map.handle, _fp(p), C.byref(intr.c()), C.byref(params.c()), int(mode),
                                    _ptr(state.expectedRange), _ptr(state.raycastResult), _ptr(state.points),
                                    _ptr(state.normals), col))
    else:
        check(lib().rfg_render_maps_list(map.handle, _fp(p), C.byref(intr.c()), C.byref(params.c()), int(mode),
                                         _ptr(state.expectedRange), _ptr(missingOnly.index),
                                         _ptr(missingOnly.count), _ptr(state.raycastResult),
                                         _ptr(state.points), _ptr(state.normals), col))
    state.pose = p.copy()
    state.intr = intr
    state.hasRaycast = True


def forward_project(state: RenderState, newPose, intr: Intrinsics, voxelSize: float,
                    map: VoxelBlockMap) -> MissingPixels:
    """forward_project (proj/src/raycast.cpp:141-188) on the device images of
    `state`; returns the pixels that must be raycast afresh."""
    missing = MissingPixels(intr.width * intr.height, intr.width)
    has = state.hasRaycast
    state.resize(intr)
    p = _pose(newPose)
    map.bind_stream()
    check(lib().rfg_forward_project(map.handle, 1 if has else 0, _ptr(state.raycastResult), _ptr(state.points),
                                    _ptr(state.normals), _fp(p), C.byref(intr.c()), voxelSize,
                                    _ptr(missing.index), _ptr(missing.count)))
    if has:
        state.pose = p.copy()
        state.intr = intr
    return missing


# ------------------------------------------------------------------ ICP
ICP_STATS = 12  # RFG_ICP_STATS
ICP_SUMS = 31   # RFG_ICP_SUMS


@dataclass
class TrackerIterationSummary:
    """SPEC.md:342-346 (TrackerIterationSummary) of the tracker's last
    evaluation, plus the run's iteration counts and outcome."""
    iterations: int          # Gauss-Newton updates, all levels
    count: int               # inliers (associated, within the gate)
    residual_sum: float      # sum r^2 over the inliers
    converged: bool          # a level stopped on ||delta|| < 1e-4
    per_level: tuple         # updates per level (finest first)
    ok: bool                 # False: too few inliers, or degenerate (init pose returned)
    inlier_fraction: float = 0.0   # inliers / valid depth pixels of the level
    hessian_det: float = 0.0       # det(H / inliers) ("after scaling")
    residual_mean: float = 0.0     # sum |r| / inliers
    valid: int = 0                 # valid depth pixels of the level

    @staticmethod
    def from_stats(st) -> "TrackerIterationSummary":
        st = np.asarray(st, np.float64)
        return TrackerIterationSummary(int(st[0]), int(st[1]), float(st[2]), bool(st[3]),
                                       (int(st[4]), int(st[5]), int(st[6])), bool(st[7]), float(st[8]),
                                       float(st[9]), float(st[10]), int(st[11]))


def track_depth(map: VoxelBlockMap, view: View, state: RenderState, init_pose, iters=(6, 10, 20),
                dist=(0.01, 0.02, 0.04), min_count: int = 10):
    """Point-to-plane ICP of the view's depth pyramid against
    the last ICP-map render in `state`.  iters/dist are indexed by pyramid
    level (0 = finest; SPEC.md:391 caps 20/10/6 coarse -> fine).  Returns
    (world->camera pose (3, 4), TrackerIterationSummary); a degenerate Hessian
    returns init_pose with summary.ok False."""
    if not state.hasRaycast:
        raise RuntimeError("track_depth needs an ICP-map render (render_maps) first")
    levels = len(view.pyramid)
    base = view.pyramid[0].depth
    # the pyramid levels are views into one contiguous buffer (build_view)
    p0 = base.data_ptr()
    expect = p0
    for lv in view.pyramid:
        if lv.depth.data_ptr() != expect:
            raise ValueError("track_depth needs a pyramid produced by build_view")
        expect += lv.depth.numel() * 4
    init = _pose(init_pose)
    rp = _pose(state.pose)
    it = (C.c_int32 * 3)(*[int(x) for x in iters])
    ds = (C.c_float * 3)(*[float(x) for x in dist])
    out = np.zeros((3, 4), np.float32)
    st = np.zeros(ICP_STATS, np.float64)
    map.bind_stream()
    check(lib().rfg_icp_track(map.handle, C.c_void_p(p0), levels, C.byref(view.calib.intrinsics_d.c()),
                              _ptr(state.points), _ptr(state.normals), _fp(rp), _fp(init), it, ds, min_count,
                              _fp(out), st.ctypes.data_as(_d)))
    return out, TrackerIterationSummary.from_stats(st)


def icp_reduce(map: VoxelBlockMap, depth_level: torch.Tensor, level: int, intr0: Intrinsics, state: RenderState,
               cam_to_world, dist: float, fixed: bool = False) -> np.ndarray:
    """One evaluation of the 31 point-to-plane sums (H upper 21, g 6, sum r^2,
    inliers, sum |r|, valid pixels): decoded float64, or with fixed=True the
    int64 fixed-point sums themselves."""
    out = np.zeros(ICP_SUMS, np.float64)
    raw = np.zeros(ICP_SUMS, np.int64)
    c2w = _pose(cam_to_world)
    rp = _pose(state.pose)
    map.bind_stream()
    check(lib().rfg_icp_reduce(map.handle, _ptr(depth_level.contiguous()), level, C.byref(intr0.c()),
                               _ptr(state.points), _ptr(state.normals), _fp(rp), _fp(c2w), dist,
                               raw.ctypes.data_as(C.POINTER(C.c_int64)), out.ctypes.data_as(_d)))
    return raw if fixed else out


# ------------------------------------------------------------- pipeline
class DeviceBuffer:
    """A raw device allocation seen by torch without a copy
    (__cuda_array_interface__); the owner keeps it alive."""

    def __init__(self, ptr: int, n: int, typestr: str = "<f4"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None, "stream": None}


class Pipeline:
    """Device-resident per-frame driver (ITMMainEngine::ProcessFrame order,
    SPEC.md:764): [ICP track] -> allocate -> integrate -> expected ranges ->
    ICP-map raycast, optionally replayed as a CUDA graph."""

    def __init__(self, map: VoxelBlockMap, intr: Intrinsics, params: SceneParams,
                 affine: DepthAffine = DepthAffine(1.0 / 5000.0, 0.0), levels: int = 3, track: bool = True,
                 iters=(6, 10, 20), dist=(0.01, 0.02, 0.04), min_count: int = 10, use_graph: bool = True,
                 profile: bool = False, bilateral: bool = False, raw_big_endian: bool = False,
                 colour: bool = False, intr_rgb: Intrinsics | None = None, extr_d_to_rgb=None):
        """colour: ITMVoxel_s_rgb fusion (the map needs a colour plane); frames
        then come with an RGB8 image, process(raw, pose, rgb=...), taken with
        intrinsics intr_rgb (default: the depth camera's) and
        extrinsics_d_to_rgb (default: identity)."""
        self.map = map
        self.intr = intr
        self.colour = colour
        cfg = _lib.PipelineConfig_()
        cfg.intr = intr.c()
        cfg.params = params.c()
        cfg.aff_scale = affine.scale
        cfg.aff_offset = affine.offset
        cfg.levels = levels
        cfg.track = 1 if track else 0
        cfg.iters = (C.c_int32 * 3)(*iters)
        cfg.dist = (C.c_float * 3)(*dist)
        cfg.min_count = min_count
        cfg.use_graph = 1 if use_graph else 0
        cfg.profile = 1 if profile else 0
        cfg.bilateral = 1 if bilateral else 0
        cfg.raw_big_endian = 1 if raw_big_endian else 0
        cfg.colour = 1 if colour else 0
        if colour:
            cfg.intr_rgb = (intr_rgb or intr).c()
            ex = np.eye(3, 4, dtype=np.float32) if extr_d_to_rgb is None else _pose(extr_d_to_rgb)
            cfg.extr_d_to_rgb = (C.c_float * 12)(*ex.reshape(-1).tolist())
        self._h = C.c_void_p()
        check(lib().rfg_pipeline_create(map.handle, C.byref(cfg), C.byref(self._h)))
        self._levels = levels
        # per-frame call state, prepared once (the end-to-end path calls
        # process / result every frame)
        L = lib()
        self._fn_host = L.rfg_pipeline_process_host
        self._fn_rgbd_host = L.rfg_pipeline_process_rgbd_host
        self._fn_result = L.rfg_pipeline_result
        self._res = (_lib.AllocStats_(), np.zeros((3, 4), np.float32), np.zeros(ICP_STATS, np.float64))
        self._res_args = (C.byref(self._res[0]), _fp(self._res[1]), self._res[2].ctypes.data_as(_d))

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib._lib is not None:
                _lib._lib.rfg_pipeline_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown: module globals may be gone
            pass

    def process(self, raw, pose=None, rgb=None):
        """raw: CUDA uint16/int16 tensor (device path) or numpy uint16 (host path).
        A device frame is ordered after the work queued on torch's current
        stream (e.g. the upload that produced it) and kept alive until the
        pipeline's stream has read it.  rgb: the (H, W, 3) uint8 colour image
        of a colour pipeline, on the same side as raw."""
        p = _fp(_pose(pose)) if pose is not None else None
        if self.colour:
            if rgb is None:
                raise ValueError("a colour pipeline needs the rgb image")
            if torch.is_tensor(raw) and raw.is_cuda:
                c = rgb if torch.is_tensor(rgb) else torch.as_tensor(np.ascontiguousarray(rgb, np.uint8))
                c = c.cuda().contiguous()
                check(lib().rfg_pipeline_process_rgbd_stream(self._h, _ptr(raw), _ptr(c), p, _stream_handle()))
            else:
                a = np.ascontiguousarray(raw, np.uint16) if not torch.is_tensor(raw) else raw.numpy()
                c = np.ascontiguousarray(rgb, np.uint8) if not torch.is_tensor(rgb) else rgb.numpy()
                check(self._fn_rgbd_host(self._h, a.ctypes.data, c.ctypes.data, p))
            return
        if torch.is_tensor(raw) and raw.is_cuda:
            check(lib().rfg_pipeline_process_raw_stream(self._h, _ptr(raw), p, _stream_handle()))
        else:
            a = np.ascontiguousarray(raw, np.uint16) if not torch.is_tensor(raw) else raw.numpy()
            check(self._fn_host(self._h, a.ctypes.data, p))

    def process_pgm(self, path: str, pose=None):
        """One frame straight from a PGM16 file (rfg_pipeline_process_pgm)."""
        p = _fp(_pose(pose)) if pose is not None else None
        check(lib().rfg_pipeline_process_pgm(self._h, path.encode(), p))

    def result(self):
        """(AllocationStats, world->camera pose (3, 4), tracker summary
        (ICP_STATS,)) of the last frame; synchronises the pipeline."""
        st, pose, icp = self._res
        check(self._fn_result(self._h, self._res_args[0], self._res_args[1], self._res_args[2]))
        return (AllocationStats(st.requested, st.allocated, st.allocFailures, st.visibleCount), pose.copy(),
                icp.copy())

    def pose_buffer(self) -> int:
        """Device pointer of the current world->camera pose (12 floats)."""
        ptr = C.c_void_p()
        check(lib().rfg_pipeline_pose_buffer(self._h, C.byref(ptr)))
        return ptr.value

    def buffers(self):
        ptrs = [C.c_void_p() for _ in range(5)]
        check(lib().rfg_pipeline_buffers(self._h, *[C.byref(p) for p in ptrs]))
        return [p.value for p in ptrs]

    def maps(self):
        """The last frame's render, as zero-copy torch views of the pipeline's
        device buffers: (expectedRange (H, W, 2), raycastResult, points,
        normals (H, W, 4)) — the outputs of render_expected_ranges +
        render_maps(kIcpMaps) at the frame's output pose (RenderState,
        proj/include/rf/raycast.hpp:15-26).  Valid after result(); the next
        process() overwrites them."""
        h, w = self.intr.height, self.intr.width
        _, rng, raycast, points, normals = self.buffers()
        view = lambda ptr, c: torch.as_tensor(DeviceBuffer(ptr, h * w * c), device="cuda").view(h, w, c)  # noqa: E731
        return view(rng, 2), view(raycast, 4), view(points, 4), view(normals, 4)

    def depth_levels(self):
        """The last frame's depth pyramid (View::depth_m + levels), zero-copy
        views of the pipeline's buffer, finest first."""
        dl = self.buffers()[0]
        out, off = [], 0
        for lv in range(self._levels):
            h, w = self.intr.height >> lv, self.intr.width >> lv
            out.append(torch.as_tensor(DeviceBuffer(dl + 4 * off, h * w), device="cuda").view(h, w))
            off += h * w
        return out

    def reset(self):
        check(lib().rfg_pipeline_reset(self._h))

    def stage_times(self) -> dict:
        ms = np.zeros(7, np.float32)
        check(lib().rfg_pipeline_stage_times(self._h, _fp(ms)))
        return dict(zip(("view", "icp", "allocate", "integrate", "ranges", "raycast", "total"), ms.tolist()))

    @property
    def stream(self) -> int:
        return int(lib().rfg_pipeline_stream(self._h) or 0)


# ------------------------------------------------------------ synthetic
def orbit_trajectory(target=(0.0, 0.15, 1.4), distance=1.4, frames=100, max_angle=0.5) -> np.ndarray:
    """proj/src/synth.cpp:173-195 (world -> camera poses, (frames, 3, 4))."""
    out = np.zeros((frames, 3, 4), np.float32)
    t = np.ascontiguousarray(target, np.float32)
    check(lib().rfg_synth_orbit_poses(_fp(t), distance, frames, max_angle, _fp(out)))
    return out


def multiroom_trajectory(frames=100) -> np.ndarray:
    out = np.zeros((frames, 3, 4), np.float32)
    check(lib().rfg_synth_multiroom_poses(frames, _fp(out)))
    return out


SCENE_SPHERE_IN_ROOM = 0
SCENE_MULTI_ROOM = 1
SCENE_CHECKER_WALL = 2


def synth_render(scene: int, pose, intr: Intrinsics, affine=DepthAffine(1.0 / 5000.0, 0.0), rgb=False):
    """synth_render_depth (proj/src/synth.cpp:136-171): (raw u16, depth m, rgb)."""
    h, w = intr.height, intr.width
    raw = np.zeros((h, w), np.uint16)
    dep = np.zeros((h, w), np.float32)
    col = np.zeros((h, w, 3), np.uint8) if rgb else None
    p = _pose(pose)
    check(lib().rfg_synth_render(scene, _fp(p), C.byref(intr.c()), affine.scale, affine.offset, 1 if rgb else 0,
                                 raw.ctypes.data_as(_u16), _fp(dep),
                                 col.ctypes.data_as(_u8) if col is not None else None))
    return raw, dep, col
