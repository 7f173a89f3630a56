"""ctypes bindings of librfg.so (include/rfg.h).

The shared library is built in-tree (paper_1708_00783_b200/librfg.so) by
`make -C paper_1708_00783_b200/csrc` / `__graft_entry__.build()`.  There is no
CPU fallback: if the library is missing, importing the compute API raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# RFG_LIB_PATH selects another build of the same library (A/B kernel variants
# in tools/); there is still no fallback if it is missing
LIB_PATH = os.environ.get("RFG_LIB_PATH") or os.path.join(PKG_DIR, "librfg.so")

RFG_OK = 0
RFG_EINVAL = -1
RFG_ECUDA = -2
RFG_ENOMEM = -3
RFG_ERANGE = -4
RFG_ESTATE = -5


class MapConfig(C.Structure):
    _fields_ = [("bucketCount", C.c_uint32), ("excessCount", C.c_uint32), ("blockCapacity", C.c_uint32),
                ("hasColour", C.c_int32)]


class Intrinsics_(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float)]


class SceneParams_(C.Structure):
    _fields_ = [("voxelSize", C.c_float), ("mu", C.c_float), ("maxW", C.c_int32),
                ("viewFrustum_min", C.c_float), ("viewFrustum_max", C.c_float),
                ("stopIntegratingAtMaxW", C.c_int32)]


class AllocStats_(C.Structure):
    _fields_ = [("requested", C.c_int32), ("allocated", C.c_int32), ("allocFailures", C.c_int32),
                ("visibleCount", C.c_int32)]


class FusionOptions_(C.Structure):
    _fields_ = [("swapping_enabled", C.c_int32), ("swap_margin_px", C.c_float)]


class PipelineConfig_(C.Structure):
    _fields_ = [("intr", Intrinsics_), ("params", SceneParams_), ("aff_scale", C.c_float),
                ("aff_offset", C.c_float), ("levels", C.c_int32), ("track", C.c_int32),
                ("iters", C.c_int32 * 3), ("dist", C.c_float * 3), ("min_count", C.c_int32),
                ("use_graph", C.c_int32), ("profile", C.c_int32), ("bilateral", C.c_int32),
                ("raw_big_endian", C.c_int32), ("colour", C.c_int32), ("intr_rgb", Intrinsics_),
                ("extr_d_to_rgb", C.c_float * 12)]


# every symbol include/rfg.h declares, with its ctypes signature
_vp = C.c_void_p
_f = C.POINTER(C.c_float)
_d = C.POINTER(C.c_double)
_i = C.POINTER(C.c_int32)
_u8 = C.POINTER(C.c_uint8)
_u16 = C.POINTER(C.c_uint16)
SIGNATURES = {
    "rfg_map_create": ([C.POINTER(MapConfig), C.c_int, C.POINTER(_vp)], C.c_int),
    "rfg_map_destroy": ([_vp], C.c_int),
    "rfg_map_clear": ([_vp], C.c_int),
    "rfg_map_set_stream": ([_vp, _vp], C.c_int),
    "rfg_map_sync": ([_vp], C.c_int),
    "rfg_map_set_shard": ([_vp, C.c_int, C.c_int, C.c_int], C.c_int),
    "rfg_last_error": ([], C.c_char_p),
    "rfg_kernel_launch_count": ([], C.c_uint64),
    "rfg_allocate_from_depth": ([_vp, _vp, C.POINTER(Intrinsics_), _f, C.POINTER(SceneParams_),
                                 C.POINTER(AllocStats_)], C.c_int),
    "rfg_integrate": ([_vp, _vp, _vp, C.POINTER(Intrinsics_), C.POINTER(Intrinsics_), _f, _f,
                       C.POINTER(SceneParams_)], C.c_int),
    "rfg_allocate_from_depth_ex": ([_vp, _vp, C.POINTER(Intrinsics_), _f, C.POINTER(SceneParams_),
                                    C.POINTER(FusionOptions_), C.POINTER(AllocStats_)], C.c_int),
    "rfg_map_reserve_block": ([_vp, C.c_int], C.c_int),
    "rfg_map_release_block": ([_vp, C.c_int], C.c_int),
    "rfg_swap_create": ([_vp, C.c_int, C.POINTER(_vp)], C.c_int),
    "rfg_swap_destroy": ([_vp], C.c_int),
    "rfg_swap_in": ([_vp, C.c_int, _i], C.c_int),
    "rfg_swap_out": ([_vp, _i], C.c_int),
    "rfg_swap_export": ([_vp, _u8, _u8], C.c_int),
    "rfg_swap_host_block": ([_vp, C.c_int, _u8], C.c_int),
    "rfg_render_expected_ranges": ([_vp, _f, C.POINTER(Intrinsics_), C.POINTER(SceneParams_), _vp], C.c_int),
    "rfg_render_icp_maps": ([_vp, _f, C.POINTER(Intrinsics_), C.POINTER(SceneParams_), _vp, _vp, _vp, _vp],
                            C.c_int),
    "rfg_forward_project": ([_vp, C.c_int, _vp, _vp, _vp, _f, C.POINTER(Intrinsics_), C.c_float, _vp, _vp], C.c_int),
    "rfg_render_icp_maps_list": ([_vp, _f, C.POINTER(Intrinsics_), C.POINTER(SceneParams_), _vp, _vp, _vp, _vp,
                                  _vp, _vp], C.c_int),
    "rfg_render_maps": ([_vp, _f, C.POINTER(Intrinsics_), C.POINTER(SceneParams_), C.c_int, _vp, _vp, _vp, _vp,
                         _vp], C.c_int),
    "rfg_render_maps_list": ([_vp, _f, C.POINTER(Intrinsics_), C.POINTER(SceneParams_), C.c_int, _vp, _vp, _vp, _vp,
                              _vp, _vp, _vp], C.c_int),
    "rfg_extract_mesh": ([_vp, C.c_float, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
    "rfg_mesh_copy": ([_vp, _vp, _vp], C.c_int),
    "rfg_mc_table": ([_i, _i], C.c_int),
    "rfg_build_view_depth": ([_vp, C.c_int, C.c_int, C.c_float, C.c_float, C.c_int, _vp, _vp], C.c_int),
    "rfg_build_view": ([_vp, _vp, C.POINTER(Intrinsics_), C.c_float, C.c_float, C.c_int, C.c_int, C.c_int, _vp, _vp,
                        _vp, _vp, _vp], C.c_int),
    "rfg_bilateral_filter": ([_vp, C.c_int, C.c_int, C.c_float, C.c_float, _vp, _vp], C.c_int),
    "rfg_compute_normals": ([_vp, C.POINTER(Intrinsics_), _vp, _vp], C.c_int),
    "rfg_rgb_to_intensity": ([_vp, C.c_int, C.c_int, _vp, _vp], C.c_int),
    "rfg_downsample_intensity": ([_vp, C.c_int, C.c_int, _vp, _vp], C.c_int),
    "rfg_read_pgm16": ([C.c_char_p, _vp, C.c_int64, _i, _i], C.c_int),
    "rfg_read_pgm16_payload": ([C.c_char_p, _vp, C.c_int64, _i, _i], C.c_int),
    "rfg_read_ppm": ([C.c_char_p, _vp, C.c_int64, _i, _i], C.c_int),
    "rfg_write_pgm16": ([C.c_char_p, _vp, C.c_int, C.c_int], C.c_int),
    "rfg_write_ppm": ([C.c_char_p, _vp, C.c_int, C.c_int], C.c_int),
    "rfg_icp_track": ([_vp, _vp, C.c_int, C.POINTER(Intrinsics_), _vp, _vp, _f, _f, _i, _f, C.c_int, _f, _d],
                      C.c_int),
    "rfg_icp_reduce": ([_vp, _vp, C.c_int, C.POINTER(Intrinsics_), _vp, _vp, _f, _f, C.c_float,
                        C.POINTER(C.c_int64), _d], C.c_int),
    "rfg_pipeline_create": ([_vp, C.POINTER(PipelineConfig_), C.POINTER(_vp)], C.c_int),
    "rfg_pipeline_destroy": ([_vp], C.c_int),
    "rfg_pipeline_process_raw": ([_vp, _vp, _f], C.c_int),
    "rfg_pipeline_process_host": ([_vp, _vp, _f], C.c_int),
    "rfg_pipeline_process_raw_stream": ([_vp, _vp, _f, _vp], C.c_int),
    "rfg_pipeline_process_pgm": ([_vp, C.c_char_p, _f], C.c_int),
    "rfg_pipeline_process_rgbd_stream": ([_vp, _vp, _vp, _f, _vp], C.c_int),
    "rfg_pipeline_process_rgbd_host": ([_vp, _vp, _vp, _f], C.c_int),
    "rfg_pipeline_result": ([_vp, C.POINTER(AllocStats_), _f, _d], C.c_int),
    "rfg_pipeline_buffers": ([_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp),
                              C.POINTER(_vp)], C.c_int),
    "rfg_pipeline_reset": ([_vp], C.c_int),
    "rfg_pipeline_stage_times": ([_vp, _f], C.c_int),
    "rfg_pipeline_stream": ([_vp], _vp),
    "rfg_pipeline_pose_buffer": ([_vp, C.POINTER(_vp)], C.c_int),
    "rfg_compose_keys": ([_vp, _f, C.c_int, C.c_int, _vp, _vp], C.c_int),
    "rfg_compose_keys_dev": ([_vp, _vp, C.c_int, C.c_int, _vp, _vp], C.c_int),
    "rfg_compose_select": ([_vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp], C.c_int),
    "rfg_icp_timers": ([_vp, C.POINTER(C.c_uint64), C.c_int], C.c_int),
    "rfg_total_entries": ([_vp], C.c_uint32),
    "rfg_export_entries": ([_vp, _i], C.c_int),
    "rfg_export_blocks": ([_vp, _i, C.c_int, _u8], C.c_int),
    "rfg_export_visible": ([_vp, _i, _u8, _i], C.c_int),
    "rfg_free_counts": ([_vp, _i, _i], C.c_int),
    "rfg_synth_orbit_poses": ([_f, C.c_float, C.c_int, C.c_float, _f], C.c_int),
    "rfg_synth_multiroom_poses": ([C.c_int, _f], C.c_int),
    "rfg_synth_render": ([C.c_int, _f, C.POINTER(Intrinsics_), C.c_float, C.c_float, C.c_int, _u16, _f, _u8],
                         C.c_int),
}

_lib = None


class RfgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"librfg error {code}: {msg}")
        self.code = code


def lib():
    """Load librfg.so (raises if it has not been built — no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {PKG_DIR}/csrc` "
                              "(the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(rc: int):
    if rc != RFG_OK:
        raise RfgError(rc, lib().rfg_last_error().decode())
    return rc


def launch_count() -> int:
    return int(lib().rfg_kernel_launch_count())
