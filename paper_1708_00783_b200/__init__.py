"""B200-native dense-fusion hot path of InfiniTAM v3 (arXiv:1708.00783).

Voxel-block hash allocation, visible-list construction, TSDF (+colour)
integration, expected-range + ICP-map raycast and the ICP 6x6 reduction as
hand-written sm_100a CUDA kernels (librfg.so, C ABI in include/rfg.h), with a
host API mirroring the reference's rf:: engine interface (fusion.py).
"""
from ._lib import LIB_PATH, RfgError, launch_count  # noqa: F401

__all__ = ["LIB_PATH", "RfgError", "launch_count"]
