"""Multi-GPU spatial sharding of the voxel-hash space.

One process per GPU (torch.distributed, NCCL over NVLink).  Each rank keeps a
full-size hash table but allocates and integrates only the blocks it owns
plus a 1-block halo (owner = hash of the block's 8^3-block super-tile mod
world; the filter runs inside k_alloc_stage1, rfg_map_set_shard).  Every rank
renders its shard; the ICP maps are then composed by a per-pixel nearest-hit
reduction — the only data-path exchange:

  keys = (float bits of hit camera-z) << 32 | rank   (rfg_compose_keys[_dev])
  all_reduce(keys, MIN)                              (NCCL, 2.46 MB @ 640x480)
  zero every pixel this rank did not win             (rfg_compose_select)
  all_reduce(raycast | points | normals, SUM)        (NCCL, 14.7 MB in place;
                                                      exact — one nonzero term
                                                      per pixel)

The ICP tracker then runs replicated on the composed maps, so tracking needs
no per-iteration collective and every rank ends the frame with the same pose.
`Composer` is the collective sequence on caller-owned tensors (the gloo
world-size-2 test drives it with CPU stand-ins for the two kernels);
`ShardedPipeline` runs it on the device-resident frame graph.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import fusion as F
from ._lib import check, lib


class Composer:
    """Nearest-hit composition of per-rank ICP maps (device kernels + NCCL)."""

    def __init__(self, rank: int, world: int, keys_fn=None, select_fn=None):
        self.rank, self.world = rank, world
        self.keys_fn = keys_fn or self._keys_gpu
        self.select_fn = select_fn or self._select_gpu

    def _keys_gpu(self, points: torch.Tensor, pose: np.ndarray) -> torch.Tensor:
        n = points.numel() // 4
        keys = torch.empty(n, dtype=torch.int64, device=points.device)
        p = np.ascontiguousarray(pose, np.float32)
        check(lib().rfg_compose_keys(C.c_void_p(points.data_ptr()), p.ctypes.data_as(C.POINTER(C.c_float)),
                                     self.rank, n, C.c_void_p(keys.data_ptr()),
                                     C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return keys

    def _select_gpu(self, keymin: torch.Tensor, raycast, points, normals):
        n = keymin.numel()
        check(lib().rfg_compose_select(C.c_void_p(keymin.data_ptr()), self.rank, n, C.c_void_p(raycast.data_ptr()),
                                       C.c_void_p(points.data_ptr()), C.c_void_p(normals.data_ptr()),
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)))

    def compose(self, pose: np.ndarray, raycast: torch.Tensor, points: torch.Tensor, normals: torch.Tensor):
        """In place: after the call every rank holds the composed maps."""
        keys = self.keys_fn(points, pose)
        dist.all_reduce(keys, op=dist.ReduceOp.MIN)
        self.select_fn(keys, raycast, points, normals)
        maps = torch.stack([raycast, points, normals])  # one collective for the three maps
        dist.all_reduce(maps, op=dist.ReduceOp.SUM)
        raycast.copy_(maps[0])
        points.copy_(maps[1])
        normals.copy_(maps[2])
        return keys


_DeviceBuffer = F.DeviceBuffer


class ShardedPipeline:
    """Per-frame driver for one rank of a spatially sharded map: the rank's
    device-resident frame graph (rfg_pipeline: build_view -> ICP on the last
    COMPOSED maps -> allocate (owned blocks + halo) -> integrate -> expected
    ranges -> raycast) followed, on the same stream, by the nearest-hit
    composition written back into the graph's map buffers, so the next
    frame tracks against the composed render.  No host round trip per frame:
    the pose stays on the device (every rank tracks on identical maps and
    frames, so every rank computes the identical pose)."""

    def __init__(self, map: F.VoxelBlockMap, intr: F.Intrinsics, params: F.SceneParams, rank: int, world: int,
                 levels: int = 3, iters=(6, 10, 20), dist=(0.01, 0.02, 0.04),
                 affine: F.DepthAffine = F.DepthAffine(1.0 / 5000.0, 0.0), min_count: int = 10,
                 use_graph: bool = True, track: bool = True):
        self.map, self.intr, self.params = map, intr, params
        self.rank, self.world = rank, world
        self.pipe = F.Pipeline(map, intr, params, affine, levels=levels, track=track, iters=iters, dist=dist,
                               min_count=min_count, use_graph=use_graph)
        self.n = intr.width * intr.height
        _, _, raycast, points, normals = self.pipe.buffers()
        assert points == raycast + 16 * self.n and normals == raycast + 32 * self.n  # one allocation
        self._ptrs = (raycast, points, normals)
        self._pose_dev = self.pipe.pose_buffer()
        self._maps = torch.as_tensor(_DeviceBuffer(raycast, 3 * 4 * self.n), device="cuda")
        self._keys = torch.empty(self.n, dtype=torch.int64, device="cuda")
        self._stream = torch.cuda.ExternalStream(self.pipe.stream)
        self.frames = 0

    @property
    def stream(self) -> int:
        return self.pipe.stream

    def reset(self):
        self.pipe.reset()
        self.frames = 0

    def maps(self):
        """(raycastResult, points, normals) of the last composed render, each
        a (H, W, 4) view of the pipeline's buffers."""
        h, w = self.intr.height, self.intr.width
        m = self._maps.view(3, h, w, 4)
        return m[0], m[1], m[2]

    def compose(self):
        """Nearest-hit composition of this rank's last render with the other
        ranks', in place, on the pipeline's stream."""
        raycast, points, normals = self._ptrs
        with torch.cuda.stream(self._stream):
            check(lib().rfg_compose_keys_dev(C.c_void_p(points), C.c_void_p(self._pose_dev), self.rank, self.n,
                                             C.c_void_p(self._keys.data_ptr()), C.c_void_p(self.pipe.stream)))
            dist.all_reduce(self._keys, op=dist.ReduceOp.MIN)
            check(lib().rfg_compose_select(C.c_void_p(self._keys.data_ptr()), self.rank, self.n, C.c_void_p(raycast),
                                           C.c_void_p(points), C.c_void_p(normals), C.c_void_p(self.pipe.stream)))
            dist.all_reduce(self._maps, op=dist.ReduceOp.SUM)  # raycast | points | normals, one collective

    def process(self, raw, pose=None):
        self.pipe.process(raw, pose)
        self.compose()
        self.frames += 1

    def result(self):
        return self.pipe.result()
