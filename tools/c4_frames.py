#!/usr/bin/env python
"""C4 frames through the frame graph (for ncu captures of the large-scene
kernels): multi-room scene, 2 mm, 2^21 buckets, 2^22 blocks, known poses."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1708_00783_b200 import fusion as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
intr = F.Intrinsics(640, 480, 525.0, 525.0, 319.5, 239.5)
poses = F.multiroom_trajectory(100)
raws = torch.from_numpy(np.stack([F.synth_render(F.SCENE_MULTI_ROOM, poses[f], intr)[0]
                                  for f in range(n)]).view(np.int16)).cuda()
m = F.VoxelBlockMap(F.VoxelBlockMapConfig(1 << 21, 1 << 19, 1 << 22))
p = F.Pipeline(m, intr, F.SceneParams(voxelSize=0.002, mu=0.02), track=False)
for f in range(n):
    p.process(raws[f], poses[f])
print(p.result()[0])
