"""Fraction of (splat, tile) pairs the render path's tile cull removes at
config-1 size: python tools/cull_stats.py"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2403_01444_b200 import _lib  # noqa: E402
from paper_2403_01444_b200.device import ptr, stream  # noqa: E402
from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer  # noqa: E402

lib = _lib.load()
sc, cache, targets = bench.build_problem(1)
tr = Stage1Trainer(sc.cloud, cache, list(zip(sc.cameras, targets)), Stage1Config())
tot, kept = 0, 0
for v in range(len(sc.cameras)):
    pairs = tr.begin(v)
    tr.render_async(v)
    cam = tr.cam_structs[v]
    nt = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    ranges = torch.zeros(2 * nt, dtype=torch.int32, device="cuda")
    lib.ss_raster_tile_lists(C.byref(cam), C.byref(tr.settings), ptr(tr.geom), ptr(tr.bins),
                             tr.bin_capacity, tr.cloud.n, ptr(ranges), None, None, stream())
    r = ranges.view(-1, 2).cpu().numpy()
    k = int((r[:, 1] - r[:, 0]).sum())
    tot += pairs
    kept += k
    print(f"view {v}: pairs {pairs} kept {k} ({k / pairs:.3f})")
print(f"total kept fraction {kept / tot:.3f}")
