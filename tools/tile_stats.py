"""Tile-list length distribution of config 1 after N Stage-1 iterations."""
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
N = int(sys.argv[1]) if len(sys.argv) > 1 else 144
sc, cache, targets = bench.build_problem(1)
tr = Stage1Trainer(sc.cloud, cache, list(zip(sc.cameras, targets)), Stage1Config())
for k in range(N):
    tr.iterate(k % 20)
v = N % 20
tr.render_async(v)
cam = tr.cam_structs[v]
nt = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
ranges = torch.zeros(2 * nt, dtype=torch.int32, device="cuda")
lib.ss_raster_tile_lists(C.byref(cam), C.byref(tr.settings), ptr(tr.geom), ptr(tr.bins),
                         tr.bin_capacity, tr.cloud.n, ptr(ranges), None, None, stream())
r = ranges.view(-1, 2).cpu().numpy()
ln = r[:, 1] - r[:, 0]
print(f"iter {N} view {v}: pairs kept {ln.sum()}, tiles {nt}, mean {ln.mean():.0f}, "
      f"p50 {np.percentile(ln, 50):.0f}, p99 {np.percentile(ln, 99):.0f}, max {ln.max()}")
t = tr.t_means.cpu().numpy()
d = t - sc.cloud["means"]
print(f"displacement |d_mu|: mean {np.linalg.norm(d, axis=1).mean():.4f}, "
      f"max {np.linalg.norm(d, axis=1).max():.4f}")
