"""Per-iteration device time of graph-replayed Stage-1 iterations over a frame
(cfg1), L2 flushed between steps, to compare against the kernel-time sums of
the ncu launch lists (gap / launch overhead inside the graph):

  python tools/step_times.py [steps] [tile_size]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer  # noqa: E402

from paper_2403_01444_b200.types import RasterSettings  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 150
ts = int(sys.argv[2]) if len(sys.argv) > 2 else 16
sc, cache, targets = bench.build_problem(1)
tr = Stage1Trainer(sc.cloud, cache, list(zip(sc.cameras, targets)),
                   Stage1Config(raster=RasterSettings(tile_size=ts)))
n = len(sc.cameras)
for k in range(20):
    tr.iterate(k % n)
tr.reset_frame()
flush = torch.empty(bench.L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
for k in range(steps):
    flush.fill_(k & 0xFF)
    ev[k][0].record()
    tr.iterate(k % n)
    ev[k][1].record()
torch.cuda.synchronize()
ms = np.array([a.elapsed_time(b) for a, b in ev])
print("mean ms %.4f" % ms.mean())
for i in list(range(0, 10)) + list(range(steps - 10, steps)):
    print(i, "%.4f" % ms[i])
