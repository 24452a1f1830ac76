"""Loss and tile-pair trajectory of a long Stage-1 run on config 1 (frame_begin
once, then N iterations over the view cycle)."""
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 300
sc, cache, targets = bench.build_problem(1)
tr = Stage1Trainer(sc.cloud, cache, list(zip(sc.cameras, targets)), Stage1Config(), history=N)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
for k in range(N):
    ev[k][0].record()
    tr.iterate(k % 20)
    ev[k][1].record()
torch.cuda.synchronize()
loss = tr.loss_hist[:N].cpu().numpy()
pairs = tr.pair_hist[:N].cpu().numpy()
ms = np.array([a.elapsed_time(b) for a, b in ev])
for k0 in range(0, N, 20):
    sl = slice(k0, k0 + 20)
    print(f"iters {k0:4d}-{k0 + 19:4d}: loss {loss[sl].mean():.5f}  pairs {pairs[sl].mean() / 1e6:.3f}M  "
          f"ms {ms[sl].mean():.3f}")
