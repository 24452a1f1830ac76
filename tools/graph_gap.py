"""GPU time of back-to-back graph-replayed Stage-1 iterations (one event pair
around the whole frame) against the sum of per-iteration event times:
  python tools/graph_gap.py"""
import sys

import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer  # noqa: E402

sc, cache, targets = bench.build_problem(1)
tr = Stage1Trainer(sc.cloud, cache, list(zip(sc.cameras, targets)), Stage1Config())
n = len(sc.cameras)
for k in range(2 * n):
    tr.iterate(k % n)
K = 150
for mode in ("per-step events", "one event pair"):
    tr.reset_frame()
    torch.cuda.synchronize()
    if mode == "per-step events":
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for k in range(K):
            ev[k][0].record()
            tr.iterate(k % n)
            ev[k][1].record()
        torch.cuda.synchronize()
        tot = sum(a.elapsed_time(b) for a, b in ev)
        span = ev[0][0].elapsed_time(ev[-1][1])
        print(f"{mode}: sum {tot / K:.4f} ms/step, span {span / K:.4f} ms/step")
    else:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for k in range(K):
            tr.iterate(k % n)
        b.record()
        torch.cuda.synchronize()
        print(f"{mode}: {a.elapsed_time(b) / K:.4f} ms/step")
