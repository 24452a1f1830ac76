"""Where does the e2e path lose time against the device-timed steps?
GPU time per step vs gaps between steps in run_from_host-style pipelining."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer  # noqa: E402

sc, cache, targets = bench.build_problem(1)
tr = Stage1Trainer(sc.cloud, cache, list(zip(sc.cameras, targets)), Stage1Config())
host = [t.cpu().pin_memory() for t in targets]
order = [k % 20 for k in range(60)]
tr.run_from_host(order[:4], host)
torch.cuda.synchronize()
# device-resident, no flush, async
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in order]
t0 = time.perf_counter()
for k, v in enumerate(order):
    ev[k][0].record()
    tr.iterate(v)
    ev[k][1].record()
host_enqueue = time.perf_counter() - t0
torch.cuda.synchronize()
wall = time.perf_counter() - t0
dev = [a.elapsed_time(b) for a, b in ev]
gaps = [ev[k][1].elapsed_time(ev[k + 1][0]) for k in range(len(order) - 1)]
span = ev[0][0].elapsed_time(ev[-1][1])
print(f"resident: mean step {np.mean(dev):.3f} ms, span/step {span / len(order):.3f}, "
      f"wall/step {1e3 * wall / len(order):.3f}, host enqueue/step {1e3 * host_enqueue / len(order):.3f}, "
      f"mean gap {np.mean(gaps):.4f} ms")
t0 = time.perf_counter()
tr.run_from_host(order, host)
wall = time.perf_counter() - t0
print(f"run_from_host: wall/step {1e3 * wall / len(order):.3f} ms")
# H2D bandwidth of one target from pinned memory
x = host[0]
d = torch.empty_like(targets[0])
for _ in range(3):
    d.view(-1)[: x.numel()].copy_(x.view(-1), non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    d.view(-1)[: x.numel()].copy_(x.view(-1), non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"H2D {x.numel() * 4 / 1e6:.1f} MB: {ms:.3f} ms = {x.numel() * 4 / ms / 1e6:.1f} GB/s, pinned={x.is_pinned()}")
# run_from_host with device events per step
tr.run_from_host(order, host)
torch.cuda.synchronize()
t0 = time.perf_counter()
tr.run_from_host(order, host)
print(f"run_from_host (warm graphs): wall/step {1e3 * (time.perf_counter() - t0) / len(order):.3f} ms")
