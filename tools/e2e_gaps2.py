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
tr.run_from_host(order, host)
for v in range(20):
    tr.iterate(v)
torch.cuda.synchronize()


def timeit(name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    print(f"{name}: {1e3 * (time.perf_counter() - t0) / len(order):.3f} ms/step", flush=True)


def a():
    for v in order:
        tr.iterate(v)


losses = torch.empty(len(order), dtype=torch.float64, pin_memory=True)


def b():
    for k, v in enumerate(order):
        tr.iterate(v)
        losses[k:k + 1].copy_(tr.loss_dev, non_blocking=True)


copy = torch.cuda.Stream()
buf = [torch.empty_like(targets[0]) for _ in range(2)]


def c():  # H2D on a side stream, unrelated buffers, resident targets
    for k, v in enumerate(order):
        with torch.cuda.stream(copy):
            buf[k & 1].view(-1)[: host[v].numel()].copy_(host[v].view(-1), non_blocking=True)
        tr.iterate(v)


timeit("graphs, resident", a)
timeit("graphs + loss D2H", b)
timeit("graphs + side-stream H2D (no deps)", c)
timeit("run_from_host", lambda: tr.run_from_host(order, host))
