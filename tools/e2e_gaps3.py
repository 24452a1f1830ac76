import sys
import time

import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer  # noqa: E402

sc, cache, targets = bench.build_problem(1)
tr = Stage1Trainer(sc.cloud, cache, list(zip(sc.cameras, targets)), Stage1Config())
order = [k % 20 for k in range(60)]


def timeit(name, graphs):
    tr.use_graphs = graphs
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in order]
    t0 = time.perf_counter()
    for k, v in enumerate(order):
        ev[k][0].record()
        tr.iterate(v)
        ev[k][1].record()
    torch.cuda.synchronize()
    dev = sum(a.elapsed_time(b) for a, b in ev) / len(order)
    print(f"{name}: wall {1e3 * (time.perf_counter() - t0) / len(order):.3f} ms/step, "
          f"device {dev:.3f} ms/step", flush=True)


for v in range(20):
    tr.iterate(v, graph=False)
timeit("eager 1", False)
timeit("graphs 1 (captures)", True)
timeit("graphs 2", True)
timeit("eager 2", False)
timeit("graphs 3", True)
