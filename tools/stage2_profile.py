"""Where Stage-2 time goes at cfg1 scale: wall clock per iteration vs the GPU
time of the same iterations (CUDA events around each iteration)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2403_01444_b200 import stage2 as S2  # noqa: E402

sc, cache, targets = bench.build_problem(1)
rng = np.random.default_rng(0)
cfg = S2.AdditionConfig(quantity_control=False)
sel = np.sort(rng.choice(len(sc.cloud["means"]), 5000, replace=False))
add = S2.spawn_gaussians(sc.cloud, sel, cfg, rng)
views = [(c, t.cpu().numpy()) for c, t in zip(sc.cameras, targets)]
S2.stage2_optimize(sc.cloud, add, views[:2], cfg, 2, np.random.default_rng(1))
torch.cuda.synchronize()
t0 = time.perf_counter()
S2.stage2_optimize(sc.cloud, add, views, cfg, 20, np.random.default_rng(1))
torch.cuda.synchronize()
print(f"wall per iteration {1e3 * (time.perf_counter() - t0) / 20:.2f} ms (incl. setup)")
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
S2.stage2_optimize(sc.cloud, add, views, cfg, 20, np.random.default_rng(1))
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
