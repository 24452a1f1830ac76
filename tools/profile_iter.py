"""One Stage-1 iteration of config 1 inside cudaProfilerStart/Stop, after
warm-up, for `ncu --profile-from-start off` captures:

  ncu --profile-from-start off --set full -o prof python tools/profile_iter.py
"""
import sys

import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 4
sc, cache, targets = bench.build_problem(cfg)
tr = Stage1Trainer(sc.cloud, cache, list(zip(sc.cameras, targets)), Stage1Config())
for k in range(warm):
    tr.iterate(k % len(sc.cameras), graph=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
tr.iterate(warm % len(sc.cameras), graph=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("pairs", int(tr.pairs_of_last(1)[0]))
