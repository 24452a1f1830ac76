"""What the late-frame Stage-1 workload looks like (diagnostic): train the
cfg1 frame to iteration K, then for the next view report the transformed
cloud's depth / footprint statistics and where the tile pairs come from."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from oracle import stage1 as O  # noqa: E402
from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer, view_order  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 144
sc, cache, targets = bench.build_problem(1)
tr = Stage1Trainer(sc.cloud, cache, list(zip(sc.cameras, targets)), Stage1Config())
order = view_order(0, 1, len(sc.cameras), 150)
for t in range(K):
    tr.iterate(order[t])
torch.cuda.synchronize()
cl = tr.transformed_cloud()
cloud = dict(means=cl.means, rotations=cl.rotations, log_scales=cl.log_scales,
             opacity_logits=cl.opacity_logits, sh=cl.sh)
v = order[K]
cam = sc.cameras[v]
pj = O.project(cloud, cam)
rect, vis = O.tile_rects(pj["mean2d"], pj["cov2d"], pj["opacity"], cam["width"], cam["height"], 16,
                         1 / 255)
area = (rect[:, 1] - rect[:, 0] + 1) * (rect[:, 3] - rect[:, 2] + 1) * vis
depth = pj["p_cam"][:, 2]
disp = np.linalg.norm(cl.means - sc.cloud["means"], axis=1)
out = {"iteration": K, "view": v, "pairs": int(area.sum()), "survivors": int(len(depth)),
       "disp_mean": float(disp.mean()), "disp_p99": float(np.quantile(disp, 0.99)),
       "depth_quantiles": [float(x) for x in np.quantile(depth, [0.001, 0.01, 0.1, 0.5])],
       "n_depth_lt_0.5": int((depth < 0.5).sum()), "n_area_gt_1000": int((area > 1000).sum()),
       "pairs_from_area_gt_1000": int(area[area > 1000].sum()),
       "pairs_from_area_gt_100": int(area[area > 100].sum()),
       "opacity_of_big": float(np.mean(pj["opacity"][area > 1000])) if (area > 1000).any() else None,
       "loss_last": tr.last_loss()}
print(json.dumps(out))
