"""Run ss_render_loss on a cfg1-sized random image pair (for ncu captures of
the SSIM kernels): python tools/loss_probe.py [reps]"""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
from paper_2403_01444_b200 import losses  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rng = np.random.default_rng(0)
img = rng.uniform(0, 1, size=(1014, 1352, 3)).astype(np.float32)
tgt = np.clip(img + rng.normal(scale=0.05, size=img.shape), 0, 1).astype(np.float32)
for _ in range(reps):
    loss, grad = losses.render_loss(img, tgt)
torch.cuda.synchronize()
print(loss)
