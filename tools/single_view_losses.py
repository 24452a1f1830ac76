import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2403_01444_b200 import scenes  # noqa: E402
from paper_2403_01444_b200.device import DeviceCloud  # noqa: E402
from paper_2403_01444_b200.ntc import NeuralTransformationCache  # noqa: E402
from paper_2403_01444_b200.rasterizer import render_device  # noqa: E402
from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer  # noqa: E402
from paper_2403_01444_b200.types import HashGridConfig  # noqa: E402

sc = scenes.config(1)
cache = NeuralTransformationCache(HashGridConfig.from_any(sc.grid), output_init="identity")
moved = scenes.moved_cloud(sc.cloud, np.random.default_rng(7), deg=1.5)
tgt = [render_device(DeviceCloud(moved), c, None, want_touch=False)[0] for c in sc.cameras[:1]]
tr = Stage1Trainer(sc.cloud, cache, list(zip(sc.cameras[:1], tgt)), Stage1Config())
losses = tr.run(iterations=60)
print(np.array2string(losses, precision=5, max_line_width=200))
