"""Event timeline of the warp-specialised decoder forward (CTA 0): when the
epilogue warps publish operands / see MMA completions and when the MMA warp
sees operands / commits, cycles relative to the first event.
  python tools/mlp_events.py"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_2403_01444_b200 import _lib, scenes  # noqa: E402
from paper_2403_01444_b200.ntc import NeuralTransformationCache  # noqa: E402
from paper_2403_01444_b200.types import HashGridConfig  # noqa: E402

lib = _lib.load()
sc = scenes.config(1)
cache = NeuralTransformationCache(HashGridConfig.from_any(sc.grid), output_init="random")
x = sc.cloud["means"]
for _ in range(3):
    cache.forward(x)
torch.cuda.synchronize()
buf = (C.c_uint64 * 256)()
lib.ss_debug_mlp_events(buf)
t = np.array(buf, dtype=np.int64).reshape(2, 128)
t0 = min(t[0][0], t[1][0])
ev = [(int(v - t0), "E") for v in t[0][:40] if v] + [(int(v - t0), "M") for v in t[1][:40] if v]
ev.sort()
for v, k in ev:
    print(f"{v:8d} {'    ' if k == 'M' else ''}{k}")
