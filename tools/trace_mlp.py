"""Stage timeline of the tcgen05 decoder kernels (CTA 0, clock64 cycles) at
config-1 size: python tools/trace_mlp.py"""
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
rng = np.random.default_rng(0)
g_mu, g_q = rng.normal(size=(len(x), 3)), rng.normal(size=(len(x), 4))
for _ in range(3):
    _, _, ctx = cache.forward(x)
    cache.backward(ctx, g_mu, g_q)
torch.cuda.synchronize()
buf = (C.c_uint64 * 128)()
lib.ss_debug_mlp_trace(buf)
t = np.array(buf, dtype=np.int64).reshape(2, 64)
for k, name in enumerate(["forward", "backward"]):
    s = t[k]
    print(name, "start->tile0", s[1] - s[0])
    for it in range(4):
        seg = s[1 + 8 * it: 9 + 8 * it]
        print(f"  tile {it}:", " ".join(f"{int(seg[j + 1] - seg[j]):7d}" if seg[j + 1] and seg[j] else "      -" for j in range(7)),
              " total", int(s[9 + 8 * it] - s[1 + 8 * it]) if s[9 + 8 * it] else "-")
