"""Cycles per tcgen05.mma (M = 128) issued back to back by one thread:
  python tools/umma_rate.py"""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_2403_01444_b200 import _lib  # noqa: E402
from paper_2403_01444_b200.device import ptr, stream  # noqa: E402

lib = _lib.load()
out = torch.zeros(2, dtype=torch.int64, device="cuda")
for kind, a_tmem, name in ((0, 0, "tf32 SS"), (0, 1, "tf32 TS"), (1, 0, "bf16 SS K-major"),
                           (3, 0, "bf16 SS MN-major"), (5, 0, "bf16 SS K-major 128B-swizzle"),
                           (9, 0, "bf16 SS K-major M=64"), (11, 0, "bf16 SS MN-major M=64"),
                           (17, 0, "bf16 3-product K=64 pattern"),
                           (33, 0, "bf16 dW GEMM M=64 MN/MN K=128"),
                           (1 | 64, 0, "bf16 SS K-major random data"),
                           (33 | 64, 0, "bf16 dW GEMM random data"),
                           (0 | 64, 0, "tf32 SS random data"), (0 | 64, 1, "tf32 TS random data")):
    for N in ((64,) if kind & 16 else ((8, 40, 64, 72, 80) if kind & 32 else ((64,) if kind & 64 else (16, 64, 128)))):
        res = []
        for count in ((24, 264) if kind & 16 else ((16, 256) if not kind & 32 else (16, 256))):
            lib.ss_debug_umma_rate(kind, N, a_tmem, count, ptr(out), stream())
            torch.cuda.synchronize()
            res.append(out.cpu().tolist())
        (t16, i16), (t256, i256) = res
        print(f"{name:30s} N={N:3d}: {(t256 - t16) / 240:6.1f} cyc/MMA (issue {(i256 - i16) / 240:5.1f})")
