"""Probe the kind::f16 (bf16) UMMA operand layouts on the device: K-major and
MN-major A/B, both LBO/SBO assignments for MN-major, M = 64 and 128."""
import sys

import numpy as np
import torch

sys.path.insert(0, '/root/repo')
from paper_2403_01444_b200 import _lib  # noqa: E402
from paper_2403_01444_b200.device import ptr, stream  # noqa: E402

lib = _lib.load()


def bf16(a):
    return torch.tensor(a, dtype=torch.float32).to(torch.bfloat16).to(torch.float64).numpy()


for M in (128, 64):
    for N in (8, 40, 72):
        for flags in (0, 1, 2, 3):
            K = 32
            a_mn, b_mn = flags & 1, (flags >> 1) & 1
            rng = np.random.default_rng(flags + N)
            A = rng.normal(size=(K, M) if a_mn else (M, K))
            B = rng.normal(size=(K, N) if b_mn else (N, K))
            opA = bf16(A).T if a_mn else bf16(A)
            opB = bf16(B) if b_mn else bf16(B).T
            ref = opA @ opB
            da = torch.tensor(A, dtype=torch.float32, device="cuda")
            db = torch.tensor(B, dtype=torch.float32, device="cuda")
            dd = torch.zeros((M, N), dtype=torch.float32, device="cuda")
            rc = lib.ss_selftest_umma(M, N, K, flags | 16, ptr(da), ptr(db), ptr(dd), stream())
            torch.cuda.synchronize()
            out = dd.cpu().numpy()
            print(f"M={M} N={N} a_mn={a_mn} b_mn={b_mn} swap={(flags >> 2) & 1} rc={rc} "
                  f"maxerr={np.abs(out - ref).max():.3e} maxout={np.abs(out).max():.3f}", flush=True)
