"""tcgen05 building blocks (csrc/umma.cuh) against host GEMMs: K-major M=128
and MN-major (transposed-tile) M=64 UMMAs with TMEM accumulators."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _tf32(a):
    b = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    b = (b + 0x1000) & 0xFFFFE000  # round to nearest (ties away), 10-bit mantissa
    return b.view(np.float32).astype(np.float64)


@pytest.mark.parametrize("test", [0, 1])
def test_umma_tf32(test):
    """K-major A and B (the only layout the kernels use), M = 128 and M = 64."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import ctypes as C

    from paper_2403_01444_b200 import _lib
    from paper_2403_01444_b200.device import ptr, stream

    lib = _lib.load()
    rng = np.random.default_rng(test)
    M, N, K = (128, 64, 32) if test == 0 else (64, 40, 64)
    a, b = rng.normal(size=(M, K)), rng.normal(size=(N, K))
    ref = _tf32(a) @ _tf32(b).T
    da = torch.tensor(a, dtype=torch.float32, device="cuda")
    db = torch.tensor(b, dtype=torch.float32, device="cuda")
    dd = torch.full(ref.shape, float("nan"), dtype=torch.float32, device="cuda")
    assert lib.ss_selftest_umma(M, N, K, 0, ptr(da), ptr(db), ptr(dd), stream()) == 0
    out = dd.cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-4)


def test_umma_tf32_a_from_tmem():
    """A operand in TMEM (tcgen05.st, row i in lane i), B K-major in smem."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_01444_b200 import _lib
    from paper_2403_01444_b200.device import ptr, stream

    lib = _lib.load()
    rng = np.random.default_rng(7)
    M, N, K = 128, 64, 64
    a, b = rng.normal(size=(M, K)), rng.normal(size=(N, K))
    ref = _tf32(a) @ _tf32(b).T
    da = torch.tensor(a, dtype=torch.float32, device="cuda")
    db = torch.tensor(b, dtype=torch.float32, device="cuda")
    dd = torch.full(ref.shape, float("nan"), dtype=torch.float32, device="cuda")
    assert lib.ss_selftest_umma(M, N, K, 32, ptr(da), ptr(db), ptr(dd), stream()) == 0
    out = dd.cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("mode,rows,hidden,cfg", [(1, 5000, 2, 1), (2, 5000, 2, 1),
                                                  (1, 250000, 2, 1), (1, 200003, 1, 1),
                                                  (1, 20000, 1, 0)])
def test_tensor_core_decoder_matches_fp32(mode, rows, hidden, cfg):
    """ss_ntc_forward with the tcgen05 decoder (3xTF32 / tf32) vs the FFMA path.
    The large cases give every CTA many tiles (both pipeline slots, odd tile
    counts, a ragged last tile)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_01444_b200 import _lib, scenes
    from paper_2403_01444_b200.ntc import NeuralTransformationCache
    from paper_2403_01444_b200.types import HashGridConfig

    lib = _lib.load()
    sc = scenes.config(cfg)  # cfg 0: 16 input features; cfg 1: 32
    cache = NeuralTransformationCache(HashGridConfig.from_any(sc.grid), hidden_layers=hidden,
                                      output_init="random")
    cache.tables[:] = np.random.default_rng(0).uniform(-0.5, 0.5, size=cache.tables.shape)
    x = sc.cloud["means"][:rows]
    lib.ss_set_mlp_mode(0)
    ref, _, _ = cache.forward(x)
    ref = np.concatenate([ref, cache.forward(x)[1]], 1)
    lib.ss_set_mlp_mode(mode)
    try:
        d_mu, d_q, _ = cache.forward(x)
    finally:
        lib.ss_set_mlp_mode(1)
    out = np.concatenate([d_mu, d_q], 1)
    tol = 2e-6 if mode == 1 else 2e-3
    assert np.abs(out - ref).max() <= tol * np.abs(ref).max()


def _bf16(a):
    import torch

    return torch.tensor(a, dtype=torch.float32).to(torch.bfloat16).double().numpy()


@pytest.mark.parametrize("M,N,flags", [(128, 64, 0), (128, 64, 2), (64, 8, 3), (64, 72, 3),
                                       (64, 40, 3), (64, 24, 1), (128, 32, 2)])
def test_umma_bf16_layouts(M, N, flags):
    """kind::f16 (bf16) UMMA: K-major and MN-major (transposed-tile) operands,
    the layouts the decoder backward uses."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_01444_b200 import _lib
    from paper_2403_01444_b200.device import ptr, stream

    lib = _lib.load()
    K = 128 if M == 64 else 32
    a_mn, b_mn = flags & 1, (flags >> 1) & 1
    rng = np.random.default_rng(M + N + flags)
    A = rng.normal(size=(K, M) if a_mn else (M, K))
    B = rng.normal(size=(K, N) if b_mn else (N, K))
    ref = (_bf16(A).T if a_mn else _bf16(A)) @ (_bf16(B) if b_mn else _bf16(B).T)
    da = torch.tensor(A, dtype=torch.float32, device="cuda")
    db = torch.tensor(B, dtype=torch.float32, device="cuda")
    dd = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    assert lib.ss_selftest_umma(M, N, K, flags | 16, ptr(da), ptr(db), ptr(dd), stream()) == 0
    np.testing.assert_allclose(dd.cpu().numpy().astype(np.float64), ref, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("cfg,hidden,rows", [(1, 2, 3001), (0, 2, 3001), (0, 1, 3001),
                                             (1, 2, 150001)])
def test_tensor_core_decoder_backward_matches_fp32(cfg, hidden, rows):
    """ss_ntc_backward with the tcgen05 decoder backward (bf16 hi/lo split) vs
    the FFMA fp32 path: every weight, bias and table gradient, norm-relative."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_01444_b200 import _lib, scenes
    from paper_2403_01444_b200.ntc import NeuralTransformationCache
    from paper_2403_01444_b200.types import HashGridConfig

    lib = _lib.load()
    sc = scenes.config(cfg)
    cache = NeuralTransformationCache(HashGridConfig.from_any(sc.grid), hidden_layers=hidden,
                                      output_init="random")
    rng = np.random.default_rng(1)
    cache.tables[:] = rng.uniform(-0.5, 0.5, size=cache.tables.shape)
    x = sc.cloud["means"][:rows]  # ragged last tile; 150001 rows: many tiles per CTA
    g_mu, g_q = rng.normal(size=(len(x), 3)), rng.normal(size=(len(x), 4))
    out = {}
    for mode in (0, 1):
        lib.ss_set_mlp_mode(mode)
        try:
            _, _, ctx = cache.forward(x)
            out[mode], _ = cache.backward(ctx, g_mu, g_q)
        finally:
            lib.ss_set_mlp_mode(1)
    for k, ref in out[0].items():
        err = np.linalg.norm(out[1][k] - ref) / max(np.linalg.norm(ref), 1e-30)
        assert err <= 2e-5, f"{k}: rel err {err:.2e}"
