"""The C-ABI library loads on a CPU-only host and exports every symbol the
header declares, with struct layouts that match the ctypes binding."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ss_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2403_01444_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        from paper_2403_01444_b200 import build

        build.build()
    return _lib.load()


def test_every_header_symbol_exported(lib):
    names = _declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n


def test_binding_covers_header():
    from paper_2403_01444_b200 import _lib

    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert set(_declared()) <= bound


def test_struct_layouts_match(lib):
    import ctypes

    from paper_2403_01444_b200 import _lib

    for i, st in enumerate(_lib.STRUCTS):
        assert lib.ss_struct_size(i) == ctypes.sizeof(st), st.__name__


def test_mlp_layout_padding(lib):
    import ctypes

    from paper_2403_01444_b200 import _lib

    m = _lib.Mlp(32, 64, 2, 7)
    lay = _lib.MlpLayout()
    assert lib.ss_mlp_get_layout(ctypes.byref(m), ctypes.byref(lay)) == 0
    assert (lay.in_pad, lay.total) == (32, 32 * 64 + 64 + 64 * 64 + 64 + 64 * 8 + 8)
    bad = _lib.Mlp(80, 64, 2, 7)
    assert lib.ss_mlp_get_layout(ctypes.byref(bad), ctypes.byref(lay)) == 1
    assert b"unsupported" in lib.ss_last_error()


def test_pack_unpack_roundtrip():
    import numpy as np

    from paper_2403_01444_b200 import _lib
    from paper_2403_01444_b200.device import mlp_layout, pack_params, unpack_params

    _lib.load()
    rng = np.random.default_rng(0)
    for shapes in ([(16, 64), (64, 64), (64, 7)], [(8, 8), (8, 7)], [(32, 40), (40, 40), (40, 7)]):
        ws = [rng.normal(size=s).astype(np.float32).astype(np.float64) for s in shapes]
        bs = [rng.normal(size=s[1]).astype(np.float32).astype(np.float64) for s in shapes]
        lay = mlp_layout(_lib.Mlp(shapes[0][0], shapes[0][1], len(shapes) - 1, 7))
        v = pack_params(ws, bs, lay)
        w2, b2 = unpack_params(v, shapes, lay)
        for a, b in zip(ws + bs, w2 + b2):
            np.testing.assert_array_equal(a, b)


def test_product_path_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2403_01444_b200.device import require_cuda

    with pytest.raises(RuntimeError):
        require_cuda()
