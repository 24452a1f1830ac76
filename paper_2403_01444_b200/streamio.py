"""NTC blob serialisation: the reference's per-frame cache
wire format, written from a reference-shaped cache or straight from the
device parameters of a Stage-1 trainer.

Format (reference streamio.py:81-150, docs/formats.md:29-99), little endian:
  header  struct "<IIIId6dIII": n_levels, n_features, table_size_log2,
          base_resolution, growth_factor (f64), aabb_min[3], aabb_max[3] (f64),
          hidden_layers, hidden_dim, n_outputs (= 7)
  tables  (L, T, F) float32
  then per layer i: W_i (fan_in, fan_out) float32, b_i (fan_out) float32

The bytes are identical to the reference's `serialize_ntc` for the same
parameters (tests/golden/ntc_blob.npz, written by the unmodified reference).
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import FormatError
from .ntc import NeuralTransformationCache
from .types import HashGridConfig

NTC_HEADER = struct.Struct("<IIIId6dIII")


def _header(grid: HashGridConfig, hidden_layers: int, hidden_dim: int, n_out: int) -> bytes:
    g = HashGridConfig.from_any(grid)
    return NTC_HEADER.pack(g.n_levels, g.n_features, g.table_size_log2, g.base_resolution,
                           float(g.growth_factor), *np.asarray(g.aabb_min, dtype=float),
                           *np.asarray(g.aabb_max, dtype=float), hidden_layers, hidden_dim, n_out)


def _pack(grid, hidden_layers, hidden_dim, tables, weights, biases) -> bytes:
    parts = [_header(grid, hidden_layers, hidden_dim, int(np.shape(weights[-1])[1])),
             np.ascontiguousarray(tables).astype("<f4").tobytes()]
    for w, b in zip(weights, biases):
        parts.append(np.ascontiguousarray(w).astype("<f4").tobytes())
        parts.append(np.ascontiguousarray(b).astype("<f4").tobytes())
    return b"".join(parts)


def serialize_ntc(cache) -> bytes:
    """Blob of a reference-shaped cache (streamio.py:84-104)."""
    return _pack(cache.grid, len(cache.weights) - 1, int(np.shape(cache.weights[0])[1]),
                 cache.tables, cache.weights, cache.biases)


def serialize_ntc_device(trainer) -> bytes:
    """Blob straight from a Stage1Trainer's device parameters (one D2H copy
    of the tables and of the packed decoder vector, no cache round trip)."""
    from .device import unpack_params

    tab = trainer.tables.view(trainer.grid_cfg.n_levels, trainer.grid_cfg.table_size,
                              trainer.grid_cfg.n_features).cpu().numpy()
    ws, bs = unpack_params(trainer.params.cpu().numpy(), trainer.w_shapes, trainer.layout)
    return _pack(trainer.grid_cfg, len(ws) - 1, int(ws[0].shape[1]), tab, ws, bs)


def deserialize_ntc(data: bytes) -> NeuralTransformationCache:
    """streamio.py:107-150: a cache holding the blob's parameters, fresh Adam."""
    if len(data) < NTC_HEADER.size:
        raise FormatError("cache payload shorter than its header")
    f = NTC_HEADER.unpack_from(data, 0)
    grid = HashGridConfig(n_levels=f[0], n_features=f[1], table_size_log2=f[2],
                          base_resolution=f[3], growth_factor=f[4], aabb_min=tuple(f[5:8]),
                          aabb_max=tuple(f[8:11]))
    hidden_layers, hidden_dim, n_out = f[11:14]
    cache = NeuralTransformationCache(grid, hidden_layers=hidden_layers, hidden_dim=hidden_dim)
    if cache.weights[-1].shape[1] != n_out:
        raise FormatError(f"cache output width {n_out} unsupported")
    # every parameter array in wire order, as float32 runs after the header
    dests = [cache.tables] + [a for wb in zip(cache.weights, cache.biases) for a in wb]
    sizes = np.array([a.size for a in dests], dtype=np.int64)
    need = NTC_HEADER.size + 4 * int(sizes.sum())
    if len(data) < need:
        raise FormatError("truncated cache payload")
    if len(data) > need:
        raise FormatError(f"cache payload has {len(data) - need} trailing bytes")
    flat = np.frombuffer(data, dtype="<f4", offset=NTC_HEADER.size).astype(np.float64)
    for a, lo, hi in zip(dests, np.cumsum(sizes) - sizes, np.cumsum(sizes)):
        a[...] = flat[lo:hi].reshape(a.shape)
    cache.reset_adam()
    return cache
