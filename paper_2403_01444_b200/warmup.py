"""NTC warm-up on the device: the reference's
`warmup_train` (ntc.py:296-333) with the same signature and batch sampling,
one `ss_ntc_warmup_step` per iteration (touched rows, tcgen05 decoder forward,
identity-pull loss losses.py:151-180, decoder backward + table scatter, lazy
Adam).

Batches are drawn on the host with the reference's numpy calls (so the same
seed gives the same points), staged through two pinned buffers and copied
host->device on the compute stream while the host draws the next batch; the
per-iteration loss sums stay on the device until the end.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .device import (empty_bytes, grid_struct, mlp_layout, mlp_struct, pack_params, ptr,
                     require_cuda, stream, to_dev, unpack_params)
from .errors import DataError
from .types import HashGridConfig


def warmup_train(cache, initial_means, noise_sigma: float, iterations: int, lr: float = 0.002,
                 batch_size: int = 65536, seed: int = 0):
    """Pull the cache toward the identity transform on noisy scene points
    (ntc.py:296-333).  Returns (parameter snapshot quantized through float32,
    per-iteration loss history); the cache is left holding the snapshot with
    fresh optimizer state."""
    means = np.asarray(initial_means, dtype=np.float64).reshape(-1, 3)
    if len(means) == 0:
        raise DataError("warmup_train needs at least one mean")
    dev = require_cuda()
    lib = _lib.load()
    grid = HashGridConfig.from_any(cache.grid)
    weights = [np.asarray(w) for w in cache.weights]
    biases = [np.asarray(b) for b in cache.biases]
    shapes = [w.shape for w in weights]
    m = mlp_struct(weights[0].shape[0], weights[0].shape[1], len(weights) - 1,
                   getattr(cache, "mlp_dtype", "f32"))
    lay = mlp_layout(m)
    gs = grid_struct(grid)
    tables = to_dev(np.asarray(cache.tables), dev=dev)
    params = to_dev(pack_params(weights, biases, lay), dev=dev)
    f32 = dict(dtype=torch.float32, device=dev)
    f64 = dict(dtype=torch.float64, device=dev)
    g_tab, g_par = torch.zeros(tables.numel(), **f32), torch.zeros(params.numel(), **f32)
    m_tab, v_tab = torch.zeros(tables.numel(), **f64), torch.zeros(tables.numel(), **f64)
    m_par, v_par = torch.zeros(params.numel(), **f64), torch.zeros(params.numel(), **f64)
    mask = torch.zeros(grid.n_levels * grid.table_size, dtype=torch.uint8, device=dev)
    step = torch.zeros(1, dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    take = min(batch_size, len(means))
    scratch = empty_bytes(lib.ss_ntc_warmup_bytes(take), dev)
    sums = torch.zeros(max(iterations, 1), **f64)
    host = [torch.empty((take, 3), dtype=torch.float32).pin_memory() for _ in range(2)]
    devb = [torch.empty((take, 3), **f32) for _ in range(2)]
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    rng = np.random.default_rng(seed)
    lo, hi = np.asarray(grid.aabb_min), np.asarray(grid.aabb_max)
    for it in range(iterations):
        sel = rng.choice(len(means), size=take, replace=False)
        batch = np.clip(means[sel] + rng.normal(scale=noise_sigma, size=(take, 3)), lo, hi)
        b = it & 1
        copied[b].synchronize()  # the copy that last read this pinned buffer is done
        host[b].numpy()[:] = batch
        devb[b].copy_(host[b], non_blocking=True)
        copied[b].record()
        _lib.check(lib.ss_ntc_warmup_step(C.byref(gs), C.byref(m), take, ptr(devb[b]), ptr(tables),
                                          ptr(params), ptr(g_tab), ptr(g_par), ptr(m_tab),
                                          ptr(v_tab), ptr(m_par), ptr(v_par), ptr(mask),
                                          ptr(step), lr, ptr(scratch), ptr(sums[it:]),
                                          ptr(status), stream()), "warmup_train")
    torch.cuda.current_stream().synchronize()
    _lib.check_flags(int(status.item()), "warmup_loss")
    history = (sums[:iterations].cpu().numpy() / take).tolist()
    cache.tables[:] = tables.view(cache.tables.shape).cpu().numpy()
    ws, bs = unpack_params(params.cpu().numpy(), shapes, lay)
    for i in range(len(ws)):
        cache.weights[i][:] = ws[i]
        cache.biases[i][:] = bs[i]
    cache.quantize_float32()
    cache.reset_adam()
    return cache.get_params(), history
