"""Drop-in for splatstream.transform (transform.py:31-135) on the GPU.

With this package's `NeuralTransformationCache` the cache forward and the
transform run as one fused kernel (ss_apply_ntc / ss_apply_ntc_backward).
Any other object exposing `.grid` and `.forward(mu, encode_ctx)` (the
reference's duck-typed stubs, test_transform.py:24-46) is honoured: its
forward output is applied by the standalone transform kernels and its
`.backward` receives the transform's vector-Jacobian product.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import DeviceCloud, ptr, require_cuda, stream, to_dev
from .ntc import NeuralTransformationCache
from .types import GaussianCloud, HashGridConfig

__all__ = ["TransformContext", "apply_ntc", "apply_ntc_backward"]


@dataclass
class TransformContext:
    cache: object
    fwd: object
    inside: np.ndarray
    d_q_raw: np.ndarray
    d_q_unit: np.ndarray
    q_src: np.ndarray
    sh_in: np.ndarray
    rotate_sh: bool
    cloud: GaussianCloud | None = None
    out7: np.ndarray | None = None


def _inside(cache, means):
    g = HashGridConfig.from_any(cache.grid)
    lo = np.asarray(g.aabb_min, dtype=np.float64)
    hi = np.asarray(g.aabb_max, dtype=np.float64)
    return np.flatnonzero(np.all((means >= lo) & (means <= hi), axis=1))


def apply_ntc(cloud, cache, rotate_sh: bool = True, encode_ctx=None):
    """transform.py:53-96: (transformed GaussianCloud, TransformContext)."""
    lib = _lib.load()
    dev = require_cuda()
    cloud = GaussianCloud.from_any(cloud)
    inside = _inside(cache, cloud.means)
    dc = DeviceCloud(cloud, dev)
    out_m, out_r, out_s = dc.means.clone(), dc.rotations.clone(), dc.sh.clone()
    rows = to_dev(inside.astype(np.int32), torch.int32, dev)
    n_in = len(inside)
    out7 = torch.zeros(max(n_in, 1), 7, dtype=torch.float32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    fwd = None
    if isinstance(cache, NeuralTransformationCache):
        _, gs, m, _, tab, par = cache._dev()
        _lib.check(lib.ss_apply_ntc(C.byref(gs), C.byref(m), C.byref(dc.struct()), n_in,
                                    ptr(rows), ptr(tab), ptr(par), int(rotate_sh), ptr(out_m),
                                    ptr(out_r), ptr(out_s), ptr(out7), ptr(status), stream()),
                   "apply_ntc")
        o7 = out7[:n_in].cpu().numpy().astype(np.float64)
        if encode_ctx is None and n_in:
            _, encode_ctx = cache.encode(cloud.means[inside])
        from .ntc import ForwardContext

        fwd = ForwardContext(encode=encode_ctx, features=np.zeros((n_in, 0)), hidden=[], out7=o7)
    else:
        d_mu, d_q, fwd = cache.forward(cloud.means[inside], encode_ctx=encode_ctx)
        o7 = np.concatenate([np.asarray(d_mu, dtype=np.float64).reshape(-1, 3),
                             np.asarray(d_q, dtype=np.float64).reshape(-1, 4)], axis=1)
        if n_in:
            out7 = to_dev(o7, dev=dev)
            _lib.check(lib.ss_transform_apply(C.byref(dc.struct()), n_in, ptr(rows), ptr(out7),
                                              int(rotate_sh), ptr(out_m), ptr(out_r), ptr(out_s),
                                              ptr(status), stream()), "apply_ntc")
    _lib.check_flags(int(status.item()))
    d_q = o7[:, 3:]
    norm = np.linalg.norm(d_q, axis=1, keepdims=True) if n_in else np.ones((0, 1))
    out = GaussianCloud(out_m.cpu().numpy(), out_r.cpu().numpy(), cloud.log_scales.copy(),
                        cloud.opacity_logits.copy(), out_s.cpu().numpy())
    ctx = TransformContext(cache=cache, fwd=fwd, inside=inside, d_q_raw=d_q,
                           d_q_unit=d_q / np.maximum(norm, 1e-300), q_src=cloud.rotations[inside],
                           sh_in=cloud.sh[inside, 1:, :].copy(), rotate_sh=rotate_sh,
                           cloud=cloud, out7=o7)
    return out, ctx


def apply_ntc_backward(ctx: TransformContext, d_means_t, d_rotations_t, d_sh_t):
    """transform.py:99-135: cache-parameter (grads, touched)."""
    lib = _lib.load()
    dev = require_cuda()
    cloud = ctx.cloud
    dc = DeviceCloud(cloud, dev)
    n_in = len(ctx.inside)
    rows = to_dev(ctx.inside.astype(np.int32), torch.int32, dev)
    dm = to_dev(np.asarray(d_means_t, dtype=np.float64), dev=dev)
    dr = to_dev(np.asarray(d_rotations_t, dtype=np.float64), dev=dev)
    ds = to_dev(np.asarray(d_sh_t, dtype=np.float64), dev=dev)
    cache = ctx.cache
    if isinstance(cache, NeuralTransformationCache):
        _, gs, m, lay, tab, par = cache._dev()
        g_tab = torch.zeros_like(tab)
        g_par = torch.zeros_like(par)
        scratch = torch.empty(max(lib.ss_apply_ntc_backward_bytes(n_in), 256), dtype=torch.uint8,
                              device=dev)
        if n_in:
            _lib.check(lib.ss_apply_ntc_backward(C.byref(gs), C.byref(m), C.byref(dc.struct()),
                                                 n_in, ptr(rows), ptr(tab), ptr(par),
                                                 int(ctx.rotate_sh), ptr(dm), ptr(dr), ptr(ds),
                                                 ptr(g_tab), ptr(g_par), ptr(scratch), stream()),
                       "apply_ntc_backward")
        from .device import unpack_params

        gt = g_tab.cpu().numpy().astype(np.float64)
        ws, bs = unpack_params(g_par.cpu().numpy(), [w.shape for w in cache.weights], lay)
        grads, touched = {}, {}
        for i in range(len(ws)):
            grads[f"w_{i}"], grads[f"b_{i}"] = ws[i], bs[i]
        for l in range(cache.grid.n_levels):
            grads[f"table_{l}"] = gt[l]
            touched[f"table_{l}"] = (ctx.fwd.encode.touched[l] if ctx.fwd.encode is not None
                                     else np.empty(0, dtype=np.int64))
        return grads, touched
    g7 = torch.zeros(max(n_in, 1), 7, dtype=torch.float32, device=dev)
    if n_in:
        o7 = to_dev(ctx.out7, dev=dev)  # alive across the launch
        _lib.check(lib.ss_transform_vjp(C.byref(dc.struct()), n_in, ptr(rows),
                                        ptr(o7), int(ctx.rotate_sh),
                                        ptr(dm), ptr(dr), ptr(ds), ptr(g7), stream()),
                   "apply_ntc_backward")
    g = g7[:n_in].cpu().numpy().astype(np.float64)
    return cache.backward(ctx.fwd, g[:, :3], g[:, 3:])
