"""Drop-in for splatstream.ntc / splatstream.optim (ntc.py:23-293, optim.py:17-72).

`NeuralTransformationCache` keeps the reference's host-visible parameter
arrays (`tables` (L,T,F), `weights[i]` (fan_in, fan_out), `biases[i]`, float64
on the float32 lattice, initialised with the same RNG sequence) so code that
reads or edits them keeps working; every compute call (encode, forward,
backward, Adam) runs in libss_b200.so on the current parameters.  The
device-resident fast path for the Stage-1 loop is `stage1.Stage1Trainer`.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .device import (empty_bytes, grid_struct, mlp_layout, mlp_struct, pack_params, ptr,
                     require_cuda, stream, to_dev, unpack_params)
from .errors import DataError
from .types import HashGridConfig

__all__ = ["HASH_PRIMES", "HashGridConfig", "EncodeContext", "ForwardContext",
           "NeuralTransformationCache", "Adam"]

HASH_PRIMES = (1, 2654435761, 805459861)  # ntc.py:23


@dataclass
class EncodeContext:
    corner_idx: np.ndarray  # (B, L, 8) int64
    corner_w: np.ndarray  # (B, L, 8)
    touched: list = field(default_factory=list)
    means: np.ndarray | None = None  # the encoded points (the device recomputes from them)


@dataclass
class ForwardContext:
    encode: EncodeContext
    features: np.ndarray
    hidden: list
    out7: np.ndarray | None = None


class NeuralTransformationCache:
    def __init__(self, grid: HashGridConfig = HashGridConfig(), hidden_layers: int = 2,
                 hidden_dim: int = 64, output_init: str = "identity", seed: int = 0,
                 mlp_dtype: str = "f32") -> None:
        # mlp_dtype (extension, keyword-only use): "f16" runs the decoder with
        # fp16 weights and activations, fp32 accumulation (BASELINE config 1);
        # parameters and Adam state stay fp32 / float64 as in the reference
        if output_init not in ("identity", "random"):
            raise DataError(f"unknown output_init {output_init!r}")
        if hidden_layers not in (1, 2) or hidden_dim > 64:
            raise DataError("the CUDA decoder supports 1-2 hidden layers of width <= 64")
        self.grid = HashGridConfig.from_any(grid)
        self.hidden_layers = hidden_layers
        self.hidden_dim = hidden_dim
        self.output_init = output_init
        if mlp_dtype not in ("f32", "f16"):
            raise DataError(f"unknown mlp_dtype {mlp_dtype!r}")
        self.mlp_dtype = mlp_dtype
        g = self.grid
        # identical RNG sequence to ntc.py:100-123
        rng = np.random.default_rng(seed)
        self.tables = rng.uniform(-1e-4, 1e-4, size=(g.n_levels, g.table_size, g.n_features))
        in_dim = g.n_levels * g.n_features
        if in_dim > 64:
            raise DataError("n_levels * n_features must be <= 64")
        self.weights, self.biases = [], []
        dims = [in_dim] + [hidden_dim] * hidden_layers
        for a, b in zip(dims[:-1], dims[1:]):
            bound = np.sqrt(6.0 / (a + b))
            self.weights.append(rng.uniform(-bound, bound, size=(a, b)))
            self.biases.append(np.zeros(b))
        if output_init == "identity":
            self.weights.append(np.zeros((dims[-1], 7)))
            ob = np.zeros(7)
            ob[3] = 1.0
            self.biases.append(ob)
        else:
            bound = np.sqrt(6.0 / (dims[-1] + 7))
            self.weights.append(rng.uniform(-bound, bound, size=(dims[-1], 7)))
            self.biases.append(rng.normal(scale=0.1, size=7))
        self.quantize_float32()
        self.adam = Adam(self._param_dict())

    # ---- parameter plumbing (ntc.py:131-158)
    def _param_dict(self) -> dict:
        p = {f"table_{l}": self.tables[l] for l in range(self.grid.n_levels)}
        for i, (w, b) in enumerate(zip(self.weights, self.biases)):
            p[f"w_{i}"] = w
            p[f"b_{i}"] = b
        return p

    def get_params(self) -> dict:
        return {k: v.copy() for k, v in self._param_dict().items()}

    def set_params(self, params: dict) -> None:
        live = self._param_dict()
        if set(params) != set(live):
            raise DataError("parameter snapshot does not match cache layout")
        for k, v in live.items():
            v[:] = params[k]

    def quantize_float32(self) -> None:
        for v in self._param_dict().values():
            v[:] = v.astype(np.float32).astype(np.float64)

    def reset_adam(self) -> None:
        self.adam.reset()

    # ---- device views of the current parameters
    def _dev(self):
        dev = require_cuda()
        m = mlp_struct(self.weights[0].shape[0], self.hidden_dim, self.hidden_layers,
                       self.mlp_dtype)
        lay = mlp_layout(m)
        return (dev, grid_struct(self.grid), m, lay, to_dev(self.tables, dev=dev),
                to_dev(pack_params(self.weights, self.biases, lay), dev=dev))

    def _touched(self, dev, gs, x_dev, n):
        lib = _lib.load()
        T = self.grid.table_size
        mask = torch.zeros(self.grid.n_levels * T, dtype=torch.uint8, device=dev)
        _lib.check(lib.ss_ntc_touched(C.byref(gs), n, ptr(x_dev), None, ptr(mask), stream()),
                   "encode")
        mk = mask.view(self.grid.n_levels, T).cpu().numpy()
        return [np.flatnonzero(mk[l]) for l in range(self.grid.n_levels)]

    # ---- encoding (ntc.py:161-216)
    def encode(self, x):
        x = np.asarray(x, dtype=np.float64).reshape(-1, 3)
        lib = _lib.load()
        dev, gs, m, lay, tab, par = self._dev()
        n, L = len(x), self.grid.n_levels
        xd = to_dev(x, dev=dev)
        idx = torch.zeros(max(n, 1), L, 8, dtype=torch.int32, device=dev)
        w = torch.zeros(max(n, 1), L, 8, dtype=torch.float32, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.check(lib.ss_ntc_encode(C.byref(gs), n, ptr(xd), ptr(idx), ptr(w), ptr(status),
                                     stream()), "encode")
        _lib.check_flags(int(status.item()))
        ctx = EncodeContext(corner_idx=idx[:n].cpu().numpy().astype(np.int64),
                            corner_w=w[:n].cpu().numpy().astype(np.float64),
                            touched=self._touched(dev, gs, xd, n), means=x.copy())
        return self._features(x), ctx

    def _run_forward(self, x):
        lib = _lib.load()
        dev, gs, m, lay, tab, par = self._dev()
        n = len(x)
        nf = self.grid.n_levels * self.grid.n_features
        out7 = torch.zeros(max(n, 1), 7, dtype=torch.float32, device=dev)
        feats = torch.zeros(max(n, 1), nf, dtype=torch.float32, device=dev)
        xd = to_dev(x, dev=dev)  # keep alive until the launch is enqueued
        _lib.check(lib.ss_ntc_forward(C.byref(gs), C.byref(m), n, ptr(xd), None,
                                      ptr(tab), ptr(par), ptr(out7), ptr(feats), stream()),
                   "forward")
        return (out7[:n].cpu().numpy().astype(np.float64),
                feats[:n].cpu().numpy().astype(np.float64))

    def _features(self, x):
        return self._run_forward(np.asarray(x, dtype=np.float64).reshape(-1, 3))[1]

    def gather_features(self, ctx: EncodeContext):
        return self._features(ctx.means)

    # ---- decoder (ntc.py:219-248)
    def forward(self, mu, encode_ctx: EncodeContext | None = None):
        mu = np.asarray(mu, dtype=np.float64).reshape(-1, 3)
        if len(mu) == 0:
            L = self.grid.n_levels
            enc = EncodeContext(np.zeros((0, L, 8), dtype=np.int64), np.zeros((0, L, 8)),
                                [np.empty(0, dtype=np.int64)] * L, mu)
            ctx = ForwardContext(enc, np.zeros((0, L * self.grid.n_features)), [], np.zeros((0, 7)))
            return np.zeros((0, 3)), np.zeros((0, 4)), ctx
        if encode_ctx is None:
            _, encode_ctx = self.encode(mu)
        out7, feats = self._run_forward(mu)
        ctx = ForwardContext(encode=encode_ctx, features=feats, hidden=[], out7=out7)
        return out7[:, :3], out7[:, 3:], ctx

    def backward(self, ctx: ForwardContext, grad_d_mu, grad_d_q):
        """ntc.py:250-288: (grads, touched) with dense per-level table gradients."""
        lib = _lib.load()
        dev, gs, m, lay, tab, par = self._dev()
        x = ctx.encode.means
        n = len(x)
        g7 = np.concatenate([np.asarray(grad_d_mu, dtype=np.float64).reshape(n, 3),
                             np.asarray(grad_d_q, dtype=np.float64).reshape(n, 4)], axis=1)
        g_tab = torch.zeros_like(tab)
        g_par = torch.zeros_like(par)
        if n:
            xd, g7d = to_dev(x, dev=dev), to_dev(g7, dev=dev)  # alive across the launch
            _lib.check(lib.ss_ntc_backward(C.byref(gs), C.byref(m), n, ptr(xd),
                                           None, ptr(tab), ptr(par), ptr(g7d),
                                           ptr(g_tab), ptr(g_par), None, stream()), "backward")
        gt = g_tab.cpu().numpy().astype(np.float64)
        ws, bs = unpack_params(g_par.cpu().numpy(), [w.shape for w in self.weights], lay)
        grads, touched = {}, {}
        for i in range(len(ws)):
            grads[f"w_{i}"] = ws[i]
            grads[f"b_{i}"] = bs[i]
        for l in range(self.grid.n_levels):
            grads[f"table_{l}"] = gt[l]
            touched[f"table_{l}"] = ctx.encode.touched[l]
        return grads, touched

    def adam_step(self, grads: dict, lr: float, touched: dict) -> None:
        self.adam.step(grads, lr, touched)


class Adam:
    """optim.py:17-72 with the update on the GPU (float64 moments, lazy rows)."""

    def __init__(self, params: dict, beta1: float = 0.9, beta2: float = 0.999,
                 eps: float = 1e-15) -> None:
        self.params = params
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.m = {k: np.zeros_like(v) for k, v in params.items()}
        self.v = {k: np.zeros_like(v) for k, v in params.items()}
        self.step_count = 0

    def step(self, grads: dict, lr, touched: dict | None = None) -> None:
        lib = _lib.load()
        dev = require_cuda()
        for key, p in self.params.items():
            g = grads.get(key)
            if g is None:
                continue
            lr_k = lr[key] if isinstance(lr, dict) else lr
            rows = touched.get(key) if touched is not None else None
            width = int(np.prod(p.shape[1:])) if p.ndim > 1 else 1
            pd = to_dev(p, dev=dev)
            gd = to_dev(np.asarray(g), dev=dev)
            md = to_dev(self.m[key], torch.float64, dev)
            vd = to_dev(self.v[key], torch.float64, dev)
            mask = None
            if rows is not None:
                mk = np.zeros(p.shape[0] if p.ndim else 1, dtype=np.uint8)
                mk[np.asarray(rows, dtype=np.int64)] = 1
                mask = to_dev(mk, torch.uint8, dev)
            step = torch.full((1,), self.step_count, dtype=torch.int32, device=dev)
            _lib.check(lib.ss_adam_step(p.size, ptr(pd), ptr(gd), ptr(md), ptr(vd), ptr(mask),
                                        width, 0, None, None, None, None, ptr(step), float(lr_k),
                                        self.beta1, self.beta2, self.eps, 0, stream()), "adam")
            p[...] = pd.cpu().numpy().reshape(p.shape)
            self.m[key][...] = md.cpu().numpy().reshape(p.shape)
            self.v[key][...] = vd.cpu().numpy().reshape(p.shape)
        self.step_count += 1

    def reset(self) -> None:
        for k in self.m:
            self.m[k][:] = 0.0
            self.v[k][:] = 0.0
        self.step_count = 0
