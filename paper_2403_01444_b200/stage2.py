"""Stage 2 on the device: the reference's frame-specific
Gaussian addition (adaptive.py:105-288) with the render/loss/backward/Adam
loop resident in HBM.

Each iteration renders the frozen transformed cloud plus the additional
Gaussians (one joint device cloud, the additional rows at its end), takes
the L1 + D-SSIM loss, runs the full-parameter raster backward (means,
rotations, log-scales, opacity logits, SH) and applies Adam with the
per-parameter learning rates to the additional rows only, accumulating the
view-space statistics.  At every epoch boundary the quantity control
(split high-gradient rows, prune dim ones; adaptive.py:155-204) runs on the
host with the reference's exact sequence of generator calls, and the device
state (joint cloud, Adam moments) is rebuilt.

`stage2_optimize` has the reference's signature and returns the optimised
additional batch and the per-iteration losses.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .device import (camera_struct, empty_bytes, pinned, ptr, require_cuda, settings_struct,
                     stream, to_dev)
from .errors import DataError, NumericalError
from .types import Camera, GaussianCloud, LossConfig, RasterSettings

_LR_KEY_BY_PARAM = {"means": "mean", "rotations": "rotation", "log_scales": "scale",
                    "opacity_logits": "opacity", "sh": "sh"}
_FIELDS = ("means", "rotations", "log_scales", "opacity_logits", "sh")


@dataclass
class AdditionConfig:
    """adaptive.py:34-77: knobs for spawning and controlling additional Gaussians."""

    tau_grad: float = 0.00015
    tau_alpha: float = 0.01
    spawn_cov_scale: float = 2.0
    split_scale_factor: float = 0.8
    init_opacity: float = 0.1
    stage2_lrs: dict = field(default_factory=lambda: {"mean": 0.0024, "sh": 0.0375,
                                                      "opacity": 0.75, "scale": 0.075,
                                                      "rotation": 0.015})
    quantity_control: bool = True
    max_additional: int = 10000

    def lr_by_param(self) -> dict:
        return {p: float(self.stage2_lrs[k]) for p, k in _LR_KEY_BY_PARAM.items()}


@dataclass
class ViewspaceStats:
    """adaptive.py:80-97."""

    norm_accum: np.ndarray
    view_count: np.ndarray

    @staticmethod
    def zeros(n: int) -> "ViewspaceStats":
        return ViewspaceStats(np.zeros(n), np.zeros(n, dtype=np.int64))

    def averages(self) -> np.ndarray:
        return self.norm_accum / np.maximum(1, self.view_count)


# ---------------------------------------------------------------- host helpers
# (gaussians.py:33-85 formulas: the split siblings are drawn on the host with
# the reference's generator calls, so the same seed gives the same rows)
def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def _unit(q):
    n = np.linalg.norm(q, axis=-1, keepdims=True)
    if np.any(n < 1e-12):
        raise NumericalError("cannot normalize near-zero quaternion")
    return q / n


def _rotmat(q):
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    return np.stack([np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
                     np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
                     np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)],
                    -2)


def _sample_around(c: dict, idx, cov_scale, rng):
    """adaptive.py:105-114: mu + R (s sqrt(c) z), z ~ N(0, I)."""
    rot = _rotmat(_unit(c["rotations"][idx]))
    sigma = np.exp(c["log_scales"][idx]) * math.sqrt(cov_scale)
    z = rng.standard_normal((len(idx), 3))
    return c["means"][idx] + np.einsum("nij,nj->ni", rot, sigma * z)


def spawn_gaussians(cloud, selected, cfg: AdditionConfig, rng) -> GaussianCloud:
    """adaptive.py:117-139: one new Gaussian per selected row at N(mu, c Sigma),
    identity rotation, opacity cfg.init_opacity, log-scales and SH copied."""
    c = _as_dict(cloud)
    sel = np.asarray(selected, dtype=np.int64)
    k = len(sel)
    rot = np.zeros((k, 4))
    rot[:, 0] = 1.0
    p = np.full(k, cfg.init_opacity)
    return GaussianCloud(_sample_around(c, sel, cfg.spawn_cov_scale, rng), rot,
                         c["log_scales"][sel].copy(), np.log(p / (1.0 - p)), c["sh"][sel].copy())


def quantity_control(add: dict, stats: ViewspaceStats, cfg: AdditionConfig, rng,
                     allow_split: bool = True):
    """adaptive.py:155-204 on host arrays: returns (cloud dict, split idx, kept mask)."""
    avg = stats.averages()
    split = np.flatnonzero(avg > cfg.tau_grad) if allow_split else np.zeros(0, np.int64)
    room = cfg.max_additional - len(add["means"])
    if len(split) > room:
        order = np.argsort(-avg[split], kind="stable")
        split = np.sort(split[order[: max(0, room)]])
    merged = {k: v.copy() for k, v in add.items()}
    if len(split) > 0:
        sib = dict(means=_sample_around(add, split, cfg.spawn_cov_scale, rng),
                   rotations=add["rotations"][split].copy(),
                   log_scales=add["log_scales"][split] + math.log(cfg.split_scale_factor),
                   opacity_logits=add["opacity_logits"][split].copy(),
                   sh=add["sh"][split].copy())
        merged["log_scales"][split] += math.log(cfg.split_scale_factor)
        merged = {k: np.concatenate([merged[k], sib[k]]) for k in _FIELDS}
    kept = _sigmoid(merged["opacity_logits"]) >= cfg.tau_alpha
    return {k: v[kept] for k, v in merged.items()}, split, kept


# ---------------------------------------------------------------- device loop
class _Joint:
    """Joint device cloud [frozen | additional] with its gradient buffers."""

    def __init__(self, frozen: dict, add: dict, dev):
        self.n_frozen, self.n_add = len(frozen["means"]), len(add["means"])
        self.n = self.n_frozen + self.n_add
        f32 = dict(dtype=torch.float32, device=dev)
        for k in _FIELDS:
            setattr(self, k, torch.cat([to_dev(frozen[k], dev=dev), to_dev(add[k], dev=dev)])
                    if self.n_add else to_dev(frozen[k], dev=dev))
        self.sh_coeffs = int(self.sh.shape[1])
        self.grads = dict(d_means=torch.zeros(self.n, 3, **f32),
                          d_rotations=torch.zeros(self.n, 4, **f32),
                          d_log_scales=torch.zeros(self.n, 3, **f32),
                          d_opacity_logits=torch.zeros(self.n, **f32),
                          d_sh=torch.zeros(self.n, self.sh_coeffs, 3, **f32),
                          viewspace=torch.zeros(self.n, **f32),
                          contributed=torch.zeros(self.n, dtype=torch.uint8, device=dev))
        self.gs = _lib.CloudGrads()
        for k, t in self.grads.items():
            setattr(self.gs, k, ptr(t))

    def struct(self) -> _lib.Cloud:
        c = _lib.Cloud()
        c.n, c.sh_coeffs = self.n, self.sh_coeffs
        for k in _FIELDS:
            setattr(c, k, ptr(getattr(self, k)))
        return c

    def additional(self) -> dict:
        return {k: getattr(self, k)[self.n_frozen:].double().cpu().numpy() for k in _FIELDS}


_GRAD_OF = {"means": "d_means", "rotations": "d_rotations", "log_scales": "d_log_scales",
            "opacity_logits": "d_opacity_logits", "sh": "d_sh"}


def _as_dict(cloud) -> dict:
    if isinstance(cloud, dict):
        return {k: np.asarray(cloud[k], dtype=np.float64) for k in _FIELDS}
    return {k: np.asarray(getattr(cloud, k), dtype=np.float64) for k in _FIELDS}


def stage2_optimize(transformed, additional, views, cfg: AdditionConfig, iterations: int, rng,
                    settings: RasterSettings = RasterSettings(),
                    loss_cfg: LossConfig = LossConfig(), background=None):
    """adaptive.py:218-288: optimise the additional Gaussians against the frozen
    transformed cloud; returns (additional GaussianCloud, per-iteration losses)."""
    if len(views) == 0:
        raise DataError("stage 2 requires at least one training view")
    add = _as_dict(additional)
    losses: list = []
    if iterations == 0 or len(add["means"]) == 0:
        return GaussianCloud(*(add[k] for k in _FIELDS)), losses
    dev = require_cuda()
    lib = _lib.load()
    frozen = _as_dict(transformed)
    cams = [Camera.from_any(c) for c, _ in views]
    cstructs = [camera_struct(c) for c in cams]
    targets = [t.to(dev, torch.float32).contiguous() if isinstance(t, torch.Tensor)
               else to_dev(np.asarray(t, dtype=np.float64), dev=dev) for _, t in views]
    sset = settings_struct(settings, background)
    lr = cfg.lr_by_param()
    f64 = dict(dtype=torch.float64, device=dev)
    H = max(c.height for c in cams)
    W = max(c.width for c in cams)
    image = torch.empty(H * W * 3, dtype=torch.float32, device=dev)
    alpha = torch.empty(H * W, dtype=torch.float32, device=dev)
    d_image = torch.empty(H * W * 3, dtype=torch.float32, device=dev)
    loss_scratch = empty_bytes(max(lib.ss_loss_bytes(c.height, c.width, 3) for c in cams), dev)
    loss_hist = torch.zeros(max(iterations, 1), **f64)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    counts = pinned(2)
    bins, bin_cap = None, 0
    n_views = len(views)
    order = rng.permutation(n_views)

    def build(add_np, m=None, v=None):
        j = _Joint(frozen, add_np, dev)
        mom = {}
        for k in _FIELDS:
            shape = (j.n_add,) + add_np[k].shape[1:]
            mom[k] = (to_dev(m[k], torch.float64, dev) if m is not None else torch.zeros(shape, **f64),
                      to_dev(v[k], torch.float64, dev) if v is not None else torch.zeros(shape, **f64))
        geom = empty_bytes(max(lib.ss_raster_geom_bytes(j.n, C.byref(cs), C.byref(sset))
                               for cs in cstructs), dev)
        return j, mom, geom

    joint, mom, geom = build(add)
    step = torch.zeros(1, dtype=torch.int32, device=dev)  # shared Adam step (optim.py:45-47)
    norm_acc = torch.zeros(joint.n_add, **f64)
    view_cnt = torch.zeros(joint.n_add, dtype=torch.int64, device=dev)
    for t in range(iterations):
        v = int(order[t % n_views])
        cam, cs = cams[v], cstructs[v]
        cl = joint.struct()
        _lib.check(lib.ss_raster_forward_begin(C.byref(cl), C.byref(cs), C.byref(sset), ptr(geom),
                                               ptr(counts), stream()), "stage2 render")
        torch.cuda.current_stream().synchronize()
        pairs = int(counts[1])
        if pairs > bin_cap or bins is None:
            bin_cap = max(int(pairs * 1.25) + 1024, 1 << 16)
            bins = empty_bytes(lib.ss_raster_bin_bytes(bin_cap, joint.n, C.byref(cs),
                                                       C.byref(sset)), dev)
        _lib.check(lib.ss_raster_forward_finish(C.byref(cl), C.byref(cs), C.byref(sset), ptr(geom),
                                                ptr(bins), pairs, ptr(image), ptr(alpha), None,
                                                stream()), "stage2 render")
        _lib.check(lib.ss_render_loss(ptr(image), ptr(targets[v]), cam.height, cam.width, 3,
                                      loss_cfg.lambda_dssim, 0.01 ** 2, 0.03 ** 2,
                                      ptr(loss_scratch), ptr(loss_hist[t:]), ptr(d_image),
                                      ptr(status), stream()), "stage2 loss")
        _lib.check(lib.ss_raster_backward(C.byref(cl), C.byref(cs), C.byref(sset), ptr(geom),
                                          ptr(bins), pairs, ptr(d_image), C.byref(joint.gs),
                                          stream()), "stage2 backward")
        # Adam on the additional rows only, one shared step count (optim.py:42-67)
        nf = joint.n_frozen
        for k in _FIELDS:
            p = getattr(joint, k)[nf:]
            g = joint.grads[_GRAD_OF[k]][nf:]
            m_k, v_k = mom[k]
            sc = torch.full((1,), 0, dtype=torch.int32, device=dev)
            sc.copy_(step)
            _lib.check(lib.ss_adam_step(p.numel(), ptr(p), ptr(g), ptr(m_k), ptr(v_k), None, 1, 0,
                                        None, None, None, None, ptr(sc), lr[k], 0.9, 0.999, 1e-15,
                                        0, stream()), "stage2 adam")
        step += 1
        norm_acc += joint.grads["viewspace"][nf:].double()
        view_cnt += joint.grads["contributed"][nf:].long()
        if (t + 1) % n_views == 0:
            if cfg.quantity_control:
                stats = ViewspaceStats(norm_acc.cpu().numpy(), view_cnt.cpu().numpy())
                cur = joint.additional()
                new, split, kept = quantity_control(cur, stats, cfg, rng,
                                                    allow_split=t + 1 + n_views <= iterations)
                m_np, v_np = {}, {}
                for k in _FIELDS:  # adaptive.py:207-215: zero moments for siblings, drop pruned
                    for src, dst in ((mom[k][0], m_np), (mom[k][1], v_np)):
                        a = src.cpu().numpy()
                        pad = np.zeros((len(split),) + a.shape[1:])
                        dst[k] = np.concatenate([a, pad])[kept]
                add = new
                if len(add["means"]) == 0:
                    joint = None
                    break
                joint, mom, geom = build(add, m_np, v_np)
            norm_acc = torch.zeros(joint.n_add, **f64)
            view_cnt = torch.zeros(joint.n_add, dtype=torch.int64, device=dev)
            order = rng.permutation(n_views)
    torch.cuda.current_stream().synchronize()
    if int(status.item()) & _lib.FLAG_NONFINITE:
        raise NumericalError("non-finite values detected in 'stage2 loss'")
    losses = loss_hist[: len(losses) or (t + 1)].cpu().numpy().tolist()
    final = add if joint is None else joint.additional()
    return GaussianCloud(*(final[k] for k in _FIELDS)), losses
