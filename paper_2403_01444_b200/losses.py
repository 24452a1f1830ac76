"""Drop-in for splatstream.losses.render_loss / ssim (losses.py:67-148) on the GPU."""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .device import empty_bytes, ptr, require_cuda, stream, to_dev
from .errors import DataError
from .types import LossConfig

__all__ = ["LossConfig", "render_loss", "render_loss_device", "ssim"]


def render_loss_device(image: torch.Tensor, target: torch.Tensor, cfg: LossConfig = LossConfig(),
                       scratch: torch.Tensor | None = None):
    """(loss_dev (1,) float64, d_image) for device images (H, W, C); no host sync."""
    lib = _lib.load()
    if image.shape != target.shape:
        raise DataError(f"render_loss shape mismatch: {tuple(image.shape)} vs {tuple(target.shape)}")
    h, w = image.shape[0], image.shape[1]
    ch = 1 if image.dim() == 2 else image.shape[2]
    if h < cfg.ssim_window or w < cfg.ssim_window:
        raise DataError("image smaller than the SSIM window")
    dev = image.device
    if scratch is None:
        scratch = empty_bytes(lib.ss_loss_bytes(h, w, ch), dev)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    grad = torch.empty_like(image)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(lib.ss_render_loss(ptr(image), ptr(target), h, w, ch, cfg.lambda_dssim,
                                  cfg.ssim_c1, cfg.ssim_c2, ptr(scratch), ptr(loss), ptr(grad),
                                  ptr(status), stream()), "render_loss")
    return loss, grad


def render_loss(rendered, target, cfg: LossConfig = LossConfig()):
    """losses.py:84-148: (float loss, grad ndarray)."""
    dev = require_cuda()
    r = np.asarray(rendered, dtype=np.float64)
    t = np.asarray(target, dtype=np.float64)
    if r.shape != t.shape:
        raise DataError(f"render_loss shape mismatch: {r.shape} vs {t.shape}")
    loss, grad = render_loss_device(to_dev(r, dev=dev), to_dev(t, dev=dev), cfg)
    return float(loss.item()), grad.cpu().numpy().astype(np.float64)


def ssim(x, y, cfg: LossConfig = LossConfig()) -> float:
    """Mean SSIM over valid windows (losses.py:67-81), via the loss kernel with lam = 1."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.shape != y.shape:
        raise DataError(f"ssim shape mismatch: {x.shape} vs {y.shape}")
    one = LossConfig(lambda_dssim=1.0, ssim_c1=cfg.ssim_c1, ssim_c2=cfg.ssim_c2)
    loss, _ = render_loss(x, y, one)
    return 1.0 - 2.0 * loss
