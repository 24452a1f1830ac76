"""The Stage-1 part of `process_frame` (pipeline.py:238-283) on the device.

Two drivers with the reference's contract -- clone the warm cache with fresh
Adam state (pipeline.py:213-219), train `stage1_iterations` iterations over
the reference's per-epoch view permutations drawn from
default_rng([seed, frame_index]), accumulate the view-space statistics over
the last epoch (adaptive.py:79-97), quantise the cache to float32 and apply it
once more (pipeline.py:281-282):

  stage1_frame         the fused, graph-replayed Stage1Trainer loop (the hot path)
  stage1_frame_dropin  the same loop written against this package's drop-in
                       modules (ntc / transform / rasterizer / losses), i.e. the
                       call pattern process_frame itself makes (pipeline.py:
                       263-277) once those names are patched into
                       splatstream.pipeline

Both return Stage1Result(cache, transformed, losses, stats_norm, stats_count).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DataError, check_finite
from .ntc import NeuralTransformationCache
from .types import GaussianCloud


@dataclass
class Stage1Result:
    cache: NeuralTransformationCache  # quantised to float32, fresh Adam state
    transformed: GaussianCloud        # apply_ntc of the final cache
    losses: np.ndarray                # per iteration
    stats_norm: np.ndarray            # ViewspaceStats.norm_accum
    stats_count: np.ndarray           # ViewspaceStats.view_count


def _clone(cache) -> NeuralTransformationCache:
    """clone_cache (pipeline.py:213-219) into this package's cache class."""
    out = NeuralTransformationCache(cache.grid, hidden_layers=len(cache.weights) - 1,
                                    hidden_dim=int(np.shape(cache.weights[0])[1]),
                                    mlp_dtype=getattr(cache, "mlp_dtype", "f32"))
    out.tables[:] = cache.tables
    for i in range(len(cache.weights)):
        out.weights[i][:] = cache.weights[i]
        out.biases[i][:] = cache.biases[i]
    out.reset_adam()
    return out


def _check(prev_cloud, views):
    if len(GaussianCloud.from_any(prev_cloud).means) == 0:
        raise DataError("previous cloud is empty")
    if len(views) == 0:
        raise DataError("frame has no training views")


def stage1_frame(prev_cloud, warm_cache, views, cfg, frame_index: int,
                 background=None) -> Stage1Result:
    """Fused device loop: Stage1Trainer.run (one CUDA graph per iteration)."""
    from .stage1 import Stage1Config, Stage1Trainer
    from .transform import apply_ntc

    _check(prev_cloud, views)
    cache = _clone(warm_cache)
    scfg = Stage1Config(stage1_iterations=cfg.stage1_iterations, ntc_lr=cfg.ntc_lr,
                        seed=cfg.seed, raster=cfg.raster, loss=cfg.loss)
    tr = Stage1Trainer(prev_cloud, cache, views, scfg, background=background)
    losses = tr.run(cfg.stage1_iterations, frame_index=frame_index)
    norm, count = tr.viewspace_stats()
    tr.export_to(cache)
    cache.quantize_float32()
    cache.reset_adam()
    transformed, _ = apply_ntc(GaussianCloud.from_any(prev_cloud), cache)
    return Stage1Result(cache, transformed, losses, norm, count)


def stage1_frame_dropin(prev_cloud, warm_cache, views, cfg, frame_index: int,
                        background=None) -> Stage1Result:
    """The reference loop's call pattern through the drop-in modules."""
    from .losses import render_loss
    from .rasterizer import rasterize_backward, rasterize_forward
    from .stage1 import view_order
    from .transform import apply_ntc, apply_ntc_backward

    _check(prev_cloud, views)
    prev = GaussianCloud.from_any(prev_cloud)
    cache = _clone(warm_cache)
    n_views = len(views)
    iters = cfg.stage1_iterations
    order = view_order(cfg.seed, frame_index, n_views, iters)
    stats_from = max(0, iters - n_views)
    norm = np.zeros(len(prev.means))
    count = np.zeros(len(prev.means), dtype=np.int64)
    losses, encode_ctx = [], None
    for t, v in enumerate(order):
        camera, target = views[v]
        transformed, tctx = apply_ntc(prev, cache, encode_ctx=encode_ctx)
        if encode_ctx is None:
            encode_ctx = tctx.fwd.encode  # frozen means: encode once per frame
        out, rctx = rasterize_forward(transformed, camera, background, cfg.raster)
        loss, d_image = render_loss(out.image, target, cfg.loss)
        check_finite("stage1 loss", np.asarray(loss))
        losses.append(float(loss))
        g = rasterize_backward(rctx, d_image)
        grads, touched = apply_ntc_backward(tctx, g.d_means, g.d_rotations, g.d_sh)
        cache.adam_step(grads, cfg.ntc_lr, touched)
        if t >= stats_from:
            norm += g.viewspace_grad_norm
            count += g.contributed.astype(np.int64)
    cache.quantize_float32()
    cache.reset_adam()
    transformed, _ = apply_ntc(prev, cache)
    return Stage1Result(cache, transformed, np.asarray(losses), norm, count)
