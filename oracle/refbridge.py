"""Adapter that runs the *unmodified* reference package on oracle-format inputs.

TEST INFRASTRUCTURE ONLY.  Usable only where `/root/reference` exists (the
build container); the GPU box never has it.  Used by `oracle/make_golden.py`
(fixture generation) and `tests/test_oracle_vs_reference.py` (pinning the
oracle restatement against the reference itself).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "splatstream"))


def load():
    """Import the reference modules (threadpool pinned by the caller, D10)."""
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from splatstream import cameras, gaussians, losses, ntc, optim, rasterizer, sh, transform

    return dict(cameras=cameras, gaussians=gaussians, losses=losses, ntc=ntc, optim=optim,
                rasterizer=rasterizer, sh=sh, transform=transform)


def ref_cloud(R, cloud):
    """Oracle cloud dict -> reference GaussianCloud (sh padded to 4 rows)."""
    sh = cloud["sh"]
    if sh.shape[1] == 1:
        sh = np.concatenate([sh, np.zeros((len(sh), 3, 3))], axis=1)
    if sh.shape[1] != 4:
        raise ValueError("the reference supports SH degree <= 1 only (gaussians.py:214)")
    return R["gaussians"].GaussianCloud(means=cloud["means"].copy(),
                                        rotations=cloud["rotations"].copy(),
                                        log_scales=cloud["log_scales"].copy(),
                                        opacity_logits=cloud["opacity_logits"].copy(),
                                        sh=sh.copy())


def ref_camera(R, cam):
    return R["cameras"].Camera(world_to_camera=cam["w2c"], fx=cam["fx"], fy=cam["fy"],
                               cx=cam["cx"], cy=cam["cy"], width=cam["width"],
                               height=cam["height"], near_clip=cam["near"])


def ref_grid(R, grid):
    return R["ntc"].HashGridConfig(n_levels=grid["levels"], n_features=grid["features"],
                                   table_size_log2=grid["log2_table"],
                                   base_resolution=grid["base"],
                                   growth_factor=grid["growth"],
                                   aabb_min=tuple(grid["lo"]), aabb_max=tuple(grid["hi"]))


def ref_cache(R, grid, tables, mlp, hidden_dim=64):
    cache = R["ntc"].NeuralTransformationCache(ref_grid(R, grid), hidden_layers=len(mlp["weights"]) - 1,
                                               hidden_dim=hidden_dim)
    cache.tables[:] = tables
    for i, (w, b) in enumerate(zip(mlp["weights"], mlp["biases"])):
        cache.weights[i][:] = w
        cache.biases[i][:] = b
    return cache


def ref_settings(R, s):
    return R["rasterizer"].RasterSettings(**s)
