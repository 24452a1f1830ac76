"""Stage-1 benchmark (BASELINE.json metric): NTC train iterations/s at 1352x1014
with 250k SH-3 Gaussians (config 1), plus render FPS (config 2) and roofline.

python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true")
    return ap.parse_args()


def make_cache(scene, output_init="identity", seed=0):
    from oracle import stage1 as O  # noqa: F401  (never used on the product path)
    return None


def build_problem(cfg_idx):
    """Scene, an identity-initialised NTC (ntc.py:100-128 init) and targets rendered
    on the device from the seeded motion field."""
    from paper_2403_01444_b200 import scenes
    from paper_2403_01444_b200.ntc import NeuralTransformationCache
    from paper_2403_01444_b200.rasterizer import render_device
    from paper_2403_01444_b200.device import DeviceCloud
    from paper_2403_01444_b200.types import HashGridConfig

    sc = scenes.config(cfg_idx)
    cache = NeuralTransformationCache(HashGridConfig.from_any(sc.grid), output_init="identity")
    moved = scenes.moved_cloud(sc.cloud, np.random.default_rng(7), axis=(0.3, 1.0, 0.2),
                               deg=1.5, shift=(0.01, -0.005, 0.008))
    dm = DeviceCloud(moved)
    targets = []
    for cam in sc.cameras:
        img = render_device(dm, cam, None, want_touch=False)[0]
        targets.append(img)
    return sc, cache, targets


def main():
    a = parse()
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.impl == "reference":
        if rank == 0:
            print(json.dumps({"impl": "reference", "unavailable": "not yet wired"}))
        return
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    from paper_2403_01444_b200 import _lib
    from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer

    lib = _lib.load()
    sc, cache, targets = build_problem(a.config)
    views = list(zip(sc.cameras, targets))
    tr = Stage1Trainer(sc.cloud, cache, views, Stage1Config())
    order = [k % len(views) for k in range(a.warmup + a.steps)]
    for k in range(a.warmup):
        tr.step(order[k])
    torch.cuda.synchronize()
    l0 = lib.ss_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pairs = []
    ev0.record()
    for k in range(a.steps):
        pairs.append(tr.step(order[a.warmup + k]))
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / a.steps
    launches = lib.ss_launch_count() - l0
    line = {"metric": "stage1_iters_per_s", "value": 1000.0 / ms, "unit": "iter/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
            "higher_is_better": True, "dtype": "f32", "data": "synthetic",
            "config": {"workload": sc.name, "gaussians": len(sc.cloud["means"]),
                       "resolution": [1352, 1014], "mean_pairs": float(np.mean(pairs))},
            "gpu_launches": launches, "loss": tr.last_loss()}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
