"""Helpers to turn tests/golden/*.npz fixtures into oracle-format dicts."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def grid(d):
    return dict(levels=int(d["grid_levels"]), features=int(d["grid_features"]),
                log2_table=int(d["grid_log2_table"]), base=int(d["grid_base"]),
                growth=float(d["grid_growth"]), lo=tuple(d["grid_lo"]), hi=tuple(d["grid_hi"]))


def cloud(d, p="cloud_"):
    return {k: d[p + k].copy() for k in ("means", "rotations", "log_scales", "opacity_logits", "sh")}


def camera(d, p="cam_"):
    fx, fy, cx, cy = d[p + "intr"]
    w, h = d[p + "size"]
    return dict(w2c=d[p + "w2c"], fx=float(fx), fy=float(fy), cx=float(cx), cy=float(cy),
                width=int(w), height=int(h), near=float(d[p + "near"]))


def mlp(d):
    n = len([k for k in d if k.startswith("mlp_w")])
    return dict(weights=[d[f"mlp_w{i}"].copy() for i in range(n)],
                biases=[d[f"mlp_b{i}"].copy() for i in range(n)])


def settings(d):
    ts, clamp, skip, stop = d["settings"]
    return dict(tile_size=int(ts), alpha_clamp=float(clamp), skip_alpha=float(skip),
                stop_transmittance=float(stop))


def norm_rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / den) if den > 0 else float(np.linalg.norm(a))
