"""Seeded synthetic Stage-1 workloads (BASELINE.json configs 0-4).

The reference measures nothing of its own, and the N3DV /
Meet Room data are not available, so every workload here is a seeded numpy
stand-in with the shapes, sizes and value distributions BASELINE.json states
(SURVEY.md section 8(d2)).  Everything is float32-lattice float64 numpy so the same
arrays can be fed to the CUDA path and to the CPU oracle.

Choices BASELINE.json leaves open, fixed here:
  * per-axis phases of the sinusoidal motion are drawn from the same rng;
  * cfg0 camera azimuths are +-35 degrees around -z (look-at origin, radius 4);
  * motion = rigid rotation R about an axis (z for cfg0) applied to means and
    composed into quaternions, plus a translation and 0.02 sin(2x + phi);
  * cfg1/2 cameras: 20 on a forward arc, yaw in [-40, 40] deg, pitch
    10 sin(2.3 a + 0.4) deg (the reference rig's pitch wobble, synth.py:72-76);
  * cfg3 cameras: 48 on the upper hemisphere (Fibonacci spiral) of radius 5;
  * cfg4 rig: 8 cameras on a ring of radius 4 around the clusters (BASELINE
    leaves it open; SURVEY.md section 8(d4) measured 4.2e9-5.1e9 tile pairs per
    view for this radius).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SH_C0 = 0.28209479177387814


def f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


@dataclass
class Scene:
    name: str
    cloud: dict
    grid: dict
    cameras: list
    sh_degree: int
    mlp_in: int
    hidden_dim: int = 64
    views_per_iteration: int = 1
    iterations: int = 150
    mlp_dtype: str = "f32"
    notes: dict = field(default_factory=dict)


def look_at(eye, width, height, fov_deg=60.0, target=(0.0, 0.0, 0.0), up=(0.0, -1.0, 0.0)):
    """Pinhole camera at `eye` looking at `target` (cameras.py:83-129 conventions:
    x right, y down, z forward; world up maps to -y)."""
    eye = np.asarray(eye, dtype=np.float64)
    zc = np.asarray(target, dtype=np.float64) - eye
    zc /= np.linalg.norm(zc)
    xc = np.cross(zc, np.asarray(up, dtype=np.float64))
    xc /= np.linalg.norm(xc)
    yc = np.cross(zc, xc)
    rot = np.stack([xc, yc, zc])
    w2c = np.eye(4)
    w2c[:3, :3] = rot
    w2c[:3, 3] = -rot @ eye
    fx = (width / 2.0) / math.tan(math.radians(fov_deg) / 2.0)
    return dict(w2c=w2c, fx=fx, fy=fx, cx=(width - 1) / 2.0, cy=(height - 1) / 2.0,
                width=int(width), height=int(height), near=0.01)


def make_cloud(rng, n, n_clusters, extent, sigma, sh_degree, log_scale=(-4.0, 0.4),
               logit=(0.0, 1.5), aniso=None):
    """Cluster mixture; draws in the order centres, labels, offsets, quats,
    log-scales, opacities, SH."""
    centres = rng.uniform(-extent, extent, size=(n_clusters, 3))
    labels = rng.integers(0, n_clusters, size=n)
    offsets = rng.normal(scale=sigma, size=(n, 3))
    means = centres[labels] + offsets
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    ls = rng.normal(log_scale[0], log_scale[1], size=(n, 3))
    if aniso is not None:
        # clamp every axis to within log(aniso) of the largest one
        top = ls.max(axis=1, keepdims=True)
        ls = np.maximum(ls, top - math.log(aniso))
    logits = rng.normal(logit[0], logit[1], size=n)
    k = (sh_degree + 1) ** 2
    sh = np.zeros((n, k, 3))
    sh[:, 0, :] = rng.uniform(0.0, 1.0, size=(n, 3))
    if k > 1:
        sh[:, 1:, :] = rng.normal(scale=0.05, size=(n, k - 1, 3))
    return dict(means=f32(means), rotations=f32(q), log_scales=f32(ls),
                opacity_logits=f32(logits), sh=f32(sh))


def fit_grid(levels, features, log2_table, base, growth, means, margin=1.5):
    """HashGridConfig with fit_grid_to_cloud's AABB (pipeline.py:348-360)."""
    lo = means.min(axis=0)
    hi = means.max(axis=0)
    c = 0.5 * (lo + hi)
    half = np.maximum(0.5 * (hi - lo) * margin, 0.25)
    return dict(levels=levels, features=features, log2_table=log2_table, base=base,
                growth=float(growth), lo=tuple(float(v) for v in c - half),
                hi=tuple(float(v) for v in c + half))


def growth_for(base, finest, levels):
    """ntc.py:57-61."""
    return 1.0 if levels <= 1 else float((finest / base) ** (1.0 / (levels - 1)))


def _quat_axis_angle(axis, deg):
    axis = np.asarray(axis, dtype=np.float64)
    axis /= np.linalg.norm(axis)
    h = math.radians(deg) / 2.0
    return np.array([math.cos(h), *(math.sin(h) * axis)])


def _quat_to_mat(q):
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def moved_cloud(cloud, rng, axis=(0.0, 0.0, 1.0), deg=2.0, shift=(0.0, 0.0, 0.0), amp=0.02):
    """Target-frame cloud: rigid rotation about the origin + shift + amp sin(2x+phi)."""
    phi = rng.uniform(0.0, 2.0 * math.pi, size=3)
    qr = _quat_axis_angle(axis, deg)
    r = _quat_to_mat(qr)
    m = cloud["means"] @ r.T + np.asarray(shift) + amp * np.sin(2.0 * cloud["means"] + phi)
    q = cloud["rotations"]
    w, x, y, z = qr
    qw, qx, qy, qz = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    q2 = np.stack([w * qw - x * qx - y * qy - z * qz, w * qx + x * qw + y * qz - z * qy,
                   w * qy - x * qz + y * qw + z * qx, w * qz + x * qy - y * qx + z * qw], 1)
    out = dict(cloud)
    out["means"] = f32(m)
    out["rotations"] = f32(q2)
    return out


def config(idx: int, seed: int = 0) -> Scene:
    rng = np.random.default_rng(seed)
    if idx == 0:
        cloud = make_cloud(rng, 20_000, 8, 2.0, 0.5, 0)
        grid = fit_grid(8, 2, 14, 16, 1.5, cloud["means"])
        cams = []
        for a in (-35.0, 35.0):
            ar = math.radians(a)
            cams.append(look_at((4 * math.sin(ar), 0.0, -4 * math.cos(ar)), 160, 120))
        return Scene("cfg0", cloud, grid, cams, 0, 16, notes=dict(motion="z2deg+sin"))
    if idx in (1, 2):
        n = 250_000 if idx == 1 else 300_000
        cloud = make_cloud(rng, n, 32, 3.0, 0.5, 3)
        grid = fit_grid(16, 2, 15, 16, growth_for(16, 2048, 16), cloud["means"])
        cams = []
        for k in range(20):
            a = math.radians(40.0) * (2.0 * k / 19 - 1.0)
            p = math.radians(10.0) * math.sin(2.3 * a + 0.4)
            cams.append(look_at((4 * math.cos(p) * math.sin(a), -4 * math.sin(p),
                                 -4 * math.cos(p) * math.cos(a)), 1352, 1014))
        return Scene(f"cfg{idx}", cloud, grid, cams, 3, 32,
                     mlp_dtype="f16" if idx == 1 else "f32")
    if idx == 3:
        cloud = make_cloud(rng, 1_000_000, 64, 4.0, 0.5, 3)
        grid = fit_grid(16, 2, 15, 16, growth_for(16, 2048, 16), cloud["means"])
        cams = []
        golden = math.pi * (3.0 - math.sqrt(5.0))
        for k in range(48):
            el = math.asin((k + 0.5) / 48 * math.sin(math.radians(75.0)))
            az = golden * k
            cams.append(look_at((5 * math.cos(el) * math.sin(az), -5 * math.sin(el),
                                 -5 * math.cos(el) * math.cos(az)), 1352, 1014))
        return Scene("cfg3", cloud, grid, cams, 3, 32, views_per_iteration=16,
                     mlp_dtype="f16")
    if idx == 4:
        cloud = make_cloud(rng, 3_000_000, 16, 4.0, 0.2, 3, log_scale=(-3.0, 0.6),
                           logit=(1.0, 1.0), aniso=10.0)
        grid = fit_grid(16, 2, 19, 16, growth_for(16, 2048, 16), cloud["means"])
        cams = []
        for k in range(8):
            a = 2 * math.pi * k / 8
            cams.append(look_at((4 * math.sin(a), -0.5, -4 * math.cos(a)), 3840, 2160))
        return Scene("cfg4", cloud, grid, cams, 3, 32, views_per_iteration=8,
                     mlp_dtype="f16")
    raise ValueError(f"unknown config {idx}")


def small_scene(seed=0, n=2000, width=64, height=48, sh_degree=1, n_views=2, levels=4,
                log2_table=10, extent=1.0):
    """A cfg0-shaped scene small enough for the float64 oracle in well under a second."""
    rng = np.random.default_rng(seed)
    cloud = make_cloud(rng, n, 4, extent, 0.4, sh_degree, log_scale=(-3.0, 0.4))
    grid = fit_grid(levels, 2, log2_table, 4, 1.5, cloud["means"])
    cams = []
    for k in range(n_views):
        a = math.radians(-30.0 + 60.0 * k / max(1, n_views - 1))
        cams.append(look_at((3.5 * math.sin(a), 0.2, -3.5 * math.cos(a)), width, height))
    return Scene("small", cloud, grid, cams, sh_degree, 2 * levels)
