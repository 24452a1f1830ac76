"""Host-side value types of the reference API, re-declared for the drop-in.

Same names, fields, validation and error behaviour as the reference
(`gaussians.py:179-287`, `cameras.py:30-129`, `ntc.py:30-61`,
`rasterizer.py:33-68`, `losses.py:21-33`); float64 numpy on the host, float32
on the device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import DataError, NumericalError


# ---------------------------------------------------------------- Gaussians
def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-np.asarray(x, dtype=np.float64)))


def inverse_sigmoid(p):
    p = np.asarray(p, dtype=np.float64)
    return np.log(p / (1.0 - p))


def quat_normalize(q, eps: float = 1e-12):
    """gaussians.py:42-48."""
    q = np.asarray(q, dtype=np.float64)
    n = np.linalg.norm(q, axis=-1, keepdims=True)
    if np.any(n < eps):
        raise NumericalError("cannot normalize near-zero quaternion")
    return q / n


@dataclass
class GaussianCloud:
    """SoA Gaussians (gaussians.py:179-216).  `sh` is (N, K, 3) with
    K = (degree+1)^2, degree <= 3 (the reference stores K = 4)."""

    means: np.ndarray
    rotations: np.ndarray
    log_scales: np.ndarray
    opacity_logits: np.ndarray
    sh: np.ndarray

    def __post_init__(self) -> None:
        self.means = np.ascontiguousarray(self.means, dtype=np.float64)
        self.rotations = np.ascontiguousarray(self.rotations, dtype=np.float64)
        self.log_scales = np.ascontiguousarray(self.log_scales, dtype=np.float64)
        self.opacity_logits = np.ascontiguousarray(self.opacity_logits, dtype=np.float64)
        self.sh = np.ascontiguousarray(self.sh, dtype=np.float64)
        n = len(self.means)
        if self.means.shape != (n, 3):
            raise ValueError(f"means must be (N, 3), got {self.means.shape}")
        if self.rotations.shape != (n, 4):
            raise ValueError(f"rotations must be (N, 4), got {self.rotations.shape}")
        if self.log_scales.shape != (n, 3):
            raise ValueError(f"log_scales must be (N, 3), got {self.log_scales.shape}")
        if self.opacity_logits.shape != (n,):
            raise ValueError(f"opacity_logits must be (N,), got {self.opacity_logits.shape}")
        if self.sh.ndim != 3 or self.sh.shape[0] != n or self.sh.shape[2] != 3 or \
                self.sh.shape[1] not in (1, 4, 9, 16):
            raise ValueError(f"sh must be (N, K, 3) with K in 1/4/9/16, got {self.sh.shape}")

    def __len__(self) -> int:
        return len(self.means)

    @property
    def sh_degree(self) -> int:
        return int(round(math.sqrt(self.sh.shape[1]))) - 1

    @property
    def opacities(self):
        return sigmoid(self.opacity_logits)

    @property
    def scales(self):
        return np.exp(self.log_scales)

    def copy(self) -> "GaussianCloud":
        return GaussianCloud(self.means.copy(), self.rotations.copy(), self.log_scales.copy(),
                             self.opacity_logits.copy(), self.sh.copy())

    def select(self, idx) -> "GaussianCloud":
        return GaussianCloud(self.means[idx], self.rotations[idx], self.log_scales[idx],
                             self.opacity_logits[idx], self.sh[idx])

    @staticmethod
    def concatenate(a: "GaussianCloud", b: "GaussianCloud") -> "GaussianCloud":
        return GaussianCloud(*(np.concatenate([getattr(a, f), getattr(b, f)]) for f in
                               ("means", "rotations", "log_scales", "opacity_logits", "sh")))

    @staticmethod
    def empty(sh_coeffs: int = 4) -> "GaussianCloud":
        return GaussianCloud(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0),
                             np.zeros((0, sh_coeffs, 3)))

    def quantize_float32(self) -> "GaussianCloud":
        """gaussians.py:275-287."""
        q = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
        return GaussianCloud(q(self.means), q(self.rotations), q(self.log_scales),
                             q(self.opacity_logits), q(self.sh))

    @staticmethod
    def from_any(c) -> "GaussianCloud":
        """Accept this class or any object with the reference's five fields."""
        if isinstance(c, GaussianCloud):
            return c
        return GaussianCloud(c.means, c.rotations, c.log_scales, c.opacity_logits, c.sh)


# ---------------------------------------------------------------- cameras
@dataclass(frozen=True)
class Camera:
    """Pinhole camera (cameras.py:30-80); x right, y down, z forward."""

    world_to_camera: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near_clip: float = 0.01

    def __post_init__(self) -> None:
        w2c = np.ascontiguousarray(self.world_to_camera, dtype=np.float64)
        if w2c.shape != (4, 4):
            raise DataError(f"world_to_camera must be 4x4, got {w2c.shape}")
        if not np.allclose(w2c[3], [0.0, 0.0, 0.0, 1.0], atol=1e-9):
            raise DataError("world_to_camera bottom row must be [0, 0, 0, 1]")
        rot = w2c[:3, :3]
        if not np.allclose(rot @ rot.T, np.eye(3), atol=1e-6):
            raise DataError("world_to_camera rotation block is not orthonormal")
        object.__setattr__(self, "world_to_camera", w2c)
        if self.width <= 0 or self.height <= 0:
            raise DataError("camera image size must be positive")
        if self.fx <= 0 or self.fy <= 0:
            raise DataError("focal lengths must be positive")
        if self.near_clip <= 0:
            raise DataError("near_clip must be positive")

    @property
    def rotation(self):
        return self.world_to_camera[:3, :3]

    @property
    def translation(self):
        return self.world_to_camera[:3, 3]

    @property
    def position(self):
        return -self.rotation.T @ self.translation

    @staticmethod
    def from_any(c) -> "Camera":
        if isinstance(c, Camera):
            return c
        if isinstance(c, dict):
            return Camera(c["w2c"], c["fx"], c["fy"], c["cx"], c["cy"], c["width"], c["height"],
                          c.get("near", 0.01))
        return Camera(c.world_to_camera, c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.near_clip)


def look_at(eye, target, up, fx, fy, cx, cy, width, height, near_clip=0.01) -> Camera:
    """cameras.py:83-129."""
    eye = np.asarray(eye, dtype=np.float64)
    zc = np.asarray(target, dtype=np.float64) - eye
    nz = np.linalg.norm(zc)
    if nz < 1e-12:
        raise DataError("look_at eye and target coincide")
    zc = zc / nz
    xc = np.cross(zc, np.asarray(up, dtype=np.float64))
    nx = np.linalg.norm(xc)
    if nx < 1e-12:
        raise DataError("look_at up direction is parallel to the view direction")
    xc = xc / nx
    yc = np.cross(zc, xc)
    rot = np.stack([xc, yc, zc])
    w2c = np.eye(4)
    w2c[:3, :3] = rot
    w2c[:3, 3] = -rot @ eye
    return Camera(w2c, fx, fy, cx, cy, width, height, near_clip)


# ---------------------------------------------------------------- hash grid
@dataclass(frozen=True)
class HashGridConfig:
    """ntc.py:30-61."""

    n_levels: int = 16
    n_features: int = 4
    table_size_log2: int = 15
    base_resolution: int = 16
    growth_factor: float = 32.0 ** (1.0 / 15.0)
    aabb_min: tuple = (-1.0, -1.0, -1.0)
    aabb_max: tuple = (1.0, 1.0, 1.0)

    def __post_init__(self) -> None:
        if self.n_levels < 1 or self.n_features < 1:
            raise DataError("hash grid needs at least one level and one feature")
        if self.growth_factor < 1.0:
            raise DataError("growth_factor must be >= 1")
        lo = np.asarray(self.aabb_min, dtype=np.float64)
        hi = np.asarray(self.aabb_max, dtype=np.float64)
        if lo.shape != (3,) or hi.shape != (3,) or not np.all(lo < hi):
            raise DataError("aabb_min must be componentwise below aabb_max")

    @property
    def table_size(self) -> int:
        return 1 << self.table_size_log2

    def resolution(self, level: int) -> int:
        """floor(base * growth**level) in float64 (ntc.py:54-55)."""
        return int(np.floor(self.base_resolution * self.growth_factor ** level))

    @staticmethod
    def growth_for(base: int, finest: int, n_levels: int) -> float:
        if n_levels <= 1:
            return 1.0
        return float((finest / base) ** (1.0 / (n_levels - 1)))

    @staticmethod
    def from_any(g) -> "HashGridConfig":
        if isinstance(g, HashGridConfig):
            return g
        if isinstance(g, dict):
            return HashGridConfig(g["levels"], g["features"], g["log2_table"], g["base"],
                                  g["growth"], tuple(g["lo"]), tuple(g["hi"]))
        return HashGridConfig(g.n_levels, g.n_features, g.table_size_log2, g.base_resolution,
                              g.growth_factor, tuple(g.aabb_min), tuple(g.aabb_max))


# ---------------------------------------------------------------- raster / loss
@dataclass(frozen=True)
class RasterSettings:
    """rasterizer.py:33-38."""

    tile_size: int = 16
    alpha_clamp: float = 0.99
    skip_alpha: float = 1.0 / 255.0
    stop_transmittance: float = 1e-4


@dataclass(frozen=True)
class LossConfig:
    """losses.py:21-33."""

    lambda_dssim: float = 0.2
    ssim_window: int = 11
    ssim_sigma: float = 1.5
    ssim_c1: float = 0.01 ** 2
    ssim_c2: float = 0.03 ** 2

    def __post_init__(self) -> None:
        if not 0.0 <= self.lambda_dssim <= 1.0:
            raise DataError("lambda_dssim must be in [0, 1]")
        if self.ssim_window % 2 != 1 or self.ssim_window < 3:
            raise DataError("ssim_window must be odd and >= 3")
        if self.ssim_window != 11 or self.ssim_sigma != 1.5:
            raise DataError("the CUDA loss is specialised for the 11x11 sigma=1.5 window")
