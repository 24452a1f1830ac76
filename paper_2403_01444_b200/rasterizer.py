"""Drop-in for splatstream.rasterizer (rasterizer.py:33-403) on the CUDA library.

Same names, signatures, return types and errors.  Inputs may be the
reference's numpy objects (copied to HBM) or DeviceCloud-backed; the contexts
keep their buffers on the device and materialise the reference's numpy fields
lazily on attribute access.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import (DeviceCloud, camera_struct, empty_bytes, pinned, ptr, require_cuda,
                     settings_struct, stream, to_dev)
from .errors import DataError
from .types import Camera, GaussianCloud, RasterSettings

__all__ = ["RasterSettings", "RenderOutput", "GradientBuffer", "RenderContext", "tile_bin",
           "rasterize_forward", "rasterize_backward"]

# Tile pairs one bin workspace holds.  A view with more pairs (config 4: 3M
# Gaussians at 3840x2160, billions of pairs) is binned and blended in bands of
# tile rows of at most this many pairs (ss_raster_*_banded).
BIN_PAIR_LIMIT = int(os.environ.get("SS_BIN_PAIR_LIMIT", str(1 << 29)))


@dataclass
class RenderOutput:
    image: np.ndarray  # (H, W, 3)
    alpha_map: np.ndarray  # (H, W)
    per_gaussian_touch_count: np.ndarray  # (N,)


@dataclass
class GradientBuffer:
    """rasterizer.py:48-68."""

    d_means: np.ndarray
    d_rotations: np.ndarray
    d_log_scales: np.ndarray
    d_opacity_logits: np.ndarray
    d_sh: np.ndarray
    viewspace_grad_norm: np.ndarray
    contributed: np.ndarray

    @staticmethod
    def zeros(n: int, sh_coeffs: int = 4) -> "GradientBuffer":
        return GradientBuffer(np.zeros((n, 3)), np.zeros((n, 4)), np.zeros((n, 3)), np.zeros(n),
                              np.zeros((n, sh_coeffs, 3)), np.zeros(n),
                              np.zeros(n, dtype=bool))


class RenderContext:
    """Device-resident replacement of the reference RenderContext
    (rasterizer.py:71-90): projected records, sort order, tile lists."""

    def __init__(self, cloud, camera, settings, background, dcloud, geom, bins, n_pairs,
                 n_survivors, bin_capacity=None):
        self.cloud = cloud
        self.camera = camera
        self.settings = settings
        self.background = background
        self._dcloud = dcloud
        self._geom = geom
        self._bins = bins
        self.n_pairs = n_pairs
        self.n_survivors = n_survivors
        self.bin_capacity = n_pairs if bin_capacity is None else bin_capacity
        self._tiles = None
        self._indices = None

    def _lists(self):
        lib = _lib.load()
        if self.n_pairs > self.bin_capacity:
            raise DataError("tile lists of a view rendered in bands are not retained "
                            f"({self.n_pairs} pairs > {self.bin_capacity}); raise "
                            "SS_BIN_PAIR_LIMIT to keep them")
        cam, s = camera_struct(self.camera), settings_struct(self.settings, self.background)
        ts = self.settings.tile_size
        ntx = (self.camera.width + ts - 1) // ts
        nty = (self.camera.height + ts - 1) // ts
        dev = self._geom.device
        ranges = torch.zeros(ntx * nty * 2, dtype=torch.int32, device=dev)
        members = torch.zeros(max(self.n_pairs, 1), dtype=torch.int32, device=dev)
        order = torch.zeros(max(self._dcloud.n, 1), dtype=torch.int32, device=dev)
        _lib.check(lib.ss_raster_tile_lists(C.byref(cam), C.byref(s), ptr(self._geom),
                                            ptr(self._bins), self.n_pairs, self._dcloud.n,
                                            ptr(ranges), ptr(members), ptr(order), stream()),
                   "tile lists")
        return ranges.view(-1, 2).cpu().numpy(), members.cpu().numpy(), order.cpu().numpy()

    @property
    def indices(self) -> np.ndarray:
        """Survivors in stable depth order (rasterizer.py:227-230)."""
        if self._indices is None:
            _, _, order = self._lists()
            self._indices = order[: self.n_survivors].astype(np.intp)
        return self._indices

    @property
    def tiles(self) -> list:
        """[(y0, y1, x0, x1, members)] for non-empty tiles, (ty, tx) order; members
        are depth ranks exactly like the reference's tile_bin (rasterizer.py:107-175)."""
        if self._tiles is None:
            ranges, members, _ = self._lists()
            self._tiles = _ranges_to_tiles(ranges, members, self.camera.width,
                                           self.camera.height, self.settings.tile_size)
        return self._tiles


def _ranges_to_tiles(ranges, members, width, height, ts):
    ntx = (width + ts - 1) // ts
    out = []
    for t in np.flatnonzero(ranges[:, 1] > ranges[:, 0]):
        ty, tx = divmod(int(t), ntx)
        a, b = ranges[t]
        out.append((ty * ts, min(ty * ts + ts, height), tx * ts, min(tx * ts + ts, width),
                    members[a:b].astype(np.intp)))
    return out


def _device_cloud(cloud):
    if isinstance(cloud, DeviceCloud):
        return cloud
    return DeviceCloud(cloud if isinstance(cloud, dict) else GaussianCloud.from_any(cloud))


def render_device(dcloud: DeviceCloud, camera, background=None,
                  settings: RasterSettings = RasterSettings(), want_touch=True):
    """Forward render of a device cloud; returns (image, alpha, touch, ctx pieces)."""
    lib = _lib.load()
    dev = require_cuda()
    camera = Camera.from_any(camera)
    cam, s = camera_struct(camera), settings_struct(settings, background)
    cl = dcloud.struct()
    geom = empty_bytes(lib.ss_raster_geom_bytes(dcloud.n, C.byref(cam), C.byref(s)), dev)
    counts = pinned(2)
    _lib.check(lib.ss_raster_forward_begin(C.byref(cl), C.byref(cam), C.byref(s), ptr(geom),
                                           ptr(counts), stream()), "rasterize_forward")
    torch.cuda.current_stream().synchronize()
    survivors, pairs = int(counts[0]), int(counts[1])
    cap = min(pairs, BIN_PAIR_LIMIT)
    bins = empty_bytes(lib.ss_raster_bin_bytes(cap, dcloud.n, C.byref(cam), C.byref(s)), dev)
    h, w = camera.height, camera.width
    image = torch.empty(h, w, 3, dtype=torch.float32, device=dev)
    alpha = torch.empty(h, w, dtype=torch.float32, device=dev)
    touch = torch.zeros(max(dcloud.n, 1), dtype=torch.int32, device=dev) if want_touch else None
    _lib.check(lib.ss_raster_forward_finish_banded(C.byref(cl), C.byref(cam), C.byref(s),
                                                   ptr(geom), ptr(bins), cap, pairs, ptr(image),
                                                   ptr(alpha), ptr(touch), stream()),
               "rasterize_forward")
    return image, alpha, touch, geom, bins, pairs, survivors, cap


def rasterize_forward(cloud, camera, background=None,
                      settings: RasterSettings = RasterSettings()):
    """rasterizer.py:214-281: (RenderOutput, RenderContext)."""
    if background is None:
        background = np.zeros(3)
    background = np.asarray(background, dtype=np.float64)
    camera = Camera.from_any(camera)
    dcloud = _device_cloud(cloud)
    image, alpha, touch, geom, bins, pairs, surv, cap = render_device(dcloud, camera, background,
                                                                      settings)
    out = RenderOutput(image=image.cpu().numpy().astype(np.float64),
                       alpha_map=alpha.cpu().numpy().astype(np.float64),
                       per_gaussian_touch_count=touch[: dcloud.n].cpu().numpy().astype(np.int64))
    ctx = RenderContext(cloud, camera, settings, background, dcloud, geom, bins, pairs, surv, cap)
    return out, ctx


def rasterize_backward(ctx: RenderContext, d_image) -> GradientBuffer:
    """rasterizer.py:284-402."""
    lib = _lib.load()
    cam_o = ctx.camera
    d_np = None if isinstance(d_image, torch.Tensor) else np.asarray(d_image, dtype=np.float64)
    shape = tuple(d_image.shape) if d_np is None else d_np.shape
    if shape != (cam_o.height, cam_o.width, 3):
        raise DataError(f"d_image shape {shape} does not match render "
                        f"{(cam_o.height, cam_o.width, 3)}")
    dc = ctx._dcloud
    n, K = dc.n, dc.sh_coeffs
    if n == 0:
        return GradientBuffer.zeros(0, K)
    dev = ctx._geom.device
    dimg = to_dev(d_image if d_np is None else d_np, dev=dev)
    f32 = dict(dtype=torch.float32, device=dev)
    bufs = dict(d_means=torch.zeros(n, 3, **f32), d_rotations=torch.zeros(n, 4, **f32),
                d_log_scales=torch.zeros(n, 3, **f32), d_opacity_logits=torch.zeros(n, **f32),
                d_sh=torch.zeros(n, K, 3, **f32), viewspace=torch.zeros(n, **f32),
                contributed=torch.zeros(n, dtype=torch.uint8, device=dev))
    g = _lib.CloudGrads()
    for k, t in bufs.items():
        setattr(g, k, ptr(t))
    cam, s = camera_struct(cam_o), settings_struct(ctx.settings, ctx.background)
    _lib.check(lib.ss_raster_backward_banded(C.byref(dc.struct()), C.byref(cam), C.byref(s),
                                             ptr(ctx._geom), ptr(ctx._bins), ctx.bin_capacity,
                                             ctx.n_pairs, ptr(dimg), C.byref(g), stream()),
               "rasterize_backward")
    h = {k: v.cpu().numpy() for k, v in bufs.items()}
    return GradientBuffer(h["d_means"].astype(np.float64), h["d_rotations"].astype(np.float64),
                          h["d_log_scales"].astype(np.float64),
                          h["d_opacity_logits"].astype(np.float64), h["d_sh"].astype(np.float64),
                          h["viewspace"].astype(np.float64), h["contributed"].astype(bool))


def tile_bin(mean2d, cov2d, opacity, width, height, tile_size, skip_alpha=1.0 / 255.0) -> list:
    """rasterizer.py:107-175 on the GPU (inputs already depth-sorted)."""
    lib = _lib.load()
    dev = require_cuda()
    mean2d = np.asarray(mean2d, dtype=np.float64).reshape(-1, 2)
    n = len(mean2d)
    cam = _lib.Camera()
    cam.width, cam.height, cam.fx, cam.fy, cam.near_clip = int(width), int(height), 1.0, 1.0, 0.01
    s = settings_struct(RasterSettings(tile_size=int(tile_size), skip_alpha=float(skip_alpha)))
    m = to_dev(mean2d, torch.float64, dev)
    cv = to_dev(np.asarray(cov2d, dtype=np.float64).reshape(-1, 2, 2), torch.float64, dev)
    op = to_dev(np.asarray(opacity, dtype=np.float64).reshape(-1), torch.float64, dev)
    geom = empty_bytes(lib.ss_raster_geom_bytes(n, C.byref(cam), C.byref(s)), dev)
    counts = pinned(2)
    _lib.check(lib.ss_tile_bin_begin(n, ptr(m), ptr(cv), ptr(op), C.byref(cam), C.byref(s),
                                     ptr(geom), ptr(counts), stream()), "tile_bin")
    torch.cuda.current_stream().synchronize()
    pairs = int(counts[1])
    bins = empty_bytes(lib.ss_raster_bin_bytes(pairs, n, C.byref(cam), C.byref(s)), dev)
    ts = int(tile_size)
    ntx, nty = (width + ts - 1) // ts, (height + ts - 1) // ts
    ranges = torch.zeros(ntx * nty * 2, dtype=torch.int32, device=dev)
    members = torch.zeros(max(pairs, 1), dtype=torch.int32, device=dev)
    _lib.check(lib.ss_tile_bin_finish(n, C.byref(cam), C.byref(s), ptr(geom), ptr(bins), pairs,
                                      ptr(ranges), ptr(members), stream()), "tile_bin")
    return _ranges_to_tiles(ranges.view(-1, 2).cpu().numpy(), members.cpu().numpy(), width,
                            height, ts)
