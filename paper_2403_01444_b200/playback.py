"""Stream playback on the device: the reference's
`materialize_frame` / `playback_render` (pipeline.py:455-482) with the folded
cloud resident in HBM.

Frame i renders the initial cloud transformed by the NTCs of records
0..i-1 in turn (each `apply_ntc` moves only the points inside that cache's
AABB, transform.py:66-68), unioned with record i-1's added Gaussians.
`DevicePlayer` walks the frames in order and folds one NTC per frame instead
of re-folding from the initial cloud.  `stream` is duck-typed like the
reference's StreamData: .header, .initial_cloud, .records (each with .ntc_blob
and .additional), .n_frames.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .device import (DeviceCloud, grid_struct, mlp_layout, mlp_struct, pack_params, ptr,
                     require_cuda, stream, to_dev)
from .errors import DataError
from .rasterizer import render_device
from .streamio import deserialize_ntc
from .types import GaussianCloud, RasterSettings


class _Cloud:
    """A device cloud assembled from tensors (DeviceCloud interface)."""

    FIELDS = DeviceCloud.FIELDS

    def __init__(self, **t):
        for k, v in t.items():
            setattr(self, k, v.contiguous())
        self.n = int(self.means.shape[0])
        self.sh_coeffs = int(self.sh.shape[1])

    struct = DeviceCloud.struct

    def to_host(self) -> GaussianCloud:
        return GaussianCloud(*(getattr(self, f).double().cpu().numpy() for f in self.FIELDS))


def _as_device(cloud, dev) -> _Cloud:
    dc = cloud if isinstance(cloud, (_Cloud, DeviceCloud)) else DeviceCloud(cloud, dev)
    return _Cloud(**{f: getattr(dc, f) for f in DeviceCloud.FIELDS})


def apply_ntc_device(dcloud: _Cloud, cache, rotate_sh: bool = True) -> _Cloud:
    """transform.py:53-96 on a device cloud: rows inside the cache's AABB get
    mu + d_mu, norm(d_q) (x) q and rotated SH; the rest are copied."""
    lib = _lib.load()
    dev = dcloud.means.device
    g = cache.grid
    lo = torch.tensor(g.aabb_min, dtype=torch.float64, device=dev)
    hi = torch.tensor(g.aabb_max, dtype=torch.float64, device=dev)
    m64 = dcloud.means.double()
    rows = torch.nonzero(((m64 >= lo) & (m64 <= hi)).all(dim=1)).flatten().int()
    out = _Cloud(means=dcloud.means.clone(), rotations=dcloud.rotations.clone(),
                 log_scales=dcloud.log_scales, opacity_logits=dcloud.opacity_logits,
                 sh=dcloud.sh.clone())
    n_in = int(rows.numel())
    if n_in == 0:
        return out
    weights = [np.asarray(w) for w in cache.weights]
    biases = [np.asarray(b) for b in cache.biases]
    m = mlp_struct(weights[0].shape[0], weights[0].shape[1], len(weights) - 1,
                   getattr(cache, "mlp_dtype", "f32"))
    tab = to_dev(np.asarray(cache.tables), dev=dev)
    par = to_dev(pack_params(weights, biases, mlp_layout(m)), dev=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    gs = grid_struct(g)
    _lib.check(lib.ss_apply_ntc(C.byref(gs), C.byref(m), C.byref(dcloud.struct()), n_in,
                                ptr(rows), ptr(tab), ptr(par), int(rotate_sh), ptr(out.means),
                                ptr(out.rotations), ptr(out.sh), None, ptr(status), stream()),
               "apply_ntc")
    _lib.check_flags(int(status.item()))
    return out


def _concat(a: _Cloud, b: _Cloud) -> _Cloud:
    if b.sh_coeffs != a.sh_coeffs:
        raise DataError("added Gaussians have a different SH degree")
    return _Cloud(**{f: torch.cat([getattr(a, f), getattr(b, f)]) for f in DeviceCloud.FIELDS})


def _check_index(stream_data, frame_index):
    if not 0 <= frame_index < stream_data.n_frames:
        raise DataError(f"frame index {frame_index} out of range [0, {stream_data.n_frames})")


def materialize_frame_device(stream_data, frame_index: int) -> _Cloud:
    _check_index(stream_data, frame_index)
    dev = require_cuda()
    cloud = _as_device(stream_data.initial_cloud, dev)
    for record in stream_data.records[:frame_index]:
        cloud = apply_ntc_device(cloud, deserialize_ntc(record.ntc_blob))
    if frame_index > 0:
        cloud = _concat(cloud, _as_device(stream_data.records[frame_index - 1].additional, dev))
    return cloud


def materialize_frame(stream_data, frame_index: int) -> GaussianCloud:
    """pipeline.py:455-468: the frame's render set (host arrays)."""
    return materialize_frame_device(stream_data, frame_index).to_host()


def playback_render(stream_data, frame_index: int, camera,
                    settings: RasterSettings = RasterSettings()) -> np.ndarray:
    """pipeline.py:471-480: the frame rendered from `camera`."""
    bg = np.asarray(stream_data.header.get("background", [0, 0, 0]), dtype=float)
    cloud = materialize_frame_device(stream_data, frame_index)
    image = render_device(cloud, camera, bg, settings, want_touch=False)[0]
    return image.cpu().numpy().astype(np.float64)


class DevicePlayer:
    """Sequential playback: frame i's base cloud is frame i-1's base folded by
    one more NTC, so a whole stream costs one apply_ntc per frame."""

    def __init__(self, stream_data, settings: RasterSettings = RasterSettings()):
        self.stream = stream_data
        self.settings = settings
        self.bg = np.asarray(stream_data.header.get("background", [0, 0, 0]), dtype=float)
        self.dev = require_cuda()
        self.base = _as_device(stream_data.initial_cloud, self.dev)
        self.index = 0

    def seek(self, frame_index: int) -> _Cloud:
        _check_index(self.stream, frame_index)
        if frame_index < self.index:
            self.base = _as_device(self.stream.initial_cloud, self.dev)
            self.index = 0
        while self.index < frame_index:
            rec = self.stream.records[self.index]
            self.base = apply_ntc_device(self.base, deserialize_ntc(rec.ntc_blob))
            self.index += 1
        if frame_index == 0:
            return self.base
        return _concat(self.base, _as_device(self.stream.records[frame_index - 1].additional,
                                             self.dev))

    def render(self, frame_index: int, camera) -> torch.Tensor:
        return render_device(self.seek(frame_index), camera, self.bg, self.settings,
                             want_touch=False)[0]
