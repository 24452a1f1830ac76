"""Device plumbing: torch tensors as caller-owned memory for the C ABI, struct
builders, parameter packing.  torch is used for allocation, streams and
collectives only -- all math runs in libss_b200.so."""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .errors import DataError
from .types import Camera, HashGridConfig, RasterSettings


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2403_01444_b200 needs a CUDA device (B200); no CPU fallback")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def ptr(t) -> C.c_void_p | None:
    """Raw device address.  The caller must keep `t` referenced until the
    launch is enqueued (a freed temporary can be reused by the next allocation)."""
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def to_dev(a, dtype=torch.float32, dev=None) -> torch.Tensor:
    dev = dev or require_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dtype).contiguous()


def empty_bytes(n: int, dev=None) -> torch.Tensor:
    return torch.empty(max(int(n), 256), dtype=torch.uint8, device=dev or require_cuda())


def grid_struct(g: HashGridConfig) -> _lib.Grid:
    g = HashGridConfig.from_any(g)
    if g.n_levels > _lib.MAX_LEVELS:
        raise DataError("at most 32 hash-grid levels")
    s = _lib.Grid()
    s.n_levels, s.n_features, s.log2_table = g.n_levels, g.n_features, g.table_size_log2
    for l in range(g.n_levels):
        s.resolution[l] = g.resolution(l)  # host float64 formula (ntc.py:54-55)
    for d in range(3):
        s.aabb_min[d] = float(g.aabb_min[d])
        s.aabb_max[d] = float(g.aabb_max[d])
    return s


MLP_DTYPES = {"f32": _lib.MLP_FP32, "f16": _lib.MLP_F16}


def mlp_struct(in_dim: int, hidden_dim: int, n_hidden: int, mlp_dtype: str = "f32") -> _lib.Mlp:
    """mlp_dtype "f16": fp16 weights / activations with fp32 accumulation
    (BASELINE config 1); "f32": the fp32-accurate decoder."""
    if mlp_dtype not in MLP_DTYPES:
        raise DataError(f"unknown mlp_dtype {mlp_dtype!r} (f32 | f16)")
    m = _lib.Mlp()
    m.in_dim, m.hidden_dim, m.n_hidden, m.out_dim = in_dim, hidden_dim, n_hidden, 7
    m.precision = MLP_DTYPES[mlp_dtype]
    return m


def mlp_layout(m: _lib.Mlp) -> _lib.MlpLayout:
    lay = _lib.MlpLayout()
    _lib.check(_lib.load().ss_mlp_get_layout(C.byref(m), C.byref(lay)), "mlp layout")
    return lay


def pack_params(weights, biases, lay: _lib.MlpLayout) -> np.ndarray:
    """Reference (fan_in, fan_out) weights -> padded device vector (include/ss_b200.h)."""
    v = np.zeros(lay.total, dtype=np.float32)
    hp, op = lay.hidden_pad, lay.out_pad
    offs = [(lay.w0, lay.b0, lay.in_pad, hp)]
    if lay.n_hidden == 2:
        offs.append((lay.w1, lay.b1, hp, hp))
    offs.append((lay.w2, lay.b2, hp, op))
    for (wo, bo, rows, cols), w, b in zip(offs, weights, biases):
        w = np.asarray(w)
        full = np.zeros((rows, cols), dtype=np.float32)
        full[: w.shape[0], : w.shape[1]] = w
        v[wo:wo + rows * cols] = full.ravel()
        v[bo:bo + len(b)] = np.asarray(b, dtype=np.float32)
    return v


def unpack_params(v: np.ndarray, shapes, lay: _lib.MlpLayout):
    """Inverse of pack_params; `shapes` = reference weight shapes."""
    hp, op = lay.hidden_pad, lay.out_pad
    offs = [(lay.w0, lay.b0, lay.in_pad, hp)]
    if lay.n_hidden == 2:
        offs.append((lay.w1, lay.b1, hp, hp))
    offs.append((lay.w2, lay.b2, hp, op))
    ws, bs = [], []
    for (wo, bo, rows, cols), (fi, fo) in zip(offs, shapes):
        full = np.asarray(v[wo:wo + rows * cols], dtype=np.float64).reshape(rows, cols)
        ws.append(full[:fi, :fo].copy())
        bs.append(np.asarray(v[bo:bo + fo], dtype=np.float64).copy())
    return ws, bs


def camera_struct(cam) -> _lib.Camera:
    cam = Camera.from_any(cam)
    s = _lib.Camera()
    for i, v in enumerate(np.asarray(cam.world_to_camera, dtype=np.float64).ravel()):
        s.w2c[i] = float(v)
    s.fx, s.fy, s.cx, s.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    s.near_clip = float(cam.near_clip)
    s.width, s.height = int(cam.width), int(cam.height)
    return s


def settings_struct(settings: RasterSettings | None, background=None) -> _lib.RasterSettings:
    st = settings or RasterSettings()
    s = _lib.RasterSettings()
    s.tile_size = int(st.tile_size)
    s.alpha_clamp, s.skip_alpha = float(st.alpha_clamp), float(st.skip_alpha)
    s.stop_transmittance = float(st.stop_transmittance)
    bg = np.zeros(3) if background is None else np.asarray(background, dtype=np.float64)
    for i in range(3):
        s.background[i] = float(bg[i])
    return s


class DeviceCloud:
    """A GaussianCloud resident in HBM as float32 SoA."""

    FIELDS = ("means", "rotations", "log_scales", "opacity_logits", "sh")

    def __init__(self, cloud, dev=None):
        dev = dev or require_cuda()
        for f in self.FIELDS:
            setattr(self, f, to_dev(getattr(cloud, f) if not isinstance(cloud, dict) else cloud[f],
                                    dev=dev))
        self.n = int(self.means.shape[0])
        self.sh_coeffs = int(self.sh.shape[1])

    def struct(self, means=None, rotations=None, sh=None) -> _lib.Cloud:
        c = _lib.Cloud()
        c.n, c.sh_coeffs = self.n, self.sh_coeffs
        c.means = ptr(means if means is not None else self.means)
        c.rotations = ptr(rotations if rotations is not None else self.rotations)
        c.log_scales = ptr(self.log_scales)
        c.opacity_logits = ptr(self.opacity_logits)
        c.sh = ptr(sh if sh is not None else self.sh)
        return c


def pinned(n: int, dtype=torch.int64) -> torch.Tensor:
    return torch.zeros(n, dtype=dtype, pin_memory=True)
