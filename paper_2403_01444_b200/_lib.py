"""ctypes binding of the C ABI in include/ss_b200.h (libss_b200.so, built in-tree).

This is the reference-side binding a maintainer of the `splatstream` package
would add: plain pointers and sizes, no torch types.  The
library is REQUIRED: importing the product path without it raises, there is no
CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import DataError, NumericalError, SplatstreamError

LIB_PATH = os.environ.get("SS_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                     "libss_b200.so")

MAX_LEVELS = 32
SS_OK, SS_ERR_DATA, SS_ERR_NUMERICAL, SS_ERR_CUDA, SS_ERR_CAPACITY = 0, 1, 2, 3, 4
FLAG_ZERO_QUAT, FLAG_NONFINITE, FLAG_OUTSIDE, FLAG_OVERFLOW = 1, 2, 4, 8

P = C.c_void_p


class Grid(C.Structure):
    _fields_ = [("n_levels", C.c_int32), ("n_features", C.c_int32), ("log2_table", C.c_int32),
                ("reserved", C.c_int32), ("resolution", C.c_int32 * MAX_LEVELS),
                ("aabb_min", C.c_double * 3), ("aabb_max", C.c_double * 3)]


MLP_FP32, MLP_F16 = 0, 1


class Mlp(C.Structure):
    _fields_ = [("in_dim", C.c_int32), ("hidden_dim", C.c_int32), ("n_hidden", C.c_int32),
                ("out_dim", C.c_int32), ("precision", C.c_int32)]


class MlpLayout(C.Structure):
    _fields_ = [("in_pad", C.c_int32), ("hidden_pad", C.c_int32), ("out_pad", C.c_int32),
                ("n_hidden", C.c_int32), ("w0", C.c_int64), ("b0", C.c_int64), ("w1", C.c_int64),
                ("b1", C.c_int64), ("w2", C.c_int64), ("b2", C.c_int64), ("total", C.c_int64)]


class Camera(C.Structure):
    _fields_ = [("w2c", C.c_double * 16), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("near_clip", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class RasterSettings(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("reserved", C.c_int32), ("alpha_clamp", C.c_double),
                ("skip_alpha", C.c_double), ("stop_transmittance", C.c_double),
                ("background", C.c_double * 3)]


class Cloud(C.Structure):
    _fields_ = [("n", C.c_int64), ("sh_coeffs", C.c_int32), ("reserved", C.c_int32),
                ("means", P), ("rotations", P), ("log_scales", P), ("opacity_logits", P),
                ("sh", P)]


class CloudGrads(C.Structure):
    _fields_ = [("d_means", P), ("d_rotations", P), ("d_log_scales", P),
                ("d_opacity_logits", P), ("d_sh", P), ("viewspace", P), ("contributed", P)]


class Stage1(C.Structure):
    _fields_ = [("grid", Grid), ("mlp", Mlp), ("settings", RasterSettings),
                ("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("lambda_dssim", C.c_double),
                ("rotate_sh", C.c_int32), ("accumulate_stats", C.c_int32),
                ("src", Cloud), ("n_in", C.c_int64), ("rows", P), ("rows_index", P),
                ("rows_pos", P),
                ("tables", P), ("params", P), ("g_tables", P), ("g_params", P),
                ("m_tables", P), ("v_tables", P), ("m_params", P), ("v_params", P),
                ("row_mask", P), ("step_dev", P),
                ("t_means", P), ("t_rotations", P), ("t_sh", P),
                ("image", P), ("alpha_map", P), ("d_image", P),
                ("d_means", P), ("d_rotations", P), ("d_sh", P),
                ("viewspace", P), ("contributed", P), ("stats_norm", P), ("stats_count", P),
                ("loss_dev", P), ("loss_history", P), ("pair_history", P),
                ("history_len", C.c_int64), ("iteration", C.c_int32), ("iter_dev", P),
                ("status", P), ("geom", P), ("bins", P), ("loss_scratch", P),
                ("ntc_scratch", P), ("bin_capacity", C.c_int64),
                ("ssim_c1", C.c_double), ("ssim_c2", C.c_double), ("loss_accum", P),
                ("defer_scatter", C.c_int32), ("reserved2", C.c_int32)]


STRUCTS = [Grid, Mlp, MlpLayout, Camera, RasterSettings, Cloud, CloudGrads, Stage1]

# (name, restype, argtypes) for every entry point declared in include/ss_b200.h
I32, I64, U64, D, SZ = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_size_t
PGrid, PMlp, PCam, PSet, PCloud = (C.POINTER(t) for t in (Grid, Mlp, Camera, RasterSettings, Cloud))
SIGNATURES = [
    ("ss_last_error", C.c_char_p, []),
    ("ss_version", I32, []),
    ("ss_struct_size", SZ, [I32]),
    ("ss_launch_count", I64, []),
    ("ss_profile_enable", I32, [I32]),
    ("ss_profile_enabled", I32, []),
    ("ss_profile_name", C.c_char_p, [I32]),
    ("ss_profile_count", I32, []),
    ("ss_profile_read", I32, [C.POINTER(D), I32]),
    ("ss_mlp_get_layout", I32, [PMlp, C.POINTER(MlpLayout)]),
    ("ss_ntc_encode", I32, [PGrid, I64, P, P, P, P, P]),
    ("ss_ntc_touched", I32, [PGrid, I64, P, P, P, P]),
    ("ss_ntc_forward", I32, [PGrid, PMlp, I64, P, P, P, P, P, P, P]),
    ("ss_ntc_backward_bytes", SZ, [PMlp]),
    ("ss_ntc_backward", I32, [PGrid, PMlp, I64, P, P, P, P, P, P, P, P, P]),
    ("ss_adam_step", I32, [I64, P, P, P, P, P, I32, I64, P, P, P, P, P, D, D, D, D, I32, P]),
    ("ss_apply_ntc", I32, [PGrid, PMlp, PCloud, I64, P, P, P, I32, P, P, P, P, P, P]),
    ("ss_apply_ntc_backward", I32, [PGrid, PMlp, PCloud, I64, P, P, P, I32, P, P, P, P, P, P,
                                    P]),
    ("ss_apply_ntc_backward_bytes", SZ, [I64]),
    ("ss_transform_apply", I32, [PCloud, I64, P, P, I32, P, P, P, P, P]),
    ("ss_transform_vjp", I32, [PCloud, I64, P, P, I32, P, P, P, P, P]),
    ("ss_raster_geom_bytes", SZ, [I64, PCam, PSet]),
    ("ss_raster_bin_bytes", SZ, [I64, I64, PCam, PSet]),
    ("ss_raster_forward_begin", I32, [PCloud, PCam, PSet, P, P, P]),
    ("ss_raster_forward_finish", I32, [PCloud, PCam, PSet, P, P, I64, P, P, P, P]),
    ("ss_raster_backward", I32, [PCloud, PCam, PSet, P, P, I64, P, C.POINTER(CloudGrads), P]),
    ("ss_raster_forward_finish_banded", I32, [PCloud, PCam, PSet, P, P, I64, I64, P, P, P, P]),
    ("ss_raster_backward_banded", I32, [PCloud, PCam, PSet, P, P, I64, I64, P,
                                        C.POINTER(CloudGrads), P]),
    ("ss_raster_tile_lists", I32, [PCam, PSet, P, P, I64, I64, P, P, P, P]),
    ("ss_tile_bin_begin", I32, [I64, P, P, P, PCam, PSet, P, P, P]),
    ("ss_tile_bin_finish", I32, [I64, PCam, PSet, P, P, I64, P, P, P]),
    ("ss_loss_bytes", SZ, [I32, I32, I32]),
    ("ss_render_loss", I32, [P, P, I32, I32, I32, D, D, D, P, P, P, P, P]),
    ("ss_ntc_warmup_bytes", SZ, [I64]),
    ("ss_ntc_warmup_step", I32, [PGrid, PMlp, I64, P, P, P, P, P, P, P, P, P, P, P, D, P, P, P,
                                 P]),
    ("ss_stage1_frame_begin", I32, [C.POINTER(Stage1), P]),
    ("ss_stage1_iter_begin", I32, [C.POINTER(Stage1), PCam, P, P]),
    ("ss_stage1_iter_finish", I32, [C.POINTER(Stage1), PCam, P, I64, P]),
    ("ss_stage1_iter_grads", I32, [C.POINTER(Stage1), PCam, P, I64, C.c_float, P]),
    ("ss_stage1_apply_adam", I32, [C.POINTER(Stage1), P]),
    ("ss_stage1_table_scatter", I32, [C.POINTER(Stage1), P]),
    ("ss_stage1_batch_view", I32, [C.POINTER(Stage1), PCam, P, C.c_float, I32, P]),
    ("ss_stage1_batch_ntc_grads", I32, [C.POINTER(Stage1), P]),
    ("ss_stage1_iter", I32, [C.POINTER(Stage1), PCam, P, C.c_float, I32, P]),
    ("ss_stage1_render", I32, [C.POINTER(Stage1), PCam, P]),
    ("ss_set_mlp_mode", I32, [I32]),
    ("ss_get_mlp_mode", I32, []),
    ("ss_selftest_umma", I32, [I32, I32, I32, I32, P, P, P, P]),
    ("ss_debug_mlp_trace", I32, [P]),
    ("ss_debug_mlp_events", I32, [P]),
    ("ss_debug_umma_rate", I32, [I32, I32, I32, I32, P, P]),
]


class LibraryMissing(SplatstreamError, ImportError):
    pass


_LIB = None


def load(path: str = LIB_PATH):
    """Load libss_b200.so (raises LibraryMissing; there is no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise LibraryMissing(
            f"{path} not found: build it with `python -m paper_2403_01444_b200.build`")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    for i, st in enumerate(STRUCTS):
        got = lib.ss_struct_size(i)
        if got != C.sizeof(st):
            raise LibraryMissing(f"ABI mismatch for {st.__name__}: lib {got} vs ctypes {C.sizeof(st)}")
    _LIB = lib
    return lib


def check(status: int, what: str = "") -> None:
    """Map an ss_status to the reference's exception hierarchy (errors.py:8-21)."""
    if status == SS_OK:
        return
    msg = (_LIB.ss_last_error().decode() if _LIB is not None else "") or what
    if status == SS_ERR_DATA:
        raise DataError(f"{what}: {msg}")
    if status == SS_ERR_NUMERICAL:
        raise NumericalError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: CUDA library error {status}: {msg}")


def check_flags(flags: int, what: str = "") -> None:
    """Device status word -> exceptions (gaussians.py:46-47, errors.py:24-29, ntc.py:167-168)."""
    if flags & FLAG_OUTSIDE:
        raise DataError("point outside the hash grid bounding box")
    if flags & FLAG_ZERO_QUAT:
        raise NumericalError("cannot normalize near-zero quaternion")
    if flags & FLAG_NONFINITE:
        raise NumericalError(f"non-finite values detected in '{what or 'stage1 loss'}'")
    if flags & FLAG_OVERFLOW:
        raise RuntimeError("tile-pair capacity overflow")
