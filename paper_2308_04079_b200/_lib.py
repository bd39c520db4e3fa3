"""ctypes binding of libgs_b200.so (declared in include/gs_rasterizer.h).

The product path has no fallback: if the shared library is missing the
import of this module raises, and every stage function fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int32, c_int64, c_size_t, c_uint32, c_void_p
from pathlib import Path

from .errors import InvalidPrimitiveError, ResourceLimitError

LIB_PATH = Path(os.environ.get("GS_B200_LIB") or Path(__file__).resolve().parent / "lib" / "libgs_b200.so")

GS_OK = 0
GS_ERR_INVALID_ARG = 1
GS_ERR_ZERO_QUATERNION = 2
GS_ERR_RESOURCE_LIMIT = 3
GS_ERR_CAPACITY = 4
GS_ERR_CUDA = 5

ABI_VERSION = 2

REC_FLOATS = 20
MODEL_FLOATS = 59
PLY_FLOATS = 62
LAYOUT_MODEL = 0
LAYOUT_PLY = 1
GRAD2D_FLOATS = 12


class GsCamera(ctypes.Structure):
    _fields_ = [
        ("rotation", c_double * 9), ("translation", c_double * 3),
        ("fx", c_double), ("fy", c_double), ("cx", c_double), ("cy", c_double),
        ("width", c_int32), ("height", c_int32), ("near_plane", c_double),
    ]


class GsParams(ctypes.Structure):
    _fields_ = [
        ("means", c_void_p), ("rotations", c_void_p), ("log_scales", c_void_p),
        ("opacity_logits", c_void_p), ("sh", c_void_p), ("n", c_int64),
    ]


class GsSplats(ctypes.Structure):
    _fields_ = [
        ("rec", c_void_p), ("depth", c_void_p), ("radii", c_void_p), ("rect", c_void_p),
        ("tiles_touched", c_void_p), ("status", c_void_p), ("n", c_int64),
    ]


class GsGrads(ctypes.Structure):
    _fields_ = [
        ("d_means", c_void_p), ("d_rotations", c_void_p), ("d_log_scales", c_void_p),
        ("d_opacity_logits", c_void_p), ("d_sh", c_void_p), ("view_pos_grad_norm", c_void_p),
    ]


class GsStats(ctypes.Structure):
    _fields_ = [("accum_pos_grad", c_void_p), ("accum_count", c_void_p), ("max_radius_frac", c_void_p)]


class GsAdamGroup(ctypes.Structure):
    _fields_ = [
        ("param", c_void_p), ("grad", c_void_p), ("exp_avg", c_void_p), ("exp_avg_sq", c_void_p),
        ("numel", c_int64), ("lr", c_float), ("lr_head", c_float), ("period", c_int32), ("head", c_int32),
    ]


class GsCloudState(ctypes.Structure):
    _fields_ = [("param", c_void_p * 5), ("exp_avg", c_void_p * 5), ("exp_avg_sq", c_void_p * 5), ("n", c_int64)]


class GsDensifyConfig(ctypes.Structure):
    _fields_ = [("grad_threshold", c_double), ("split_scale_threshold", c_double), ("split_log_factor", c_double),
                ("prune_alpha", c_double), ("prune_world_scale", c_double), ("prune_screen_fraction", c_double),
                ("prune_big", c_int32), ("reset_opacity", c_int32), ("reset_logit", c_float)]


# (name, restype, argtypes) — the full exported surface of gs_rasterizer.h
SIGNATURES = [
    ("gs_abi_version", c_int32, []),
    ("gs_status_string", ctypes.c_char_p, [c_int32]),
    ("gs_last_cuda_error", c_int32, [ctypes.c_char_p, c_size_t]),
    ("gs_fp32_fma_probe", c_int32, [c_void_p, c_int32, c_int32, c_void_p]),
    ("gs_preprocess_forward", c_int32, [POINTER(GsParams), POINTER(GsCamera), c_int32, POINTER(GsSplats), c_void_p]),
    ("gs_bin_workspace_size", c_int32, [c_int64, c_int32, c_int32, c_int64, POINTER(c_size_t)]),
    ("gs_bin_and_sort", c_int32, [POINTER(GsSplats), c_int32, c_int32, c_void_p, c_size_t, c_int64, c_void_p,
                                  c_void_p, c_void_p, POINTER(c_int64), c_void_p]),
    ("gs_bin_and_sort_async", c_int32, [POINTER(GsSplats), c_int32, c_int32, c_void_p, c_size_t, c_int64,
                                        c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("gs_blend_forward", c_int32, [POINTER(GsSplats), c_void_p, c_void_p, c_int32, c_int32, POINTER(c_float),
                                   c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("gs_blend_backward", c_int32, [c_void_p, POINTER(GsSplats), c_void_p, c_void_p, c_void_p, c_void_p, c_int32,
                                    c_int32, POINTER(c_float), c_void_p, c_void_p]),
    ("gs_preprocess_backward", c_int32, [POINTER(GsParams), POINTER(GsCamera), c_int32, POINTER(GsSplats),
                                         c_void_p, POINTER(GsGrads), c_int32, POINTER(GsStats), c_void_p]),
    ("gs_preprocess_backward_adam", c_int32, [POINTER(GsParams), POINTER(GsCamera), c_int32, POINTER(GsSplats),
                                              c_void_p, POINTER(GsAdamGroup), c_double, c_double, c_double,
                                              c_double, c_double, POINTER(GsStats), POINTER(GsGrads), c_void_p]),
    ("gs_preprocess_backward_adam_guarded", c_int32, [POINTER(GsParams), POINTER(GsCamera), c_int32,
                                                      POINTER(GsSplats), c_void_p, POINTER(GsAdamGroup), c_double,
                                                      c_double, c_double, c_double, c_double, POINTER(GsStats),
                                                      POINTER(GsGrads), c_void_p, c_void_p]),
    ("gs_preprocess_backward_adam_project", c_int32, [POINTER(GsParams), POINTER(GsCamera), c_int32,
                                                      POINTER(GsSplats), c_void_p, POINTER(GsAdamGroup), c_double,
                                                      c_double, c_double, c_double, c_double, POINTER(GsStats),
                                                      POINTER(GsGrads), c_void_p, POINTER(GsCamera), c_int32,
                                                      POINTER(GsSplats), c_void_p]),
    ("gs_step_guard", c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("gs_blend_backward_ordered", c_int32, [c_void_p, POINTER(GsSplats), c_void_p, c_void_p, c_void_p, c_void_p,
                                            c_int32, c_int32, POINTER(c_float), c_void_p, c_void_p, c_void_p]),
    ("gs_blend_forward_ordered", c_int32, [POINTER(GsSplats), c_void_p, c_void_p, c_int32, c_int32, POINTER(c_float),
                                           c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                           c_void_p]),
    ("gs_tile_schedule", c_int32, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
    ("gs_blend_backward_scheduled", c_int32, [c_void_p, POINTER(GsSplats), c_void_p, c_void_p, c_void_p, c_void_p,
                                              c_int32, c_int32, POINTER(c_float), c_void_p, c_void_p, c_void_p]),
    ("gs_blend_backward_schedule", c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p]),
    ("gs_blend_backward_accumulate", c_int32, [c_void_p, POINTER(GsSplats), c_void_p, c_void_p, c_void_p, c_void_p,
                                               c_int32, c_int32, POINTER(c_float), c_void_p, c_void_p, c_void_p]),
    ("gs_blend_backward_det_workspace_size", c_int32, [c_int64, c_int32, c_int32, c_int64, POINTER(c_size_t)]),
    ("gs_blend_backward_deterministic", c_int32, [c_void_p, POINTER(GsSplats), c_void_p, c_void_p, c_void_p, c_void_p,
                                                  c_int32, c_int32, POINTER(c_float), c_void_p, c_void_p, c_size_t,
                                                  c_int64, c_void_p, c_void_p]),
    ("gs_forward", c_int32, [POINTER(GsParams), POINTER(GsCamera), c_int32, POINTER(GsSplats), c_void_p, c_size_t,
                             c_int64, c_void_p, c_void_p, c_void_p, POINTER(c_float), c_int32, c_void_p, c_void_p,
                             c_void_p, c_void_p, c_void_p, c_void_p]),
    ("gs_backward", c_int32, [c_void_p, POINTER(GsParams), POINTER(GsCamera), c_int32, POINTER(GsSplats), c_void_p,
                              c_void_p, c_void_p, c_void_p, POINTER(c_float), c_void_p, c_void_p, POINTER(GsGrads),
                              POINTER(GsStats), c_void_p]),
    ("gs_backward_prepared", c_int32, [c_void_p, POINTER(GsParams), POINTER(GsCamera), c_int32, POINTER(GsSplats),
                                       c_void_p, c_void_p, c_void_p, c_void_p, POINTER(c_float), c_void_p, c_void_p,
                                       POINTER(GsGrads), POINTER(GsStats), c_void_p]),
    ("gs_densify_workspace_size", c_int32, [c_int64, POINTER(c_size_t)]),
    ("gs_densify_classify", c_int32, [POINTER(GsCloudState), POINTER(GsStats), POINTER(GsDensifyConfig), c_void_p,
                                      c_size_t, POINTER(c_int64), POINTER(c_int64), c_void_p]),
    ("gs_densify_apply", c_int32, [POINTER(GsCloudState), POINTER(GsStats), POINTER(GsDensifyConfig), c_int64,
                                   c_int64, c_void_p, c_void_p, c_size_t, POINTER(GsCloudState), POINTER(c_int64),
                                   c_void_p]),
    ("gs_loss_workspace_size", c_int32, [c_int32, c_int32, POINTER(c_size_t)]),
    ("gs_l1_dssim_loss", c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_double, c_void_p, c_size_t, c_void_p,
                                   c_void_p, c_void_p]),
    ("gs_pack_records", c_int32, [POINTER(GsParams), c_int32, c_void_p, c_void_p]),
    ("gs_unpack_records", c_int32, [c_void_p, POINTER(GsParams), c_void_p]),
    ("gs_knn_workspace_size", c_int32, [c_int64, c_int64, POINTER(c_size_t)]),
    ("gs_knn_mean_distance", c_int32, [c_void_p, c_int64, c_int32, c_int64, c_void_p, c_size_t, c_void_p,
                                       c_void_p]),
    ("gs_adam_step", c_int32, [POINTER(GsAdamGroup), c_int32, c_double, c_double, c_double, c_double, c_double,
                               c_void_p]),
    ("gs_adam_step_guarded", c_int32, [POINTER(GsAdamGroup), c_int32, c_double, c_double, c_double, c_double,
                                       c_double, c_void_p, c_void_p]),
    ("gs_preprocess_backward_guarded", c_int32, [POINTER(GsParams), POINTER(GsCamera), c_int32, POINTER(GsSplats),
                                                 c_void_p, POINTER(GsGrads), c_int32, POINTER(GsStats), c_void_p,
                                                 c_void_p]),
]

_lib = None


def load(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library; raise if it is not built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"B200 rasterizer library not found at {p}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = ctypes.CDLL(str(p))
    for name, restype, argtypes in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    if lib.gs_abi_version() != ABI_VERSION:
        raise RuntimeError("libgs_b200.so ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


def last_cuda_error() -> str:
    buf = ctypes.create_string_buffer(256)
    load().gs_last_cuda_error(buf, 256)
    return buf.value.decode()


def check(status: int, what: str) -> None:
    """Map a gs_status to the reference's exception types."""
    if status == GS_OK:
        return
    if status == GS_ERR_ZERO_QUATERNION:
        raise InvalidPrimitiveError("zero-norm quaternion cannot be normalized")
    if status == GS_ERR_RESOURCE_LIMIT:
        raise ResourceLimitError(f"{what}: tile or instance count exceeds the supported limit")
    if status == GS_ERR_INVALID_ARG:
        raise ValueError(f"{what}: invalid argument")
    if status == GS_ERR_CUDA:
        raise RuntimeError(f"{what}: CUDA error: {last_cuda_error()}")
    raise RuntimeError(f"{what}: status {status}")


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()
