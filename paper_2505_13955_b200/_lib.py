"""ctypes binding of the C ABI in include/tomofuse_b200.h.

The library is required: there is no CPU fallback anywhere in this package.
If libtomofuse_b200.so is missing, importing the compute entry points raises
(build it with `python -m paper_2505_13955_b200.build`).
"""

from __future__ import annotations

import ctypes
import os

from . import build as _build

_lib = None

TF_OK, TF_ERR_INVALID_ARGUMENT, TF_ERR_CUDA, TF_ERR_UNSUPPORTED, TF_ERR_OOM = 0, 1, 2, 3, 4
TF_F32, TF_F64 = 0, 1
TF_BP_ACCUMULATE, TF_BP_FINALIZE, TF_BP_KERNEL_V1 = 1, 2, 4
KIND = {"ramlak": 0, "shepplogan": 1}


class TfGeometry(ctypes.Structure):
    _fields_ = [
        ("n_proj", ctypes.c_int32), ("n_rows", ctypes.c_int32), ("n_chan", ctypes.c_int32),
        ("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
        ("offset_chan", ctypes.c_int32), ("scan_mode", ctypes.c_int32), ("reserved", ctypes.c_int32),
        ("angle_span", ctypes.c_double), ("pixel_pitch", ctypes.c_double),
        ("voxel_pitch", ctypes.c_double),
    ]


# name -> (restype, argtypes); mirrors include/tomofuse_b200.h exactly
_vp, _i, _i64, _d, _f = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_float
_pg = ctypes.POINTER(TfGeometry)
SIGNATURES = {
    "tf_error_string": (ctypes.c_char_p, [_i]),
    "tf_last_error": (ctypes.c_char_p, []),
    "tf_version": (_i, []),
    "tf_filter_multiplier": (_i, [_i, _i64, _d, _vp]),
    "tf_offset_weights": (_i, [_pg, _i, _vp]),
    "tf_filter_plan_create": (_i, [_i, _i, _i64, _d, _d, ctypes.POINTER(_vp)]),
    "tf_filter_plan_destroy": (_i, [_vp]),
    "tf_filter": (_i, [_vp, _vp, _vp, _i64, _f, _i, _i, _vp, _vp, _vp]),
    "tf_filter_stage": (_i, [_vp, _vp, _vp, _vp, _i64, _f, _i, _i, _vp, _vp, _vp]),
    "tf_filter_peers": (_i, [_vp, _vp, ctypes.c_int64, ctypes.c_float, _i, _i, _vp, _vp, _vp]),
    "tf_filter_stage_peers": (_i, [_vp, _vp, _vp, _i64, _f, _i, _i, _vp, _vp, _vp]),
    "tf_preprocess": (_i, [_vp, _i, _vp, _i64, _d, _vp]),
    "tf_bp_plan_create": (_i, [_pg, _i, ctypes.POINTER(_vp)]),
    "tf_bp_plan_destroy": (_i, [_vp]),
    "tf_bp_stage_bytes": (_i64, [_vp, _i]),
    "tf_bp_stage": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp]),
    "tf_backproject": (_i, [_vp, _vp, _i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp]),
    "tf_bp_smem_bytes_per_update": (_i, [_vp, _i, ctypes.POINTER(ctypes.c_double)]),
    "tf_backproject_reduce": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _vp, _i, _vp]),
    "tf_bp_finalize": (_i, [_vp, _vp, _i, _vp]),
    "tf_bp_kernel_info": (_i, [_vp, _i, _i, _i, _i, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]),
    "tf_bp_tc_supported": (_i, [_vp]),
    "tf_bp_tc_taps_bytes": (_i64, [_vp, _i, _i]),
    "tf_bp_tc_stage": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _d, _vp, _i64, _vp]),
    "tf_bp_tc_set_exponent": (_i, [_vp, _vp, _i, _d, _vp]),
    "tf_backproject_tc": (_i, [_vp, _vp, _i64, _i, _i, _i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp]),
    "tf_bp_tc_work": (_i, [_vp, _i, _i, _i, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "tf_filter_taps": (_i, [_vp, _vp, _vp, _vp, _i64, _i64, _f, _i, _vp]),
    "tf_filter_tap_bound": (_i, [_vp, _d, ctypes.POINTER(_d)]),
    "tf_quantize": (_i, [_vp, _i, _vp, _i64, _d, _d, _vp]),
    "tf_phantom_sinogram": (_i, [_pg, _i, _i, _i, _i, _d, _d, _vp, _vp]),
    "tf_forward_project": (_i, [_pg, _vp, _vp, _vp]),
    "tf_copy2d_async": (_i, [_vp, ctypes.c_size_t, _vp, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t, _vp]),
}


class TfError(RuntimeError):
    pass


def lib_path() -> str:
    return _build.SO


def lib():
    """Load (never silently skip) the CUDA library."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: the tomofuse-b200 CUDA library is required "
                "(no CPU fallback). Build it with `python -m paper_2505_13955_b200.build`.")
        L = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == TF_OK:
        return
    L = lib()
    detail = (L.tf_last_error() or b"").decode()
    if status == TF_ERR_INVALID_ARGUMENT:
        raise ValueError(detail)
    raise TfError(f"{L.tf_error_string(status).decode()}: {detail}")


def geometry(params, dims) -> TfGeometry:
    return TfGeometry(
        n_proj=params.n_proj, n_rows=params.n_rows, n_chan=params.n_chan,
        nx=dims.nx, ny=dims.ny, offset_chan=int(params.offset_chan),
        scan_mode=int(params.scan_mode), reserved=0,
        angle_span=float(params.angle_span), pixel_pitch=float(params.pixel_pitch),
        voxel_pitch=float(dims.voxel_pitch))
