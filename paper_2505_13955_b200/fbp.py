"""GPU filtered back-projection -- drop-in for `tomofuse.fbp`.

Same public names, signatures, argument meaning, return shapes/dtypes and
ValueError texts as `/root/reference/pkg/src/tomofuse/fbp.py`; every compute
call goes through the sm_100a C ABI (`include/tomofuse_b200.h`).  There is no
CPU path: without a CUDA device / the built library these functions raise.

Inputs may be numpy arrays (results come back as numpy, like the reference)
or CUDA torch tensors (results stay on the device, for device-resident
pipelines).  Arithmetic: filtering and back-projection accumulate in fp32
with fp64-accurate detector coordinates (relative L2 vs the reference's
float64 output <= 1e-5, tests/test_gpu_parity.py); preprocess, quantize,
offset_weights and filter_multiplier are fp64 and match the reference
bit-for-bit (quantize, offset_weights) or to 1e-15.
"""

from __future__ import annotations

import ctypes
import functools
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, lib
from .geometry import AcquisitionParams, ScanMode, VolumeDims

LOG_CLAMP_COUNTS = 1.0  # fbp.py:26


@dataclass(frozen=True)
class FilterSpec:
    """Ramp filter configuration (fbp.py:29-60)."""

    kind: str = "ramlak"
    padding: int | None = None
    blur_sigma: float = 0.0

    def __post_init__(self):
        if self.kind not in ("ramlak", "shepplogan"):
            raise ValueError(f"unknown filter kind {self.kind!r}")
        if self.blur_sigma < 0:
            raise ValueError("blur_sigma must be >= 0")

    def padded_length(self, n_chan: int) -> int:
        need = 2 * n_chan
        if self.padding is not None:
            if self.padding < need:
                raise ValueError(
                    f"padding {self.padding} below required {need} for {n_chan} channels")
            return self.padding
        return 1 << max(0, (need - 1).bit_length())


@dataclass(frozen=True)
class HuWindow:
    """Intensity window mapped onto the full uint16 range (fbp.py:63-72)."""

    lo: float
    hi: float

    def __post_init__(self):
        if not self.lo < self.hi:
            raise ValueError(f"window requires lo < hi, got [{self.lo}, {self.hi}]")


# ---------------------------------------------------------------- plumbing
def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2505_13955_b200 requires a CUDA device (no CPU fallback)")
    return torch


def _stream():
    return ctypes.c_void_p(_torch().cuda.current_stream().cuda_stream)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _dtype_name(x) -> str:
    """'float32', 'float64', ... for numpy arrays and torch tensors alike."""
    return str(x.dtype).replace("torch.", "")


def _device_array(x, dtype="float32"):
    """Contiguous CUDA tensor of `dtype` holding x (numpy or torch)."""
    torch = _torch()
    tdt = getattr(torch, dtype)
    if _is_tensor(x):
        return x.to(device="cuda", dtype=tdt).contiguous()
    a = np.ascontiguousarray(np.asarray(x), dtype=np.dtype(dtype))
    return torch.from_numpy(a).to("cuda")


def _finish(t, like_tensor: bool, np_dtype):
    """Return a device tensor as the caller's array kind / dtype."""
    if like_tensor:
        torch = _torch()
        return t.to(getattr(torch, np.dtype(np_dtype).name))
    return t.cpu().numpy().astype(np_dtype, copy=False)


class _FilterPlan:
    def __init__(self, n_chan, kind, padded, pixel_pitch, blur_sigma):
        h = ctypes.c_void_p()
        check(lib().tf_filter_plan_create(n_chan, _lib.KIND[kind], padded, pixel_pitch, blur_sigma,
                                          ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        if getattr(self, "handle", None) and _lib._lib is not None:
            _lib._lib.tf_filter_plan_destroy(self.handle)


class _BPPlan:
    def __init__(self, params, dims, feather_band):
        h = ctypes.c_void_p()
        self.geom = _lib.geometry(params, dims)
        check(lib().tf_bp_plan_create(ctypes.byref(self.geom), feather_band, ctypes.byref(h)))
        self.handle = h

    def stage_bytes(self, n_rows: int) -> int:
        return int(lib().tf_bp_stage_bytes(self.handle, n_rows))

    def __del__(self):
        if getattr(self, "handle", None) and _lib._lib is not None:
            _lib._lib.tf_bp_plan_destroy(self.handle)


@functools.lru_cache(maxsize=16)
def _filter_plan(device, n_chan, kind, padded, pixel_pitch, blur_sigma):
    return _FilterPlan(n_chan, kind, padded, pixel_pitch, blur_sigma)


@functools.lru_cache(maxsize=16)
def _bp_plan(device, params: AcquisitionParams, dims_key, feather_band):
    nx, ny, voxel_pitch = dims_key
    return _BPPlan(params, VolumeDims(nx=nx, ny=ny, nz=params.n_rows, voxel_pitch=voxel_pitch),
                   feather_band)


def filter_plan(n_chan: int, spec: "FilterSpec", pixel_pitch: float = 1.0) -> _FilterPlan:
    padded = spec.padded_length(n_chan)  # validates like fbp.py:48-60
    return _filter_plan(_torch().cuda.current_device(), n_chan, spec.kind, int(padded),
                        float(pixel_pitch), float(spec.blur_sigma))


def bp_plan(params, dims, feather_band: int = 32) -> _BPPlan:
    params = _as_params(params)
    return _bp_plan(_torch().cuda.current_device(), params,
                    (dims.nx, dims.ny, float(dims.voxel_pitch)), int(feather_band))


def _as_params(p) -> AcquisitionParams:
    """Accept the reference's AcquisitionParams (duck-typed) as well as ours."""
    if isinstance(p, AcquisitionParams):
        return p
    return AcquisitionParams(n_proj=p.n_proj, n_rows=p.n_rows, n_chan=p.n_chan,
                             angle_span=p.angle_span, pixel_pitch=p.pixel_pitch,
                             scan_mode=ScanMode(int(p.scan_mode)), offset_chan=p.offset_chan)


# ---------------------------------------------------------------- public API
def preprocess(raw, i0: float):
    """Beer-Lambert depth -ln(max(raw, 1)/i0) (fbp.py:75-83), fp64 on the GPU."""
    if i0 <= 0:
        raise ValueError(f"i0 must be positive, got {i0}")
    torch = _torch()
    tensor_in = _is_tensor(raw)
    a = raw if tensor_in else np.asarray(raw)
    use64 = _dtype_name(a) != "float32"  # the reference reads counts as float64
    src = _device_array(a, "float64" if use64 else "float32")
    out = torch.empty(src.shape, dtype=torch.float64, device="cuda")
    check(lib().tf_preprocess(_ptr(src), _lib.TF_F64 if use64 else _lib.TF_F32, _ptr(out),
                              src.numel(), float(i0), _stream()))
    return out if tensor_in else out.cpu().numpy()


def filter_kernel(kind: str, padded: int) -> np.ndarray:
    """Band-limited spatial kernel on the circular padded grid (fbp.py:86-102).
    A host-side table (not on the hot path); the GPU filter derives its own
    spectrum in the C library (tf_filter_multiplier)."""
    m = np.arange(padded)
    d = np.where(m <= padded // 2, m, m - padded).astype(np.float64)
    if kind == "ramlak":
        h = np.zeros(padded)
        odd = d % 2 != 0
        h[odd] = -1.0 / (np.pi ** 2 * d[odd] ** 2)
        h[0] = 0.25
        return h
    return -2.0 / (np.pi ** 2 * (4.0 * d ** 2 - 1.0))


def filter_multiplier(kind: str, padded: int, pixel_pitch: float = 1.0) -> np.ndarray:
    """rfft-domain multiplier Re(rfft(kernel))/pitch (fbp.py:105-116), fp64,
    computed by the C library."""
    if kind not in _lib.KIND:
        raise ValueError(f"unknown filter kind {kind!r}")
    out = np.empty(padded // 2 + 1, dtype=np.float64)
    check(lib().tf_filter_multiplier(_lib.KIND[kind], int(padded), float(pixel_pitch),
                                     out.ctypes.data_as(ctypes.c_void_p)))
    return out


def ramp_filter(sino, spec: FilterSpec, pixel_pitch: float = 1.0):
    """Filter every (angle, row) line along channels (fbp.py:119-131).
    Returns float64 like the reference (computed in fp32 on the GPU)."""
    torch = _torch()
    tensor_in = _is_tensor(sino)
    shape = tuple(sino.shape) if tensor_in else np.shape(sino)
    n_chan = shape[-1]
    plan = filter_plan(n_chan, spec, pixel_pitch)
    src = _device_array(sino, "float32")
    n_lines = src.numel() // max(n_chan, 1)
    out = torch.empty(src.shape, dtype=torch.float32, device="cuda")
    check(lib().tf_filter(plan.handle, _ptr(src), _ptr(out), n_lines, 0.0, 0, 0, None, None,
                          _stream()))
    return _finish(out, tensor_in, np.float64)


def fov_radius_channels(params: AcquisitionParams) -> float:
    """Scanned field-of-view radius in channels (fbp.py:134-144)."""
    half = (params.n_chan - 1) / 2.0
    if params.scan_mode == ScanMode.NORMAL:
        return half
    return half + abs(params.offset_chan)


def offset_weights(params: AcquisitionParams, band: int = 32) -> np.ndarray:
    """Offset-scan feather normalised against the conjugate channel
    (fbp.py:147-183), fp64 from the C library."""
    params = _as_params(params)
    g = _lib.geometry(params, VolumeDims(2, 2, 1))
    out = np.empty(params.n_chan, dtype=np.float64)
    check(lib().tf_offset_weights(ctypes.byref(g), int(band), out.ctypes.data_as(ctypes.c_void_p)))
    return out


def _tensor_path(plan) -> bool:
    """K2 on the tensor cores when the geometry allows it (the default);
    TF_BP_TENSOR=0 selects the CUDA-core kernel."""
    import os

    return os.environ.get("TF_BP_TENSOR", "1") != "0" and bool(lib().tf_bp_tc_supported(plan.handle))


def _bp_device(src_rows, params, dims, angles, tile, feather_band):
    """Stage + back-project device rows (n_proj, k, n_chan) -> (k, ny, nx) fp32.
    Tensor path: tap planes of angles [a0, a1) with per-row exponents from
    the rows' own data (row independence, test_fbp.py:180-191)."""
    torch = _torch()
    plan = bp_plan(params, dims, feather_band)
    k = src_rows.shape[1]
    vol = torch.empty((k, dims.ny, dims.nx), dtype=torch.float32, device="cuda")
    if (tile[1] - tile[0]) * (tile[3] - tile[2]) < dims.nx * dims.ny:
        vol.zero_()  # voxels outside the tile are zero (fbp.py:236)
    s = _stream()
    a0, a1 = angles
    x0, x1, y0, y1 = tile
    if _tensor_path(plan):
        nb = int(lib().tf_bp_tc_taps_bytes(plan.handle, k, a1 - a0))
        taps = torch.empty(nb, dtype=torch.uint8, device="cuda")
        check(lib().tf_bp_tc_stage(plan.handle, _ptr(src_rows), k, 0, k, a0, a1, 0.0, _ptr(taps), nb, s))
        check(lib().tf_backproject_tc(plan.handle, _ptr(taps), nb, a0, a1, k, _ptr(vol), a0, a1, x0, x1, y0, y1,
                                      _lib.TF_BP_FINALIZE, s))
        return vol
    stage = torch.empty(plan.stage_bytes(k), dtype=torch.uint8, device="cuda")
    check(lib().tf_bp_stage(plan.handle, _ptr(src_rows), k, 0, k, _ptr(stage), s))
    check(lib().tf_backproject(plan.handle, _ptr(stage), k, _ptr(vol), a0, a1, x0, x1, y0, y1,
                               _lib.TF_BP_FINALIZE, s))
    return vol


def back_project(sino, dims: VolumeDims, params: AcquisitionParams, rows=None, angles=None,
                 tile=None, feather_band: int = 32, dtype=np.float64):
    """Back-project filtered lines into a partial volume (fbp.py:186-252).

    Returns (r1 - r0, ny, nx) of `dtype`, zero outside `tile` and outside the
    scanned field of view; accumulation runs in ascending angle order.
    """
    tensor_in = _is_tensor(sino)
    if not tensor_in:
        sino = np.asarray(sino)
    shape = tuple(sino.shape)
    if shape != (params.n_proj, params.n_rows, params.n_chan):
        raise ValueError(
            f"sinogram shape {shape} does not match params "
            f"({params.n_proj}, {params.n_rows}, {params.n_chan})")
    r0, r1 = rows if rows is not None else (0, params.n_rows)
    a0, a1 = angles if angles is not None else (0, params.n_proj)
    x0, x1, y0, y1 = tile if tile is not None else (0, dims.nx, 0, dims.ny)
    if not (0 <= r0 <= r1 <= params.n_rows):
        raise ValueError(f"row range ({r0}, {r1}) out of bounds")
    if not (0 <= a0 <= a1 <= params.n_proj):
        raise ValueError(f"angle range ({a0}, {a1}) out of bounds")
    if not (0 <= x0 <= x1 <= dims.nx and 0 <= y0 <= y1 <= dims.ny):
        raise ValueError(f"tile ({x0}, {x1}, {y0}, {y1}) out of bounds")
    if r1 == r0 or a1 == a0 or x1 == x0 or y1 == y0:
        z = np.zeros((r1 - r0, dims.ny, dims.nx), dtype=dtype)
        if tensor_in:
            torch = _torch()
            return torch.from_numpy(z).to("cuda")
        return z
    src = _device_array(sino[:, r0:r1], "float32")
    vol = _bp_device(src, params, dims, (a0, a1), (x0, x1, y0, y1), feather_band)
    return _finish(vol, tensor_in, dtype)


def quantize(volume, window: HuWindow):
    """Window + round-half-even to uint16 (fbp.py:255-259), fp64 on the GPU,
    bit-identical to the reference for the same input values."""
    torch = _torch()
    tensor_in = _is_tensor(volume)
    v = volume if tensor_in else np.asarray(volume)
    is32 = _dtype_name(v) == "float32"
    src = _device_array(v, "float32" if is32 else "float64")
    out = torch.empty(src.shape, dtype=torch.uint16, device="cuda")
    check(lib().tf_quantize(_ptr(src), _lib.TF_F32 if is32 else _lib.TF_F64, _ptr(out), src.numel(),
                            float(window.lo), float(window.hi), _stream()))
    return out if tensor_in else out.cpu().numpy()


def reconstruct(depth_sino, dims: VolumeDims, params: AcquisitionParams, spec: FilterSpec | None = None,
                feather_band: int = 32, dtype=np.float64):
    """Serial FBP of an optical-depth sinogram (fbp.py:262-275): filter and
    back-project on the device without a host round trip."""
    torch = _torch()
    spec = spec if spec is not None else FilterSpec()
    tensor_in = _is_tensor(depth_sino)
    shape = tuple(depth_sino.shape) if tensor_in else np.shape(depth_sino)
    if shape != (params.n_proj, params.n_rows, params.n_chan):
        raise ValueError(
            f"sinogram shape {shape} does not match params "
            f"({params.n_proj}, {params.n_rows}, {params.n_chan})")
    plan = filter_plan(params.n_chan, spec, params.pixel_pitch)
    src = _device_array(depth_sino, "float32")
    bplan = bp_plan(params, dims, feather_band)
    n_lines = src.numel() // params.n_chan
    if _tensor_path(bplan):
        # K1 straight into the tap planes (per-row exponents from the depth data), then K2-TC
        nb = int(lib().tf_bp_tc_taps_bytes(bplan.handle, params.n_rows, params.n_proj))
        taps = torch.empty(nb, dtype=torch.uint8, device="cuda")
        vol = torch.empty((params.n_rows, dims.ny, dims.nx), dtype=torch.float32, device="cuda")
        s = _stream()
        check(lib().tf_filter_taps(plan.handle, bplan.handle, _ptr(src), _ptr(taps), nb, n_lines, 0.0,
                                   params.n_rows, s))
        check(lib().tf_backproject_tc(bplan.handle, _ptr(taps), nb, 0, params.n_proj, params.n_rows, _ptr(vol), 0,
                                      params.n_proj, 0, dims.nx, 0, dims.ny, _lib.TF_BP_FINALIZE, s))
        return _finish(vol, tensor_in, dtype)
    filt = torch.empty_like(src)
    check(lib().tf_filter(plan.handle, _ptr(src), _ptr(filt), n_lines, 0.0, 0, 0, None, None, _stream()))
    vol = _bp_device(filt, params, dims, (0, params.n_proj), (0, dims.nx, 0, dims.ny), feather_band)
    return _finish(vol, tensor_in, dtype)
