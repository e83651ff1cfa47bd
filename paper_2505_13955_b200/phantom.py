"""Synthetic inputs and the forward projector on the GPU.

* `project_volume` / `forward_project`: drop-ins for the reference's
  phantom.project_volume / forward_project (phantom.py:188-255) -- the
  transpose of the back-projection interpolation (K5, csrc/project.cu), so
  the pair FP/BP is adjoint like the reference's (test_phantom.py:134-146).
* `shepp_logan_raw`: analytic 3-D Shepp-Logan raw counts (K4) for benches.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import check, lib
from .fbp import _as_params, _device_array, _finish, _is_tensor, _stream, _torch
from .geometry import VolumeDims


def project_volume(volume, params):
    """Line integrals of a (nz, ny, nx) volume -> (n_proj, n_rows, n_chan),
    voxel pitch = detector pitch and FoV-masked as phantom.py:199-255.
    Returns float64 like the reference (computed in fp32)."""
    torch = _torch()
    params = _as_params(params)
    tensor_in = _is_tensor(volume)
    shape = tuple(volume.shape) if tensor_in else np.shape(volume)
    nz, ny, nx = shape
    if params.n_rows != nz:
        raise ValueError(f"params.n_rows ({params.n_rows}) must equal volume slices ({nz})")
    dims = VolumeDims(nx=nx, ny=ny, nz=nz, voxel_pitch=params.pixel_pitch)
    src = _device_array(volume, "float32")
    out = torch.empty((params.n_proj, nz, params.n_chan), dtype=torch.float32, device="cuda")
    g = _lib.geometry(params, dims)
    check(lib().tf_forward_project(ctypes.byref(g), ctypes.c_void_p(src.data_ptr()),
                                   ctypes.c_void_p(out.data_ptr()), _stream()))
    return _finish(out, tensor_in, np.float64)


def forward_project(m, params):
    """Discrete Radon transform of a microstructure's attenuation volume
    (phantom.py:188-196): `m.attenuation_volume()` projected on the GPU."""
    return project_volume(m.attenuation_volume(), params)


def shepp_logan_raw(params, dims, out=None, a0=0, a1=None, r0=0, r1=None, i0=1e5, mu_max=3.5e-4):
    """Analytic 3-D Shepp-Logan raw counts i0*exp(-p), fp32 on the device."""
    from .engine import phantom_raw

    torch = _torch()
    a1 = params.n_proj if a1 is None else a1
    r1 = params.n_rows if r1 is None else r1
    if out is None:
        out = torch.empty((a1 - a0, r1 - r0, params.n_chan), dtype=torch.float32, device="cuda")
    return phantom_raw(params, dims, out, a0, a1, r0, r1, i0, mu_max)
