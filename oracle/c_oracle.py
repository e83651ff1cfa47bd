"""ctypes binding of oracle/liboracle_fbp.so -- TEST INFRASTRUCTURE ONLY.

The C restatement is bit-identical to the reference's float64 (and float32)
back-projection and is fast enough (pthreads over rows) to check sampled
rows of the 2048^3 configuration in seconds.  Loaded only by tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline leg.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_fbp.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        dp = ctypes.POINTER(ctypes.c_double)
        i, d = ctypes.c_int, ctypes.c_double
        L.oracle_back_project.argtypes = [dp, i, i, i, i, i, d, d, d, i, i, i, i, i, i, i,
                                          i, i, dp, i]
        L.oracle_back_project.restype = i
        L.oracle_ramp_filter.argtypes = [dp, dp, ctypes.c_long, i, i, d, d, i]
        L.oracle_preprocess.argtypes = [dp, dp, ctypes.c_long, d]
        L.oracle_quantize.argtypes = [dp, ctypes.POINTER(ctypes.c_uint16), ctypes.c_long, d, d]
        L.oracle_offset_weights.argtypes = [dp, i, i, i]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _threads(n):
    return n if n else (os.cpu_count() or 1)


def back_project(sino_rows, geom, angle_range=None, tile=None, feather_band=32,
                 use_f32=False, threads=0):
    """sino_rows: (n_proj, k, n_chan) -- only the rows to reconstruct."""
    s = np.ascontiguousarray(sino_rows, dtype=np.float64)
    n_proj, k, n = s.shape
    nx, ny = geom["nx"], geom["ny"]
    a0, a1 = angle_range if angle_range is not None else (0, n_proj)
    x0, x1, y0, y1 = tile if tile is not None else (0, nx, 0, ny)
    out = np.empty((k, ny, nx), dtype=np.float64)
    rc = lib().oracle_back_project(_p(s), n_proj, k, n, nx, ny, geom["span"],
                                   geom["pixel_pitch"], geom["voxel_pitch"],
                                   geom["offset_chan"], a0, a1, x0, x1, y0, y1,
                                   feather_band, int(use_f32), _p(out), _threads(threads))
    if rc != 0:
        raise ValueError("feather band must be >= 1 channel")
    return out.astype(np.float32) if use_f32 else out


def ramp_filter(sino, kind="ramlak", pixel_pitch=1.0, blur_sigma=0.0, threads=0):
    s = np.ascontiguousarray(sino, dtype=np.float64)
    out = np.empty_like(s)
    n = s.shape[-1]
    lib().oracle_ramp_filter(_p(s), _p(out), s.size // n, n, 0 if kind == "ramlak" else 1,
                             pixel_pitch, blur_sigma, _threads(threads))
    return out


def preprocess(raw, i0):
    r = np.ascontiguousarray(raw, dtype=np.float64)
    out = np.empty_like(r)
    lib().oracle_preprocess(_p(r), _p(out), r.size, i0)
    return out


def quantize(v, lo, hi):
    a = np.ascontiguousarray(v, dtype=np.float64)
    q = np.empty(a.shape, dtype=np.uint16)
    lib().oracle_quantize(_p(a), q.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)), a.size, lo, hi)
    return q


def offset_weights(n, offset_chan, band=32):
    w = np.empty(n, dtype=np.float64)
    lib().oracle_offset_weights(_p(w), n, offset_chan, band)
    return w


def fbp_rows(raw_rows, geom, i0=1e5, kind="ramlak", feather_band=32, use_f32=False, threads=0):
    """preprocess -> ramp filter -> BP of sampled raw rows (n_proj, k, n_chan)."""
    depth = preprocess(raw_rows, i0)
    filt = ramp_filter(depth, kind, geom["pixel_pitch"], threads=threads)
    if use_f32:
        filt = filt.astype(np.float32)
    return back_project(filt, geom, feather_band=feather_band, use_f32=use_f32, threads=threads)
