"""SINO / VOL containers (formats.py of the reference) and file-to-file
reconstruction on the GPU.

Byte layouts are the reference's (formats.py:1-37), little-endian:
  SINO: "TSIN", u32 version, u32 n_proj, u32 n_rows, u32 n_chan, u8 scan_mode,
        i32 offset_chan, f32 angle_span (29 B), then f32 samples angle-major;
  VOL:  "TVOL", u32 nx, u32 ny, u32 nz, f32 voxel_pitch (20 B), then u16 z-major.
Writes are atomic (temporary sibling + rename, formats.py:44-51).

`reconstruct_file` is the GPU counterpart of `tomofuse reconstruct`
(cli.py:153-159 without the modeled pipeline): the SINO payload is read
straight into pinned host memory, streamed through
engine.StreamedReconstructor in z-sub-slabs, quantized on the device (K3)
and written as a VOL file.
"""

from __future__ import annotations

import os
import struct
from pathlib import Path

import numpy as np

from .geometry import AcquisitionParams, ScanMode, VolumeDims

SINO_MAGIC, VOL_MAGIC, SINO_VERSION = b"TSIN", b"TVOL", 1
SINO_HEADER = struct.Struct("<4sIIIIBif")  # 29 bytes
VOL_HEADER = struct.Struct("<4sIIIf")      # 20 bytes


class FormatError(ValueError):
    pass


def atomic_write(path, chunks) -> None:
    """Write `chunks` (bytes-like objects) to a temporary sibling, fsync,
    rename into place."""
    path = Path(path)
    tmp = path.with_name(path.name + ".tmp")
    with open(tmp, "wb") as fh:
        for c in chunks:
            fh.write(c)
        fh.flush()
        os.fsync(fh.fileno())
    os.replace(tmp, path)


def sino_header(params: AcquisitionParams) -> bytes:
    return SINO_HEADER.pack(SINO_MAGIC, SINO_VERSION, params.n_proj, params.n_rows, params.n_chan,
                            int(params.scan_mode), int(params.offset_chan), float(params.angle_span))


def read_sino_header(path, pixel_pitch: float = 1.0) -> AcquisitionParams:
    path = Path(path)
    try:
        with open(path, "rb") as fh:
            head = fh.read(SINO_HEADER.size)
    except FileNotFoundError:
        raise FormatError(f"missing file: {path}")
    if len(head) < SINO_HEADER.size:
        raise FormatError(f"malformed header: {path} truncated")
    magic, version, n_proj, n_rows, n_chan, mode, offset, span = SINO_HEADER.unpack(head)
    if magic != SINO_MAGIC:
        raise FormatError(f"malformed header: {path} is not a SINO file")
    if version != SINO_VERSION:
        raise FormatError(f"malformed header: unsupported SINO version {version}")
    params = AcquisitionParams(n_proj=n_proj, n_rows=n_rows, n_chan=n_chan, angle_span=float(span),
                               pixel_pitch=pixel_pitch, scan_mode=ScanMode(mode), offset_chan=offset)
    expected = SINO_HEADER.size + n_proj * n_rows * n_chan * 4
    size = path.stat().st_size
    if size != expected:
        raise FormatError(f"malformed payload: {path} holds {size - SINO_HEADER.size} bytes, "
                          f"expected {expected - SINO_HEADER.size}")
    return params


def read_sino(path, pixel_pitch: float = 1.0):
    """Reference-compatible reader: (float64 array, params) (formats.py:81-108)."""
    params = read_sino_header(path, pixel_pitch)
    data = np.fromfile(path, dtype="<f4", offset=SINO_HEADER.size)
    return data.reshape(params.n_proj, params.n_rows, params.n_chan).astype(np.float64), params


def read_sino_pinned(path, pixel_pitch: float = 1.0):
    """SINO payload read straight into a pinned host tensor (fp32, no
    float64 detour) -- the input of engine.StreamedReconstructor."""
    import torch

    params = read_sino_header(path, pixel_pitch)
    buf = torch.empty((params.n_proj, params.n_rows, params.n_chan), dtype=torch.float32, pin_memory=True)
    view = memoryview(buf.numpy()).cast("B")
    with open(path, "rb") as fh:
        fh.seek(SINO_HEADER.size)
        got = 0
        while got < len(view):
            n = fh.readinto(view[got:])
            if not n:
                raise FormatError(f"malformed payload: {path} truncated")
            got += n
    return buf, params


def write_sino(path, sino, params: AcquisitionParams) -> None:
    s = np.asarray(sino, dtype="<f4")
    if s.shape != (params.n_proj, params.n_rows, params.n_chan):
        raise FormatError(f"sinogram shape {s.shape} does not match params "
                          f"({params.n_proj}, {params.n_rows}, {params.n_chan})")
    atomic_write(path, [sino_header(params), np.ascontiguousarray(s).tobytes()])


def write_vol(path, volume, voxel_pitch: float = 1.0) -> None:
    v = volume.numpy() if hasattr(volume, "numpy") else np.asarray(volume)
    if v.ndim != 3 or v.dtype != np.uint16:
        raise FormatError("volume must be a 3D uint16 array (z, y, x)")
    nz, ny, nx = v.shape
    atomic_write(path, [VOL_HEADER.pack(VOL_MAGIC, nx, ny, nz, float(voxel_pitch)),
                        memoryview(np.ascontiguousarray(v, dtype="<u2")).cast("B")])


def read_vol(path):
    path = Path(path)
    try:
        blob = path.read_bytes()
    except FileNotFoundError:
        raise FormatError(f"missing file: {path}")
    if len(blob) < VOL_HEADER.size:
        raise FormatError(f"malformed header: {path} truncated")
    magic, nx, ny, nz, pitch = VOL_HEADER.unpack_from(blob)
    if magic != VOL_MAGIC:
        raise FormatError(f"malformed header: {path} is not a VOL file")
    body = blob[VOL_HEADER.size:]
    if len(body) != nx * ny * nz * 2:
        raise FormatError(f"malformed payload: {path} holds {len(body)} bytes, expected {nx * ny * nz * 2}")
    return (np.frombuffer(body, dtype="<u2").reshape(nz, ny, nx).copy(),
            VolumeDims(nx=nx, ny=ny, nz=nz, voxel_pitch=float(pitch)))


def reconstruct_file(sino_path, vol_path, pixel_pitch: float = 1.0, i0: float = 1e5,
                     window=(0.0, 4e-4), spec=None, feather_band: int = 32, slab_rows: int = 256,
                     device=None):
    """SINO (raw counts) -> VOL (uint16), entirely through the GPU path.
    Returns (VolumeDims, seconds spent in the GPU pipeline)."""
    import time

    import torch

    from .engine import StreamedReconstructor

    raw, params = read_sino_pinned(sino_path, pixel_pitch)
    dims = VolumeDims(nx=params.n_chan, ny=params.n_chan, nz=params.n_rows, voxel_pitch=pixel_pitch)
    eng = StreamedReconstructor(params, dims, spec, i0=i0, feather_band=feather_band, slab_rows=slab_rows,
                                device=device)
    out = torch.empty((params.n_rows, dims.ny, dims.nx), dtype=torch.uint16, pin_memory=True)
    t0 = time.perf_counter()
    eng.run(raw, out, quantize=window)
    torch.cuda.synchronize(eng.device)
    dt = time.perf_counter() - t0
    write_vol(vol_path, out, pixel_pitch)
    return dims, dt
