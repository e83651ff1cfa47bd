"""CPU oracle for the FBP hot path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

This module is a numpy restatement of the reference reconstruction chain
(`/root/reference/pkg/src/tomofuse/fbp.py` + `geometry.py`).  It exists only
so that `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg
have a checker / CPU timing arm.  The product path
(`paper_2505_13955_b200`) never imports it; a product call that lands here
would void the parity claims, so the package has no import of `oracle`.

Parity pinning: every function below is checked against golden vectors that
`tests/golden/make_golden.py` produced by importing the reference package
itself (`tests/test_cpu_host.py`, the oracle-vs-golden tests).  Third-party arithmetic the reference
delegates to:

* numpy.fft.rfft/irfft (pocketfft, numpy 2.3.5 here) -- used the same way
  below, and additionally pinned by the O(n^2) spatial-convolution oracle the
  reference's own tests use (`pkg/tests/test_fbp.py:66-75`).
* scipy.ndimage.gaussian_filter1d (scipy 1.18.1) -- restated below from its
  published algorithm (radius int(truncate*sigma+0.5), normalised Gaussian,
  correlate with mode="nearest"), pinned against scipy in the golden script.

Float-order notes (what makes the fp64 restatement bit-identical to the
reference): the detector coordinate is evaluated as
`((x-cx)*cos + (y-cy)*sin) * scale + axis` exactly as
`geometry.py:148-153`, angles are `k * (span / n_proj)` (`geometry.py:69-70`),
and accumulation is `acc += g0 + g1` in ascending angle order
(`fbp.py:233-245`).
"""

from __future__ import annotations

import math

import numpy as np

LOG_CLAMP = 1.0  # fbp.py:26 (counts clamped to one before the log)


# ---------------------------------------------------------------------------
# geometry (geometry.py:27-153)


def angles(n_proj: int, span: float) -> np.ndarray:
    """theta_k = k * (span / n_proj)  -- geometry.py:69-70."""
    step = span / n_proj
    return np.arange(n_proj) * step


def axis_channel(n_chan: int, offset_chan: int) -> float:
    """(n_chan-1)/2 - offset  -- geometry.py:60-67."""
    return (n_chan - 1) / 2.0 - offset_chan


def ray_coordinate(x, y, theta, n_chan, offset_chan, nx, ny, voxel_pitch, pixel_pitch):
    """Continuous channel of the ray through (x, y) -- geometry.py:142-153."""
    cx = (nx - 1) / 2.0
    cy = (ny - 1) / 2.0
    s = voxel_pitch / pixel_pitch
    u = (np.asarray(x, dtype=np.float64) - cx) * math.cos(theta)
    u = u + (np.asarray(y, dtype=np.float64) - cy) * math.sin(theta)
    return u * s + axis_channel(n_chan, offset_chan)


# ---------------------------------------------------------------------------
# preprocessing + filtering (fbp.py:75-131)


def preprocess(raw, i0: float) -> np.ndarray:
    """Beer-Lambert depth -ln(max(raw,1)/i0), float64 -- fbp.py:75-83."""
    if i0 <= 0:
        raise ValueError(f"i0 must be positive, got {i0}")
    r = np.maximum(np.asarray(raw, dtype=np.float64), LOG_CLAMP)
    return -np.log(r / i0)


def padded_length(n_chan: int, padding=None) -> int:
    """next pow2 >= 2n, or validated explicit padding -- fbp.py:48-60."""
    need = 2 * n_chan
    if padding is not None:
        if padding < need:
            raise ValueError(f"padding {padding} below required {need} for {n_chan} channels")
        return int(padding)
    return 1 << max(0, (need - 1).bit_length())


def kernel_tap(kind: str, d: int) -> float:
    """Band-limited spatial ramp kernel at integer lag d -- fbp.py:86-102."""
    if kind == "ramlak":
        if d == 0:
            return 0.25
        return -1.0 / (math.pi ** 2 * d * d) if d % 2 else 0.0
    return -2.0 / (math.pi ** 2 * (4.0 * d * d - 1.0))


def filter_kernel(kind: str, padded: int) -> np.ndarray:
    """Circular kernel on the padded grid -- fbp.py:86-102."""
    m = np.arange(padded)
    lag = np.where(m <= padded // 2, m, m - padded).astype(np.float64)
    if kind == "ramlak":
        h = np.where(lag % 2 != 0, -1.0 / (np.pi ** 2 * np.where(lag == 0, 1.0, lag) ** 2), 0.0)
        h[0] = 0.25
        return h
    return -2.0 / (np.pi ** 2 * (4.0 * lag ** 2 - 1.0))


def filter_multiplier(kind: str, padded: int, pixel_pitch: float = 1.0) -> np.ndarray:
    """Re(rfft(kernel)) / pitch -- fbp.py:105-116."""
    return np.real(np.fft.rfft(filter_kernel(kind, padded))) / pixel_pitch


def gaussian_blur_nearest(s: np.ndarray, sigma: float, truncate: float = 4.0) -> np.ndarray:
    """Restatement of scipy.ndimage.gaussian_filter1d(mode="nearest") along
    the last axis (scipy 1.18.1: radius int(truncate*sigma+0.5), weights
    exp(-x^2/(2 sigma^2)) normalised; symmetric so correlate == convolve).
    Used by the reference at fbp.py:125-126."""
    radius = int(truncate * float(sigma) + 0.5)
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    w = np.exp(-0.5 / (float(sigma) ** 2) * x ** 2)
    w = w / w.sum()
    n = s.shape[-1]
    idx = np.clip(np.arange(n)[:, None] + np.arange(-radius, radius + 1)[None, :], 0, n - 1)
    return np.tensordot(s[..., idx], w, axes=([-1], [0]))


def ramp_filter(sino, kind="ramlak", padding=None, blur_sigma=0.0, pixel_pitch=1.0):
    """Per-line zero-padded FFT ramp filter, float64 -- fbp.py:119-131."""
    s = np.asarray(sino, dtype=np.float64)
    n = s.shape[-1]
    if blur_sigma > 0:
        s = gaussian_blur_nearest(s, blur_sigma)
    p = padded_length(n, padding)
    spec = np.fft.rfft(s, n=p, axis=-1) * filter_multiplier(kind, p, pixel_pitch)
    return np.fft.irfft(spec, n=p, axis=-1)[..., :n]


def ramp_filter_direct(line, kind="ramlak", pixel_pitch=1.0) -> np.ndarray:
    """O(n^2) linear convolution with taps |d| <= n-1 (equal to the circular
    padded convolution because padding >= 2n); the reference tests' own
    oracle shape (pkg/tests/test_fbp.py:66-75)."""
    x = np.asarray(line, dtype=np.float64)
    n = x.shape[-1]
    taps = np.array([kernel_tap(kind, d) for d in range(-(n - 1), n)])
    out = np.empty_like(x)
    for i in range(n):
        out[..., i] = x @ taps[(i - np.arange(n)) + (n - 1)]
    return out / pixel_pitch


# ---------------------------------------------------------------------------
# back-projection (fbp.py:134-252)


def fov_radius(n_chan: int, offset_chan: int, offset_scan: bool) -> float:
    """fbp.py:134-144."""
    half = (n_chan - 1) / 2.0
    return half + abs(offset_chan) if offset_scan else half


def offset_weights(n_chan: int, offset_chan: int, offset_scan: bool, band: int = 32) -> np.ndarray:
    """Feathered conjugate-normalised redundancy weights -- fbp.py:147-183."""
    if not offset_scan:
        return np.ones(n_chan)
    if band < 1:
        raise ValueError("feather band must be >= 1 channel")
    c0 = axis_channel(n_chan, offset_chan)
    c = np.arange(n_chan, dtype=np.float64)
    near = c if offset_chan > 0 else (n_chan - 1) - c
    own = np.clip(near / band, 0.0, 1.0)
    mirror = 2.0 * c0 - c
    ok = (mirror >= 0) & (mirror <= n_chan - 1)
    mnear = mirror if offset_chan > 0 else (n_chan - 1) - mirror
    other = np.where(ok, np.clip(np.where(ok, mnear, 0.0) / band, 0.0, 1.0), 0.0)
    tot = own + other
    return np.where(tot > 0, own / np.where(tot > 0, tot, 1.0), 0.0)


def back_project(sino, geom: dict, rows=None, angle_range=None, tile=None,
                 feather_band=32, dtype=np.float64) -> np.ndarray:
    """Voxel-driven linear-interpolation BP -- fbp.py:186-252.

    `geom` keys: n_proj n_rows n_chan span pixel_pitch offset_scan
    offset_chan nx ny voxel_pitch.  `sino` is (n_proj, n_rows, n_chan).
    Returns (r1-r0, ny, nx) in `dtype`; zero outside the tile and the FoV.
    """
    g = geom
    s = np.asarray(sino)
    if s.shape != (g["n_proj"], g["n_rows"], g["n_chan"]):
        raise ValueError(f"sinogram shape {s.shape} does not match params "
                         f"({g['n_proj']}, {g['n_rows']}, {g['n_chan']})")
    r0, r1 = rows if rows is not None else (0, g["n_rows"])
    a0, a1 = angle_range if angle_range is not None else (0, g["n_proj"])
    x0, x1, y0, y1 = tile if tile is not None else (0, g["nx"], 0, g["ny"])
    nx, ny, n = g["nx"], g["ny"], g["n_chan"]
    out = np.zeros((r1 - r0, ny, nx), dtype=dtype)
    if r1 == r0 or a1 == a0 or x1 == x0 or y1 == y0:
        return out
    w = offset_weights(n, g["offset_chan"], g["offset_scan"], feather_band).astype(dtype)
    th = angles(g["n_proj"], g["span"])
    xs = np.arange(x0, x1)
    ys = np.arange(y0, y1)[:, None]
    acc = np.zeros((r1 - r0, y1 - y0, x1 - x0), dtype=dtype)
    for k in range(a0, a1):
        t = ray_coordinate(xs, ys, th[k], n, g["offset_chan"], nx, ny,
                           g["voxel_pitch"], g["pixel_pitch"])
        lo = np.floor(t).astype(np.int64)
        fr = (t - lo).astype(dtype)
        ok0 = (lo >= 0) & (lo < n)
        ok1 = (lo + 1 >= 0) & (lo + 1 < n)
        line = s[k, r0:r1].astype(dtype, copy=False) * w
        v0 = line[:, np.where(ok0, lo, 0)] * np.where(ok0, 1.0 - fr, 0.0)
        v1 = line[:, np.where(ok1, lo + 1, 0)] * np.where(ok1, fr, 0.0)
        acc += v0 + v1
    cx, cy = (nx - 1) / 2.0, (ny - 1) / 2.0
    sc = g["voxel_pitch"] / g["pixel_pitch"]
    rr = ((xs - cx) ** 2 + (ys - cy) ** 2) * sc ** 2
    acc[:, rr > fov_radius(n, g["offset_chan"], g["offset_scan"]) ** 2] = 0
    out[:, y0:y1, x0:x1] = acc * dtype(g["span"] / g["n_proj"])
    return out


def quantize(volume, lo: float, hi: float) -> np.ndarray:
    """Window to uint16 with round-half-even -- fbp.py:255-259."""
    v = np.asarray(volume, dtype=np.float64)
    return np.round(np.clip((v - lo) / (hi - lo), 0.0, 1.0) * 65535.0).astype(np.uint16)


def make_geom(n_proj, n_rows, n_chan, nx=None, ny=None, span=math.pi, pixel_pitch=1.0,
              voxel_pitch=1.0, offset_chan=0) -> dict:
    return dict(n_proj=n_proj, n_rows=n_rows, n_chan=n_chan, span=span,
                pixel_pitch=pixel_pitch, offset_scan=offset_chan != 0,
                offset_chan=offset_chan, nx=nx or n_chan, ny=ny or n_chan,
                voxel_pitch=voxel_pitch)


def fbp_rows(raw_rows, geom, i0=1e5, kind="ramlak", feather_band=32, dtype=np.float64):
    """The parity oracle call of SURVEY §8c on a row sample: raw counts of
    the sampled rows (n_proj, k, n_chan) -> volume slices (k, ny, nx).
    Rows are independent (pkg/tests/test_fbp.py:180-191) so sampled rows are
    an exact check of those slices."""
    depth = preprocess(raw_rows, i0)
    filt = ramp_filter(depth, kind, None, 0.0, geom["pixel_pitch"])
    if dtype == np.float32:
        filt = filt.astype(np.float32)
    g = dict(geom)
    g["n_rows"] = filt.shape[1]
    return back_project(filt, g, feather_band=feather_band, dtype=dtype)
