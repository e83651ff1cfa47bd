"""numpy restatement of the K4 analytic Shepp-Logan raw counts -- TEST /
BASELINE INFRASTRUCTURE ONLY (inputs for the CPU-baseline timing arm when no
GPU-generated rows are at hand).  Same ellipsoids and conventions as
paper_2505_13955_b200/csrc/misc.cu::phantom_kernel, evaluated in fp64."""

from __future__ import annotations

import numpy as np

# {rho, a, b, c, x0, y0, z0, phi_deg}
ELLIPSOIDS = np.array([
    [1.0, 0.6900, 0.920, 0.810, 0.00, 0.0000, 0.00, 0.0],
    [-0.8, 0.6624, 0.874, 0.780, 0.00, -0.0184, 0.00, 0.0],
    [-0.2, 0.1100, 0.310, 0.220, 0.22, 0.0000, 0.00, -18.0],
    [-0.2, 0.1600, 0.410, 0.280, -0.22, 0.0000, 0.00, 18.0],
    [0.1, 0.2100, 0.250, 0.410, 0.00, 0.3500, -0.15, 0.0],
    [0.1, 0.0460, 0.046, 0.050, 0.00, 0.1000, 0.25, 0.0],
    [0.1, 0.0460, 0.046, 0.050, 0.00, -0.1000, 0.25, 0.0],
    [0.1, 0.0460, 0.023, 0.050, -0.08, -0.6050, 0.00, 0.0],
    [0.1, 0.0230, 0.023, 0.020, 0.00, -0.6060, 0.00, 0.0],
    [0.1, 0.0230, 0.046, 0.020, 0.06, -0.6050, 0.00, 0.0],
])


def raw_counts(n_proj, n_rows, n_chan, nx, ny, angles, rows, span=np.pi, pixel_pitch=12.0,
               voxel_pitch=12.0, offset_chan=0, i0=1e5, mu_max=3.5e-4) -> np.ndarray:
    """(len(angles), len(rows), n_chan) float32 raw counts."""
    step = span / n_proj
    axis = (n_chan - 1) / 2.0 - offset_chan
    scale = voxel_pitch / pixel_pitch
    rph = 0.48 * min(nx, ny)
    rphz = 0.48 * n_rows
    th = np.asarray(angles, dtype=np.float64)[:, None, None] * step
    zn = ((np.asarray(rows, dtype=np.float64) - (n_rows - 1) / 2.0) / rphz)[None, :, None]
    u = ((np.arange(n_chan) - axis) / scale / rph)[None, None, :]
    acc = np.zeros((len(angles), len(rows), n_chan))
    for rho, a, b, c, x0, y0, z0, phi in ELLIPSOIDS:
        kk = 1.0 - ((zn - z0) / c) ** 2
        sk = np.sqrt(np.clip(kk, 0.0, None))
        A, B = a * sk, b * sk
        ph = th - np.deg2rad(phi)
        a2 = A * A * np.cos(ph) ** 2 + B * B * np.sin(ph) ** 2
        up = u - (x0 * np.cos(th) + y0 * np.sin(th))
        d = a2 - up * up
        ok = (kk > 0) & (d > 0)
        acc += np.where(ok, rho * 2 * A * B * np.sqrt(np.where(ok, d, 0.0)) / np.where(ok, a2, 1.0), 0.0)
    return (i0 * np.exp(-acc * rph * voxel_pitch * mu_max)).astype(np.float32)
