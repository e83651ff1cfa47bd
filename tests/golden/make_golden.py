"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden_fbp.npz.  Every array in it is the output of an
unmodified `tomofuse` call (reference `pkg/src/tomofuse/fbp.py`,
`geometry.py`, `phantom.py`, scipy/numpy as pinned below), so the oracle and
the CUDA path are checked against the reference's own numbers, and the GPU
box (where /root/reference is absent) only needs this file.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import scipy  # noqa: E402
from tomofuse import fbp, phantom  # noqa: E402
from tomofuse.fbp import FilterSpec, HuWindow  # noqa: E402
from tomofuse.geometry import AcquisitionParams, ScanMode, VolumeDims, ray_coordinate  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_fbp.npz")


def params(n_proj, n_rows, n_chan, offset=0, span=None, pitch=1.0):
    mode = ScanMode.OFFSET if offset else ScanMode.NORMAL
    span = span if span is not None else (2 * math.pi if offset else math.pi)
    return AcquisitionParams(n_proj=n_proj, n_rows=n_rows, n_chan=n_chan,
                             angle_span=span, pixel_pitch=pitch,
                             scan_mode=mode, offset_chan=offset)


def geom_record(p: AcquisitionParams, d: VolumeDims) -> dict:
    return dict(n_proj=p.n_proj, n_rows=p.n_rows, n_chan=p.n_chan, span=p.angle_span,
                pixel_pitch=p.pixel_pitch, offset_chan=p.offset_chan,
                nx=d.nx, ny=d.ny, nz=d.nz, voxel_pitch=d.voxel_pitch)


def main():
    g = {}
    meta = {"numpy": np.__version__, "scipy": scipy.__version__, "cases": {}}

    # --- geometry: ray_coordinate (geometry.py:142-153)
    for name, p, d in [
        ("geo_normal", params(10, 4, 9), VolumeDims(7, 7, 4)),
        ("geo_offset", params(10, 4, 16, offset=4), VolumeDims(9, 11, 4, voxel_pitch=1.3)),
    ]:
        xs = np.arange(d.nx)[None, :]
        ys = np.arange(d.ny)[:, None]
        th = p.angles()
        g[name] = np.stack([ray_coordinate(xs, ys, t, p, d) for t in th])
        g[name + "_angles"] = th
        meta["cases"][name] = geom_record(p, d)

    # --- preprocess (fbp.py:75-83)
    rng = np.random.default_rng(7)
    raw = rng.uniform(0, 2e5, size=(3, 4, 16)).astype(np.float32)
    raw[0, 0, :4] = [0.0, 0.5, 1.0, 1.5]
    g["pre_raw"] = raw
    g["pre_out"] = fbp.preprocess(raw, 1e5)

    # --- filter multiplier (fbp.py:105-116)
    for kind in ("ramlak", "shepplogan"):
        for P in (16, 64, 256, 4096):
            g[f"mult_{kind}_{P}"] = fbp.filter_multiplier(kind, P, 1.0)
        g[f"mult_{kind}_256_p12"] = fbp.filter_multiplier(kind, 256, 12.0)

    # --- ramp filter (fbp.py:119-131)
    x = rng.normal(size=(3, 4, 24))
    g["rf_in"] = x
    g["rf_ramlak"] = fbp.ramp_filter(x, FilterSpec("ramlak"))
    g["rf_shepplogan"] = fbp.ramp_filter(x, FilterSpec("shepplogan"))
    g["rf_ramlak_pitch12"] = fbp.ramp_filter(x, FilterSpec("ramlak"), 12.0)
    g["rf_ramlak_pad100"] = fbp.ramp_filter(x, FilterSpec("ramlak", padding=100))
    g["rf_blur1p5"] = fbp.ramp_filter(x, FilterSpec("ramlak", blur_sigma=1.5))
    g["rf_blur0p4_sl"] = fbp.ramp_filter(x, FilterSpec("shepplogan", blur_sigma=0.4))
    x2 = rng.normal(size=(2, 3, 300))
    g["rf_in300"] = x2
    g["rf_300"] = fbp.ramp_filter(x2, FilterSpec("ramlak"))

    # --- offset weights (fbp.py:147-183)
    for off, band, n in [(16, 8, 64), (-20, 32, 96), (5, 1, 40), (-3, 8, 24)]:
        g[f"ow_{off}_{band}_{n}"] = fbp.offset_weights(params(8, 1, n, offset=off), band)

    # --- back projection (fbp.py:186-252): assorted geometries and ranges
    bp_cases = [
        ("bp_small", params(12, 5, 24), VolumeDims(24, 24, 5), {}),
        ("bp_ranges", params(21, 6, 24), VolumeDims(24, 24, 6),
         dict(rows=(1, 5), angles=(3, 17), tile=(2, 19, 4, 22))),
        ("bp_rect", params(17, 3, 20), VolumeDims(31, 26, 3), {}),
        ("bp_pitch", params(15, 2, 32, pitch=1.0), VolumeDims(28, 28, 2, voxel_pitch=1.3), {}),
        ("bp_offset", params(40, 2, 64, offset=16), VolumeDims(96, 96, 2), dict(feather_band=8)),
        ("bp_offset_neg", params(36, 3, 48, offset=-11), VolumeDims(64, 60, 3), {}),
        ("bp_odd_span", params(13, 2, 18, span=2.3), VolumeDims(18, 18, 2), {}),
    ]
    for name, p, d, kw in bp_cases:
        s = rng.normal(size=(p.n_proj, p.n_rows, p.n_chan))
        g[name + "_sino"] = s
        g[name + "_f64"] = fbp.back_project(s, d, p, dtype=np.float64, **kw)
        g[name + "_f32"] = fbp.back_project(s.astype(np.float32), d, p, dtype=np.float32, **kw)
        rec = geom_record(p, d)
        rec["kw"] = {k: list(v) if isinstance(v, tuple) else v for k, v in kw.items()}
        meta["cases"][name] = rec

    # --- quantize (fbp.py:255-259)
    v = np.concatenate([np.linspace(-1e-4, 5e-4, 1001),
                        np.array([0.0, 4e-4, 2e-4, 2e-4 * (1 + 1e-12)])])
    g["q_in"] = v.astype(np.float32).astype(np.float64)
    g["q_out"] = fbp.quantize(g["q_in"][None, None, :], HuWindow(0.0, 4e-4))[0, 0]

    # --- end-to-end FBP on the reference's own microstructure phantom
    n, n_proj, nz = 48, 60, 6
    pitch = 12.0
    p = params(n_proj, nz, n, pitch=pitch)
    d = VolumeDims(n, n, nz, voxel_pitch=pitch)
    micro = phantom.generate_microstructure(d, 0.25, 0.04, seed=1)
    counts = phantom.intensity_sinogram(micro, p, phantom.DegradationSpec(seed=1))
    counts = counts.astype(np.float32)
    g["e2e_raw"] = counts
    depth = fbp.preprocess(counts, 1e5)
    filt = fbp.ramp_filter(depth, FilterSpec(), p.pixel_pitch)
    g["e2e_f64"] = fbp.back_project(filt, d, p, dtype=np.float64)
    g["e2e_f32"] = fbp.back_project(filt.astype(np.float32), d, p, dtype=np.float32)
    g["e2e_recon"] = fbp.reconstruct(depth, d, p)
    g["e2e_q"] = fbp.quantize(g["e2e_f32"], HuWindow(0.0, 4e-4))
    meta["cases"]["e2e"] = geom_record(p, d)

    # --- offset-scan end-to-end (SURVEY §8d secondary case)
    n, n_proj, nz, off = 40, 64, 3, 10
    p = params(n_proj, nz, n, offset=off, pitch=pitch)
    d = VolumeDims(n + 2 * off, n + 2 * off, nz, voxel_pitch=pitch)
    micro = phantom.generate_microstructure(d, 0.25, 0.04, seed=2)
    counts = phantom.intensity_sinogram(micro, p, phantom.DegradationSpec(seed=2))
    counts = counts.astype(np.float32)
    g["e2eoff_raw"] = counts
    depth = fbp.preprocess(counts, 1e5)
    filt = fbp.ramp_filter(depth, FilterSpec(), p.pixel_pitch)
    g["e2eoff_f64"] = fbp.back_project(filt, d, p, dtype=np.float64)
    meta["cases"]["e2eoff"] = geom_record(p, d)

    # --- pipeline.run (pipeline.py:119-324), the caller the shim rebinds:
    # 2x2x1 simulated ranks (row slabs x angle chunks), float32 volumes + uint16
    from tomofuse import pipeline
    from tomofuse.fabric import Fabric, StorageModel
    from tomofuse.geometry import Specimen, SpecimenSet
    from tomofuse.partition import RankGrid

    n, n_proj = 40, 36
    p = params(n_proj, n, n)
    d = VolumeDims(n, n, n)
    micro = phantom.generate_microstructure(d, 0.25, 0.03, seed=3)
    counts = phantom.intensity_sinogram(
        micro, p, phantom.DegradationSpec(poisson_flux=1e5, seed=3, poisson_enabled=False))
    counts = counts.astype(np.float32)
    sset = SpecimenSet(specimens=(Specimen(params=p, dims=d, specimen_id="s0"),))
    cfg = pipeline.PipelineConfig(grid=RankGrid(2, 2, 1), i0=1e5, hu_window=HuWindow(0.0, 4e-4))
    res = pipeline.run(sset, {"s0": counts}, cfg, Fabric(n_ranks=cfg.grid.total), StorageModel())
    g["pipe_raw"] = counts
    g["pipe_vol"] = res.volumes["s0"]
    g["pipe_q"] = res.quantized["s0"]
    meta["cases"]["pipe"] = dict(geom_record(p, d), grid=[2, 2, 1])

    # --- forward projector phantom.project_volume (phantom.py:199-255)
    for name, p in [("fp_normal", params(6, 3, 24)), ("fp_offset", params(10, 2, 30, offset=7)),
                     ("fp_pitch", params(9, 2, 20, pitch=2.5))]:
        n = p.n_chan
        vol = rng.random((p.n_rows, n + 4, n + 2))
        g[name + "_vol"] = vol
        g[name + "_sino"] = phantom.project_volume(vol, p)
        meta["cases"][name] = geom_record(p, VolumeDims(n + 2, n + 4, p.n_rows, voxel_pitch=p.pixel_pitch))

    # --- on-disk containers (formats.py): the reference's own bytes
    import tempfile

    from tomofuse import formats

    with tempfile.TemporaryDirectory() as td:
        sp, vp = os.path.join(td, "a.sino"), os.path.join(td, "a.vol")
        formats.write_sino(sp, g["pipe_raw"], params(36, 40, 40))
        formats.write_vol(vp, g["pipe_q"], 12.0)
        g["file_sino"] = np.frombuffer(open(sp, "rb").read(), dtype=np.uint8)
        g["file_vol"] = np.frombuffer(open(vp, "rb").read(), dtype=np.uint8)

    g["meta_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
