"""CPU-only checks: the oracle against the reference's golden vectors, the
C-ABI library (loads, exports every declared symbol, host-side plan math),
and the host logic of the API mirror (validation / error texts)."""

import math
import os
import re

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from conftest import ROOT, oracle_geom, ref_objects, rel_l2


# ---------------------------------------------------------------- oracle pinning
BP_CASES = ["bp_small", "bp_ranges", "bp_rect", "bp_pitch", "bp_offset", "bp_offset_neg",
            "bp_odd_span"]


@pytest.mark.parametrize("name", BP_CASES)
@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_oracle_bp_bit_exact_vs_reference(golden, name, dt):
    from oracle import c_oracle as C
    from oracle import fbp_oracle as O

    g, meta = golden
    rec = meta["cases"][name]
    geom = oracle_geom(rec)
    kw = rec["kw"]
    sino = g[name + "_sino"]
    sino = sino if dt == np.float64 else sino.astype(np.float32)
    ref = g[name + ("_f64" if dt == np.float64 else "_f32")]
    rows, ang, tile = kw.get("rows"), kw.get("angles"), kw.get("tile")
    band = kw.get("feather_band", 32)
    o = O.back_project(sino, geom, rows=rows, angle_range=ang, tile=tile, feather_band=band, dtype=dt)
    assert np.array_equal(o, ref)
    r0, r1 = rows if rows else (0, rec["n_rows"])
    c = C.back_project(sino[:, r0:r1], geom, angle_range=ang, tile=tile, feather_band=band,
                       use_f32=dt == np.float32)
    assert np.array_equal(c.astype(dt), ref)


def test_oracle_filters_vs_reference(golden):
    from oracle import c_oracle as C
    from oracle import fbp_oracle as O

    g, _ = golden
    x = g["rf_in"]
    assert np.array_equal(O.ramp_filter(x), g["rf_ramlak"])
    assert np.array_equal(O.ramp_filter(x, "shepplogan"), g["rf_shepplogan"])
    assert np.array_equal(O.ramp_filter(x, padding=100), g["rf_ramlak_pad100"])
    assert np.abs(O.ramp_filter(x, blur_sigma=1.5) - g["rf_blur1p5"]).max() < 1e-14
    assert np.abs(C.ramp_filter(x) - g["rf_ramlak"]).max() < 1e-13
    assert np.abs(C.ramp_filter(x, "shepplogan", blur_sigma=0.4) - g["rf_blur0p4_sl"]).max() < 1e-13
    assert np.abs(C.ramp_filter(x, pixel_pitch=12.0) - g["rf_ramlak_pitch12"]).max() < 1e-14
    for kind in ("ramlak", "shepplogan"):
        for P in (16, 64, 256, 4096):
            assert np.array_equal(O.filter_multiplier(kind, P), g[f"mult_{kind}_{P}"])


def test_oracle_direct_convolution_matches_fft(golden):
    """The O(n^2) spatial oracle of pkg/tests/test_fbp.py:66-75 agrees."""
    from oracle import fbp_oracle as O

    g, _ = golden
    assert np.abs(O.ramp_filter_direct(g["rf_in"]) - g["rf_ramlak"]).max() < 1e-13


def test_oracle_misc_vs_reference(golden):
    from oracle import c_oracle as C
    from oracle import fbp_oracle as O

    g, meta = golden
    assert np.array_equal(O.preprocess(g["pre_raw"], 1e5), g["pre_out"])
    assert np.abs(C.preprocess(g["pre_raw"], 1e5) - g["pre_out"]).max() < 1e-15
    assert np.array_equal(O.quantize(g["q_in"], 0.0, 4e-4), g["q_out"])
    assert np.array_equal(C.quantize(g["q_in"], 0.0, 4e-4), g["q_out"])
    for k in g.files:
        if k.startswith("ow_"):
            _, off, band, n = k.split("_")
            assert np.array_equal(O.offset_weights(int(n), int(off), True, int(band)), g[k])
            assert np.array_equal(C.offset_weights(int(n), int(off), int(band)), g[k])
    for case in ("e2e", "e2eoff"):
        geom = oracle_geom(meta["cases"][case])
        assert np.array_equal(O.fbp_rows(g[case + "_raw"], geom), g[case + "_f64"])
        assert rel_l2(C.fbp_rows(g[case + "_raw"], geom), g[case + "_f64"]) < 1e-13
    geom = oracle_geom(meta["cases"]["e2e"])
    assert np.array_equal(O.fbp_rows(g["e2e_raw"], geom, dtype=np.float32), g["e2e_f32"])


def test_oracle_ray_coordinate_vs_reference(golden):
    from oracle import fbp_oracle as O

    g, meta = golden
    for name in ("geo_normal", "geo_offset"):
        rec = meta["cases"][name]
        xs = np.arange(rec["nx"])[None, :]
        ys = np.arange(rec["ny"])[:, None]
        th = O.angles(rec["n_proj"], rec["span"])
        assert np.array_equal(th, g[name + "_angles"])
        t = np.stack([O.ray_coordinate(xs, ys, a, rec["n_chan"], rec["offset_chan"], rec["nx"],
                                       rec["ny"], rec["voxel_pitch"], rec["pixel_pitch"]) for a in th])
        assert np.array_equal(t, g[name])


# ---------------------------------------------------------------- the C ABI library
def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "tomofuse_b200.h")).read()
    return sorted(set(re.findall(r"TF_API\s+[\w\s\*]+?\b(tf_\w+)\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2505_13955_b200 import _lib

    names = _declared_symbols()
    assert len(names) >= 15
    L = _lib.lib()
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_lib.SIGNATURES)
    assert L.tf_version() >= 1


def test_library_filter_multiplier_host_math(golden):
    import ctypes

    from paper_2505_13955_b200 import _lib

    g, _ = golden
    L = _lib.lib()
    for kind in ("ramlak", "shepplogan"):
        for P, pitch, key in [(16, 1.0, f"mult_{kind}_16"), (4096, 1.0, f"mult_{kind}_4096"),
                              (256, 12.0, f"mult_{kind}_256_p12")]:
            out = np.empty(P // 2 + 1)
            assert L.tf_filter_multiplier(_lib.KIND[kind], P, pitch,
                                          out.ctypes.data_as(ctypes.c_void_p)) == 0
            assert np.abs(out - g[key]).max() < 1e-14


def test_library_offset_weights_bit_exact(golden):
    from paper_2505_13955_b200 import fbp
    from paper_2505_13955_b200.geometry import AcquisitionParams, ScanMode

    g, _ = golden
    for k in g.files:
        if k.startswith("ow_"):
            _, off, band, n = k.split("_")
            p = AcquisitionParams(n_proj=8, n_rows=1, n_chan=int(n), angle_span=2 * math.pi,
                                  scan_mode=ScanMode.OFFSET, offset_chan=int(off))
            assert np.array_equal(fbp.offset_weights(p, int(band)), g[k])
    assert np.all(fbp.offset_weights(AcquisitionParams(n_proj=8, n_rows=1, n_chan=64)) == 1.0)
    with pytest.raises(ValueError, match="feather band"):
        fbp.offset_weights(AcquisitionParams(n_proj=8, n_rows=1, n_chan=64, angle_span=2 * math.pi,
                                             scan_mode=ScanMode.OFFSET, offset_chan=4), 0)


def test_filter_multiplier_dc_bound():  # pkg/tests/test_fbp.py:78-86 (multiplier half)
    from paper_2505_13955_b200 import fbp

    padded = fbp.FilterSpec().padded_length(16)
    for kind in ("ramlak", "shepplogan"):
        m = fbp.filter_multiplier(kind, padded)
        assert 0 <= m[0] < 2.0 / padded
    with pytest.raises(ValueError):
        fbp.filter_multiplier("hann", 16)


def test_non_pow2_multiplier_matches_numpy():
    from oracle import fbp_oracle as O
    from paper_2505_13955_b200 import fbp

    for P in (100, 90):
        assert np.abs(fbp.filter_multiplier("ramlak", P) - O.filter_multiplier("ramlak", P)).max() < 1e-13


# ---------------------------------------------------------------- host logic of the API mirror
def test_filter_spec_validation():  # test_fbp.py:122-127
    from paper_2505_13955_b200.fbp import FilterSpec, HuWindow

    with pytest.raises(ValueError):
        FilterSpec(padding=16).padded_length(16)
    assert FilterSpec().padded_length(100) == 256
    with pytest.raises(ValueError):
        FilterSpec(kind="hann")
    with pytest.raises(ValueError):
        FilterSpec(blur_sigma=-1)
    with pytest.raises(ValueError):
        HuWindow(lo=1.0, hi=1.0)


def test_back_project_validation_and_empty_ranges():  # test_fbp.py:142-147 + fbp.py:205-223
    from paper_2505_13955_b200 import fbp
    from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims

    p, d = AcquisitionParams(n_proj=8, n_rows=4, n_chan=16), VolumeDims(16, 16, 4)
    s = np.ones((8, 4, 16))
    # empty ranges are answered without touching the device
    assert np.all(fbp.back_project(s, d, p, angles=(3, 3)) == 0)
    assert fbp.back_project(s, d, p, rows=(2, 2)).shape == (0, 16, 16)
    with pytest.raises(ValueError, match="does not match params"):
        fbp.back_project(np.ones((8, 4, 15)), d, p)
    with pytest.raises(ValueError, match="row range"):
        fbp.back_project(s, d, p, rows=(3, 5))
    with pytest.raises(ValueError, match="angle range"):
        fbp.back_project(s, d, p, angles=(-1, 2))
    with pytest.raises(ValueError, match="tile"):
        fbp.back_project(s, d, p, tile=(0, 17, 0, 16))
    with pytest.raises(ValueError, match="i0 must be positive"):
        fbp.preprocess(s, 0.0)


def test_geometry_conventions():  # pkg/tests/test_geometry.py:18-73
    from paper_2505_13955_b200.geometry import (AcquisitionParams, ScanMode, VolumeDims,
                                                check_consistent, ray_coordinate, split_range)

    p, d = AcquisitionParams(n_proj=10, n_rows=4, n_chan=9), VolumeDims(7, 7, 4)
    for th in np.linspace(0, 2 * math.pi, 17):
        assert ray_coordinate(3.0, 3.0, th, p, d) == pytest.approx(4.0, abs=1e-12)
    po = AcquisitionParams(n_proj=10, n_rows=4, n_chan=16, angle_span=2 * math.pi,
                           scan_mode=ScanMode.OFFSET, offset_chan=4)
    assert ray_coordinate(4.0, 4.0, 1.234, po, VolumeDims(9, 9, 4)) == pytest.approx(7.5 - 4, abs=1e-12)
    p4, d4 = AcquisitionParams(n_proj=4, n_rows=4, n_chan=4), VolumeDims(4, 4, 4)
    assert ray_coordinate(0, 0, math.pi / 2, p4, d4) == pytest.approx(0.0, abs=1e-12)
    assert np.allclose(AcquisitionParams(n_proj=6, n_rows=2, n_chan=4).angles(), np.arange(6) * math.pi / 6)
    with pytest.raises(ValueError):
        AcquisitionParams(n_proj=0, n_rows=1, n_chan=4)
    with pytest.raises(ValueError):
        AcquisitionParams(n_proj=1, n_rows=1, n_chan=8, offset_chan=2)
    with pytest.raises(ValueError):
        AcquisitionParams(n_proj=1, n_rows=1, n_chan=8, scan_mode=ScanMode.OFFSET, offset_chan=9)
    with pytest.raises(ValueError):
        VolumeDims(nx=1, ny=4, nz=4)
    with pytest.raises(ValueError):
        check_consistent(AcquisitionParams(n_proj=2, n_rows=5, n_chan=4), VolumeDims(4, 4, 4))
    assert split_range(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert split_range(2048, 8)[-1] == (1792, 2048)


@settings(max_examples=60, deadline=None)
@given(x=st.integers(0, 15), y=st.integers(0, 15), theta=st.floats(0, math.pi, allow_nan=False))
def test_half_turn_mirrors_about_detector_center(x, y, theta):  # test_geometry.py:52-63
    from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims, ray_coordinate

    p, d = AcquisitionParams(n_proj=8, n_rows=2, n_chan=21), VolumeDims(16, 16, 2)
    c = (p.n_chan - 1) / 2
    t0 = ray_coordinate(x, y, theta, p, d)
    t1 = ray_coordinate(x, y, theta + math.pi, p, d)
    assert t1 - c == pytest.approx(-(t0 - c), abs=1e-9)


def test_geometry_matches_oracle(golden):
    from paper_2505_13955_b200.geometry import ray_coordinate

    g, meta = golden
    for name in ("geo_normal", "geo_offset"):
        p, d = ref_objects(meta["cases"][name])
        xs = np.arange(d.nx)[None, :]
        ys = np.arange(d.ny)[:, None]
        t = np.stack([ray_coordinate(xs, ys, a, p, d) for a in p.angles()])
        assert np.array_equal(t, g[name])


def test_product_package_never_imports_oracle():
    """The product path must not route through the checker."""
    pkg = os.path.join(ROOT, "paper_2505_13955_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_shim_rebinds_reference_surface():
    """shim.install() rebinds tomofuse.fbp.* and the names pipeline.py:30
    imported, and uninstall() restores them (fake modules: no reference
    needed at run time)."""
    import types

    from paper_2505_13955_b200 import fbp as gpu
    from paper_2505_13955_b200 import shim

    def orig(*a, **k):
        return "cpu"

    fbp_mod = types.ModuleType("tomofuse.fbp")
    pipe_mod = types.ModuleType("tomofuse.pipeline")
    for name in ("preprocess", "ramp_filter", "back_project", "quantize", "reconstruct",
                 "filter_multiplier", "offset_weights"):
        setattr(fbp_mod, name, orig)
    for name in ("preprocess", "ramp_filter", "back_project", "quantize"):
        setattr(pipe_mod, name, orig)
    mods = {"tomofuse.fbp": fbp_mod, "tomofuse.pipeline": pipe_mod}
    done = shim.install(mods)
    assert "tomofuse.pipeline.back_project" in done and "tomofuse.fbp.reconstruct" in done
    assert pipe_mod.back_project is gpu.back_project and fbp_mod.quantize is gpu.quantize
    shim.uninstall(mods)
    assert pipe_mod.back_project is orig and fbp_mod.reconstruct is orig


def test_shim_binds_the_real_reference_modules():
    """shim.install() on the unmodified reference package (baseline/_ref,
    tools/install_reference.sh): every name pipeline.py:30 and fbp.py:75-275
    expose is rebound, a module importing `from tomofuse.fbp import
    back_project` afterwards (as test_fbp.py does) gets the GPU function,
    and uninstall() restores the reference.  No compute: runs on CPU."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ref = os.path.join(root, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "tomofuse")):
        pytest.skip("baseline/_ref not installed (tools/install_reference.sh)")
    code = """
import tomofuse.fbp as F, tomofuse.pipeline as P
from paper_2505_13955_b200 import shim, fbp as G
orig = {n: getattr(F, n) for n in shim.REBIND}
done = shim.install()
assert len(done) == 11, done
for n, mods in shim.REBIND.items():
    for m in mods:
        assert getattr(__import__(m, fromlist=['x']), n) is getattr(G, n), (m, n)
from tomofuse.fbp import back_project, ramp_filter
assert back_project is G.back_project and ramp_filter is G.ramp_filter
shim.uninstall()
assert all(getattr(F, n) is f for n, f in orig.items())
assert P.back_project.__module__ == 'tomofuse.fbp'
print('SHIM_OK')
"""
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ref, root]))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0 and "SHIM_OK" in r.stdout, r.stderr[-2000:]


def test_oracle_matches_reference_pipeline_run(golden):
    """pipeline.run over a 2x2 simulated grid == the serial float32 chain
    (pkg/tests/test_pipeline.py:102-112 tolerance 1e-5), through the oracle."""
    from oracle import fbp_oracle as O

    g, meta = golden
    geom = oracle_geom(meta["cases"]["pipe"])
    serial = O.fbp_rows(g["pipe_raw"], geom, dtype=np.float32)
    scale = np.abs(serial).max()
    assert np.abs(serial - g["pipe_vol"]).max() <= 1e-5 * scale


def test_formats_bytes_match_reference(golden, tmp_path):
    """SINO/VOL writers produce the reference's exact bytes; readers parse
    the reference's files (formats.py:30-134)."""
    from paper_2505_13955_b200 import formats
    from paper_2505_13955_b200.geometry import AcquisitionParams

    g, _ = golden
    p = AcquisitionParams(n_proj=36, n_rows=40, n_chan=40)
    sp, vp = tmp_path / "x.sino", tmp_path / "x.vol"
    formats.write_sino(sp, g["pipe_raw"], p)
    assert sp.read_bytes() == g["file_sino"].tobytes()
    formats.write_vol(vp, g["pipe_q"], 12.0)
    assert vp.read_bytes() == g["file_vol"].tobytes()
    ref_sino = tmp_path / "ref.sino"
    ref_sino.write_bytes(g["file_sino"].tobytes())
    data, params = formats.read_sino(ref_sino, pixel_pitch=12.0)
    assert data.dtype == np.float64 and np.array_equal(data, g["pipe_raw"].astype(np.float64))
    assert (params.n_proj, params.n_rows, params.n_chan, params.pixel_pitch) == (36, 40, 40, 12.0)
    vol, dims = formats.read_vol(vp)
    assert np.array_equal(vol, g["pipe_q"]) and dims.voxel_pitch == 12.0
    bad = tmp_path / "bad.sino"
    bad.write_bytes(g["file_sino"].tobytes()[:-4])
    with pytest.raises(ValueError, match="malformed payload"):
        formats.read_sino(bad)
    bad.write_bytes(b"XXXX" + g["file_sino"].tobytes()[4:])
    with pytest.raises(ValueError, match="not a SINO"):
        formats.read_sino(bad)
    with pytest.raises(ValueError, match="missing file"):
        formats.read_sino(tmp_path / "none.sino")


def test_cli_error_mapping(tmp_path):
    """Input errors exit 2 with the reference's prefixes (cli.py:264-285),
    before any GPU work."""
    from paper_2505_13955_b200.__main__ import main

    bad = tmp_path / "bad.sino"
    bad.write_bytes(b"nonsense")
    assert main(["reconstruct", str(bad), "--out", str(tmp_path / "o")]) == 2
    assert main(["reconstruct", str(tmp_path / "missing.sino"), "--out", str(tmp_path / "o")]) == 2


@pytest.mark.parametrize("R0,R1,S", [(0, 2048, 256), (0, 1024, 256), (0, 1100, 256), (512, 1024, 256),
                                     (0, 300, 256), (0, 96, 256), (0, 4096, 128), (7, 999, 64),
                                     (0, 512, 256), (0, 256, 256), (1536, 2048, 256), (0, 130, 256)])
def test_streamed_sub_slabs_cover_rows_once(R0, R1, S):
    """engine.StreamedReconstructor.sub_slabs: contiguous, disjoint, in order,
    covering [R0, R1); never longer than slab_rows; with a ramp (any range of
    >= 128 rows: the middle slab size halves until the ramp fits), the first and
    last slabs are 32 rows and each next slab at most doubles (so its H2D
    hides under the current slab's compute)."""
    from paper_2505_13955_b200.engine import StreamedReconstructor

    class Eng:
        tensor = False

    class Cfg:
        slab_rows = S
        eng = Eng()

    cuts = StreamedReconstructor.sub_slabs(Cfg(), R0, R1)
    assert cuts[0][0] == R0 and cuts[-1][1] == R1
    assert all(a < b for a, b in cuts)
    assert all(cuts[i][1] == cuts[i + 1][0] for i in range(len(cuts) - 1))
    sizes = [b - a for a, b in cuts]
    assert max(sizes) <= S
    if R1 - R0 >= 128 and S >= 64:  # the ramp fits once the middle slab may shrink to 64 rows
        assert sizes[0] == 32 and sizes[-1] == 32
        assert all(sizes[i + 1] <= 2 * sizes[i] for i in range(len(sizes) // 2))


@pytest.mark.parametrize("R0,R1,S", [(0, 2048, 256), (0, 1100, 256), (512, 1024, 256), (0, 96, 256)])
def test_streamed_sub_slabs_tensor_core_uniform(R0, R1, S):
    """Tensor-core K2: uniform slab_rows sub-slabs (a short slab costs a
    whole MMA row block), the last one ragged."""
    from paper_2505_13955_b200.engine import StreamedReconstructor

    class Eng:
        tensor = True

    class Cfg:
        slab_rows = S
        eng = Eng()

    cuts = StreamedReconstructor.sub_slabs(Cfg(), R0, R1)
    assert cuts[0][0] == R0 and cuts[-1][1] == R1
    assert all(cuts[i][1] == cuts[i + 1][0] for i in range(len(cuts) - 1))
    assert all(b - a == S for a, b in cuts[:-1]) and 0 < cuts[-1][1] - cuts[-1][0] <= S


@pytest.mark.parametrize("n,n_proj,k,free_gb,expect", [
    (2048, 1800, 256, 178, None),      # C3: a whole-scan 256-row sub-slab fits
    (8192, 7200, 256, 178, "chunk"),   # C5: it does not; chunks sized from the free memory
    (8192, 7200, 256, 130, "chunk"),
    (8192, 7200, 512, 178, "raise"),   # the fp32 + uint16 slabs alone exceed the device
])
def test_streamed_angle_chunk_sizing(monkeypatch, n, n_proj, k, free_gb, expect):
    """StreamedReconstructor._chunk("auto"): no chunking when 2 raw buffers + tap planes of the
    whole scan fit beside the volume slabs; otherwise the largest multiple of 16 angles that
    fits (free memory less 4 GiB); an explicit chunk rounds down to 16 and disables itself when
    it covers the scan."""
    import torch

    from paper_2505_13955_b200 import engine
    from paper_2505_13955_b200.engine import StreamedReconstructor
    from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims

    monkeypatch.setattr(torch.cuda, "mem_get_info", lambda dev=None: (int(free_gb * 1e9), int(180e9)))
    monkeypatch.setattr(torch.cuda, "memory_reserved", lambda dev=None: 0)
    monkeypatch.setattr(torch.cuda, "memory_allocated", lambda dev=None: 0)
    monkeypatch.setattr(engine, "tensor_default", lambda: True)

    class Cfg:
        params = AcquisitionParams(n_proj=n_proj, n_rows=n, n_chan=n, pixel_pitch=12.0)
        dims = VolumeDims(n, n, n, voxel_pitch=12.0)
        slab_rows = k

    cfg = Cfg()
    cfg.torch = torch
    cfg.device = None
    if expect == "raise":
        with pytest.raises(ValueError):
            StreamedReconstructor._chunk(cfg, "auto", None)
        return
    a = StreamedReconstructor._chunk(cfg, "auto", None)
    if expect is None:
        assert a is None
    else:
        line = k * n * 4
        budget = free_gb * 1e9 - (4 << 30) - k * n * n * 6
        assert a % 16 == 0 and 16 <= a < n_proj
        assert 3 * line * a <= budget < 3 * line * (a + 16)
    assert StreamedReconstructor._chunk(cfg, 100, None) == 96
    assert StreamedReconstructor._chunk(cfg, n_proj, None) is None
    assert StreamedReconstructor._chunk(cfg, "auto", False) is None  # CUDA-core K2: never chunked


def test_hostnuma_cpulist_parse():
    """hostnuma._parse_cpulist reads sysfs local_cpulist syntax."""
    from paper_2505_13955_b200.hostnuma import _parse_cpulist

    assert _parse_cpulist("0-3,8,10-11\n") == {0, 1, 2, 3, 8, 10, 11}
    assert _parse_cpulist("5") == {5}
    assert _parse_cpulist("") == set()
