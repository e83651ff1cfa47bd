import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden_fbp.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture(scope="session")
def golden():
    g = np.load(GOLDEN)
    meta = json.loads(bytes(g["meta_json"]).decode())
    return g, meta


def ref_objects(rec):
    """(params, dims) of a golden case, built with this package's geometry."""
    from paper_2505_13955_b200.geometry import AcquisitionParams, ScanMode, VolumeDims

    off = rec["offset_chan"]
    p = AcquisitionParams(n_proj=rec["n_proj"], n_rows=rec["n_rows"], n_chan=rec["n_chan"],
                          angle_span=rec["span"], pixel_pitch=rec["pixel_pitch"],
                          scan_mode=ScanMode.OFFSET if off else ScanMode.NORMAL, offset_chan=off)
    d = VolumeDims(nx=rec["nx"], ny=rec["ny"], nz=rec["nz"], voxel_pitch=rec["voxel_pitch"])
    return p, d


def oracle_geom(rec):
    from oracle import fbp_oracle as O

    return O.make_geom(rec["n_proj"], rec["n_rows"], rec["n_chan"], rec["nx"], rec["ny"],
                       rec["span"], rec["pixel_pitch"], rec["voxel_pitch"], rec["offset_chan"])


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
