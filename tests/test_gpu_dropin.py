"""The drop-in on a B200: the reference's OWN test files (test_fbp.py,
test_pipeline.py, test_acceptance.py, unmodified, installed into
baseline/_ref by tools/install_reference.sh) run with every tomofuse.fbp /
tomofuse.pipeline reconstruction binding replaced by this package
(shim.install(), loaded as a pytest plugin before the test modules import
their names).  So pipeline.run's stage 2/4 (pipeline.py:163-237) and
fbp.back_project / reconstruct (fbp.py:186-275) execute on the GPU through
the C ABI -- the tensor-core K2 where the geometry allows it."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _run(files, extra=()):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.isdir(os.path.join(REF, "tomofuse")):
        pytest.skip("baseline/_ref not installed (tools/install_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(ROOT, "tests"), ROOT, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-p", "dropin_plugin", "-q", "-p", "no:cacheprovider",
           "--rootdir", os.path.join(REF, "tests"), *extra,
           *[os.path.join(REF, "tests", f) for f in files]]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=os.path.join(REF, "tests"), env=env)
    print(r.stdout[-6000:], r.stderr[-3000:])
    return r


def test_reference_fbp_suite_through_shim():
    """tests/test_fbp.py of the reference: preprocess, ramp filter (spatial
    and impulse oracles, DC, linearity, padding), back-projection (zero,
    empty ranges, angle additivity, tile/row restriction, row independence,
    disc fidelity, offset completeness), offset weights, quantize."""
    r = _run(["test_fbp.py"])
    assert r.returncode == 0, r.stdout[-3000:]
    assert "drop-in: tomofuse.fbp.back_project -> paper_2505_13955_b200.fbp" in r.stdout, r.stdout[-2000:]


def test_reference_pipeline_suite_through_shim():
    """tests/test_pipeline.py: pipeline.run on 1x1x1 ... 1x4x4 grids against
    the serial fbp chain at 1e-5 (test_pipeline.py:102-112), bitwise equality
    over group sizes / overlap and block / cyclic mappings (:115-137), the
    offset-scan grid, traces and accounting."""
    r = _run(["test_pipeline.py"])
    assert r.returncode == 0, r.stdout[-3000:]
    assert "tomofuse.pipeline.back_project -> paper_2505_13955_b200.fbp" in r.stdout


def test_reference_acceptance_suite_through_shim():
    """tests/test_acceptance.py: the reference's acceptance criteria with the
    reconstruction on the GPU (distributed == serial, disc fidelity,
    segmentation on the reconstructed volume, adjointness, ...)."""
    r = _run(["test_acceptance.py"])
    assert r.returncode == 0, r.stdout[-3000:]
    assert "tomofuse.pipeline.back_project -> paper_2505_13955_b200.fbp" in r.stdout
