"""pytest plugin for running the UNMODIFIED reference test-suite through the
drop-in: loaded with `-p dropin_plugin` before the reference's test modules
are imported (test_fbp.py binds `from tomofuse.fbp import back_project, ...`
at import, pipeline.py:30 binds the same names), it calls shim.install() so
every binding the tests and the pipeline see is the sm_100a implementation.
Used by tests/test_gpu_dropin.py; test infrastructure only."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    import tomofuse.fbp  # noqa: F401  the reference package (baseline/_ref on PYTHONPATH)
    import tomofuse.pipeline  # noqa: F401

    from paper_2505_13955_b200 import shim

    bound = shim.install()
    config._dropin_bound = bound
    assert "tomofuse.pipeline.back_project" in bound and "tomofuse.fbp.back_project" in bound, bound


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    import tomofuse.fbp
    import tomofuse.pipeline

    terminalreporter.write_line(
        f"drop-in: tomofuse.fbp.back_project -> {tomofuse.fbp.back_project.__module__}, "
        f"tomofuse.pipeline.back_project -> {tomofuse.pipeline.back_project.__module__} "
        f"({len(config._dropin_bound)} bindings replaced)")
