"""tomofuse-b200: B200-native FBP reconstruction hot path of ROVAI
(arXiv 2505.13955), a drop-in for the reference `tomofuse.fbp` API.

    from paper_2505_13955_b200 import fbp, geometry
    vol = fbp.reconstruct(depth, dims, params)          # sm_100a kernels

See DESIGN.md (data layout, kernels, rooflines) and INTEGRATION.md (how the
reference binds the C ABI in include/tomofuse_b200.h).
"""

from . import geometry  # noqa: F401
from .geometry import AcquisitionParams, ScanMode, VolumeDims, check_consistent, ray_coordinate  # noqa: F401

__all__ = ["geometry", "fbp", "engine", "AcquisitionParams", "ScanMode", "VolumeDims",
           "check_consistent", "ray_coordinate"]


def __getattr__(name):
    # fbp / engine need torch + the CUDA library; import lazily so the host
    # logic (geometry, build) stays importable on a CPU-only box.
    if name in ("fbp", "engine", "distributed", "shim"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
