"""Drop-in installation into the reference package.

    import tomofuse
    from paper_2505_13955_b200 import shim
    shim.install()            # tomofuse.fbp.* and tomofuse.pipeline.* now run on the B200

The reference has no plugin registry; its reconstruction surface is the
module-level functions of `tomofuse.fbp` (fbp.py:75-275).  `pipeline.py:30`
imports them by name at import time, so both modules' bindings are replaced
(SURVEY.md §8b).  The replacements take the reference's own dataclasses
(AcquisitionParams, VolumeDims, FilterSpec, HuWindow) unchanged -- they are
read by attribute -- and keep return shapes, dtypes and ValueError texts.
`uninstall()` restores the originals.
"""

from __future__ import annotations

import importlib
import sys

# name -> replaced in these modules (fbp.py:75-275; pipeline.py:30)
REBIND = {
    "preprocess": ("tomofuse.fbp", "tomofuse.pipeline"),
    "ramp_filter": ("tomofuse.fbp", "tomofuse.pipeline"),
    "back_project": ("tomofuse.fbp", "tomofuse.pipeline"),
    "quantize": ("tomofuse.fbp", "tomofuse.pipeline"),
    "reconstruct": ("tomofuse.fbp",),
    "filter_multiplier": ("tomofuse.fbp",),
    "offset_weights": ("tomofuse.fbp",),
}

_saved: dict[tuple[str, str], object] = {}


def install(modules: dict | None = None) -> list[str]:
    """Rebind the reference's FBP entry points to the GPU implementations.

    `modules` maps module names to module objects (defaults to importing
    them); returns the list of "module.name" bindings replaced.
    """
    from . import fbp as gpu

    done = []
    for name, targets in REBIND.items():
        for modname in targets:
            mod = (modules or {}).get(modname)
            if mod is None:
                mod = sys.modules.get(modname) or importlib.import_module(modname)
            if not hasattr(mod, name):
                continue
            key = (modname, name)
            if key not in _saved:
                _saved[key] = getattr(mod, name)
            setattr(mod, name, getattr(gpu, name))
            done.append(f"{modname}.{name}")
    return done


def uninstall(modules: dict | None = None) -> None:
    for (modname, name), fn in list(_saved.items()):
        mod = (modules or {}).get(modname) or sys.modules.get(modname)
        if mod is not None:
            setattr(mod, name, fn)
        del _saved[(modname, name)]
