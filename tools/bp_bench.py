"""Micro-benchmark of the back-projection kernel variants (dev tool).

    TF_BP_VARIANT=k python tools/bp_bench.py --n 2048 --proj 1800 --rows 128 [--v1]
"""
import argparse, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_13955_b200 import _lib
from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw
from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--proj", type=int, default=1800)
ap.add_argument("--rows", type=int, default=128)
ap.add_argument("--v1", action="store_true")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
p = AcquisitionParams(n_proj=a.proj, n_rows=a.rows, n_chan=a.n, pixel_pitch=12.0)
d = VolumeDims(a.n, a.n, a.rows, voxel_pitch=12.0)
eng = SlabReconstructor(p, d, i0=1e5)
raw = torch.empty((a.proj, a.rows, a.n), device="cuda")
phantom_raw(p, d, raw)
eng.stage_rows(eng.filter(raw))
flags = _lib.TF_BP_FINALIZE | (_lib.TF_BP_KERNEL_V1 if a.v1 else 0)
for _ in range(2):
    eng.backproject(flags=flags)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    eng.backproject(flags=flags)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
import ctypes
bpu, exe = ctypes.c_double(), ctypes.c_int64()
_lib.lib().tf_bp_kernel_info(eng.bplan.handle, flags, a.rows, 0, a.proj, ctypes.byref(bpu), ctypes.byref(exe))
exec_upd = exe.value
ref = eng.backproject(flags=_lib.TF_BP_FINALIZE | _lib.TF_BP_KERNEL_V1).clone()
out = eng.backproject(flags=flags)
rel = float((out - ref).norm() / ref.norm())
print(json.dumps({"variant": "v1" if a.v1 else os.environ.get("TF_BP_VARIANT", "default"), "n": a.n, "proj": a.proj,
                  "rows": a.rows, "ms": round(ms, 3), "gups_exec": round(exec_upd / ms / 1e6, 1),
                  "upd_per_clk_sm_at1965": round(exec_upd / ms / 1e-3 / 148 / 1.965e9, 2), "rel_vs_v1": rel}))
