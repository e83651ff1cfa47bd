"""Micro-benchmark of K1 (dev tool): natural vs fused z-blocked output."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw
from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--proj", type=int, default=1800)
ap.add_argument("--rows", type=int, default=256)
a = ap.parse_args()
p = AcquisitionParams(n_proj=a.proj, n_rows=a.rows, n_chan=a.n, pixel_pitch=12.0)
d = VolumeDims(a.n, a.n, a.rows, voxel_pitch=12.0)
eng = SlabReconstructor(p, d, i0=1e5)
raw = torch.empty((a.proj, a.rows, a.n), device="cuda")
phantom_raw(p, d, raw)
out = torch.empty_like(raw)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
nat = t(lambda: eng.filter(raw, out=out))
fused = t(lambda: eng.filter_stage(raw))
stage = t(lambda: eng.stage_rows(out))
gb = raw.numel() * 4 / 1e9
print(json.dumps({"shape": list(raw.shape), "natural_ms": round(nat, 3), "fused_stage_ms": round(fused, 3),
                  "stage_kernel_ms": round(stage, 3), "natural_GBps_rw": round(2 * gb / nat * 1e3, 1),
                  "scaled_to_C3_natural_ms": round(nat * 2048 / a.rows, 1),
                  "scaled_to_C3_fused_ms": round(fused * 2048 / a.rows, 1)}))
