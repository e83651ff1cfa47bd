"""Dev tool: compare a K2 variant against V1 on a small problem (debugging)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_13955_b200 import _lib
from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw
from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims
n, n_proj, rows = (int(x) for x in sys.argv[1:4])
p = AcquisitionParams(n_proj=n_proj, n_rows=rows, n_chan=n, pixel_pitch=12.0)
d = VolumeDims(n, n, rows, voxel_pitch=12.0)
eng = SlabReconstructor(p, d, i0=1e5)
raw = torch.empty((n_proj, rows, n), device="cuda"); phantom_raw(p, d, raw)
eng.filter_stage(raw)
ref = eng.backproject(flags=_lib.TF_BP_FINALIZE | _lib.TF_BP_KERNEL_V1).clone()
out = eng.backproject(flags=_lib.TF_BP_FINALIZE).clone()
diff = (out - ref).abs()
print("rel", float((out - ref).norm() / ref.norm()), "bad voxels", int((diff > 1e-6 * ref.abs().max()).sum()), "of", diff.numel())
bad = (diff > 1e-6 * ref.abs().max()).nonzero()
if len(bad): print("first bad", bad[:10].tolist())
