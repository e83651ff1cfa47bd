import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2505_13955_b200 import _lib
from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw
from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims
p = AcquisitionParams(n_proj=90, n_rows=64, n_chan=128); d = VolumeDims(128, 128, 64)
eng = SlabReconstructor(p, d, i0=1e5)
raw = torch.empty((90, 64, 128), device='cuda'); phantom_raw(p, d, raw)
filt = eng.filter(raw); eng.stage_rows(filt)
v4 = eng.backproject(5, 6, flags=0).clone()
v1 = eng.backproject(5, 6, flags=_lib.TF_BP_KERNEL_V1).clone()
np.savez('gpurun_out/dbg_v4b.npz', v4=v4.cpu().numpy(), v1=v1.cpu().numpy(), filt=filt.cpu().numpy())
