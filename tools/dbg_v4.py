import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2505_13955_b200 import _lib
from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw
from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims
p = AcquisitionParams(n_proj=90, n_rows=64, n_chan=128); d = VolumeDims(128, 128, 64)
eng = SlabReconstructor(p, d, i0=1e5)
raw = torch.empty((90, 64, 128), device='cuda'); phantom_raw(p, d, raw)
filt = eng.filter(raw); eng.stage_rows(filt)
v4 = eng.backproject().clone()
v1 = eng.backproject(flags=_lib.TF_BP_FINALIZE | _lib.TF_BP_KERNEL_V1).clone()
diff = (v4 - v1).abs()
nz = diff > 0
print('n differ', int(nz.sum()), 'of', diff.numel(), 'max', float(diff.max()), 'rel', float(diff.max()/v1.abs().max()))
idx = nz.nonzero()[:20].cpu().numpy()
print(idx)
print('z hist', np.bincount(nz.nonzero()[:,0].cpu().numpy() % 32, minlength=32))
print('x mod 16', np.bincount(nz.nonzero()[:,2].cpu().numpy() % 16, minlength=16))
print('y mod 16', np.bincount(nz.nonzero()[:,1].cpu().numpy() % 16, minlength=16))
for a in [(0,1),(0,2),(5,6),(0,90)]:
    v4 = eng.backproject(a[0],a[1]).clone(); v1 = eng.backproject(a[0],a[1],flags=_lib.TF_BP_FINALIZE | _lib.TF_BP_KERNEL_V1).clone()
    print(a, int(((v4-v1).abs()>0).sum()))
