"""Reproduce: CUDA-graph capture of a tensor-core engine, then a fresh engine."""
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw  # noqa: E402
from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims  # noqa: E402

n, n_proj = 64, 70
p = AcquisitionParams(n_proj=n_proj, n_rows=40, n_chan=n)
d = VolumeDims(n, n, 40)
eng = SlabReconstructor(p, d, i0=1e5)
raw = torch.empty((n_proj, 40, n), device="cuda")
phantom_raw(p, d, raw)
graph = eng.capture(raw)
raw.mul_(0.97)
graph.replay()
torch.cuda.synchronize()
got = eng.vol.clone()
ref = SlabReconstructor(p, d, i0=1e5).run(raw)
torch.cuda.synchronize()
print("graph==eager", bool(torch.equal(got, ref)), float((got - ref).norm() / ref.norm()), flush=True)
for case in [(90, 64, 128), (90, 64, 128)]:
    pa = AcquisitionParams(n_proj=case[0], n_rows=case[1], n_chan=case[2])
    da = VolumeDims(case[2], case[2], case[1])
    r2 = torch.empty((case[0], case[1], case[2]), device="cuda")
    phantom_raw(pa, da, r2)
    e1 = SlabReconstructor(pa, da, i0=1e5, tensor=True)
    tc = e1.run(r2)
    torch.cuda.synchronize()
    hdr = e1.tc_ws[:8].view(torch.int32).cpu().tolist()
    cc = SlabReconstructor(pa, da, i0=1e5, tensor=False).run(r2)
    print("after graph: tc max", float(tc.abs().max()), "cc max", float(cc.abs().max()), "hdr", hdr,
          "rel", float((tc - cc).norm() / cc.norm()), flush=True)
