"""Repeat tensor-core vs CUDA-core K2 on small cases in one process (flakiness hunt)."""
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw  # noqa: E402
from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


for it in range(6):
    for (n_proj, rows, nch, nx, ny) in [(90, 64, 128, 128, 128), (37, 45, 61, 61, 53), (40, 300, 64, 64, 64)]:
        p = AcquisitionParams(n_proj=n_proj, n_rows=rows, n_chan=nch)
        d = VolumeDims(nx, ny, rows)
        raw = torch.empty((n_proj, rows, nch), device="cuda")
        phantom_raw(p, d, raw)
        e1 = SlabReconstructor(p, d, i0=1e5, tensor=True)
        tc = e1.run(raw).cpu().numpy()
        ex = int(e1.tc_ws[4:8].view(torch.int32).item())
        cc = SlabReconstructor(p, d, i0=1e5, tensor=False).run(raw).cpu().numpy()
        bad = np.argwhere(np.abs(tc - cc) > 1e-3 * np.abs(cc).max())
        print(it, (n_proj, rows, nch), "exp", ex, "rel", rel(tc, cc), "nbad", len(bad),
              "first bad", bad[:3].tolist(), flush=True)
