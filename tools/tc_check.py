"""Tensor-core back-projection (K2-TC) vs the CUDA-core default kernel:
agreement, parity against the C oracle on sampled rows, and timing.

    python tools/tc_check.py [--n 256 --n-proj 180 --rows 64 --oracle-rows 2]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_13955_b200 import _lib  # noqa: E402
from paper_2505_13955_b200._lib import check, lib  # noqa: E402
from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw  # noqa: E402
from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--n-proj", type=int, default=180)
    ap.add_argument("--rows", type=int, default=64)
    ap.add_argument("--oracle-rows", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dbg", action="store_true", help="print the kernel's per-role wait-cycle counters")
    ap.add_argument("--pitch", type=float, default=12.0)
    a = ap.parse_args()
    n, k = a.n, a.rows
    p = AcquisitionParams(n_proj=a.n_proj, n_rows=n, n_chan=n, pixel_pitch=a.pitch)
    d = VolumeDims(n, n, n, voxel_pitch=a.pitch)
    r0 = n // 2 - k // 2
    eng = SlabReconstructor(p, d, i0=1e5, rows=(0, k))
    raw = torch.empty((a.n_proj, k, n), dtype=torch.float32, device="cuda")
    phantom_raw(p, d, raw, r0=r0, r1=r0 + k)
    eng.filter_stage(raw)
    ref = eng.backproject().clone()
    L = lib()
    h = eng.bplan.handle
    wsb = L.tf_bp_tc_workspace_bytes(h, k, 0, a.n_proj)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    vol = torch.full_like(ref, float("nan"))
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def prep():
        check(L.tf_bp_tc_prepare(h, ctypes.c_void_p(eng.stage.data_ptr()), k, 0, a.n_proj, 0.0,
                                 ctypes.c_void_p(ws.data_ptr()), st))

    def bp():
        check(L.tf_backproject_tc(h, ctypes.c_void_p(ws.data_ptr()), 0, a.n_proj, k, ctypes.c_void_p(vol.data_ptr()),
                                  0, a.n_proj, 0, n, 0, n, _lib.TF_BP_FINALIZE, st))

    dbg = torch.zeros(1024 * 8, dtype=torch.int64, device="cuda")
    if a.dbg:
        check(L.tf_bp_tc_debug(ctypes.c_void_p(dbg.data_ptr())))
    prep()
    bp()
    torch.cuda.synchronize()
    check(L.tf_bp_tc_debug(None))
    if a.dbg:
        d8 = dbg.view(1024, 8).cpu().numpy().astype(np.float64)
        d8 = d8[d8[:, 0] > 0]
        names = ["mma_total", "", "", "w_total", "mma_wait_accfree", "mma_wait_full", "mma_wait_afull",
                 "w_wait_empty"]
        print(json.dumps({"dbg_ctas": len(d8), **{nm: round(float(d8[:, i].mean()) / a.n_proj, 1)
                                                 for i, nm in enumerate(names) if nm}, "unit": "clk per angle"}))
    first = vol.clone()
    bp()
    torch.cuda.synchronize()
    deterministic = bool(torch.equal(first, vol))
    e = int(torch.tensor(ws[4:8].cpu().numpy().view(np.int32))[0])
    diff = (vol - ref).double()
    rel = float(diff.norm() / ref.double().norm())
    out = {"n": n, "n_proj": a.n_proj, "rows": k, "exp": e, "deterministic": deterministic, "nan": int(torch.isnan(vol).sum()),
           "rel_l2_vs_default": rel, "max_abs_vs_default": float(diff.abs().max()),
           "ref_max": float(ref.abs().max())}

    def timed(fn):
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return min(ts)

    out["default_ms"] = round(timed(lambda: eng.backproject()), 3)
    out["tc_prepare_ms"] = round(timed(prep), 3)
    out["tc_bp_ms"] = round(timed(bp), 3)
    upd = a.n_proj * k * n * n
    out["default_gups_full"] = round(upd / out["default_ms"] / 1e6, 1)
    out["tc_gups_full"] = round(upd / out["tc_bp_ms"] / 1e6, 1)
    if a.oracle_rows:
        from oracle import c_oracle as C
        from oracle import fbp_oracle as O

        rows = [k // 2, k - 1][: a.oracle_rows]
        geom = O.make_geom(a.n_proj, len(rows), n, pixel_pitch=a.pitch, voxel_pitch=a.pitch)
        oref = C.fbp_rows(raw[:, rows].cpu().numpy(), geom)
        got = vol[rows].cpu().numpy().astype(np.float64)
        dft = ref[rows].cpu().numpy().astype(np.float64)
        out["rel_l2_tc_vs_oracle"] = float(np.linalg.norm(got - oref) / np.linalg.norm(oref))
        out["max_abs_tc_vs_oracle"] = float(np.abs(got - oref).max())
        out["rel_l2_default_vs_oracle"] = float(np.linalg.norm(dft - oref) / np.linalg.norm(oref))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
