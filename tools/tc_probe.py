"""Where K2-TC's cycles go: per-role wait counters of bp_tc_kernel from the
probe build (tools/micro/tc_probe.cu), averaged over the probed CTAs and
expressed per MMA item.

    python tools/tc_probe.py [--n 2048 --n-proj 1800 --rows 256]

Slots: 0 TMA total, 1 TMA wait(empty); 2 MMA total, 3 MMA wait(full),
4 MMA wait(accfree), 5 MMA issue (fence + elect + 3 MMA + commits +
syncwarp), 6 items; 7/10 weight warp (group 0 / group 3) total, 8/11
wait(empty), 9/12 flush; 13 group 0's end-of-round flush + epilogue + grid barrier.
"""

from __future__ import annotations

import argparse
import ctypes
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SO = os.path.join(ROOT, "tools", "micro", "libtomofuse_probe.so")


def build(defines=(), src=None):
    csrc = os.path.join(ROOT, "paper_2505_13955_b200", "csrc")
    srcs = [s for s in sorted(glob.glob(os.path.join(csrc, "*.cu"))) if not s.endswith("bp_tc.cu")]
    srcs.append(os.path.join(ROOT, "tools", "micro", "tc_probe.cu"))
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler",
           "-fPIC", "-shared", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr", "-I",
           os.path.join(ROOT, "include"), "-I", csrc, *[f"-D{d}" for d in defines],
           *([f'-DTF_TC_SRC="{os.path.abspath(src)}"'] if src else []), "-o", so_path(defines, src), *srcs]
    subprocess.run(cmd, check=True)


def so_path(defines=(), src=None):
    tag = "_".join([d.lower() for d in defines] + ([os.path.splitext(os.path.basename(src))[0]] if src else []))
    return SO if not tag else SO.replace(".so", "_" + tag + ".so")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--n-proj", type=int, default=1800)
    ap.add_argument("--rows", type=int, default=256)
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--define", action="append", default=[], help="e.g. TF_TC_PROBE_NO_TMA")
    ap.add_argument("--src", default=None, help="alternative bp_tc.cu (A/B timing)")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    so = so_path(a.define, a.src)
    if a.build or not os.path.exists(so):
        build(a.define, a.src)
    import numpy as np
    import torch

    from paper_2505_13955_b200 import _lib

    L = ctypes.CDLL(so)
    for name, (res, args) in _lib.SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    L.tf_bp_tc_probe.argtypes = [ctypes.c_void_p]
    _lib._lib = L  # the engine now calls the probe build
    from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw
    from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims

    n, k = a.n, a.rows
    p = AcquisitionParams(n_proj=a.n_proj, n_rows=n, n_chan=n, pixel_pitch=12.0)
    d = VolumeDims(n, n, n, voxel_pitch=12.0)
    raw = torch.empty((a.n_proj, k, n), dtype=torch.float32, device="cuda")
    r0 = n // 2 - k // 2
    phantom_raw(p, d, raw, r0=r0, r1=r0 + k)
    eng = SlabReconstructor(p, d, i0=1e5, rows=(0, k), tensor=True)
    eng.filter_stage(raw)
    eng.backproject()
    buf = torch.zeros(1024 * 16, dtype=torch.int64, device="cuda")
    L.tf_bp_tc_probe(ctypes.c_void_p(buf.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.backproject()
    e1.record()
    torch.cuda.synchronize()
    L.tf_bp_tc_probe(None)
    best = e0.elapsed_time(e1)
    for _ in range(a.reps - 1):
        e0.record()
        eng.backproject()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    v = buf.view(1024, 16).cpu().numpy().astype(np.float64)
    v = v[v[:, 2] > 0]
    w = eng.bp_work()
    ms = best
    if len(v) == 0:  # uninstrumented build (-DTF_TC_NOPROBE): timing only
        print(json.dumps({"variant": (",".join(a.define) or "full") + (f" src={os.path.basename(a.src)}" if a.src else ""), "n": n, "n_proj": a.n_proj, "rows": k,
                          "ms": round(ms, 3), "clk_per_item_at_1965": round(ms / 1e3 * 1.965e9 * 148 / w["mma_items"], 1)}))
        return
    items = v[:, 6]
    per = lambda j: float(np.mean(v[:, j] / items))  # noqa: E731
    out = {"variant": ",".join(a.define) or "full", "n": n, "n_proj": a.n_proj, "rows": k, "ctas": int(len(v)), "ms": round(e0.elapsed_time(e1), 3),
           "items_per_cta": float(items.mean()), "unit": "clk per item",
           "tma_total": per(0), "tma_wait_empty": per(1),
           "mma_total": per(2), "mma_wait_full": per(3), "mma_wait_accfree": per(4), "mma_issue": per(5),
           "w0_total": per(7), "w0_wait_empty": per(8), "w0_flush": per(9),
           "w3_total": per(10), "w3_wait_empty": per(11), "w3_flush": per(12),
           "w0_round_tail": per(13)}
    out["ms_best"] = round(best, 3)
    out["variant"] = out["variant"] + (f" src={os.path.basename(a.src)}" if a.src else "")
    print(json.dumps({k2: (round(x, 1) if isinstance(x, float) else x) for k2, x in out.items()}), flush=True)


if __name__ == "__main__":
    main()
