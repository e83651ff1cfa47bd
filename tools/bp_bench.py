"""Micro-benchmark of one back-projection launch (dev tool): the tensor-core
K2 (default), the CUDA-core pair kernel, or its two-tap reference-order V1.

    python tools/bp_bench.py --n 2048 --proj 1800 --rows 256 [--kernel tc|cuda|v1]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2505_13955_b200 import _lib
    from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw
    from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--proj", type=int, default=1800)
    ap.add_argument("--rows", type=int, default=256)
    ap.add_argument("--kernel", choices=("tc", "cuda", "v1"), default="tc")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    p = AcquisitionParams(n_proj=a.proj, n_rows=a.rows, n_chan=a.n, pixel_pitch=12.0)
    d = VolumeDims(a.n, a.n, a.rows, voxel_pitch=12.0)
    eng = SlabReconstructor(p, d, i0=1e5, tensor=a.kernel == "tc")
    raw = torch.empty((a.proj, a.rows, a.n), device="cuda")
    phantom_raw(p, d, raw)
    eng.filter_stage(raw)
    flags = _lib.TF_BP_FINALIZE | (_lib.TF_BP_KERNEL_V1 if a.kernel == "v1" else 0)
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
    print(json.dumps({"kernel": a.kernel, "n": a.n, "proj": a.proj, "rows": a.rows, "ms": round(ms, 3),
                      "gups": round(a.proj * a.rows * a.n * a.n / ms / 1e6, 1)}))


if __name__ == "__main__":
    main()
