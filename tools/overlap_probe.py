"""Probe: does K1 (filter, on a high-priority stream) hide under K2
(back-projection) when they run concurrently on independent row chunks?

    python tools/overlap_probe.py [--rows 256]

Prints K2 alone, K1 alone, and K2 || K1 times (CUDA events, ms)."""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw  # noqa: E402
from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims  # noqa: E402


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--n-proj", type=int, default=1800)
    ap.add_argument("--rows", type=int, default=256)
    ap.add_argument("--k1-per-k2", type=int, default=1, help="K1 chunks launched beside one K2 chunk")
    a = ap.parse_args()
    n, k = a.n, a.rows
    p = AcquisitionParams(n_proj=a.n_proj, n_rows=n, n_chan=n, pixel_pitch=12.0)
    d = VolumeDims(n, n, n, voxel_pitch=12.0)
    A = SlabReconstructor(p, d, i0=1e5, rows=(0, k))
    B = SlabReconstructor(p, d, i0=1e5, rows=(0, k))
    raw = torch.empty((a.n_proj, k, n), dtype=torch.float32, device="cuda")
    phantom_raw(p, d, raw, r0=n // 2 - k // 2, r1=n // 2 + k // 2)
    A.filter_stage(raw)
    lo, hi = torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1)
    cur = torch.cuda.current_stream()

    def k2():
        A.backproject()

    def k1():
        for _ in range(a.k1_per_k2):
            B.filter_stage(raw)

    def both():
        lo.wait_stream(cur)
        hi.wait_stream(cur)
        A.backproject(stream=lo)
        for _ in range(a.k1_per_k2):
            B.filter_stage(raw, stream=hi)
        cur.wait_stream(lo)
        cur.wait_stream(hi)

    k2()
    k1()
    both()
    t2, t1, tb = timed(k2), timed(k1), timed(both)
    vol_ref = A.vol.clone()
    both()
    torch.cuda.synchronize()
    print(json.dumps({"rows": k, "k2_ms": round(t2, 3), "k1_ms": round(t1, 3), "both_ms": round(tb, 3),
                      "hidden_frac": round((t2 + t1 - tb) / t1, 3),
                      "bitwise": bool(torch.equal(vol_ref, A.vol))}), flush=True)


if __name__ == "__main__":
    main()
