"""Precision of K2-TC variants (probe builds) against the f64 oracle on full
detector-row slices: python tools/precision_probe.py --define X [--config c3] [--rows 2]"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    import numpy as np
    import torch

    import tc_probe
    from bench import CONFIGS, I0, PITCH, geometry
    from paper_2505_13955_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--define", action="append", default=[])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--rows", type=int, default=2)
    a = ap.parse_args()
    so = tc_probe.so_path(a.define + ["TF_TC_NOPROBE"])
    if not os.path.exists(so):
        tc_probe.build(a.define + ["TF_TC_NOPROBE"])
    L = ctypes.CDLL(so)
    for name, (res, args) in _lib.SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    _lib._lib = L
    from oracle import c_oracle as C
    from oracle import fbp_oracle as O
    from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw

    cfg = CONFIGS[a.config]
    p, d = geometry(cfg)
    n, n_proj = cfg["n"], cfg["n_proj"]
    rows = [n // 2, n // 3 + 5, n // 5 + 11][: a.rows]
    got, raws = [], []
    raw = torch.empty((n_proj, 1, n), dtype=torch.float32, device="cuda")
    for r in rows:
        phantom_raw(p, d, raw, r0=r, r1=r + 1, i0=I0)
        raws.append(raw[:, 0].cpu().numpy())
        eng = SlabReconstructor(p, d, i0=I0, rows=(r, r + 1), tensor=True)
        got.append(eng.run(raw)[0].cpu().numpy().astype(np.float64))
    ref = C.fbp_rows(np.stack(raws, axis=1), O.make_geom(n_proj, len(rows), n, pixel_pitch=PITCH, voxel_pitch=PITCH))
    got = np.stack(got)
    print(json.dumps({"variant": ",".join(a.define) or "default", "config": a.config, "rows": rows,
                      "rel_l2": float(np.linalg.norm(got - ref) / np.linalg.norm(ref)),
                      "max_abs_rel": float(np.abs(got - ref).max() / np.abs(ref).max())}), flush=True)


if __name__ == "__main__":
    main()
