"""One full-volume K1 + K2 step of a config (default C3) and nothing else:
the command the ncu captures of profiles/ run (launch list, --set full of
bp_tc_kernel / ramp_filter_r8).

    python tools/bp_launch.py [--config c3] [--rows R] [--tensor 0|1] [--reps 1]
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import CONFIGS, I0, geometry
    from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--rows", type=int, default=None)
    ap.add_argument("--tensor", type=int, default=1)
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    p, d = geometry(cfg)
    k = a.rows or cfg["n"]
    r0 = (cfg["n"] - k) // 2
    eng = SlabReconstructor(p, d, i0=I0, rows=(r0, r0 + k), tensor=bool(a.tensor))
    raw = torch.empty((cfg["n_proj"], k, cfg["n"]), dtype=torch.float32, device="cuda")
    phantom_raw(p, d, raw, r0=r0, r1=r0 + k)
    for _ in range(a.reps):
        eng.run(raw)
    torch.cuda.synchronize()
    print("ok", float(eng.vol[k // 2].abs().max()))


if __name__ == "__main__":
    main()
