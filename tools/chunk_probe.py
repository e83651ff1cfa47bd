"""Does L2 locality limit K2-TC?  Times the C3 back-projection as one launch
and as angle-chunked launches chained with TF_BP_ACCUMULATE (the resident
CTAs' angle phases then spread over one chunk instead of the whole scan),
with the SM clock sampled by nvidia-smi during each variant.

    python tools/chunk_probe.py [rows]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import CONFIGS, I0, Clocks, geometry
    from paper_2505_13955_b200 import _lib
    from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw

    cfg = CONFIGS["c3"]
    p, d = geometry(cfg)
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    eng = SlabReconstructor(p, d, i0=I0, rows=(0, k))
    raw = torch.empty((cfg["n_proj"], k, cfg["n"]), dtype=torch.float32, device="cuda")
    phantom_raw(p, d, raw, r0=0, r1=k)
    eng.filter_stage(raw)
    del raw
    n_proj = cfg["n_proj"]
    for chunk in (n_proj, 448, 224, 112):
        cuts = list(range(0, n_proj, chunk)) + [n_proj]

        def run():
            for i, (a, b) in enumerate(zip(cuts[:-1], cuts[1:])):
                flags = (_lib.TF_BP_ACCUMULATE if i else 0) | (_lib.TF_BP_FINALIZE if b == n_proj else 0)
                eng.backproject(a, b, flags=flags)

        run()
        torch.cuda.synchronize()
        clk = Clocks(0)
        clk.start()
        time.sleep(0.2)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run()
        e1.record()
        torch.cuda.synchronize()
        c = clk.stop()
        ms = e0.elapsed_time(e1) / 3
        print(json.dumps({"rows": k, "chunk": chunk, "launches": len(cuts) - 1, "ms": round(ms, 2),
                          "sm_mhz": c.get("sm_mhz"), "power_w_max": c.get("power_w_max"),
                          "reasons": c.get("reasons")}), flush=True)


if __name__ == "__main__":
    main()
