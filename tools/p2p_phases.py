"""Per-phase device times of one N-GPU z-slab step (the `p2p` exchange of
bench.py): K1 storing into the owners over NVLink (with the entry
barrier), the exchange barrier, the owner's tap staging, K2.  Run under
torchrun, one rank per GPU:

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/p2p_phases.py [--config c3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    from bench import CONFIGS, I0, geometry
    from paper_2505_13955_b200.distributed import ZSlabReconstructor
    from paper_2505_13955_b200.engine import phantom_raw

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--exchange", default="p2p")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    rank, local = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    p, d = geometry(CONFIGS[a.config])
    eng = ZSlabReconstructor(p, d, i0=I0, exchange_mode=a.exchange, device=dev)
    raw = torch.empty(eng.chunk_shape(), dtype=torch.float32, device=dev)
    phantom_raw(p, d, raw, a0=eng.a0, a1=eng.a1)
    names = ["filter", "exchange", "stage", "backproject"]
    acc = {k: [] for k in names}
    for rep in range(a.reps + 1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        dist.barrier()
        torch.cuda.synchronize()
        ev[0].record()
        eng.filter(raw)
        ev[1].record()
        eng.exchange()
        ev[2].record()
        eng.stage()
        ev[3].record()
        eng.local.backproject()
        ev[4].record()
        torch.cuda.synchronize()
        if rep:
            for i, k in enumerate(names):
                acc[k].append(ev[i].elapsed_time(ev[i + 1]))
    out = {k: round(sum(v) / len(v), 2) for k, v in acc.items()}
    out["total"] = round(sum(out.values()), 2)
    g = [None] * dist.get_world_size()
    dist.all_gather_object(g, out)
    if rank == 0:
        for r, o in enumerate(g):
            print(json.dumps({"rank": r, "world": len(g), "exchange": a.exchange, "ms": o}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
