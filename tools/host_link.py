"""Host-link probe: concurrent pinned H2D + D2H per rank, with and without
binding the rank (and its first-touch pinned pages) to the GPU's NUMA node.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/host_link.py [--bind]

Prints one JSON line per rank and an aggregate line on rank 0."""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_13955_b200.hostnuma import bind_to_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bind", action="store_true")
    ap.add_argument("--gb", type=float, default=2.0)
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    info = bind_to_device(local) if a.bind else None
    n = int(a.gb * 2 ** 30) // 4
    h_in = torch.empty(n, dtype=torch.float32, pin_memory=True).fill_(1.0)
    h_out = torch.empty(n, dtype=torch.float32, pin_memory=True).fill_(0.0)
    d_in = torch.empty(n, dtype=torch.float32, device="cuda")
    d_out = torch.ones(n, dtype=torch.float32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for mode in ("h2d", "d2h", "both"):
        times = []
        for it in range(a.iters + 1):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            s1.wait_event(e0)
            s2.wait_event(e0)
            if mode in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d_in.copy_(h_in, non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h_out.copy_(d_out, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
            if it:
                times.append(e0.elapsed_time(e1) / 1e3)
        t = torch.tensor([min(times)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        nbytes = n * 4 * (2 if mode == "both" else 1)
        res[mode] = {"rank_gbs": round(nbytes / min(times) / 1e9, 1),
                     "aggregate_gbs": round(world * nbytes / t.item() / 1e9, 1)}
    print(json.dumps({"rank": rank, "world": world, "bind": info, **res}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
