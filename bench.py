#!/usr/bin/env python
"""Benchmark: FBP reconstruction of the 2048^3 / 1800-projection volume (C3).

    python bench.py [--gpus N --steps K --warmup W]            # our sm_100a path
    python bench.py --impl reference ...                        # CPU reference arm
    torchrun --nproc-per-node N bench.py --gpus N ...           # z-slab multi-GPU

A step = one complete reconstruction of the volume: raw counts (resident in
HBM) -> K1 Beer-Lambert + ramp filter -> [N>1: row-slab exchange, by
default K1's own stores into the owner GPU over NVLink] -> z-block staging
-> K2 back-projection -> fp32 volume.  `value` is whole-job
GUPS (voxel x projection updates / s, N_p*N^3 convention of
pipeline.py:225-227) over the max-over-ranks device time; `e2e` is the same
through host pinned buffers (H2D of the raw counts + D2H of the volume inside
every timed step).  Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FDK backprojection GUPS & s/volume at 2048³ (1/2/4/8 B200) vs CPU ref"
CONFIGS = {
    "c1": dict(n=128, n_proj=180),
    "c2": dict(n=512, n_proj=720),
    "c3": dict(n=2048, n_proj=1800),
    "c4": dict(n=4096, n_proj=3600),
    "c5": dict(n=8192, n_proj=7200),  # N_p assumed (~0.88 N)
}
PITCH = 12.0   # um (config.py:40,47)
I0 = 1e5       # config.py:59
SM_COUNT = 148
# per SM per clock, measured: conflict-free LDS.128 over all 148 SMs, each SM timed on its own
# clock64 (tools/micro/smem_rate.cu -> profiles/r01_smem_rate.jsonl; nominal 128)
SMEM_BYTES_PER_CLK = 127.69
TX = TY = 16   # BP tile (csrc/backproject.cu)
ZB = 32


EXCHANGE_STEP = {
    "": "K1 Beer-Lambert+ramp+feather -> z-blocked staging -> K2 back-projection",
    "alltoall": "K1 Beer-Lambert+ramp+feather -> z-blocked staging per owner slab -> NCCL row-slab all-to-all "
                "landing in the owner's staging buffer -> K2 back-projection",
    "p2p": "K1 Beer-Lambert+ramp -> natural rows stored straight into the owner GPU's buffer over NVLink "
           "(symmetric memory; the all-to-all is K1's store stream) -> owner stages (feather) -> K2",
    "p2p-zblocked": "K1 Beer-Lambert+ramp+feather -> z-blocked rows stored straight into the owner's staging "
                    "buffer over NVLink -> K2",
    "allgather": "K1 Beer-Lambert+ramp -> NCCL all-gather of natural rows -> owner stages its rows -> K2",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--exchange", default="p2p",
                    choices=["alltoall", "allgather", "p2p", "p2p-zblocked", "angles-p2p", "angles-nccl"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--slab-rows", type=int, default=256)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--stream", action="store_true",
                    help="z-sub-slab streaming mode (automatic when the per-GPU slab exceeds HBM)")
    ap.add_argument("--rows", type=int, default=None,
                    help="streaming mode: reconstruct only this many rows per GPU (bounded sample)")
    ap.add_argument("--cpu-angles", type=int, default=None,
                    help="angles per CPU-baseline sample (default sized for ~10 s)")
    return ap.parse_args()


def geometry(cfg):
    from paper_2505_13955_b200.geometry import AcquisitionParams, VolumeDims

    n, n_proj = cfg["n"], cfg["n_proj"]
    p = AcquisitionParams(n_proj=n_proj, n_rows=n, n_chan=n, pixel_pitch=PITCH)
    d = VolumeDims(n, n, n, voxel_pitch=PITCH)
    return p, d


def workload_desc(cfg):
    n, n_proj = cfg["n"], cfg["n_proj"]
    return (f"{n}^3 volume from {n_proj} parallel-beam projections of {n}x{n}, span pi, "
            f"Ram-Lak, pitch {PITCH:g} um, i0 {I0:g}")


# ---------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.path = tempfile.mktemp(prefix="clocks_", suffix=".csv")
        self.proc = None

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "200"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power)}


# ---------------------------------------------------------------- CPU reference arm
def _cpu_worker(args):
    """One process: the reference chain (numpy port, fp32 pipeline path of
    pipeline.py:176-222) on one detector row and the first `na` angles."""
    raw_row, n_proj_full, n, na = args
    import numpy as np

    from oracle import fbp_oracle as O

    span = math.pi * na / n_proj_full  # same angular positions as the full scan
    geom = O.make_geom(na, 1, n, pixel_pitch=PITCH, voxel_pitch=PITCH, span=span)
    t0 = time.perf_counter()
    depth = O.preprocess(raw_row, I0)
    filt = O.ramp_filter(depth, pixel_pitch=PITCH).astype(np.float32)
    O.back_project(filt, geom, dtype=np.float32)
    return time.perf_counter() - t0


def cpu_reference(cfg, steps, warmup, na=None, raw_rows=None):
    """Times the reference algorithm (oracle numpy port) on all host cores:
    one process per core, each a full slice x `na` angles.  Returns
    (GUPS per step list, info)."""
    import multiprocessing as mp

    import numpy as np

    from oracle import phantom_cpu

    n, n_proj = cfg["n"], cfg["n_proj"]
    cores = os.cpu_count() or 1
    if na is None:  # ~8-10 s per step at ~0.03 GUPS per core
        na = max(4, min(n_proj, int(2.5e8 / (n * n))))
    rows = np.linspace(0, n - 1, cores).astype(int)
    if raw_rows is None:
        raw = phantom_cpu.raw_counts(n_proj, n, n, n, n, np.arange(na), rows, pixel_pitch=PITCH,
                                     voxel_pitch=PITCH, i0=I0)
    else:
        raw = raw_rows[:na]
    jobs = [(raw[:, i:i + 1, :].copy(), n_proj, n, na) for i in range(len(rows))]
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    ctx = mp.get_context("fork")
    gups = []
    with ctx.Pool(cores) as pool:
        pool.map(_cpu_worker, [(j[0][:1], n_proj, n, 1) for j in jobs])  # fork + import warm-up
        for it in range(warmup + steps):
            t0 = time.perf_counter()
            pool.map(_cpu_worker, jobs, chunksize=1)
            dt = time.perf_counter() - t0
            if it >= warmup:
                gups.append(len(jobs) * na * n * n / dt / 1e9)
    cpu_model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu_model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    info = {"cores": cores, "kind": "port",
            "sample": (f"{len(jobs)} processes x 1 detector row x first {na} of {n_proj} angles x full "
                       f"{n}x{n} slice (preprocess + ramp_filter + back_project float32, numpy port of "
                       f"fbp.py in oracle/fbp_oracle.py); rows {rows.tolist()}; CPU {cpu_model}"),
            "updates_per_step": len(jobs) * na * n * n}
    return gups, info


def run_reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    gups, info = cpu_reference(cfg, args.steps, args.warmup, args.cpu_angles)
    v = statistics.mean(gups)
    n, n_proj = cfg["n"], cfg["n_proj"]
    total = n_proj * n ** 3
    line = {
        "metric": METRIC, "value": round(v, 6), "unit": "GUPS", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(info["updates_per_step"] / (v * 1e9) * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (analytic 3-D Shepp-Logan raw counts)", "impl": "reference",
        "config": {"workload": workload_desc(cfg), "volume": [n, n, n], "n_proj": n_proj},
        "s_per_volume_extrapolated": round(total / (v * 1e9), 1),
        "cpu_baseline": {"value": round(v, 6), "unit": "GUPS", "cores": info["cores"], "kind": info["kind"],
                         "sample": info["sample"]},
        "e2e": {"value": round(v, 6), "unit": "GUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def executed_updates(d, n_proj, k):
    """Updates the BP kernel really executes: tiles wholly outside the FoV
    are skipped (same fp64 test as bp_kernel), rows padded to 32."""
    import numpy as np

    cx, cy = (d.nx - 1) / 2.0, (d.ny - 1) / 2.0
    R2 = ((d.nx - 1) / 2.0) ** 2  # normal scan, n_chan == nx, scale 1
    active = 0
    for ty in range(0, d.ny, TY):
        for tx in range(0, d.nx, TX):
            xs = np.arange(tx, min(tx + TX, d.nx))
            ys = np.arange(ty, min(ty + TY, d.ny))
            rr = ((xs[None, :] - cx) ** 2 + (ys[:, None] - cy) ** 2)
            if (rr <= R2).any():
                active += 1
    return active * TX * TY * n_proj * (-(-k // ZB) * ZB), active


def run_streamed(args, cfg, world, rank, local, dev):
    """Volumes larger than (aggregate) HBM -- configs C4/C5: each GPU walks
    its z-slab in sub-slabs; per sub-slab the raw counts are generated on the
    device (K4; the host cannot hold a 1.9 TB C5 sinogram), filtered straight
    into staging (K1), back-projected (K2), quantized (K3) and the uint16
    slab is copied into a pinned host ring (2 slabs), overlapped on 2 streams."""
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2505_13955_b200 import _lib
    from paper_2505_13955_b200._lib import check, lib
    from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw
    from paper_2505_13955_b200.geometry import split_range

    p, d = geometry(cfg)
    n, n_proj = cfg["n"], cfg["n_proj"]
    r0, r1 = split_range(n, world)[rank]
    if args.rows:
        r1 = min(r1, r0 + args.rows)
    S = min(args.slab_rows, r1 - r0)
    eng = SlabReconstructor(p, d, i0=I0, rows=(0, S), device=dev)
    raw = torch.empty((n_proj, S, n), dtype=torch.float32, device=dev)
    q = [torch.empty((S, n, n), dtype=torch.uint16, device=dev) for _ in range(2)]
    ring = [torch.empty((S, n, n), dtype=torch.uint16, pin_memory=True) for _ in range(2)]
    s_comp = torch.cuda.current_stream(dev)
    s_d2h = torch.cuda.Stream(dev)
    d2h_done = [None, None]
    bp_events = []

    def one_pass(record=False):
        for i, s0 in enumerate(range(r0, r1, S)):
            k = min(S, r1 - s0)
            b = i % 2
            src = raw.view(-1)[: n_proj * k * n].view(n_proj, k, n)
            phantom_raw(p, d, src, r0=s0, r1=s0 + k, i0=I0)
            check(lib().tf_filter_stage(eng.fplan.handle, eng.bplan.handle, ctypes.c_void_p(src.data_ptr()),
                                        ctypes.c_void_p(eng.stage.data_ptr()), n_proj * k, I0, k, 0, None, None,
                                        ctypes.c_void_p(s_comp.cuda_stream)))
            if d2h_done[b] is not None:
                s_comp.wait_event(d2h_done[b])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s_comp)
            check(lib().tf_backproject(eng.bplan.handle, ctypes.c_void_p(eng.stage.data_ptr()), k,
                                       ctypes.c_void_p(eng.vol.data_ptr()), 0, n_proj, 0, n, 0, n,
                                       _lib.TF_BP_FINALIZE, ctypes.c_void_p(s_comp.cuda_stream)))
            e1.record(s_comp)
            if record:
                bp_events.append((e0, e1, k))
            check(lib().tf_quantize(ctypes.c_void_p(eng.vol.data_ptr()), _lib.TF_F32,
                                    ctypes.c_void_p(q[b].data_ptr()), k * n * n, 0.0, 4e-4,
                                    ctypes.c_void_p(s_comp.cuda_stream)))
            ev = torch.cuda.Event()
            ev.record(s_comp)
            s_d2h.wait_event(ev)
            with torch.cuda.stream(s_d2h):
                ring[b][:k].copy_(q[b][:k], non_blocking=True)
            dd = torch.cuda.Event()
            dd.record(s_d2h)
            d2h_done[b] = dd
        s_comp.wait_stream(s_d2h)

    for _ in range(args.warmup):
        one_pass()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record()
    for _ in range(args.steps):
        one_pass(record=True)
    eb.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t = torch.tensor([ea.elapsed_time(eb) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    rows_all = (r1 - r0) * world if args.rows else n
    upd = n_proj * rows_all * n * n
    bp_ms = sum(e0.elapsed_time(e1) for e0, e1, _ in bp_events)
    bp_upd = sum(n_proj * k * n * n for _, _, k in bp_events)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(upd / (ms / 1e3) / 1e9, 3), "unit": "GUPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "strong" if not args.rows else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (analytic 3-D Shepp-Logan raw counts generated on device per sub-slab)",
            "config": {"workload": workload_desc(cfg), "volume": [n, n, n], "n_proj": n_proj,
                       "mode": f"z-sub-slab streaming ({S} rows), uint16 volume D2H into a 2-slab pinned ring",
                       "rows_per_gpu": r1 - r0, "sample": bool(args.rows),
                       "s_per_volume_extrapolated": round(ms / 1e3 * n / rows_all, 2)},
            "roofline": {"bound": "smem", "kernel": "bp_kernel (K2)",
                         "bp_gups_full_count": round(bp_upd / (bp_ms / 1e3) / 1e9, 1)},
            "clocks": clk, "gpu_launches": 5 * len(bp_events) // max(1, args.steps) * args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return
    if args.stream or cfg["n"] >= 4096 and int(os.environ.get("WORLD_SIZE", "1")) * 180e9 < 2.2 * 4 * cfg["n"] ** 3:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "WARN")
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        if world > 1:
            dist.init_process_group("nccl", device_id=dev)
        run_streamed(args, cfg, world, rank, local, dev)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2505_13955_b200.engine import SlabReconstructor, phantom_raw

    os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep stdout to the one JSON line
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        from paper_2505_13955_b200.hostnuma import bind_to_device

        numa = bind_to_device(local)  # pinned e2e buffers on the GPU's node (no-op on 1-node hosts)
    else:
        numa = None
    p, d = geometry(cfg)
    n, n_proj = cfg["n"], cfg["n_proj"]
    total_updates = n_proj * n * n * n

    # ---- setup: engine + synthetic raw counts generated on the device (K4)
    bp_a0, bp_a1 = 0, n_proj  # angles K2 runs on this rank
    angle_split = world > 1 and args.exchange.startswith("angles-")
    if world > 1 and args.exchange.startswith("angles-"):
        # P_proj: angle-split partials reduced onto the z-slab owners
        from paper_2505_13955_b200.distributed import AngleSplitReconstructor

        eng = slab = AngleSplitReconstructor(p, d, i0=I0, reduce=args.exchange[len("angles-"):], device=dev)
        raw = torch.empty(eng.chunk_shape(), dtype=torch.float32, device=dev)
        phantom_raw(p, d, raw, a0=eng.a0, a1=eng.a1)
        k_rows = n
        bp_a0, bp_a1 = eng.a0, eng.a1

        def step_parts():
            bp_ev[0].record()
            eng.run(raw)  # K1, K2 with the reduction in its epilogue (or + NCCL), finalize
            bp_ev[1].record()
    elif world > 1:
        from paper_2505_13955_b200.distributed import ZSlabReconstructor

        try:
            eng = ZSlabReconstructor(p, d, i0=I0, exchange_mode=args.exchange, device=dev)
        except Exception as e:  # symmetric memory unavailable: same z-slab path, NCCL all-to-all
            if not args.exchange.startswith("p2p"):
                raise
            print(f"p2p exchange unavailable ({e}); using alltoall", file=sys.stderr)
            args.exchange = "alltoall"
            eng = ZSlabReconstructor(p, d, i0=I0, exchange_mode=args.exchange, device=dev)
        raw = torch.empty(eng.chunk_shape(), dtype=torch.float32, device=dev)
        phantom_raw(p, d, raw, a0=eng.a0, a1=eng.a1)
        slab = eng.local
        k_rows = eng.r1 - eng.r0

        def step_parts():
            eng.filter(raw)
            eng.exchange()
            eng.stage()  # owner: natural rows -> tap planes (tensor K2) or z-blocked staging
            bp_ev[0].record()
            eng.local.backproject()
            bp_ev[1].record()
    else:
        eng = slab = SlabReconstructor(p, d, i0=I0, device=dev)
        raw = torch.empty((n_proj, n, n), dtype=torch.float32, device=dev)
        phantom_raw(p, d, raw)
        k_rows = n

        def step_parts():
            eng.filter_stage(raw)  # K1 fused: Beer-Lambert + ramp + feather -> tap planes (or staging)
            bp_ev[0].record()
            eng.backproject()
            bp_ev[1].record()

    torch.cuda.synchronize()
    bp_ev = [torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
    for _ in range(args.warmup):
        step_parts()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---- timed region: K device-resident steps
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    tensor = bool(getattr(slab, "tensor", False)) and not angle_split
    for e in evs:
        bp_ev = [e[1], e[2]]
        e[0].record()
        step_parts()
        e[3].record()
    torch.cuda.synchronize()
    if tensor:  # the MMA items K2 issues per launch (same window test as the kernel, tf_bp_tc_work)
        ksteps_per_launch = slab.bp_work(bp_a0, bp_a1)["mma_items"]
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [e[0].elapsed_time(e[3]) for e in evs]
    bp_ms = [e[1].elapsed_time(e[2]) for e in evs]
    t_tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_tot, op=dist.ReduceOp.MAX)
    ms_per_step = t_tot.item() / args.steps
    gups = total_updates / (ms_per_step / 1e3) / 1e9

    # ---- roofline of the dominant kernel (K2 BP) on this rank
    bp_avg_ms = statistics.mean(bp_ms)
    exec_upd, active_tiles = executed_updates(d, n_proj, k_rows)
    sm_mhz = clk.get("sm_mhz") or 1965.0
    smem_peak = SMEM_BYTES_PER_CLK * SM_COUNT * sm_mhz * 1e6 / 1e9  # GB/s
    from paper_2505_13955_b200._lib import TF_BP_FINALIZE, lib as _tf_lib

    bpu, exe = ctypes.c_double(), ctypes.c_int64()
    _tf_lib().tf_bp_kernel_info(slab.bplan.handle, TF_BP_FINALIZE, k_rows, bp_a0, bp_a1, ctypes.byref(bpu),
                                ctypes.byref(exe))
    bytes_per_update = bpu.value
    exec_upd = exe.value  # the library's own count: FoV-active tiles x tile voxels x padded rows x angles
    smem_achieved = exec_upd * bytes_per_update / (bp_avg_ms / 1e3) / 1e9
    fp32_peak_tflops = 128 * 2 * SM_COUNT * sm_mhz * 1e6 / 1e12
    fp32_achieved = exec_upd * 4 / (bp_avg_ms / 1e3) / 1e12
    slab_updates = n_proj * k_rows * n * n
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    stage_bytes = slab.stage.numel()
    vol_elems = slab.vol.numel() if hasattr(slab, "vol") else n * n * n
    hbm_alg = stage_bytes + vol_elems * 4  # one pass over the staged slab + the volume write
    traffic = None  # ncu dram bytes of this kernel/config, captured separately (profiles/)
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", f"bp_traffic_{args.config}.json")))
        if world == 1:
            traffic = {"bytes_per_launch": tr["dram_bytes_per_launch"], "algorithmic_bytes": hbm_alg,
                       "ratio": round(tr["dram_bytes_per_launch"] / hbm_alg, 2), "source": tr["source"]}
    except (OSError, KeyError, ValueError):
        pass

    # ---- e2e through host pinned buffers: StreamedReconstructor (public API)
    e2e = None
    if not args.no_e2e:
        from paper_2505_13955_b200.engine import StreamedReconstructor
        from paper_2505_13955_b200.geometry import split_range

        ke = args.e2e_steps if args.e2e_steps is not None else max(1, min(args.steps, 2))
        er0, er1 = split_range(n, world)[rank]
        ek = er1 - er0
        h_raw = torch.empty((n_proj, ek, n), dtype=torch.float32, pin_memory=True)
        if world == 1:
            h_raw.copy_(raw)
        else:  # this rank's detector rows, all angles (generated once, then kept on the host)
            tmp = torch.empty((n_proj, ek, n), dtype=torch.float32, device=dev)
            phantom_raw(p, d, tmp, r0=er0, r1=er1)
            h_raw.copy_(tmp)
            del tmp
        h_vol = torch.empty((ek, n, n), dtype=torch.float32, pin_memory=True)
        streamed = StreamedReconstructor(p, d, i0=I0, slab_rows=args.slab_rows, device=dev)

        def e2e_step():
            streamed.run(h_raw, h_vol, row_range=(er0, er1), host_row0=er0)

        e2e_step()  # warm the copy path
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record()
        for _ in range(ke):
            e2e_step()
        eb.record()
        torch.cuda.synchronize()
        te = torch.tensor([ea.elapsed_time(eb) / ke], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = te.item()
        if world == 1 and rank == 0:  # the host-fed volume must equal the device-resident one
            a_, b_ = h_vol[n // 2], slab.vol[n // 2].cpu()
            if getattr(slab, "tensor", False):  # sub-slabs pick their own fp16 tap scale: fp32 roundoff
                same = bool(float((a_ - b_).norm() / b_.norm()) < 1e-6)
            else:
                same = bool(torch.equal(a_, b_))
        else:
            same = None
        e2e = {"value": round(total_updates / (e2e_ms / 1e3) / 1e9, 3), "unit": "GUPS",
               "h2d_bytes_per_step": int(h_raw.numel() * 4), "d2h_bytes_per_step": int(h_vol.numel() * 4),
               "s_per_volume": round(e2e_ms / 1e3, 4), "steps": ke,
               "path": f"engine.StreamedReconstructor: pinned host sinogram -> {args.slab_rows}-row z-sub-slabs, "
                       "H2D / kernels / D2H on 3 streams (double-buffered); bytes are per rank",
               "matches_device_resident_volume": same,
               "host_numa": numa}
        del streamed

    # ---- parity spot check on the bench data (rank 0): 2 rows x 256^2 centre tile vs the C oracle
    parity = None
    if rank == 0 and not args.no_parity and world == 1:
        try:
            from oracle import c_oracle as C
            from oracle import fbp_oracle as O

            rows = [n // 2, n // 3]
            t = min(256, n)
            x0 = (n - t) // 2
            raw_rows = raw[:, rows].cpu().numpy()
            filt = O.ramp_filter(O.preprocess(raw_rows, I0), pixel_pitch=PITCH)
            geom = O.make_geom(n_proj, len(rows), n, pixel_pitch=PITCH, voxel_pitch=PITCH)
            tile = (x0, x0 + t, x0, x0 + t)
            ref = C.back_project(filt, geom, tile=tile)[:, x0:x0 + t, x0:x0 + t]
            got = slab.vol[rows][:, x0:x0 + t, x0:x0 + t].cpu().numpy().astype(np.float64)
            parity = {"rel_l2_vs_f64_oracle": float(np.linalg.norm(got - ref) / np.linalg.norm(ref)),
                      "max_abs": float(np.abs(got - ref).max()), "rows": rows, "tile": list(tile)}
        except Exception as ex:  # never let the checker break the bench line
            parity = {"error": repr(ex)}

    # ---- CPU baseline (rank 0, N=1 only): the reference chain on the same raw rows
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        na = args.cpu_angles or max(4, min(n_proj, int(2.5e8 / (n * n))))
        rows_idx = np.linspace(0, n - 1, cores).astype(int)
        raw_rows = raw[:na][:, rows_idx].cpu().numpy()
        g_cpu, info = cpu_reference(cfg, 1, 0, na, raw_rows=raw_rows)
        v = g_cpu[0]
        cpu_baseline = {"value": round(v, 6), "unit": "GUPS", "cores": info["cores"], "kind": info["kind"],
                        "sample": info["sample"] + " (same raw rows the GPU consumed)",
                        "s_per_volume_extrapolated": round(total_updates / (v * 1e9), 1)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    tc_roof = None
    if tensor:
        # tensor-core K2: per angle and CTA (121 voxels padded to M = 128, x 128 rows) 3 fp16 MMAs of 128 x 128 x 16
        # per K-step (T_hi W_hi + T_hi W_lo + T_lo W_hi), 1 or 2 K-steps by the tile's window
        flops = ksteps_per_launch * 3 * 2 * 128 * 128 * 16
        tflops = flops / (bp_avg_ms / 1e3) / 1e12
        pk = peaks.get("bf16_tflops_sustained") or 1420.9
        tc_roof = {
            "bound": "tensor",
            "kernel": "bp_tc_kernel (K2, tcgen05)",
            "achieved": round(tflops, 1),
            "peak": pk,
            "unit": "TFLOP/s",
            "frac": round(tflops / pk, 4),
            "frac_of_burst": round(tflops / (peaks.get("bf16_tflops") or 1684.4), 4),
            "traffic": None,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (dense fp16 MMA runs at the bf16 rate; "
                           "K2 is a 1-2 s kernel inside the step)",
            "flops_per_launch": flops,
            "flops_note": "executed MMA FLOPs of the GEMM formulation D[voxel][row] += W[voxel][chan] T[chan][row]: "
                          "K-steps counted on the device (tf_bp_tc_count) x 3 split products x 2*128*128*16",
            "mma_ksteps_per_launch": ksteps_per_launch,
            "bp_ms_per_launch": round(bp_avg_ms, 3),
            "bp_gups_full_count": round(slab_updates / (bp_avg_ms / 1e3) / 1e9, 1),
            # per angle and CTA (11 x 11 voxels x 128 rows = 15488 updates), one K-step (97% of angles):
            # TMA writes 2 x 128 rows x 16 ch x 2 B = 8 KB and the MMAs read B 3 x 4 KB; weights come
            # from TMEM: 20 KB / 15488 updates
            "smem_bytes_per_update": 1.32,
            "hbm_gbs_algorithmic": round(hbm_alg / (bp_avg_ms / 1e3) / 1e9, 1),
            "hbm_peak_measured": peaks.get("hbm_gbs"),
        }
    line = {
        "metric": METRIC,
        "value": round(gups, 3),
        "unit": "GUPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 3),
        "s_per_volume": round(ms_per_step / 1e3, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (analytic 3-D Shepp-Logan raw counts generated on device, i0=1e5)",
        "config": {"workload": workload_desc(cfg), "volume": [n, n, n], "n_proj": n_proj,
                   "parallelism": (f"angle-split x{world} ({args.exchange}: partials reduced onto z-slab owners)"
                                   if angle_split else
                                   f"z-slab x{world}" + (f" ({args.exchange} exchange)" if world > 1 else "")),
                   "l2": "inputs larger than L2 (raw %.1f GB, volume %.1f GB per step)" % (
                       raw.numel() * 4 / 1e9, vol_elems * 4 / 1e9),
                   "step": ("K1 Beer-Lambert+ramp+feather -> z-blocked staging -> K2 back-projection of this "
                            "rank's angles over the whole volume, epilogue adds into each row's owner "
                            "(NVLink peer memory, or + NCCL reduce-scatter) -> FoV/scale finalize"
                            if angle_split else
                            EXCHANGE_STEP.get(args.exchange if world > 1 else "", EXCHANGE_STEP[""]))},
        "roofline": tc_roof if tensor else {
            "bound": "smem",
            "kernel": "bp_kernel (K2)",
            "achieved": round(smem_achieved, 1),
            "peak": round(smem_peak, 1),
            "unit": "GB/s",
            "frac": round(smem_achieved / smem_peak, 4),
            "traffic": traffic["bytes_per_launch"] if traffic else None,
            "traffic_detail": traffic,
            "peak_source": "measured 127.69 B/clk/SM (conflict-free LDS.128, tools/micro/smem_rate.cu, "
                           "profiles/r01_smem_rate.jsonl) x 148 SMs x measured median SM clock "
                           "(shared-memory data path; no tensor-core or HBM bound applies, SURVEY 8d)",
            "roof_updates_per_s_e9": round(smem_peak / bytes_per_update, 1),
            "algorithmic_bytes_per_update": bytes_per_update,
            "bytes_note": "smem bytes the K2 variant gathers per update: 8 = two fp32 taps; 6 = x-pair "
                          "kernel (3 taps shared by 2 voxels, taps held in registers)",
            "bp_ms_per_launch": round(bp_avg_ms, 3),
            "executed_updates_per_launch": exec_upd,
            "active_tiles": active_tiles,
            "bp_gups_executed": round(exec_upd / (bp_avg_ms / 1e3) / 1e9, 1),
            "bp_gups_full_count": round(slab_updates / (bp_avg_ms / 1e3) / 1e9, 1),
            "fp32_tflops": round(fp32_achieved, 2),
            "fp32_frac": round(fp32_achieved / fp32_peak_tflops, 4),
            "hbm_gbs_algorithmic": round(hbm_alg / (bp_avg_ms / 1e3) / 1e9, 1),
            "hbm_peak_measured": peaks.get("hbm_gbs"),
        },
        "clocks": clk,
        # our kernels per step: K1 + K2, + tf_bp_stage (allgather, p2p) or + tf_bp_finalize (angle split)
        # (+2 with the tensor-core K2: tc_absmax_kernel for the fp16 tap scale, tc_convert_kernel)
        "gpu_launches": ((3 if (world > 1 and (args.exchange in ("allgather", "p2p") or angle_split)) else 2)
                         + (2 if tensor else 0)) * args.steps,
    }
    if e2e is not None:
        line["e2e"] = e2e
    if cpu_baseline is not None:
        line["cpu_baseline"] = cpu_baseline
    if parity is not None:
        line["parity"] = parity
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
