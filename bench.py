#!/usr/bin/env python
"""Benchmark: FBP reconstruction of the 2048^3 / 1800-projection volume (C3).

    python bench.py [--gpus N --steps K --warmup W]            # our sm_100a path
    python bench.py --impl reference ...                        # CPU reference arm
    torchrun --nproc-per-node N bench.py --gpus N ...           # z-slab multi-GPU
    python bench.py --config c4|c5 [--rows R]                   # slab-streamed (> HBM) configs

A step = one complete reconstruction of the volume: raw counts (resident in
HBM) -> K1 Beer-Lambert + ramp filter + feather, written straight into K2's
fp16 tap planes -> [N>1: row-slab exchange, K1's own stores into the owner
GPU over NVLink, owner stages its rows] -> K2 back-projection on the tensor
cores -> fp32 volume.  `value` is whole-job GUPS (voxel x projection updates
/ s, the N_p*N^3 convention of pipeline.py:225-227) over the max-over-ranks
device time; `e2e` is the same through the public streaming API with host
pinned buffers (H2D of the raw counts + D2H of the volume inside every timed
step).  Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
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
REF = os.path.join(ROOT, "baseline", "_ref")  # the unmodified reference (tools/install_reference.sh)

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
FP32_FMA_PER_CLK = 128       # per SM
TC_F16_FLOP_PER_CLK = 8192   # dense fp16 MMA per SM per clock (tools/micro/umma_probe.cu: 128x256x16 in 128 clk)

EXCHANGE_STEP = {
    "": "K1 Beer-Lambert+ramp+feather -> fp16 hi/lo tap planes -> K2 tensor-core back-projection",
    "alltoall": "K1 Beer-Lambert+ramp+feather -> z-blocked staging per owner slab -> NCCL row-slab all-to-all "
                "landing in the owner's staging buffer -> K2 (CUDA-core kernel)",
    "p2p": "K1 Beer-Lambert+ramp -> natural rows stored straight into the owner GPU's buffer over NVLink "
           "(symmetric memory; the all-to-all is K1's store stream) -> owner stages its rows into tap planes "
           "(feather, raw-count bound) -> K2 tensor-core back-projection",
    "p2p-zblocked": "K1 Beer-Lambert+ramp+feather -> z-blocked rows stored straight into the owner's staging "
                    "buffer over NVLink -> K2 (CUDA-core kernel)",
    "allgather": "K1 Beer-Lambert+ramp -> NCCL all-gather of natural rows -> owner stages its rows into tap "
                 "planes -> K2 tensor-core back-projection",
    "p2p-chunked": "per ascending angle chunk: K1 Beer-Lambert+ramp of this rank's share -> natural rows stored into "
                   "the owners' receive buffers over NVLink -> owner stages the chunk into tap planes -> K2 "
                   "tensor-core back-projection with TF_BP_ACCUMULATE (bitwise the single pass)",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--exchange", default="p2p",
                    choices=["alltoall", "allgather", "p2p", "p2p-zblocked", "p2p-chunked", "angles-p2p",
                             "angles-nccl"])
    ap.add_argument("--chunk", type=int, default=None, help="p2p-chunked: angles per chunk (multiple of 16)")
    ap.add_argument("--e2e-steps", type=int, default=None, help="default: --steps")
    ap.add_argument("--slab-rows", type=int, default=256)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--parity-rows", type=int, default=8, help="full slices checked against the f64 oracle")
    ap.add_argument("--stream", action="store_true",
                    help="z-sub-slab streaming mode (automatic when the per-GPU slab exceeds HBM)")
    ap.add_argument("--rows", type=int, default=None,
                    help="streaming mode: reconstruct only this many rows per specimen and GPU (bounded sample)")
    ap.add_argument("--specimens", type=int, default=2, help="streaming mode: synthetic specimens per batch")
    ap.add_argument("--angle-chunk", default="auto",
                    help="streaming mode: angles per H2D/K1/K2 chunk of a sub-slab ('auto': only when a whole scan "
                         "does not fit)")
    ap.add_argument("--cpu-seconds", type=float, default=6.0, help="target CPU seconds per reference sample")
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


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


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


# ---------------------------------------------------------------- CPU reference (baseline/_ref)
_SHARED: dict = {}  # set in the parent before the fork: the sample's raw rows and geometry


def _ref_import():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import tomofuse.fbp as RF  # the UNMODIFIED reference package
    import tomofuse.geometry as RG

    return RF, RG


def _ref_worker(job):
    """One process: the reference chain on its contiguous row slab
    [r0, r1) of the sample, through the reference's own `rows=` argument:
    fbp.preprocess -> fbp.ramp_filter (timed) -> fbp.back_project(float32,
    the pipeline.py:106 dtype) and optionally float64 (the oracle), timed."""
    r0, r1, do64 = job
    import numpy as np

    RF, _ = _ref_import()
    raw, params, dims = _SHARED["raw"], _SHARED["params"], _SHARED["dims"]
    t0 = time.perf_counter()
    depth = RF.preprocess(raw[:, r0:r1], I0)
    filt = RF.ramp_filter(depth, RF.FilterSpec(), params.pixel_pitch)
    t1 = time.perf_counter()
    sino = np.zeros((params.n_proj, params.n_rows, params.n_chan), dtype=np.float32)
    sino[:, r0:r1] = filt.astype(np.float32)  # pipeline.py:178 astype(float32)
    t2 = time.perf_counter()
    RF.back_project(sino, dims, params, rows=(r0, r1), dtype=np.float32)
    t3 = time.perf_counter()
    t64 = None
    if do64:
        s64 = np.zeros(sino.shape, dtype=np.float64)
        s64[:, r0:r1] = filt
        t4 = time.perf_counter()
        RF.back_project(s64, dims, params, rows=(r0, r1), dtype=np.float64)
        t64 = time.perf_counter() - t4
    return t1 - t0, t3 - t2, t64


def ref_sample(cfg, seconds, rows_per_proc=8):
    """(cores, angles, rows) of the CPU sample: one contiguous slab of
    `rows_per_proc` rows per core, spread over the volume, and enough of the
    scan's first angles for ~`seconds` of float32 back_project per process
    at ~0.03 GUPS per core."""
    import numpy as np

    n, n_proj = cfg["n"], cfg["n_proj"]
    cores = os.cpu_count() or 1
    na = max(1, min(n_proj, int(round(seconds * 0.03e9 / (rows_per_proc * n * n)))))
    starts = np.linspace(0, n - rows_per_proc, cores).astype(int)
    rows = np.concatenate([np.arange(s, s + rows_per_proc) for s in starts])
    return cores, na, rows


class CpuReference:
    """The reference's own CPU path (baseline/_ref tomofuse.fbp) on all host
    cores: one forked process per core, each a contiguous
    slab of `rows_per_proc` (>= 8) detector rows through back_project's
    `rows=` argument, the first `na` angles of the scan (same angular
    positions), full n x n slices; extrapolated linearly to the volume."""

    def __init__(self, cfg, raw_rows, cores, na, rows_per_proc=8):
        import multiprocessing as mp

        _, RG = _ref_import()
        n, n_proj = cfg["n"], cfg["n_proj"]
        self.cores, self.k, self.na, self.n, self.n_proj = cores, rows_per_proc, na, n, n_proj
        R = cores * rows_per_proc
        span = math.pi * na / n_proj  # k * span / na = k * pi / n_proj: the scan's first na angles
        params = RG.AcquisitionParams(n_proj=na, n_rows=R, n_chan=n, angle_span=span, pixel_pitch=PITCH)
        dims = RG.VolumeDims(nx=n, ny=n, nz=R, voxel_pitch=PITCH)
        _SHARED.update(raw=raw_rows, params=params, dims=dims)
        os.environ.setdefault("OMP_NUM_THREADS", "1")
        self.pool = mp.get_context("fork").Pool(cores)
        self.pool.map(_ref_worker, [(0, 1, False)] * cores)  # fork + import warm-up
        self.cpu_model = ""
        try:
            for line in open("/proc/cpuinfo"):
                if line.startswith("model name"):
                    self.cpu_model = line.split(":", 1)[1].strip()
                    break
        except OSError:
            pass

    def step(self, do64=False):
        """One parallel pass over the sample: rates over the pool's wall time."""
        jobs = [(i * self.k, (i + 1) * self.k, do64) for i in range(self.cores)]
        t0 = time.perf_counter()
        res = self.pool.map(_ref_worker, jobs, chunksize=1)
        wall = time.perf_counter() - t0
        upd = self.cores * self.k * self.na * self.n * self.n
        lines = self.cores * self.k * self.na
        out = {"chain_f32_gups": upd / wall / 1e9, "bp_f32_gups": upd / max(r[1] for r in res) / 1e9,
               "ramp_filter_msamples_per_s": lines * self.n / max(r[0] for r in res) / 1e6, "wall_s": wall}
        if do64:
            out["chain_f32_gups"] = None  # the pass also ran float64
            out["bp_f64_gups"] = upd / max(r[2] for r in res) / 1e9
        return out

    def sample_desc(self):
        return (f"{self.cores} processes x {self.k} contiguous detector rows (rows= of fbp.back_project) x first "
                f"{self.na} of {self.n_proj} angles x full {self.n}x{self.n} slices: unmodified tomofuse.fbp "
                f"(baseline/_ref) preprocess -> ramp_filter -> back_project float32 (the pipeline dtype); "
                f"float64 back_project and ramp_filter timed separately; extrapolated linearly to the volume; "
                f"CPU {self.cpu_model}")

    def close(self):
        self.pool.close()
        self.pool.join()


def run_reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if not os.path.isdir(os.path.join(REF, "tomofuse")):
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref not installed "
                                                              "(tools/install_reference.sh)"}))
        return
    from oracle import phantom_cpu  # synthetic input for the sample (not the thing timed)

    n, n_proj = cfg["n"], cfg["n_proj"]
    cores, na, rows = ref_sample(cfg, args.cpu_seconds)
    raw = phantom_cpu.raw_counts(n_proj, n, n, n, n, range(na), rows, pixel_pitch=PITCH, voxel_pitch=PITCH, i0=I0)
    ref = CpuReference(cfg, raw, cores, na)
    gups = []
    for it in range(args.warmup + args.steps):
        r = ref.step()
        if it >= args.warmup:
            gups.append(r["chain_f32_gups"])
    r64 = ref.step(do64=True)
    ref.close()
    v = statistics.mean(gups)
    total = n_proj * n ** 3
    upd_step = ref.cores * ref.k * ref.na * n * n
    line = {
        "metric": METRIC, "value": round(v, 6), "unit": "GUPS", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(upd_step / (v * 1e9) * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (analytic 3-D Shepp-Logan raw counts)", "impl": "reference",
        "config": {"workload": workload_desc(cfg), "volume": [n, n, n], "n_proj": n_proj},
        "s_per_volume_extrapolated": round(total / (v * 1e9), 1),
        "cpu_baseline": {"value": round(v, 6), "unit": "GUPS", "cores": ref.cores, "kind": "reference",
                         "sample": ref.sample_desc(), "rows_per_process": ref.k,
                         "bp_f32_gups": round(r64["bp_f32_gups"], 6), "bp_f64_gups": round(r64["bp_f64_gups"], 6),
                         "ramp_filter_msamples_per_s": round(r64["ramp_filter_msamples_per_s"], 2)},
        "e2e": {"value": round(v, 6), "unit": "GUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- roofline of K2
def roofline(slab, bp_a0, bp_a1, k_rows, bp_ms, sm_mhz, peaks, tag):
    """executed updates / t over min(R_fp32, R_smem(B)) at the
    measured SM clock, B = algorithmic shared-memory tap bytes per update.
    For the tensor-core K2 the tensor pipe's own busy fraction (MMA clocks of
    the items the kernel issues / SM clocks) is reported beside it."""
    f = (sm_mhz or 1965.0) * 1e6
    w = slab.bp_work(bp_a0, bp_a1, k_rows)
    t = bp_ms / 1e3
    upd_s = w["executed_updates"] / t
    r_fp32 = FP32_FMA_PER_CLK / 2 * SM_COUNT * f  # 2 FMA per update
    tensor = bool(getattr(slab, "tensor", False))
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", f"bp_traffic_{tag}.json")))
        if tr.get("tensor", False) == tensor:
            traffic = tr
    except (OSError, ValueError):
        pass
    out = {"bound": "fp32", "unit": "TFLOP/s"}
    if tensor:
        nr = 256 if k_rows > 128 else 128
        tap_bytes = w["mma_items"] * 2 * nr * 16 * 2  # TMA: T_hi + T_lo boxes per item into shared memory
        B = tap_bytes / w["executed_updates"]
        mma_flops = w["mma_items"] * 3 * 2 * 128 * nr * 16
        out["kernel"] = "bp_tc_kernel (K2, tcgen05)"
        out["tensor_pipe"] = {
            "frac": round(w["mma_clocks"] / SM_COUNT / f / t, 4), "mma_items_per_launch": w["mma_items"],
            "mma_clocks_per_launch": w["mma_clocks"],
            "note": "items x 3 fp16 MMAs of 128 x N x 16 at N/2 clk each (N = rows per CTA), over 148 SMs x the "
                    "measured clock x K2's time: how busy the tensor pipe is",
            "mma_tflops_executed": round(mma_flops / t / 1e12, 1),
            "mma_peak_tflops_at_clock": round(TC_F16_FLOP_PER_CLK * SM_COUNT * f / 1e12, 1),
            "bf16_tflops_sustained_measured": peaks.get("bf16_tflops_sustained"),
            "bf16_measured_at_mhz": (peaks.get("clocks_under_load") or {}).get("sm_mhz_median")}
    else:
        B = w.get("smem_bytes_per_update") or 6.0
        out["kernel"] = "bp_kernel (K2, CUDA cores)"
    r_smem = SMEM_BYTES_PER_CLK * SM_COUNT * f / B
    roof = min(r_fp32, r_smem)
    out.update({
        "achieved": round(upd_s * 4 / 1e12, 3), "peak": round(roof * 4 / 1e12, 3),
        "frac": round(upd_s / roof, 4),
        "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
        "traffic_detail": traffic,
        "peak_source": (f"SURVEY 8(d): min(R_fp32, R_smem(B)) at the measured median SM clock {sm_mhz} MHz; "
                        f"R_fp32 = 64 updates/clk/SM (2 FMA per update, 128 FMA/clk) x 148 SMs; R_smem = "
                        f"127.69 B/clk/SM (measured LDS.128 roof, profiles/r01_smem_rate.jsonl) x 148 / B; "
                        f"TFLOP/s here are 4 x updates/s (fp32-equivalent)"),
        "algorithmic_smem_bytes_per_update": round(B, 4),
        "roof_updates_per_s_e9": round(roof / 1e9, 1), "r_fp32_updates_per_s_e9": round(r_fp32 / 1e9, 1),
        "r_smem_updates_per_s_e9": round(r_smem / 1e9, 1),
        "executed_updates_per_launch": w["executed_updates"],
        "executed_updates_note": "voxel x angle x row updates of the FoV-active tiles (out-of-FoV tiles skip the "
                                 "angle loop), tile voxels clipped to the volume",
        "bp_ms_per_launch": round(bp_ms, 3),
        "bp_gups_executed": round(upd_s / 1e9, 1),
    })
    return out


# ---------------------------------------------------------------- parity
def parity_rows(n, count, seed=0):
    """{0, N/2, N-1} + seeded random rows."""
    import numpy as np

    base = sorted({0, n // 2, n - 1})
    rest = np.setdiff1d(np.arange(n), base)
    extra = np.random.default_rng(seed).choice(rest, size=min(len(rest), max(0, count - len(base))), replace=False)
    return sorted(base + [int(r) for r in extra])


def parity_check(slab, raw, n_proj, n, count):
    """Full n x n slices of rows {0, N/2, N-1} + seeded rows vs the float64
    oracle (the reference chain restated in C, bit-identical to
    tomofuse.fbp -- tests/test_cpu_host.py) on the same raw counts; the
    error is split into K1 (our fp32 filtered rows vs the oracle's f64
    filter) and BP (the f64 oracle back-projection of OUR filtered rows vs
    our volume) on the first three rows."""
    import numpy as np
    import torch

    from oracle import c_oracle as C
    from oracle import fbp_oracle as O

    rows = parity_rows(n, count)
    raw_rows = raw[:, rows].cpu().numpy()
    geom = O.make_geom(n_proj, len(rows), n, pixel_pitch=PITCH, voxel_pitch=PITCH)
    t0 = time.perf_counter()
    ref = C.fbp_rows(raw_rows, geom)
    got = slab.vol[rows].cpu().numpy().astype(np.float64)
    # rows outside the phantom's z extent reconstruct to exactly zero: no relative error there
    per = [float(np.linalg.norm(got[i] - ref[i]) / np.linalg.norm(ref[i])) for i in range(len(rows))
           if np.linalg.norm(ref[i]) > 0]
    out = {"rows": rows, "slices": "full", "tolerance": 1e-5,
           "rel_l2_vs_f64_oracle": float(np.linalg.norm(got - ref) / np.linalg.norm(ref)),
           "rel_l2_per_row_max": max(per) if per else 0.0, "zero_rows": len(rows) - len(per),
           "max_abs": float(np.abs(got - ref).max()),
           "max_abs_over_max_ref": float(np.abs(got - ref).max() / np.abs(ref).max())}
    sub = rows[:3]
    fg = slab.filter(raw[:, sub].contiguous(),
                     out=torch.empty((n_proj, len(sub), n), device=raw.device)).cpu().numpy().astype(np.float64)
    f64 = C.ramp_filter(C.preprocess(raw_rows[:, :3], I0), "ramlak", PITCH)
    out["k1_rel_l2"] = float(np.linalg.norm(fg - f64) / np.linalg.norm(f64))
    g3 = O.make_geom(n_proj, 3, n, pixel_pitch=PITCH, voxel_pitch=PITCH)
    bp_of_ours = C.back_project(fg, g3)
    out["bp_rel_l2"] = float(np.linalg.norm(got[:3] - bp_of_ours) / np.linalg.norm(bp_of_ours))
    out["oracle_s"] = round(time.perf_counter() - t0, 1)
    return out


def parity_check_multi(vol, r0, r1, p, d, n_proj, n, count):
    """N > 1: each rank checks the parity rows its z-slab owns (full slices,
    raw counts of ALL angles regenerated by K4 for just those rows -- the
    phantom is analytic, so they equal the rows every rank filtered) against
    the float64 oracle; rank 0 aggregates.  The K1/BP split is N=1 only."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from oracle import c_oracle as C
    from oracle import fbp_oracle as O
    from paper_2505_13955_b200.engine import phantom_raw

    rows = parity_rows(n, count)
    mine = [r for r in rows if r0 <= r < r1]
    t0 = time.perf_counter()
    stats, err = [], None
    try:  # never skip the collective below: an exception on one rank must not hang the others
        if mine:
            raw = torch.empty((n_proj, 1, n), dtype=torch.float32, device=vol.device)
            raw_rows = np.empty((n_proj, len(mine), n), dtype=np.float32)
            for i, r in enumerate(mine):
                phantom_raw(p, d, raw, r0=r, r1=r + 1, i0=I0)
                raw_rows[:, i] = raw[:, 0].cpu().numpy()
            ref = C.fbp_rows(raw_rows, O.make_geom(n_proj, len(mine), n, pixel_pitch=PITCH, voxel_pitch=PITCH))
            for i, r in enumerate(mine):
                got = vol[r - r0].cpu().numpy().astype(np.float64)
                dif = got - ref[i]
                stats.append((r, float((dif ** 2).sum()), float((ref[i] ** 2).sum()), float(np.abs(dif).max()),
                              float(np.abs(ref[i]).max())))
    except Exception as ex:
        err = repr(ex)
    gathered = [None] * dist.get_world_size()
    dist.all_gather_object(gathered, (stats, err))
    errs = [e for _, e in gathered if e]
    if errs:
        return {"error": errs[0]}
    gathered = [g for g, _ in gathered]
    allst = sorted(x for g in gathered for x in g)
    d2, r2 = sum(x[1] for x in allst), sum(x[2] for x in allst)
    per = [float(np.sqrt(x[1] / x[2])) for x in allst if x[2] > 0]
    return {"rows": [x[0] for x in allst], "slices": "full", "tolerance": 1e-5,
            "rel_l2_vs_f64_oracle": float(np.sqrt(d2 / r2)) if r2 > 0 else 0.0,
            "rel_l2_per_row_max": max(per) if per else 0.0, "zero_rows": len(allst) - len(per),
            "max_abs": max(x[3] for x in allst), "max_abs_over_max_ref": max(x[3] for x in allst) / max(x[4] for x in allst),
            "checked_by": "each rank its own z-slab's rows", "oracle_s": round(time.perf_counter() - t0, 1)}


# ---------------------------------------------------------------- streamed (> HBM) configs
def run_streamed(args, cfg, world, rank, local, dev):
    """Volumes larger than (aggregate) HBM -- configs C4/C5: a batch of
    synthetic specimens, each streamed through engine.StreamedReconstructor
    (the public host-fed API): pinned host raw counts -> H2D per z-sub-slab
    -> K1 into tap planes -> K2 (tensor cores) -> K3 quantize -> uint16 D2H
    into a pinned host volume, three streams overlapped.  The raw counts are
    generated once before timing (K4 on the device, copied to pinned host
    memory); a bounded sample of rows per specimen and GPU."""
    import torch
    import torch.distributed as dist

    from paper_2505_13955_b200.engine import StreamedReconstructor, phantom_raw
    from paper_2505_13955_b200.geometry import split_range

    p, d = geometry(cfg)
    n, n_proj = cfg["n"], cfg["n_proj"]
    r0, r1 = split_range(n, world)[rank]
    rows = min(args.rows or (r1 - r0), r1 - r0)
    S = min(args.slab_rows, rows)
    specimens = []
    tmp = torch.empty((n_proj, S, n), dtype=torch.float32, device=dev)
    for s in range(args.specimens):
        # specimen s: the phantom at its own contrast (mu_max) and row band
        s0 = r0 + (s * 97) % max(1, (r1 - r0) - rows + 1)
        h = torch.empty((n_proj, rows, n), dtype=torch.float32, pin_memory=True)
        for q0 in range(0, rows, S):
            q1 = min(rows, q0 + S)
            v = tmp[:, : q1 - q0]
            phantom_raw(p, d, v, r0=s0 + q0, r1=s0 + q1, i0=I0, mu_max=3.5e-4 * (1.0 - 0.1 * s))
            h[:, q0:q1].copy_(v)
        specimens.append((s0, h, torch.empty((rows, n, n), dtype=torch.uint16, pin_memory=True)))
    del tmp
    torch.cuda.empty_cache()
    free_gb = torch.cuda.mem_get_info(dev)[0] / 1e9
    ac = args.angle_chunk if args.angle_chunk == "auto" else int(args.angle_chunk)
    st = StreamedReconstructor(p, d, i0=I0, slab_rows=S, device=dev, angle_chunk=ac)
    jobs = [(h_raw, h_vol, (s0, s0 + rows), s0) for s0, h_raw, h_vol in specimens]

    def one_pass():  # the batch as one sub-slab stream (StreamedReconstructor.run_batch)
        st.run_batch(jobs, quantize=(0.0, 4e-4))

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
        one_pass()
    eb.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t = torch.tensor([ea.elapsed_time(eb) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    upd = n_proj * rows * n * n * world * args.specimens
    s_per_spec = ms / 1e3 / args.specimens * (r1 - r0) / rows  # one specimen's full volume on these GPUs
    if rank == 0:
        sub = st.sub_slabs(specimens[0][0], specimens[0][0] + rows)
        line = {
            "metric": METRIC, "value": round(upd / (ms / 1e3) / 1e9, 3), "unit": "GUPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (analytic 3-D Shepp-Logan raw counts, one contrast per specimen, in pinned host "
                    "memory before timing)",
            "config": {"workload": workload_desc(cfg), "volume": [n, n, n], "n_proj": n_proj,
                       "mode": (f"batch of {args.specimens} specimens, each {rows} rows per GPU host-streamed in "
                                f"{S}-row z-sub-slabs as one stream (StreamedReconstructor.run_batch: H2D / K1 "
                                f"taps + K2 tensor cores + K3 quantize / uint16 D2H on 3 streams"
                                + (f"; each sub-slab's angles in chunks of {st.angle_chunk} chained with "
                                   f"TF_BP_ACCUMULATE" if st.angle_chunk else "") + ")"),
                       "angle_chunk": st.angle_chunk, "device_free_gb_at_setup": round(free_gb, 1),
                       "rows_per_gpu_per_specimen": rows, "sample": rows < (r1 - r0),
                       "s_per_specimen_volume_extrapolated": round(s_per_spec, 2)},
            "e2e": {"value": round(upd / (ms / 1e3) / 1e9, 3), "unit": "GUPS",
                    "h2d_bytes_per_step": sum(h.numel() * 4 for _, h, _ in specimens),
                    "d2h_bytes_per_step": sum(v.numel() * 2 for _, _, v in specimens),
                    "path": "host pinned raw counts -> GPU -> host pinned uint16 volume, every step"},
            # per angle chunk: K1's exponent fill, K1, K2; per sub-slab: the FoV-zero pass and K3
            "clocks": clk, "gpu_launches": (3 * -(-n_proj // (st.angle_chunk or n_proj)) + 2) * len(sub)
                                           * args.specimens * args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------- our arm
def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return
    import torch
    import torch.distributed as dist

    os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep stdout to the one JSON line
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.stream or cfg["n"] >= 4096 and world * 180e9 < 2.2 * 4 * cfg["n"] ** 3:
        run_streamed(args, cfg, world, rank, local, dev)
        return

    from paper_2505_13955_b200.engine import SlabReconstructor, StreamedReconstructor, phantom_raw
    from paper_2505_13955_b200.geometry import split_range

    numa = None
    if world > 1:
        from paper_2505_13955_b200.hostnuma import bind_to_device

        numa = bind_to_device(local)  # pinned e2e buffers on the GPU's node (no-op on 1-node hosts)
    p, d = geometry(cfg)
    n, n_proj = cfg["n"], cfg["n_proj"]
    total_updates = n_proj * n * n * n

    # ---- setup: engine + synthetic raw counts generated on the device (K4)
    bp_a0, bp_a1 = 0, n_proj  # angles K2 runs on this rank
    angle_split = world > 1 and args.exchange.startswith("angles-")
    if angle_split:
        # P_proj: angle-split partials reduced onto the z-slab owners (CUDA-core K2 reduce epilogue)
        from paper_2505_13955_b200.distributed import AngleSplitReconstructor

        eng = slab = AngleSplitReconstructor(p, d, i0=I0, reduce=args.exchange[len("angles-"):], device=dev)
        raw = torch.empty(eng.chunk_shape(), dtype=torch.float32, device=dev)
        phantom_raw(p, d, raw, a0=eng.a0, a1=eng.a1)
        k_rows = n
        bp_a0, bp_a1 = eng.a0, eng.a1
        launches = 3  # K1 -> staging, K2 + reduce epilogue, finalize

        def step_parts():
            bp_ev[0].record()
            eng.run(raw)
            bp_ev[1].record()
    elif world > 1 and (args.exchange == "p2p-chunked" or (
            args.exchange == "p2p" and 4.0 * (2 * n_proj * (n / world) * n + (n / world) * n * n + n_proj / world * n * n)
            > 0.8 * torch.cuda.get_device_properties(dev).total_memory)):
        # the whole scan's receive + tap buffers do not fit next to the slab (C4): angle-chunked exchange
        from paper_2505_13955_b200.distributed import ChunkedZSlabReconstructor

        args.exchange = "p2p-chunked"
        raw_bytes = 4.0 * (n_proj / world) * n * n
        eng = ChunkedZSlabReconstructor(p, d, i0=I0, chunk=args.chunk, device=dev,
                                        budget_bytes=torch.cuda.mem_get_info(dev)[0] - raw_bytes - 4e9)
        raw = torch.empty(eng.chunk_shape(), dtype=torch.float32, device=dev)
        for (pa, pb), o in zip(eng.rank_angles(), eng.offsets):
            if pb > pa:
                phantom_raw(p, d, raw[o: o + pb - pa], a0=pa, a1=pb)
        slab = eng.local
        k_rows = eng.r1 - eng.r0
        launches = 4 * len(eng.chunks)  # per chunk: K1, exponent fill + tap staging, K2

        def step_parts():
            bp_ev[0].record()
            eng.run(raw)
            bp_ev[1].record()
    elif world > 1:
        from paper_2505_13955_b200.distributed import ZSlabReconstructor

        try:
            eng = ZSlabReconstructor(p, d, i0=I0, exchange_mode=args.exchange, device=dev)
        except Exception as e:  # symmetric memory unavailable: same z-slab path over NCCL all-gather
            if not args.exchange.startswith("p2p"):
                raise
            print(f"p2p exchange unavailable ({e}); using allgather", file=sys.stderr)
            args.exchange = "allgather"
            eng = ZSlabReconstructor(p, d, i0=I0, exchange_mode=args.exchange, device=dev)
        raw = torch.empty(eng.chunk_shape(), dtype=torch.float32, device=dev)
        phantom_raw(p, d, raw, a0=eng.a0, a1=eng.a1)
        slab = eng.local
        k_rows = eng.r1 - eng.r0
        # K1, [owner staging: exponent fill + tap staging | nothing], K2
        launches = {"p2p": 4, "allgather": 4, "alltoall": 2, "p2p-zblocked": 2}[args.exchange]

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
        launches = 3 if slab.tensor else 2  # K1 (+ the exponent fill of the tap planes), K2

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

    # ---- timed region: K device-resident steps (inputs >> L2)
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for e in evs:
        bp_ev = [e[1], e[2]]
        e[0].record()
        step_parts()
        e[3].record()
    torch.cuda.synchronize()
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
    bp_avg_ms = statistics.mean(bp_ms)
    roof = None
    chunked = args.exchange == "p2p-chunked" and world > 1
    if not angle_split and not chunked:
        roof = roofline(slab, bp_a0, bp_a1, k_rows, bp_avg_ms, clk.get("sm_mhz"), load_peaks(),
                        args.config if world == 1 else f"{args.config}_n{world}")

    # ---- e2e through host pinned buffers: StreamedReconstructor (public API), --e2e-steps steps
    e2e = None
    if not args.no_e2e and not angle_split and not chunked:
        ke = args.e2e_steps if args.e2e_steps is not None else args.steps
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

        def e2e_step(join):
            # back-to-back steps stream like a serving pipeline: step i's last D2H overlaps step
            # i + 1's first H2D (every step still moves its own raw counts in and volume out)
            streamed.run(h_raw, h_vol, row_range=(er0, er1), host_row0=er0, join=join)

        e2e_step(True)  # warm the copy path
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record()
        for _ in range(ke):
            e2e_step(False)
        streamed.join()  # the timed region ends after the last step's D2H
        eb.record()
        torch.cuda.synchronize()
        te = torch.tensor([ea.elapsed_time(eb) / ke], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = te.item()
        same = None
        if world == 1:  # the host-fed volume equals the device-resident one, bit for bit (sampled slices)
            same = bool(all(torch.equal(h_vol[r], slab.vol[r].cpu()) for r in parity_rows(n, 8)))
        e2e = {"value": round(total_updates / (e2e_ms / 1e3) / 1e9, 3), "unit": "GUPS",
               "h2d_bytes_per_step": int(h_raw.numel() * 4), "d2h_bytes_per_step": int(h_vol.numel() * 4),
               "s_per_volume": round(e2e_ms / 1e3, 4), "steps": ke,
               "vs_device_resident": round(e2e_ms / ms_per_step, 4),
               "path": f"engine.StreamedReconstructor: pinned host sinogram -> {args.slab_rows}-row z-sub-slabs, "
                       "H2D / kernels / D2H on 3 streams (double-buffered), consecutive steps pipelined "
                       "(a step's last D2H overlaps the next step's first H2D); bytes are per rank",
               "matches_device_resident_volume_bitwise": same,
               "host_numa": numa}
        del streamed

    # ---- parity on the bench data (rank 0, N=1): full slices vs the f64 oracle
    parity = None
    if rank == 0 and not args.no_parity and world == 1:
        try:
            parity = parity_check(slab, raw, n_proj, n, args.parity_rows)
        except Exception as ex:  # never let the checker break the bench line
            parity = {"error": repr(ex)}
    elif world > 1 and not args.no_parity and not angle_split:
        try:  # z-slabs: every rank checks the rows it owns
            parity = parity_check_multi(slab.vol, eng.r0, eng.r1, p, d, n_proj, n, args.parity_rows)
        except Exception as ex:
            parity = {"error": repr(ex)}

    # ---- CPU baseline (rank 0, N=1 only): the unmodified reference on the same raw rows
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if not os.path.isdir(os.path.join(REF, "tomofuse")):
            cpu_baseline = {"error": "baseline/_ref not installed (tools/install_reference.sh)"}
        else:
            try:
                cores, na, rows = ref_sample(cfg, args.cpu_seconds)
                raw_rows = raw[:na][:, torch.from_numpy(rows).to(raw.device)].cpu().numpy()
                ref = CpuReference(cfg, raw_rows, cores, na)
                r32 = ref.step()
                r64 = ref.step(do64=True)
                ref.close()
                v = r32["chain_f32_gups"]
                cpu_baseline = {"value": round(v, 6), "unit": "GUPS", "cores": ref.cores, "kind": "reference",
                                "sample": ref.sample_desc() + " (the raw rows the GPU consumed)",
                                "rows_per_process": ref.k,
                                "bp_f32_gups": round(r32["bp_f32_gups"], 6),
                                "bp_f64_gups": round(r64["bp_f64_gups"], 6),
                                "ramp_filter_msamples_per_s": round(r32["ramp_filter_msamples_per_s"], 2),
                                "s_per_volume_extrapolated": round(total_updates / (v * 1e9), 1)}
            except Exception as ex:
                cpu_baseline = {"error": repr(ex)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
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
                   "chunks": (len(eng.chunks) if chunked else None),
                   "parallelism": (f"angle-split x{world} ({args.exchange}: partials reduced onto z-slab owners)"
                                   if angle_split else
                                   f"z-slab x{world}" + (f" ({args.exchange} exchange)" if world > 1 else "")),
                   "k2": "tensor cores" if getattr(slab, "tensor", False) else "CUDA cores",
                   "l2": "inputs larger than L2 (raw %.1f GB, volume %.1f GB per step)" % (
                       raw.numel() * 4 / 1e9, n * n * k_rows * 4 / 1e9),
                   "step": ("K1 Beer-Lambert+ramp+feather -> z-blocked staging -> K2 back-projection of this "
                            "rank's angles over the whole volume, epilogue adds into each row's owner "
                            "(NVLink peer memory, or + NCCL reduce-scatter) -> FoV/scale finalize"
                            if angle_split else
                            EXCHANGE_STEP.get(args.exchange if world > 1 else "", EXCHANGE_STEP[""]))},
        "roofline": roof,
        "clocks": clk,
        "gpu_launches": launches * args.steps,
        "bp_share_of_step": round(bp_avg_ms / statistics.mean(step_ms), 4),
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
