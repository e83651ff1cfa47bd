"""Device-resident FBP engine: the reconstruction stage of `pipeline.run`
(`/root/reference/pkg/src/tomofuse/pipeline.py:163-237`) as one GPU pass.

One `SlabReconstructor` owns the HBM buffers for a row slab [r0, r1) of one
specimen and runs, all on one CUDA stream:

    raw counts (n_proj, k, n_chan) fp32
      --K1 tf_filter--> filtered (Beer-Lambert + ramp, fp32)
      --tf_bp_stage--> z-blocked staging (feather folded in)
      --K2 tf_backproject--> volume (k, ny, nx) fp32
      [--K3 tf_quantize--> uint16]

which is exactly `preprocess -> ramp_filter -> astype(float32) ->
back_project(dtype=float32)` of pipeline.py:176-222 / fbp.reconstruct.
Buffers are allocated once; `run()` never allocates, so the step can be
timed (and CUDA-graph captured) without allocator noise.
"""

from __future__ import annotations

import ctypes
import os

from . import _lib
from ._lib import check, lib
from .fbp import FilterSpec, bp_plan, filter_plan
from .geometry import AcquisitionParams, VolumeDims


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def tensor_default() -> bool:
    """K2 on the tensor cores (tf_backproject_tc) unless TF_BP_TENSOR=0."""
    return os.environ.get("TF_BP_TENSOR", "1") != "0"


class SlabReconstructor:
    """HBM buffers and kernels of one row slab.  K2 runs on the tensor cores
    (tap planes written by K1 directly, tf_filter_taps -> tf_backproject_tc)
    unless `tensor=False` / TF_BP_TENSOR=0 selects the CUDA-core kernel
    (fp32 z-blocked staging, tf_filter_stage -> tf_backproject)."""

    def __init__(self, params: AcquisitionParams, dims: VolumeDims, spec: FilterSpec | None = None,
                 i0: float = 1e5, feather_band: int = 32, rows: tuple[int, int] | None = None,
                 device=None, in_place_filter: bool = False, stage=None, tensor: bool | None = None,
                 n_angles: int | None = None):
        import torch

        self.torch = torch
        self.params, self.dims = params, dims
        self.spec = spec if spec is not None else FilterSpec()
        self.i0 = float(i0)
        self.r0, self.r1 = rows if rows is not None else (0, params.n_rows)
        self.k = self.r1 - self.r0
        self.n_angles = params.n_proj if n_angles is None else int(n_angles)  # angles the taps buffer holds
        self.device = torch.device(device if device is not None else "cuda")
        with torch.cuda.device(self.device):
            self.fplan = filter_plan(params.n_chan, self.spec, params.pixel_pitch)
            self.bplan = bp_plan(params, dims, feather_band)
            self.in_place = in_place_filter
            self._filt = None  # natural-layout filtered rows, only for the unfused path
            sup = bool(lib().tf_bp_tc_supported(self.bplan.handle))
            if tensor and not sup:
                raise ValueError("tensor-core back-projection needs voxel_pitch / pixel_pitch <= 2.12")
            self.tensor = sup and (tensor_default() if tensor is None else bool(tensor))
            self.stage = self.taps = None
            if self.tensor:
                nb = int(lib().tf_bp_tc_taps_bytes(self.bplan.handle, self.k, self.n_angles))
                if stage is not None:
                    stage = stage.view(torch.uint8).view(-1)
                    if stage.numel() < nb:
                        raise ValueError(f"tap buffer too small: {stage.numel()} < {nb} bytes")
                    self.taps = stage[:nb]
                else:
                    self.taps = torch.empty(nb, dtype=torch.uint8, device=self.device)
            else:
                need = self.bplan.stage_bytes(self.k)
                if stage is not None:  # caller-provided (e.g. NVLink-mapped symmetric memory)
                    stage = stage.view(torch.uint8).view(-1)
                    if stage.numel() < need:
                        raise ValueError(f"staging buffer too small: {stage.numel()} < {need} bytes")
                    self.stage = stage[:need]
                else:
                    self.stage = torch.empty(need, dtype=torch.uint8, device=self.device)
            self.vol = torch.empty((self.k, dims.ny, dims.nx), dtype=torch.float32, device=self.device)

    @property
    def filt(self):
        if self._filt is None:
            self._filt = self.torch.empty((self.params.n_proj, self.k, self.params.n_chan),
                                          dtype=self.torch.float32, device=self.device)
        return self._filt

    def tap_bound(self, i0=None) -> float:
        """The |T| bound K1 uses for raw counts (tf_filter_tap_bound): every
        producer of tap planes from raw counts scales by the same 2^e."""
        b = ctypes.c_double()
        check(lib().tf_filter_tap_bound(self.fplan.handle, self.i0 if i0 is None else float(i0), ctypes.byref(b)))
        return b.value

    # -- individual kernels (stream = torch current stream unless given)
    def _s(self, stream):
        st = stream if stream is not None else self.torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(st.cuda_stream)

    def filter(self, raw, out=None, stream=None, i0=None):
        """K1 on raw counts (or depth when i0 <= 0) -> natural-layout fp32 rows."""
        out = out if out is not None else (raw if self.in_place else self.filt)
        n_lines = raw.numel() // self.params.n_chan
        check(lib().tf_filter(self.fplan.handle, _ptr(raw), _ptr(out), n_lines,
                              self.i0 if i0 is None else float(i0), 0, 0, None, None, self._s(stream)))
        return out

    def filter_stage(self, raw, stream=None, i0=None, n_rows=None):
        """Fused K1: raw counts (A, k, n_chan) -> Beer-Lambert -> ramp filter
        -> feather -> K2's input (tap planes, or z-blocked staging for the
        CUDA-core kernel), no filtered copy."""
        k = self.k if n_rows is None else n_rows
        n_lines = raw.numel() // self.params.n_chan
        i0 = self.i0 if i0 is None else float(i0)
        if self.tensor:
            check(lib().tf_filter_taps(self.fplan.handle, self.bplan.handle, _ptr(raw), _ptr(self.taps),
                                       self.taps.numel(), n_lines, i0, k, self._s(stream)))
        else:
            check(lib().tf_filter_stage(self.fplan.handle, self.bplan.handle, _ptr(raw), _ptr(self.stage), n_lines,
                                        i0, k, 0, None, None, self._s(stream)))

    def stage_rows(self, filt, rows_per_angle=None, r0=0, stream=None, a0=0, a1=None, t_bound=None):
        """Filtered natural rows [r0, r0 + k) of angles [a0, a1) -> K2's input.
        Tensor path: tap planes scaled from `t_bound` (default: the raw-count
        bound of this slab's i0, so rows staged after an exchange match K1's
        own tap planes bit for bit); t_bound <= 0 takes per-row data maxima."""
        rpa = rows_per_angle if rows_per_angle is not None else self.k
        if self.tensor:
            a1 = self.params.n_proj if a1 is None else a1
            tb = self.tap_bound() if t_bound is None else float(t_bound)
            check(lib().tf_bp_tc_stage(self.bplan.handle, _ptr(filt), rpa, r0, r0 + self.k, a0, a1, tb,
                                       _ptr(self.taps), self.taps.numel(), self._s(stream)))
            return
        check(lib().tf_bp_stage(self.bplan.handle, _ptr(filt), rpa, r0, r0 + self.k, _ptr(self.stage),
                                self._s(stream)))

    def backproject(self, a0=0, a1=None, flags=_lib.TF_BP_FINALIZE, stream=None, vol=None, n_rows=None,
                    taps_a0=0, taps_a1=None):
        """K2 over angles [a0, a1) of the staged rows (n_rows, default the
        slab's); the tap planes hold angles [taps_a0, taps_a1)."""
        a1 = self.params.n_proj if a1 is None else a1
        vol = self.vol if vol is None else vol
        k = self.k if n_rows is None else n_rows
        if self.tensor and not flags & _lib.TF_BP_KERNEL_V1:
            ta1 = self.n_angles + taps_a0 if taps_a1 is None else taps_a1
            check(lib().tf_backproject_tc(self.bplan.handle, _ptr(self.taps), self.taps.numel(), taps_a0, ta1, k,
                                          _ptr(vol), a0, a1, 0, self.dims.nx, 0, self.dims.ny, flags,
                                          self._s(stream)))
            return vol
        if self.stage is None:
            raise ValueError("the CUDA-core kernel needs the fp32 staging buffer (tensor=False)")
        check(lib().tf_backproject(self.bplan.handle, _ptr(self.stage), k, _ptr(vol), a0, a1,
                                   0, self.dims.nx, 0, self.dims.ny, flags, self._s(stream)))
        return vol

    def quantize(self, lo, hi, out, stream=None):
        check(lib().tf_quantize(_ptr(self.vol), _lib.TF_F32, _ptr(out), self.vol.numel(), float(lo),
                                float(hi), self._s(stream)))
        return out

    def run(self, raw, stream=None):
        """raw: device (n_proj, k, n_chan) fp32 counts -> self.vol."""
        self.filter_stage(raw, stream=stream)
        return self.backproject(stream=stream)

    def capture(self, raw):
        """Record run(raw) -- K1 into K2's input, K2 into self.vol -- as a
        CUDA graph and return it; `graph.replay()` re-runs the step on
        whatever `raw` holds then, with one launch from the host.  The
        library call path allocates nothing, so it is capture-safe."""
        torch = self.torch
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            self.run(raw)  # warm-up outside the graph (kernel attributes, tensor-map encoder)
        torch.cuda.current_stream(self.device).wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            self.run(raw)
        return graph

    def bp_work(self, a0=0, a1=None, n_rows=None) -> dict:
        """What K2 executes for angles [a0, a1): voxel x angle x row updates of
        the FoV-active tiles, and on the tensor path the MMA items and the
        tensor-pipe clocks (tf_bp_tc_work / tf_bp_kernel_info)."""
        a1 = self.params.n_proj if a1 is None else a1
        k = self.k if n_rows is None else n_rows
        if self.tensor:
            it, up, clk = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
            check(lib().tf_bp_tc_work(self.bplan.handle, k, a0, a1, ctypes.byref(it), ctypes.byref(up),
                                      ctypes.byref(clk)))
            return {"executed_updates": up.value, "mma_items": it.value, "mma_clocks": clk.value}
        bpu, exe = ctypes.c_double(), ctypes.c_int64()
        check(lib().tf_bp_kernel_info(self.bplan.handle, _lib.TF_BP_FINALIZE, k, a0, a1, ctypes.byref(bpu),
                                      ctypes.byref(exe)))
        return {"executed_updates": exe.value, "smem_bytes_per_update": bpu.value}

    def updates(self) -> int:
        """Voxel x projection updates of one run (pipeline.py:225-227 convention)."""
        return self.params.n_proj * self.k * self.dims.nx * self.dims.ny


def phantom_raw(params: AcquisitionParams, dims: VolumeDims, out, a0=0, a1=None, r0=0, r1=None,
                i0=1e5, mu_max=3.5e-4, stream=None):
    """Analytic 3-D Shepp-Logan raw counts (K4) into device tensor `out`
    of shape (a1-a0, r1-r0, n_chan)."""
    import torch

    a1 = params.n_proj if a1 is None else a1
    r1 = params.n_rows if r1 is None else r1
    g = _lib.geometry(params, dims)
    st = stream if stream is not None else torch.cuda.current_stream()
    check(lib().tf_phantom_sinogram(ctypes.byref(g), a0, a1, r0, r1, float(i0), float(mu_max),
                                    _ptr(out), ctypes.c_void_p(st.cuda_stream)))
    return out


class StreamedReconstructor:
    """Host-fed FBP: pinned host sinogram in, pinned host volume out, with
    the copies hidden under compute (the reference's four-stage pipeline of
    pipeline.py:311-349, realised with CUDA streams instead of a model).

    The volume is processed in z-sub-slabs of `slab_rows` rows.  For slab i:
      h2d stream : strided 2-D copy of rows [r0, r1) of every angle -> raw[i%2]
      comp stream: K1 filter -> stage -> K2 back-projection -> vol[i%2]
      d2h stream : vol[i%2] -> host rows [r0, r1)
    Events order the double-buffered raw/vol buffers, so slab i+1's H2D and
    slab i-1's D2H overlap slab i's kernels.  HBM use is bounded by the
    sub-slab size, so this is also the path for volumes larger than HBM.
    """

    def __init__(self, params: AcquisitionParams, dims: VolumeDims, spec: FilterSpec | None = None,
                 i0: float = 1e5, feather_band: int = 32, slab_rows: int = 256, device=None,
                 tensor: bool | None = None, angle_chunk: int | str | None = "auto"):
        import torch

        self.torch = torch
        self.params, self.dims = params, dims
        self.device = torch.device(device if device is not None else "cuda")
        self.slab_rows = min(slab_rows, params.n_rows)
        k = self.slab_rows
        with torch.cuda.device(self.device):
            self.angle_chunk = self._chunk(angle_chunk, tensor)
            A = self.angle_chunk or params.n_proj
            self.eng = SlabReconstructor(params, dims, spec, i0, feather_band, rows=(0, k),
                                         device=self.device, tensor=tensor, n_angles=A)
            if self.angle_chunk and not self.eng.tensor:
                raise ValueError("angle chunks need the tensor-core K2 (blocks of 16 absolute angles chain exactly)")
            shape = (A, k, params.n_chan)
            self.raw = [torch.empty(shape, dtype=torch.float32, device=self.device) for _ in range(2)]
            self.vol = [self.eng.vol, None]  # the second fp32 slab only without quantize (allocated on use)
            self.s_h2d = torch.cuda.Stream(self.device)
            self.s_comp = torch.cuda.Stream(self.device)
            self.s_d2h = torch.cuda.Stream(self.device)
        # buffer parity and the events guarding the double buffers persist across calls, so
        # back-to-back calls with join=False overlap one call's last D2H with the next one's
        # first H2D (the pipeline fills and drains once per sequence of calls)
        self._n = 0  # raw-buffer parity (per H2D chunk)
        self._m = 0  # output-buffer parity (per sub-slab)
        self._raw_free = [None, None]
        self._out_free = [None, None]

    def _chunk(self, angle_chunk, tensor):
        """Angles per H2D / K1 / K2 chunk of a sub-slab (None: all).  "auto"
        chunks only when the double-buffered raw counts, the tap planes and
        the fp32 + uint16 volume slabs of whole-scan sub-slabs would not fit
        in the device's free memory less 4 GiB (C5: 7200 x 8192 x 256-row
        sub-slabs); chunks are multiples of 16 angles, so chaining them with
        TF_BP_ACCUMULATE gives the single-pass volume bit for bit."""
        p, d, k = self.params, self.dims, self.slab_rows
        if angle_chunk is None or (tensor is False) or (tensor is None and not tensor_default()):
            return None
        if angle_chunk != "auto":  # a chunk covering the scan is no chunking
            return None if int(angle_chunk) >= p.n_proj else max(16, int(angle_chunk) // 16 * 16)
        free, _ = self.torch.cuda.mem_get_info(self.device)
        # blocks the caching allocator holds but no tensor uses are free for these buffers too
        free += self.torch.cuda.memory_reserved(self.device) - self.torch.cuda.memory_allocated(self.device)
        line = k * p.n_chan * 4  # raw fp32 and fp16 hi/lo taps: 4 B per sample each
        fixed = k * d.nx * d.ny * (4 + 2)  # fp32 slab + the uint16 slab
        budget = free - (4 << 30) - fixed  # a 4 GiB margin for the plan, workspaces and the allocator
        if 3 * line * p.n_proj <= budget:
            return None
        a = int(budget // (3 * line)) // 16 * 16
        if a < 16:
            raise ValueError(f"a {k}-row sub-slab does not fit in device memory; lower slab_rows")
        return a

    def sub_slabs(self, R0, R1):
        """Sub-slab boundaries.  Tensor-core K2: uniform `slab_rows` slabs
        (a short slab costs a full 128/256-row MMA block, so a ramp of small
        slabs would waste tensor work; the un-overlapped fill and drain are
        one slab's H2D and D2H).  CUDA-core K2: full slabs in the middle and
        a geometric ramp at both ends (32, 64, 128, ... rows) so that the
        fill (first H2D) and drain (last D2H) are one 32-row slab each,
        while every next slab's H2D still hides under the current slab's
        compute; when the range is too short for the ramp up to `slab_rows`
        (a z-slab of one GPU among several: 512 rows at N=4), the middle
        slab size halves until the ramp fits."""
        S = self.slab_rows
        if self.eng.tensor:
            return [(r, min(r + S, R1)) for r in range(R0, R1, S)]

        def ramp_to(s):
            r, e = [], 32
            while e < s:
                r.append(e)
                e *= 2
            return r

        ramp = []
        s = S
        while s >= 64:
            if R1 - R0 >= 2 * sum(ramp_to(s)) + s:
                S, ramp = s, ramp_to(s)
                break
            s //= 2
        cuts, r = [], R0
        for e in ramp:
            cuts.append((r, r + e))
            r += e
        tail = R1 - sum(ramp)
        while r < tail:
            cuts.append((r, min(r + S, tail)))
            r = cuts[-1][1]
        for e in reversed(ramp):
            cuts.append((r, r + e))
            r += e
        assert r == R1
        return cuts

    def _copy2d(self, dst, dpitch, src, spitch, width, height, stream):
        check(lib().tf_copy2d_async(ctypes.c_void_p(dst), dpitch, ctypes.c_void_p(src), spitch, width, height,
                                    ctypes.c_void_p(stream.cuda_stream)))

    def run(self, raw_host, vol_host, row_range=None, host_row0=0, quantize=None, join=True):
        """raw_host: pinned (n_proj, H, n_chan) fp32 counts holding detector
        rows [host_row0, host_row0 + H); vol_host: pinned (R, ny, nx) fp32
        receiving volume rows `row_range` = [r0, r1) (default: all rows), or
        uint16 when `quantize` = (lo, hi) (K3 runs per slab on the device, so
        only 2 B/voxel cross PCIe).  With `angle_chunk` each sub-slab's
        angles stream in chunks (H2D / K1 / K2 with TF_BP_ACCUMULATE), which
        lets whole-width sub-slabs fit when the scan does not (C5).  Work is queued on this object's streams
        (ordered after the current stream); returns the last D2H event.
        join=False leaves the work on this object's streams (the caller
        waits on the returned event or calls join()), so the next call's
        first H2D overlaps this call's last D2H."""
        return self.run_batch([(raw_host, vol_host, row_range, host_row0)], quantize, join)

    def join(self):
        """Make the current stream wait for everything queued on this object's streams."""
        cur = self.torch.cuda.current_stream(self.device)
        for s in (self.s_h2d, self.s_comp, self.s_d2h):
            cur.wait_stream(s)

    def run_batch(self, jobs, quantize=None, join=True):
        """A batch of specimens (the reference's SpecimenSet groups,
        pipeline.py:119-161) as ONE sub-slab stream: jobs = [(raw_host,
        vol_host, row_range, host_row0), ...], each as in run().  The next
        specimen's first H2D overlaps the previous one's last sub-slab, so
        the pipeline fills and drains once per batch, not per specimen."""
        torch = self.torch
        p, d = self.params, self.dims
        n = p.n_chan
        line = n * 4
        plane = d.nx * d.ny * (2 if quantize is not None else 4)
        if quantize is not None and getattr(self, "_q", None) is None:
            self._q = torch.empty(self.vol[0].shape, dtype=torch.uint16, device=self.device)
        if quantize is None and self.vol[1] is None:
            self.vol[1] = torch.empty_like(self.vol[0])
        cur = torch.cuda.current_stream(self.device)
        for s in (self.s_h2d, self.s_comp, self.s_d2h):
            s.wait_stream(cur)
        raw_free, out_free = self._raw_free, self._out_free
        A = self.angle_chunk or p.n_proj
        chunks = [(a, min(a + A, p.n_proj)) for a in range(0, p.n_proj, A)]
        done = None
        tasks = []
        for raw_host, vol_host, row_range, host_row0 in jobs:
            R0, R1 = row_range if row_range is not None else (0, p.n_rows)
            tasks += [(raw_host, vol_host, R0, host_row0, r0, r1) for r0, r1 in self.sub_slabs(R0, R1)]
        for raw_host, vol_host, R0, host_row0, r0, r1 in tasks:
            k = r1 - r0
            o = self._m % 2
            self._m += 1
            # with K3 the fp32 slab is consumed on the compute stream itself: one buffer suffices
            vol = self.vol[0] if quantize is not None else self.vol[o]
            for a, b in chunks:
                rb = self._n % 2
                self._n += 1
                # H2D: rows [r0, r1) of angles [a, b) (b - a strided chunks)
                if raw_free[rb] is not None:
                    self.s_h2d.wait_event(raw_free[rb])
                self._copy2d(self.raw[rb].data_ptr(), k * line,
                             raw_host.data_ptr() + (a * raw_host.shape[1] + r0 - host_row0) * line,
                             raw_host.shape[1] * line, k * line, b - a, self.s_h2d)
                h2d_done = torch.cuda.Event()
                h2d_done.record(self.s_h2d)
                # compute: K1 into the tap planes of this chunk, K2 over its angles
                self.s_comp.wait_event(h2d_done)
                self.eng.filter_stage(self.raw[rb].view(-1)[: (b - a) * k * n], stream=self.s_comp, n_rows=k)
                ev = torch.cuda.Event()
                ev.record(self.s_comp)
                raw_free[rb] = ev
                if a == 0 and quantize is None and out_free[o] is not None:
                    self.s_comp.wait_event(out_free[o])  # vol[o]'s previous D2H
                flags = (_lib.TF_BP_ACCUMULATE if a > 0 else 0) | (_lib.TF_BP_FINALIZE if b == p.n_proj else 0)
                self.eng.backproject(a0=a, a1=b, flags=flags, stream=self.s_comp, vol=vol, n_rows=k, taps_a0=a,
                                     taps_a1=b)
            src_vol = vol
            if quantize is not None:  # fbp.quantize on the device (K3) into the one uint16 slab
                lo, hi = quantize
                o = 0
                if out_free[0] is not None:
                    self.s_comp.wait_event(out_free[0])  # its previous D2H (far shorter than a sub-slab)
                check(lib().tf_quantize(_ptr(vol), _lib.TF_F32, _ptr(self._q), k * d.nx * d.ny,
                                        float(lo), float(hi), ctypes.c_void_p(self.s_comp.cuda_stream)))
                src_vol = self._q
            comp_done = torch.cuda.Event()
            comp_done.record(self.s_comp)
            # D2H: contiguous volume slab
            self.s_d2h.wait_event(comp_done)
            self._copy2d(vol_host.data_ptr() + (r0 - R0) * plane, plane, src_vol.data_ptr(), plane, plane, k,
                         self.s_d2h)
            ev = torch.cuda.Event()
            ev.record(self.s_d2h)
            out_free[o] = ev
            done = ev
        if join:
            self.join()
        return done

    def updates(self, row_range=None) -> int:
        r0, r1 = row_range if row_range is not None else (0, self.params.n_rows)
        return self.params.n_proj * (r1 - r0) * self.dims.nx * self.dims.ny
