"""Multi-GPU z-slab reconstruction (one process per GPU, NCCL over NVLink).

Replaces the reference's simulated P_row partition (partition.py:221,
PAPER.md:253-255) and its in-process `Fabric` (fabric.py:25-127) with real
devices:

* rank g owns detector rows / volume slices `split_range(n_rows, N)[g]`
  and back-projects ALL angles for them -- rows are independent
  (pkg/tests/test_fbp.py:180-191), so there is no reduction and the N-GPU
  volume is bitwise the 1-GPU volume;
* rank g ingests and filters the angle chunk `split_range(n_proj, N)[g]`
  (all rows), i.e. 1/N of the projections, as north_star prescribes;
* filtered rows reach their owner through one collective:
    - "alltoall" (default, minimal bytes): K1 writes its output already in
      K2's z-blocked staging layout, grouped per destination slab, so a
      single `all_to_all_single` lands every owner's rows angle-ordered
      directly in its staging buffer (no separate staging pass);
    - "p2p" (fused compute + exchange): every rank's receive buffer is
      symmetric memory mapped over NVLink; K1's epilogue stores each
      destination slab's rows, natural layout, straight into the owner's
      buffer (tf_filter_peers, one contiguous run per line: coalesced
      NVLink stores), so the all-to-all IS the filter's store stream; the
      owner then stages its rows locally (tf_bp_stage).  Two symmetric-
      memory barriers per step order it (previous step's staging done
      before overwrite; all stores landed before staging);
    - "p2p-zblocked": as "p2p" but K1 stores straight into the owner's
      staging layout (tf_filter_stage_peers): no staging pass, but 8-byte
      scattered remote stores;
    - "allgather" (north_star's literal variant): `all_gather_into_tensor`
      of the natural-layout chunks, N x the bytes, owners stage their rows.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import check, lib
from .engine import SlabReconstructor
from .fbp import FilterSpec
from .geometry import AcquisitionParams, VolumeDims, split_range


ZB, ZP = 32, 36  # z-block rows and padded row pitch of K2's staging layout (csrc/common.cuh)


def _rows_elems(k: int, n_chan: int, zblocked: bool) -> int:
    """Elements one angle of a k-row slab occupies: natural rows or z-blocks."""
    return (-(-k // ZB)) * n_chan * ZP if zblocked else k * n_chan


def exchange_layout(world: int, rank: int, n_proj: int, n_rows: int, n_chan: int, zblocked: bool = False):
    """Row-slab all-to-all layout for `rank`.

    Returns (slabs, chunks, slab_row0, slab_base, in_splits, out_splits):
    element offsets of each destination's block in the send buffer
    (slab-major: [dest][angle][rows of the dest slab]) and the split sizes of
    `all_to_all_single`, in elements.  With `zblocked` the rows of a slab are
    K2's staging layout ([zb][chan][36]), so what lands on the owner is its
    staging buffer, angle-ordered.
    """
    slabs = split_range(n_rows, world)
    chunks = split_range(n_proj, world)
    a0, a1 = chunks[rank]
    A = a1 - a0
    r0, r1 = slabs[rank]
    per = [_rows_elems(e - s, n_chan, zblocked) for s, e in slabs]
    slab_row0 = [s for s, _ in slabs] + [n_rows]
    slab_base = [A * sum(per[:i]) for i in range(world)]
    in_splits = [A * q for q in per]
    out_splits = [(ce - cs) * per[rank] for cs, ce in chunks]
    return slabs, chunks, slab_row0, slab_base, in_splits, out_splits


def slab_major(chunk, slabs):
    """Host/torch restatement of K1's slab-major output mapping (test helper
    and documentation of tf_filter's slab map): (A, n_rows, n_chan) ->
    flat [dest][A][rows_in_slab][n_chan]."""
    import torch

    return torch.cat([chunk[:, s:e].reshape(-1) for s, e in slabs])


def zblocked(rows, weights=None):
    """Host/torch restatement of K2's staging layout (tf_bp_stage /
    tf_filter_stage): (A, k, n_chan) -> flat [A][zb][n_chan][36], rows padded
    to 32 with zeros, pad floats 32..35 zero, optional per-channel feather."""
    import torch

    A, k, n = rows.shape
    nzb = -(-k // ZB)
    x = rows if weights is None else rows * weights
    out = torch.zeros((A, nzb * ZB, n), dtype=rows.dtype, device=rows.device)
    out[:, :k] = x
    out = out.view(A, nzb, ZB, n).permute(0, 1, 3, 2)  # [A][zb][n][32]
    full = torch.zeros((A, nzb, n, ZP), dtype=rows.dtype, device=rows.device)
    full[..., :ZB] = out
    return full.reshape(-1)


def tap_planes(rows, weights, bound):
    """Host/torch restatement of K2-TC's tap planes (tf_filter_taps /
    tf_bp_tc_stage with a bound): (A, k, n_chan) fp32 filtered rows ->
    flat bytes [A][hi, lo][k/8][n_chan][8] fp16 of (rows * weights) * 2^e,
    e = 14 - floor(log2(bound)), hi = fp16(x), lo = fp16(x - hi); rows past
    k in the last 8-row group are zero here (the kernels leave them
    unwritten).  The workspace header (per-row exponents) is not included."""
    import math

    import torch

    A, k, n = rows.shape
    e = min(100, max(-100, 14 - (math.frexp(bound)[1] - 1)))
    x = (rows * weights) * (2.0 ** e)
    hi = x.to(torch.float16)
    lo = (x - hi.float()).to(torch.float16)
    R8 = -(-k // 8)
    out = torch.zeros((A, 2, R8 * 8, n), dtype=torch.float16, device=rows.device)
    out[:, 0, :k] = hi
    out[:, 1, :k] = lo
    return out.view(A, 2, R8, 8, n).permute(0, 1, 2, 4, 3).contiguous().view(torch.uint8).reshape(-1)


def exchange(send, recv, in_splits, out_splits, group=None):
    import torch.distributed as dist

    dist.all_to_all_single(recv, send, output_split_sizes=out_splits, input_split_sizes=in_splits,
                           group=group)


class ZSlabReconstructor:
    """Per-rank state of an N-GPU z-slab reconstruction."""

    def __init__(self, params: AcquisitionParams, dims: VolumeDims, spec: FilterSpec | None = None,
                 i0: float = 1e5, feather_band: int = 32, exchange_mode: str = "alltoall",
                 group=None, device=None):
        import torch
        import torch.distributed as dist

        self.torch = torch
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.mode = exchange_mode
        self.params, self.dims = params, dims
        n_proj, n_rows, n_chan = params.n_proj, params.n_rows, params.n_chan
        (self.slabs, self.chunks, row0, base, self.in_splits,
         self.out_splits) = exchange_layout(self.world, self.rank, n_proj, n_rows, n_chan,
                                            zblocked=exchange_mode == "alltoall")
        self.a0, self.a1 = self.chunks[self.rank]
        self.r0, self.r1 = self.slabs[self.rank]
        self.device = torch.device(device if device is not None else "cuda")
        if exchange_mode == "allgather":
            sizes = {e - s for s, e in self.chunks}
            if len(sizes) != 1:
                raise ValueError("allgather exchange needs n_proj divisible by the world size")
        elif exchange_mode not in ("alltoall", "p2p", "p2p-zblocked"):
            raise ValueError(f"unknown exchange mode {exchange_mode!r}")
        A = self.a1 - self.a0
        self.symm = None
        self.recv = None
        stage = None
        if exchange_mode.startswith("p2p"):
            import torch.distributed._symmetric_memory as symm

            zb = exchange_mode == "p2p-zblocked"
            per = [_rows_elems(e - s, n_chan, zb) for s, e in self.slabs]  # floats per angle per slab
            buf = symm.empty(n_proj * max(per), dtype=torch.float32, device=self.device)
            self.symm = symm.rendezvous(buf, group if group is not None else dist.group.WORLD)
            # slab s's rows of my angles go to rank s's buffer at angle a0
            dst = [int(self.symm.buffer_ptrs[s]) + self.a0 * per[s] * 4 for s in range(self.world)]
            self._dst = (ctypes.c_void_p * self.world)(*dst)
            if zb:
                stage = buf  # lands directly in the owner's staging layout
            else:
                k = self.r1 - self.r0
                self.recv = buf[: n_proj * k * n_chan].view(n_proj, k, n_chan)
        # local slab engine; for "alltoall" / "p2p-zblocked" its fp32 staging buffer is the exchange
        # landing zone (CUDA-core K2); "p2p" / "allgather" land natural rows that the owner stages
        # into tap planes for the tensor-core K2 with the raw-count bound (bitwise K1's own taps)
        zblocked_landing = exchange_mode in ("alltoall", "p2p-zblocked")
        self.local = SlabReconstructor(params, dims, spec, i0, feather_band, rows=(self.r0, self.r1),
                                       device=self.device, stage=stage,
                                       tensor=False if zblocked_landing else None)
        if exchange_mode.startswith("p2p"):
            self.send = None
        else:
            self.send = torch.empty(sum(self.in_splits) if exchange_mode == "alltoall" else A * n_rows * n_chan,
                                    dtype=torch.float32, device=self.device)
        if exchange_mode == "allgather":
            self.gathered = torch.empty((n_proj, n_rows, n_chan), dtype=torch.float32,
                                        device=self.device)
            self._map = None
        else:
            self.gathered = None
            self._map = ((ctypes.c_int32 * len(row0))(*row0), (ctypes.c_int64 * len(base))(*base))

    def chunk_shape(self):
        return (self.a1 - self.a0, self.params.n_rows, self.params.n_chan)

    def _s(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def filter(self, raw_chunk):
        """K1 over this rank's angle chunk, written in the exchange layout:
        z-blocked staging per destination slab (alltoall) or natural rows
        (allgather)."""
        p = self.params
        n_lines = raw_chunk.numel() // p.n_chan
        if self.mode.startswith("p2p"):
            row0, _ = self._map
            self.symm.barrier(channel=0)  # owners finished reading their buffer (previous step)
            if self.mode == "p2p":
                check(lib().tf_filter_peers(self.local.fplan.handle, ctypes.c_void_p(raw_chunk.data_ptr()),
                                            n_lines, self.local.i0, p.n_rows, self.world, row0, self._dst,
                                            self._s()))
            else:
                check(lib().tf_filter_stage_peers(self.local.fplan.handle, self.local.bplan.handle,
                                                  ctypes.c_void_p(raw_chunk.data_ptr()), n_lines, self.local.i0,
                                                  p.n_rows, self.world, row0, self._dst, self._s()))
            return
        if self._map is None:
            check(lib().tf_filter(self.local.fplan.handle, ctypes.c_void_p(raw_chunk.data_ptr()),
                                  ctypes.c_void_p(self.send.data_ptr()), n_lines, self.local.i0,
                                  0, 0, None, None, self._s()))
        else:
            row0, base = self._map
            check(lib().tf_filter_stage(self.local.fplan.handle, self.local.bplan.handle,
                                        ctypes.c_void_p(raw_chunk.data_ptr()), ctypes.c_void_p(self.send.data_ptr()),
                                        n_lines, self.local.i0, p.n_rows, self.world, row0, base, self._s()))

    def exchange(self):
        import torch.distributed as dist

        if self.mode.startswith("p2p"):  # the stores already landed; wait until every peer's have
            self.symm.barrier(channel=0)
            return
        if self.mode == "allgather":
            dist.all_gather_into_tensor(self.gathered.view(-1), self.send, group=self.group)
        else:  # lands directly in this rank's staging buffer
            exchange(self.send, self.local.stage.view(self.torch.float32), self.in_splits, self.out_splits,
                     self.group)

    def stage(self):
        if self.mode == "allgather":
            self.local.stage_rows(self.gathered, rows_per_angle=self.params.n_rows, r0=self.r0)
        elif self.mode == "p2p":
            self.local.stage_rows(self.recv, rows_per_angle=self.r1 - self.r0, r0=0)

    def run(self, raw_chunk):
        """raw_chunk: device (A, n_rows, n_chan) fp32 counts of this rank's
        angles -> this rank's volume slab (k, ny, nx) in self.local.vol."""
        self.filter(raw_chunk)
        self.exchange()
        self.stage()
        return self.local.backproject()

    def updates(self) -> int:
        return self.local.updates()

    def exchange_bytes(self) -> int:
        """Bytes this rank receives from peers per run."""
        if self.mode == "allgather":
            return int(np.prod(self.chunk_shape())) * 4 * (self.world - 1)
        return sum(s for i, s in enumerate(self.out_splits) if i != self.rank) * 4


class AngleSplitReconstructor:
    """P_proj partitioning: angle-parallel partial volumes, reduced onto the
    z-slab owners (the reference's projection split with
    `Fabric.reduce_scatter_block`, pipeline.py:239-275 / fabric.py:67-101).

    Rank g filters and back-projects ONLY its angle chunk
    `split_range(n_proj, N)[g]`, over every row of the volume, and ends up
    owning rows `split_range(n_rows, N)[g]` summed over all ranks' angles,
    then finalized (FoV mask + angle weight).  Worth it when z-slabs run
    short (n_rows < N x 32-row blocks), where z-slabs would leave z-blocks
    half empty; otherwise `ZSlabReconstructor` moves far fewer bytes.

    reduce="p2p" (default): every rank's slab is symmetric memory mapped over
        NVLink and K2's epilogue adds each row's partial sums straight into
        the owner's slab (tf_backproject_reduce) -- the reduce-scatter is the
        back-projection's store stream, overlapped with the other tiles'
        angle loops.  Two symmetric-memory barriers order a step.
    reduce="nccl": K2 writes the full partial volume (owner-padded layout),
        then one `reduce_scatter_tensor` (sum).

    Summation order across ranks differs from the 1-GPU ascending order, so
    results agree with it to fp32 rounding (not bitwise, unlike z-slabs).
    """

    def __init__(self, params: AcquisitionParams, dims: VolumeDims, spec: FilterSpec | None = None,
                 i0: float = 1e5, feather_band: int = 32, reduce: str = "p2p", group=None, device=None):
        import torch
        import torch.distributed as dist

        from .fbp import bp_plan, filter_plan

        if reduce not in ("p2p", "nccl"):
            raise ValueError(f"unknown reduce mode {reduce!r}")
        self.torch = torch
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > 8:
            raise ValueError("angle-split reduction supports at most 8 ranks")
        self.mode = reduce
        self.params, self.dims = params, dims
        self.spec = spec if spec is not None else FilterSpec()
        self.i0 = float(i0)
        self.device = torch.device(device if device is not None else "cuda")
        self.slabs = split_range(params.n_rows, self.world)
        self.chunks = split_range(params.n_proj, self.world)
        self.a0, self.a1 = self.chunks[self.rank]
        self.r0, self.r1 = self.slabs[self.rank]
        self.kmax = max(e - s for s, e in self.slabs)
        n_rows, n_chan, plane = params.n_rows, params.n_chan, dims.nx * dims.ny
        with torch.cuda.device(self.device):
            self.fplan = filter_plan(n_chan, self.spec, params.pixel_pitch)
            self.bplan = bp_plan(params, dims, feather_band)
        A = self.a1 - self.a0
        nzb = -(-n_rows // ZB)
        self.angle_bytes = nzb * n_chan * ZP * 4
        self.stage = torch.empty(max(A, 1) * self.angle_bytes, dtype=torch.uint8, device=self.device)
        row0 = [s for s, _ in self.slabs] + [n_rows]
        self._row0 = (ctypes.c_int32 * len(row0))(*row0)
        if reduce == "p2p":
            import torch.distributed._symmetric_memory as symm

            self.slab = symm.empty((self.kmax, dims.ny, dims.nx), dtype=torch.float32, device=self.device)
            self.symm = symm.rendezvous(self.slab, group if group is not None else dist.group.WORLD)
            dst = [int(self.symm.buffer_ptrs[s]) for s in range(self.world)]
            self.partial = None
        else:
            self.symm = None
            self.slab = torch.empty((self.kmax, dims.ny, dims.nx), dtype=torch.float32, device=self.device)
            self.partial = torch.empty((self.world * self.kmax, dims.ny, dims.nx), dtype=torch.float32,
                                       device=self.device)
            base = self.partial.data_ptr()
            dst = [base + s * self.kmax * plane * 4 for s in range(self.world)]
        self._dst = (ctypes.c_void_p * self.world)(*dst)

    def chunk_shape(self):
        return (self.a1 - self.a0, self.params.n_rows, self.params.n_chan)

    def _s(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def run(self, raw_chunk):
        """raw_chunk: device (A, n_rows, n_chan) fp32 counts of this rank's
        angles -> this rank's finalized volume slab (k, ny, nx)."""
        import torch.distributed as dist

        p = self.params
        n_lines = raw_chunk.numel() // p.n_chan
        check(lib().tf_filter_stage(self.fplan.handle, self.bplan.handle, ctypes.c_void_p(raw_chunk.data_ptr()),
                                    ctypes.c_void_p(self.stage.data_ptr()), n_lines, self.i0, p.n_rows, 0, None,
                                    None, self._s()))
        if self.mode == "p2p":
            self.slab.zero_()
            self.symm.barrier(channel=0)  # every owner zeroed (and done reading the last step)
        else:
            self.partial.zero_()
        check(lib().tf_backproject_reduce(self.bplan.handle, ctypes.c_void_p(self.stage.data_ptr()), p.n_rows, self.a0, self.a1, self.world,
                                          self._row0, self._dst, 0, self._s()))
        if self.mode == "p2p":
            self.symm.barrier(channel=0)  # every rank's adds have landed
        else:
            dist.reduce_scatter_tensor(self.slab, self.partial, group=self.group)
        k = self.r1 - self.r0
        check(lib().tf_bp_finalize(self.bplan.handle, ctypes.c_void_p(self.slab.data_ptr()), k, self._s()))
        return self.slab[:k]

    def updates(self) -> int:
        return (self.a1 - self.a0) * self.params.n_rows * self.dims.nx * self.dims.ny


def chunk_plan(n_proj: int, world: int, rank: int, chunk: int):
    """Angle chunks [j C, (j + 1) C) of the scan, this rank's share of each
    (`split_range(len, world)[rank]`, absolute angles) and the offsets of the
    shares in the rank's concatenated raw input."""
    chunks = [(a, min(a + chunk, n_proj)) for a in range(0, n_proj, chunk)]
    parts = []
    for a, b in chunks:
        n = b - a  # split_range semantics (the first n % world shares one longer); empty shares allowed
        q, r = divmod(n, world)
        s = rank * q + min(rank, r)
        parts.append((a + s, a + s + q + (1 if rank < r else 0)))
    offsets = [0]
    for pa, pb in parts:
        offsets.append(offsets[-1] + pb - pa)
    return chunks, parts, offsets


class ChunkedZSlabReconstructor:
    """Z-slabs at C4 scale (4096^3 x 3600 on 4-8 GPUs): the p2p row-slab
    exchange run over ascending angle chunks, so the receive and tap buffers
    hold one chunk instead of the whole scan and the raw counts can stream
    in from pinned host memory.

    The angle range is cut into chunks [j C, (j + 1) C) with C a multiple of
    16.  For chunk j, rank g filters its share `split_range(len, N)[g]` of
    the chunk (so every rank ingests and filters 1/N of the projections,
    north_star); K1's epilogue stores each owner's rows straight into the
    owner's symmetric-memory receive buffer over NVLink (tf_filter_peers);
    after a device-side barrier each owner stages the chunk's rows into tap
    planes with the raw-count bound (tf_bp_tc_stage) and back-projects the
    chunk on the tensor cores with TF_BP_ACCUMULATE (the last chunk also
    FINALIZE).  Chunks ascend and start at multiples of 16 angles -- the
    tensor-core kernel's absolute RN flush blocks -- so the N-GPU volume is
    bitwise the 1-GPU single-pass volume.  This is the reference's
    angle-chunked work units (pipeline.py:210-222, partition.py:200-260) on
    real devices.

    Raw counts: `run(raw)` with a device tensor holding this rank's angles
    (`rank_angles()`, concatenated), or `run(raw_host)` with a pinned host
    tensor of the same shape: each chunk's part is copied on a side stream
    (double-buffered) while the previous chunk back-projects.
    """

    def __init__(self, params: AcquisitionParams, dims: VolumeDims, spec: FilterSpec | None = None,
                 i0: float = 1e5, feather_band: int = 32, chunk: int | None = None, group=None, device=None,
                 budget_bytes: float | None = None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        self.torch = torch
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.params, self.dims = params, dims
        n_proj, n_rows, n_chan = params.n_proj, params.n_rows, params.n_chan
        self.device = torch.device(device if device is not None else "cuda")
        self.slabs = split_range(n_rows, self.world)
        self.r0, self.r1 = self.slabs[self.rank]
        k = self.r1 - self.r0
        kmax = max(e - s for s, e in self.slabs)
        if chunk is None:
            # per angle of a chunk: receive rows + tap planes (4 B/sample each) + two raw part buffers
            per_angle = 4.0 * kmax * n_chan * 2 + 2 * 4.0 * n_rows * n_chan / self.world
            free = torch.cuda.mem_get_info(self.device)[0] if budget_bytes is None else budget_bytes
            vol = 4.0 * k * dims.nx * dims.ny
            chunk = int(max(16, (0.85 * free - vol) / per_angle) // 16 * 16)
        if chunk % 16:
            raise ValueError("angle chunks must be multiples of 16 angles (the tensor core flush blocks)")
        self.C = min(chunk, -(-n_proj // 16) * 16)
        self.chunks, self.parts, self.offsets = chunk_plan(n_proj, self.world, self.rank, self.C)
        with torch.cuda.device(self.device):
            self.local = SlabReconstructor(params, dims, spec, i0, feather_band, rows=(self.r0, self.r1),
                                           device=self.device, tensor=True, n_angles=self.C)
            buf = symm.empty(self.C * kmax * n_chan, dtype=torch.float32, device=self.device)
            self.symm = symm.rendezvous(buf, group if group is not None else dist.group.WORLD)
            self.recv = buf[: self.C * k * n_chan]
            self.raw_buf = None
            self.s_h2d = torch.cuda.Stream(self.device)
        self._row0 = (ctypes.c_int32 * (self.world + 1))(*([s for s, _ in self.slabs] + [n_rows]))
        self._ptrs = [int(self.symm.buffer_ptrs[s]) for s in range(self.world)]
        self._ks = [e - s for s, e in self.slabs]
        self.bound = self.local.tap_bound()

    def rank_angles(self):
        """This rank's angle ranges, one per chunk; run()'s raw input holds them concatenated."""
        return list(self.parts)

    def chunk_shape(self):
        return (self.offsets[-1], self.params.n_rows, self.params.n_chan)

    def _s(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def run(self, raw):
        """raw: (A, n_rows, n_chan) fp32 counts of rank_angles(), on this device
        or in pinned host memory -> this rank's volume slab in self.local.vol."""
        torch = self.torch
        p = self.params
        n_chan = p.n_chan
        host = not raw.is_cuda
        cur = torch.cuda.current_stream(self.device)
        if host and self.raw_buf is None:
            mx = max(pb - pa for pa, pb in self.parts)
            self.raw_buf = [torch.empty((max(mx, 1), p.n_rows, n_chan), dtype=torch.float32, device=self.device)
                            for _ in range(2)]
        k = self.r1 - self.r0
        free_ev = [None, None]
        copied = [None, None]

        def copy(j):
            b = j % 2
            pa, pb = self.parts[j]
            if j < 2:
                self.s_h2d.wait_stream(cur)
            if free_ev[b] is not None:
                self.s_h2d.wait_event(free_ev[b])
            with torch.cuda.stream(self.s_h2d):
                self.raw_buf[b][: pb - pa].copy_(raw[self.offsets[j]: self.offsets[j + 1]], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.s_h2d)
            copied[b] = ev

        if host:
            copy(0)
        last = len(self.chunks) - 1
        for j, ((ca, cb), (pa, pb)) in enumerate(zip(self.chunks, self.parts)):
            if host:
                if j + 1 <= last:
                    copy(j + 1)
                cur.wait_event(copied[j % 2])
                src = self.raw_buf[j % 2][: pb - pa]
            else:
                src = raw[self.offsets[j]: self.offsets[j + 1]]
            # owners finished staging the previous chunk out of their receive buffers
            self.symm.barrier(channel=0)
            if pb > pa:
                # slab s's rows of my part land in rank s's buffer at the part's angle offset in the chunk
                dst = (ctypes.c_void_p * self.world)(*[self._ptrs[s] + (pa - ca) * self._ks[s] * n_chan * 4
                                                       for s in range(self.world)])
                check(lib().tf_filter_peers(self.local.fplan.handle, ctypes.c_void_p(src.data_ptr()),
                                            (pb - pa) * p.n_rows, self.local.i0, p.n_rows, self.world, self._row0,
                                            dst, self._s()))
            if host:
                ev = torch.cuda.Event()
                ev.record(cur)
                free_ev[j % 2] = ev
            self.symm.barrier(channel=0)  # every rank's stores into my buffer have landed
            n = cb - ca
            self.local.stage_rows(self.recv[: n * k * n_chan].view(n, k, n_chan), rows_per_angle=k, r0=0,
                                  a0=0, a1=n, t_bound=self.bound)
            flags = (_lib.TF_BP_ACCUMULATE if j else 0) | (_lib.TF_BP_FINALIZE if j == last else 0)
            self.local.backproject(ca, cb, flags=flags, taps_a0=ca, taps_a1=cb)
        return self.local.vol

    def updates(self) -> int:
        return self.local.updates()
