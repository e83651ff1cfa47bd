"""Multi-process (gloo, CPU) checks of the z-slab exchange host logic used by
paper_2505_13955_b200.distributed on NCCL: split sizes, the slab-major send
layout K1 writes, and the angle-ordered landing layout owners stage from."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _full(n_proj, n_rows, n_chan):
    a = torch.arange(n_proj, dtype=torch.float32)[:, None, None] * 1e4
    r = torch.arange(n_rows, dtype=torch.float32)[None, :, None] * 1e2
    c = torch.arange(n_chan, dtype=torch.float32)[None, None, :]
    return a + r + c


def _worker(rank, world, port, shape, q, zb=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_13955_b200.distributed import exchange, exchange_layout, slab_major, zblocked

        n_proj, n_rows, n_chan = shape
        full = _full(*shape)
        slabs, chunks, row0, base, ins, outs = exchange_layout(world, rank, *shape, zblocked=zb)
        a0, a1 = chunks[rank]
        r0, r1 = slabs[rank]
        if zb:  # K1's fused output: one z-blocked staging array per destination slab
            send = torch.cat([zblocked(full[a0:a1, s:e]) for s, e in slabs])
        else:
            send = slab_major(full[a0:a1], slabs)
        assert send.numel() == sum(ins)
        assert base == [sum(ins[:i]) for i in range(world)]
        recv = torch.empty(sum(outs))
        exchange(send, recv, ins, outs)
        want = zblocked(full[:, r0:r1]) if zb else full[:, r0:r1].reshape(-1)
        ok = torch.equal(recv, want)
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape,zb", [(2, (12, 10, 8), False), (3, (7, 11, 5), False),
                                           (2, (1800 // 60, 64, 16), False), (2, (12, 70, 8), True),
                                           (3, (7, 40, 5), True), (8, (30, 20, 6), False)])
def test_row_slab_all_to_all_layout(world, shape, zb):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, q, zb)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res


def test_exchange_layout_bytes():
    from paper_2505_13955_b200.distributed import exchange_layout

    # C3 at 8 GPUs: every rank sends 7/8 of its filtered chunk
    slabs, chunks, row0, base, ins, outs = exchange_layout(8, 3, 1800, 2048, 2048)
    assert chunks[3] == (675, 900) and slabs[3] == (768, 1024)
    assert sum(ins) == 225 * 2048 * 2048
    assert sum(outs) == 1800 * 256 * 2048
    assert row0 == [0, 256, 512, 768, 1024, 1280, 1536, 1792, 2048]


def _chunk_worker(rank, world, port, shape, chunk, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_13955_b200.distributed import chunk_plan, exchange
        from paper_2505_13955_b200.geometry import split_range

        n_proj, n_rows, n_chan = shape
        full = _full(*shape)
        slabs = split_range(n_rows, world)
        r0, r1 = slabs[rank]
        chunks, parts, offsets = chunk_plan(n_proj, world, rank, chunk)
        plans = [chunk_plan(n_proj, world, r, chunk) for r in range(world)]
        raw = torch.cat([full[a:b] for a, b in parts]) if offsets[-1] else full[:0]
        assert raw.shape[0] == offsets[-1]
        ok = True
        for j, ((ca, cb), (pa, pb)) in enumerate(zip(chunks, parts)):
            mine = raw[offsets[j]: offsets[j + 1]]  # this rank's part, as run() slices its input
            send = torch.cat([mine[:, s:e].reshape(-1) for s, e in slabs])
            ins = [(pb - pa) * (e - s) * n_chan for s, e in slabs]
            outs = [(plans[r][1][j][1] - plans[r][1][j][0]) * (r1 - r0) * n_chan for r in range(world)]
            recv = torch.empty(sum(outs))
            exchange(send, recv, ins, outs)
            # rank r's rows land at its part's angle offset in the chunk (run()'s dst pointers)
            for r in range(world):
                qa, qb = plans[r][1][j]
                off = (qa - ca) * (r1 - r0) * n_chan
                ok &= off == sum(outs[:r])
            ok &= torch.equal(recv, full[ca:cb, r0:r1].reshape(-1))
            ok &= ca % 16 == 0 and all(plans[r][0][j] == (ca, cb) for r in range(world))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape,chunk", [(3, (50, 11, 5), 16), (2, (100, 10, 6), 32), (8, (90, 20, 5), 32)])
def test_chunked_zslab_exchange_plan(world, shape, chunk):
    """ChunkedZSlabReconstructor's host logic (chunk_plan + the receive
    offsets run() uses for K1's peer stores): every owner's receive buffer
    holds exactly the chunk's angles of its rows, angle-ordered, and every
    chunk starts at a multiple of 16 angles."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunk_worker, args=(r, world, port, shape, chunk, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res
