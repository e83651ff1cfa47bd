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
                                           (3, (7, 40, 5), True)])
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
