"""Host logic of the row-band exchange (paper_1309_3848_b200/bands.py) with
world_size 2 and 3 over gloo on CPU: every rank receives the concatenation of
every rank's records (its own included, counts differing per rank) and the
neighbours' edge rows land in the right halo buffers."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1309_3848_b200.bands import DistExchange
        ex = DistExchange()
        rb, cap = 16, 8
        n = rank + 1  # rank r emits r + 1 records
        rec = torch.zeros(cap * rb, dtype=torch.uint8)
        for i in range(n):
            rec[i * rb:(i + 1) * rb] = rank * 16 + i
        allrec, nall = ex.records(rec, torch.tensor([n], dtype=torch.int32), rb)
        W = 5
        top = torch.full((2 * W,), 100 + rank, dtype=torch.int16)
        bot = torch.full((2 * W,), 200 + rank, dtype=torch.int16)
        tr = torch.full((2 * W,), -1, dtype=torch.int16)
        br = torch.full((2 * W,), -1, dtype=torch.int16)
        ex.halo(top, bot, tr, br)
        q.put((rank, int(nall.item()), allrec.view(-1, rb)[:, 0].tolist(), int(tr[0]), int(br[0])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_records_and_halos(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [rk * 16 + i for rk in range(world) for i in range(rk + 1)]
    for rank in range(world):
        _, nall, first_bytes, tr, br = res[rank]
        assert nall == sum(range(1, world + 1))
        assert first_bytes == want
        assert tr == (200 + rank - 1 if rank > 0 else -1)       # bottom rows of the band above
        assert br == (100 + rank + 1 if rank + 1 < world else -1)  # top rows of the band below
