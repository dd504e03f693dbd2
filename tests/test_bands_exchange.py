"""Host plumbing of the row-band bootstrap (paper_1309_3848_b200/bands.py)
over gloo on CPU, world sizes 2 and 3: every rank receives every rank's blob
in rank order, and rank 0's NCCL id reaches every rank."""
import os
import socket

import pytest
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
        from paper_1309_3848_b200 import bands
        blob = bytes([rank]) * (16 + rank)  # blobs of different contents and sizes
        allb = bands.exchange_blobs(blob)
        idb = bands.broadcast_id(b"id-of-rank-0" if rank == 0 else None)
        q.put((rank, allb, idb))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bootstrap_exchange(world):
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
    want = [bytes([r]) * (16 + r) for r in range(world)]
    for rank in range(world):
        assert res[rank][1] == want
        assert res[rank][2] == b"id-of-rank-0"
