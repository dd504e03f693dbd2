"""Row-band runs of one large frame (include/seeds.h, "Row-band mode"): the
schedule and the exchange between bands.  Plumbing only -- every step of the
refinement runs in the CUDA kernels behind seeds_band_*; this module moves
the sparse delta records and the two-row label halos between bands.

Two exchanges with one interface:
  * DistExchange: one band per rank over torch.distributed (NCCL on GPUs; the
    same code runs on CPU tensors with gloo, which is how tests/ cover it).
  * local_run: every band in this process on one GPU ("virtual ranks"), used
    to check that any number of bands gives the one-GPU result bit for bit.
"""
from __future__ import annotations


class DistExchange:
    """Record all-gather and halo send/recv between the ranks of `group`
    (rank r refines band r).  Tensors may live on CUDA (NCCL) or CPU (gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def records(self, rec_out, n_out, rb=16):
        """Every band's records, concatenated (this band's included): returns
        (uint8 tensor of n * rb bytes, int32 tensor [n]).  The counts go first,
        then every rank sends max(count) records' worth of its buffer."""
        import torch
        dist = self.dist
        counts = [torch.zeros_like(n_out) for _ in range(self.world)]
        dist.all_gather(counts, n_out, group=self.group)
        cnt = [int(c.item()) for c in counts]
        m = max(1, max(cnt))
        send = rec_out[:m * rb].contiguous()
        recv = [torch.empty_like(send) for _ in range(self.world)]
        dist.all_gather(recv, send, group=self.group)
        parts = [recv[r][:cnt[r] * rb] for r in range(self.world)]
        allrec = torch.cat(parts) if sum(cnt) else rec_out[:0]
        return allrec, torch.tensor([sum(cnt)], dtype=torch.int32, device=n_out.device)

    def halo(self, top_send, bottom_send, top_recv, bottom_recv):
        """Send this band's first rows up (to rank - 1) and last rows down (to
        rank + 1); receive the neighbours' into top_recv / bottom_recv."""
        dist = self.dist
        ops = []
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, top_send, self.rank - 1, group=self.group))
            ops.append(dist.P2POp(dist.irecv, top_recv, self.rank - 1, group=self.group))
        if self.rank + 1 < self.world:
            ops.append(dist.P2POp(dist.isend, bottom_send, self.rank + 1, group=self.group))
            ops.append(dist.P2POp(dist.irecv, bottom_recv, self.rank + 1, group=self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()


def dist_run(band, image, labels_out, init_labels=None, exchange=None, stream=None):
    """Refine `image` (the whole frame, on this rank's GPU) as band `band.band`
    of `band.n_bands`; writes this band's rows of labels_out."""
    import torch
    ex = exchange or DistExchange()
    W = band.width
    dev = image.device
    rec_out = torch.empty(band.record_capacity * band.record_bytes, dtype=torch.uint8, device=dev)
    n_out = torch.zeros(1, dtype=torch.int32, device=dev)
    top_s, bot_s, top_r, bot_r = (torch.empty(2 * W, dtype=torch.int16, device=dev) for _ in range(4))
    band.seed(image, init_labels, stream=stream)
    rec_in, n_in = None, None
    for s in range(band.subsweeps):
        band.subsweep(s, rec_in, n_in, rec_out, n_out, stream=stream)
        rec_in, n_in = ex.records(rec_out, n_out, band.record_bytes)
        band.halo(False, top_s, bot_s, stream=stream)
        ex.halo(top_s, bot_s, top_r, bot_r)
        band.halo(True, top_r if band.band > 0 else None, bot_r if band.band + 1 < band.n_bands else None,
                  stream=stream)
    band.finish(rec_in, n_in, labels_out, stream=stream)
    return labels_out


def local_run(bands, image, init_labels=None, stream=None):
    """Every band of a run in this process (one GPU): the same schedule and
    exchange as dist_run, with the ranks' messages replaced by tensor copies."""
    import torch
    W, H = bands[0].width, bands[0].height
    dev = image.device
    labels = torch.empty((H, W), dtype=torch.int32, device=dev)
    outs = [torch.empty(b.record_capacity * b.record_bytes, dtype=torch.uint8, device=dev) for b in bands]
    cnts = [torch.zeros(1, dtype=torch.int32, device=dev) for _ in bands]
    tops = [torch.empty(2 * W, dtype=torch.int16, device=dev) for _ in bands]
    bots = [torch.empty(2 * W, dtype=torch.int16, device=dev) for _ in bands]
    for b in bands:
        b.seed(image, init_labels, stream=stream)
    S = bands[0].subsweeps
    rec_in, n_in = None, None
    for s in range(S):
        for i, b in enumerate(bands):
            b.subsweep(s, rec_in, n_in, outs[i], cnts[i], stream=stream)
        cnt = [int(c.item()) for c in cnts]
        parts = [outs[i][:cnt[i] * bands[i].record_bytes] for i in range(len(bands))]
        rec_in = torch.cat(parts) if sum(cnt) else outs[0][:0]
        n_in = torch.tensor([sum(cnt)], dtype=torch.int32, device=dev)
        for i, b in enumerate(bands):
            b.halo(False, tops[i], bots[i], stream=stream)
        for i, b in enumerate(bands):
            b.halo(True, bots[i - 1] if i > 0 else None, tops[i + 1] if i + 1 < len(bands) else None,
                   stream=stream)
    for b in bands:
        b.finish(rec_in, n_in, labels, stream=stream)
    return labels
