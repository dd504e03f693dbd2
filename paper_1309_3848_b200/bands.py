"""Row-band runs of one large frame over several GPUs (include/seeds.h,
"Row-band mode"): bootstrap plumbing only.  The exchange itself -- owner-band
histogram updates and halo label rows written into peer memory, one barrier
per sub-sweep -- happens inside the persistent kernel; this module only gets
every rank the others' CUDA IPC handles:

  * bootstrap="nccl": rank 0 makes an NCCL unique id, torch.distributed
    broadcasts it, the library's own one-off NCCL all-gather exchanges the
    handles (seeds_create_banded with an id);
  * bootstrap="caller": the handle blobs travel over torch.distributed
    (all_gather_object: NCCL or gloo), then seeds_band_connect.
"""
from __future__ import annotations


def exchange_blobs(blob: bytes, group=None) -> list:
    """Every rank's blob, in rank order (torch.distributed, any backend)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, blob, group=group)
    return out


def broadcast_id(idb: bytes | None, group=None) -> bytes:
    """Rank 0's bytes on every rank (torch.distributed, any backend)."""
    import torch.distributed as dist
    obj = [idb]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def make_band(width, height, channels, n_superpixels, n_levels, bins_per_channel, smoothness_prior,
              iters_per_level, group=None, bootstrap="nccl"):
    """This rank's SeedsBand of a world-rank run (one GPU per rank)."""
    import torch.distributed as dist
    from .seeds import SeedsBand, nccl_unique_id
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    args = (width, height, channels, n_superpixels, n_levels, bins_per_channel, smoothness_prior, iters_per_level,
            rank, world)
    if world == 1:
        return SeedsBand(*args)
    if bootstrap == "nccl":
        idb = broadcast_id(nccl_unique_id() if rank == 0 else None, group)
        return SeedsBand(*args, nccl_id=idb)
    band = SeedsBand(*args)
    band.connect(exchange_blobs(band.export(), group))
    return band
