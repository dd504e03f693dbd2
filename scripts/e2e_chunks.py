"""e2e (seeds_batch_host, pinned buffers, copies inside the timed region) of
a batch config for several seeds_set_host_chunks values, CUDA events on the
calling stream.  Usage: e2e_chunks.py [cfg] [chunks,...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1309_3848_b200 import configs  # noqa: E402
from paper_1309_3848_b200.seeds import Seeds  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
ks = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8,16").split(",")]
f = configs.frames(cfg)
p = configs.params(cfg)
s = Seeds(f.shape[2], f.shape[1], f.shape[3], *[p[k] for k in (
    "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
h = torch.from_numpy(f).pin_memory()
o = torch.empty(f.shape[:3], dtype=torch.int32).pin_memory()
st = torch.cuda.current_stream()
ref = None
for k in ks:
    s.set_host_chunks(k)
    for _ in range(2):
        s.batch_host(h.numpy(), o.numpy(), stream=st)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    n = 5
    torch.cuda.synchronize()
    ev[0].record(st)
    for _ in range(n):
        s.batch_host(h.numpy(), o.numpy(), stream=st)
    ev[1].record(st)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / n
    if ref is None:
        ref = o.clone()
    assert torch.equal(ref, o), "chunked results differ"
    print(f"{cfg} chunks {k:2d}: {ms:7.2f} ms per batch, e2e {f.shape[0] * f.shape[1] * f.shape[2] / ms / 1e3:7.1f} Mpx/s")
