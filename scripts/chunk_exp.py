"""Experiment (not product code): c3 batch as one launch vs L2-sized chunks."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1309_3848_b200 import configs
from paper_1309_3848_b200.seeds import Seeds
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
f = configs.frames(cfg)
p = configs.params(cfg)
d = torch.from_numpy(f).cuda()
n = d.shape[0]
s = Seeds(f.shape[2], f.shape[1], f.shape[3], *[p[k] for k in (
    "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
ref = s.batch(d).clone()
for ch in [n, n // 2, n // 4, n // 8, n // 16]:
    if ch < 1: continue
    outs = []
    for _ in range(2):
        for i in range(0, n, ch): s.batch(d[i:i + ch])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    R = 3
    for _ in range(R):
        for i in range(0, n, ch): outs.append(s.batch(d[i:i + ch]))
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    ok = torch.equal(torch.cat(outs[-(n // ch):]), ref) if n % ch == 0 else None
    print(f"{cfg} chunk {ch}: {ms:.2f} ms per batch, {n * f.shape[1] * f.shape[2] / ms / 1e3:.0f} Mpx/s, same={ok}", flush=True)
