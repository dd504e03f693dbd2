"""Time the seed alone: runs with iters_per_level = 0 (quantise, grid labels,
histograms, emit) of a config, CUDA events, median of 20.  usage: seed_time.py cfg [frames]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1309_3848_b200 import configs  # noqa: E402
from paper_1309_3848_b200.seeds import Seeds  # noqa: E402

cfg = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
f = configs.frames(cfg, n=n) if n else configs.frames(cfg, n=1)
p = configs.params(cfg)
s = Seeds(f.shape[2], f.shape[1], f.shape[3], p["n_superpixels"], p["n_levels"], p["bins_per_channel"],
          p["smoothness_prior"], 0)
d = torch.from_numpy(f).cuda()
for _ in range(3):
    s.batch(d)
ts = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s.batch(d)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
print(f"{cfg} x{f.shape[0]} seed+emit (I=0): median {ts[10] * 1e3:.1f} us  min {ts[0] * 1e3:.1f} us  lib {os.environ.get('SEEDS_LIB', 'in-tree')}")
