"""Run one config a few times in one mode (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1309_3848_b200 import configs
from paper_1309_3848_b200.seeds import Seeds
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
mode = sys.argv[2] if len(sys.argv) > 2 else "grid"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
nfr = int(sys.argv[4]) if len(sys.argv) > 4 else 1
imgs = configs.frames(cfg, n=nfr)
p = configs.params(cfg)
n, H, W, C = imgs.shape
s = Seeds(W, H, C, *[p[k] for k in ("n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
s.set_mode(mode)
d = torch.from_numpy(imgs).cuda()
for _ in range(reps):
    out = s.batch(d)
torch.cuda.synchronize()
print("ok", cfg, mode, s.info)
