"""One small run for compute-sanitizer (scripts/gpu_sanitize.sh):
  san_case.py cold CFG [NFRAMES] [MODE]   -- cold batch run
  san_case.py badinit                     -- c1 warm start with out-of-range labels (expects SEEDS_ESTATE)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1309_3848_b200 import configs  # noqa: E402
from paper_1309_3848_b200.seeds import Seeds, SeedsError  # noqa: E402

what = sys.argv[1]
cfg = sys.argv[2] if len(sys.argv) > 2 else "c1"
nf = int(sys.argv[3]) if len(sys.argv) > 3 else 1
mode = sys.argv[4] if len(sys.argv) > 4 else "grid"
f = configs.frames(cfg if what == "cold" else "c1", n=nf)
p = configs.params(cfg if what == "cold" else "c1")
n, H, W, C = f.shape
s = Seeds(W, H, C, *[p[k] for k in ("n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior",
                                    "iters_per_level")])
s.set_mode(mode)
d = torch.from_numpy(f).cuda()
lab = s.batch(d)
if what == "badinit":
    bad = lab.clone()
    bad[0, 5, 5] = 100000
    bad[0, 6, 6] = -3
    s.batch(d, init_labels=bad)
    try:
        s.sync()
        print("NO ERROR RAISED")
        sys.exit(1)
    except SeedsError as e:
        print("flagged:", e)
torch.cuda.synchronize()
print("ok", what, cfg, nf, mode, s.info.grid_ctas, s.info.grid_tiles)
