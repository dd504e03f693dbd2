"""Per-kernel-class device time of one config (seeds_profile): seed / frame
(k_grid) / emit, averaged over 10 runs.  usage: kinds.py cfg [frames]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1309_3848_b200 import configs  # noqa: E402
from paper_1309_3848_b200.seeds import Seeds  # noqa: E402

cfg = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
f = configs.frames(cfg, n=n)
p = configs.params(cfg)
s = Seeds(f.shape[2], f.shape[1], f.shape[3], *[p[k] for k in (
    "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
d = torch.from_numpy(f).cuda()
for _ in range(3):
    s.batch(d)
s.profile(True)
prof = None
for _ in range(10):
    s.batch(d)
    prof = s.profile_collect()
print(cfg, f"x{n}", " ".join(f"{k} {v[0] / 10 * 1e3:.1f}us/{v[1] // 10}" for k, v in prof.items() if v[1]))
