"""k_tile1 prologue phases (tracing build, SEEDS_LIB=scripts/alt_trace.so):
row 0 stamps 2 launch, 3 seed pass done, 4 first barrier passed, 5 flush done,
6 item build done, 1 second barrier passed -- mean / max over CTAs, cycles."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1309_3848_b200 import configs  # noqa: E402
from paper_1309_3848_b200.seeds import Seeds  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
img = configs.frames(cfg)[0]
p = configs.params(cfg)
s = Seeds(img.shape[1], img.shape[0], img.shape[2], *[p[k] for k in (
    "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
s.debug_trace(True)
d = torch.from_numpy(img).cuda()
for _ in range(3):
    s.iterate(d)
torch.cuda.synchronize()
tr = s.debug_trace(True).astype(np.float64)
r0 = tr[:, 0, :]
act = r0[:, 2] != 0
r0 = r0[act]
names = [(2, 3, "blob + seed pass"), (3, 4, "barrier 1"), (4, 5, "flush + zero"), (5, 6, "item build"), (6, 1, "barrier 2")]
for a, b, n in names:
    v = r0[:, b] - r0[:, a]
    print(f"{n:18s} mean {v.mean():8.0f} max {v.max():8.0f} min {v.min():8.0f}")
print(f"{'total':18s} mean {(r0[:, 1] - r0[:, 2]).mean():8.0f}")
# per level of the item build (stamps 7 + l at each level's start, thread 0's view)
L = s.info.levels_eff
pts = [5] + [7 + l for l in range(L)] + [6]
for a, b in zip(pts[:-1], pts[1:]):
    v = r0[:, b] - r0[:, a]
    print(f"  item build {a}->{b}: mean {v.mean():7.0f} max {v.max():7.0f}")
