"""Time the LAB pre-pass alone (seeds_rgb_to_lab, reading M3) on the c5 frame:
6 B/px of algorithmic traffic (3 in, 3 out) against the HBM peak."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1309_3848_b200 import configs  # noqa: E402
from paper_1309_3848_b200.seeds import Seeds  # noqa: E402

pk = os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")
hbm = json.load(open(pk))["hbm_gbs"] if os.path.exists(pk) else 6650.0
img = torch.from_numpy(configs.frames("c5", n=1)[0]).cuda()
s = Seeds(64, 64, 3, 4, 1, 4, 0, 1)
out = s.rgb_to_lab(img)
for _ in range(3):
    s.rgb_to_lab(img)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20
e0.record()
for _ in range(n):
    s._lib.seeds_rgb_to_lab(s._ctx, img.data_ptr(), img.numel() // 3, out.data_ptr(), None)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
px = img.numel() // 3
print(json.dumps({"kernel": "k_rgb2lab", "pixels": px, "ms": ms, "gbs": 6 * px / ms / 1e6,
                  "hbm_frac": 6 * px / ms / 1e6 / hbm}))
