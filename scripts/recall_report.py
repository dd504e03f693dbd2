"""P15 report: boundary recall (epsilon = 1) of the c4 video's labels against
the moving mosaic's region edges (the synthetic ground truth), for frame t of
clip 0 refined cold and warm-started from frame t-1's labels (reading O9),
and the final H.  Runs the CPU oracle (whose labels the GPU reproduces bit for
bit); writes profiles/r01/c4_recall.json."""
import json
import os
import sys

import numpy as np
from scipy import ndimage

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1309_3848_b200 import configs, mosaic  # noqa: E402


def edges(lab):
    e = np.zeros(lab.shape, bool)
    e[:, :-1] |= lab[:, 1:] != lab[:, :-1]
    e[:-1, :] |= lab[1:, :] != lab[:-1, :]
    return e


def recall(gt, lab, eps=1):
    g = edges(gt)
    s = ndimage.maximum_filter(edges(lab).astype(np.uint8), size=2 * eps + 1).astype(bool)
    return float((g & s).sum() / max(1, g.sum()))


c = configs.CONFIGS["c4"]
p = configs.params("c4")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
frames, regions = mosaic.moving_mosaic(n, c["W"], c["H"], c["R"], c["sigma"], seed=1000 * c["index"],
                                       grad=c["grad"], C=c["C"])
out = []
prev = None
for t in range(n):
    cold = oracle.run(frames[t], **p)
    warm = oracle.run(frames[t], **p, init_labels=prev) if prev is not None else cold
    rc, rw = recall(regions[t], cold.labels), recall(regions[t], warm.labels)
    Hc = oracle.energy(cold.labels, frames[t], p["bins_per_channel"], cold.k_act)[0]
    Hw = oracle.energy(warm.labels, frames[t], p["bins_per_channel"], warm.k_act)[0]
    out.append({"t": t, "recall_cold": rc, "recall_warm": rw, "H_cold": Hc, "H_warm": Hw})
    print(f"t={t} recall cold {rc:.3f} warm {rw:.3f}  H cold {Hc:.2f} warm {Hw:.2f}")
    prev = warm.labels
with open(os.path.join(ROOT, "profiles", "r01", "c4_recall.json"), "w") as f:
    json.dump({"config": "c4 clip 0 (gamma=0, K=1000, L=5, I=4)", "epsilon": 1, "frames": out}, f, indent=1)
