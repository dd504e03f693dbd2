"""Per-CTA clock64 trace of one grid-mode run: work and barrier cycles
per sub-sweep (max / min over CTAs), summarised per phase group.
Usage: [NF=frames] trace.py [cfg] [mode] [HxW crop]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1309_3848_b200 import configs  # noqa: E402
from paper_1309_3848_b200.seeds import Seeds  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
mode = sys.argv[2] if len(sys.argv) > 2 else "grid"
NF = int(os.environ.get("NF", "1"))  # frames per run (multi-tile plans)
img = configs.frames(cfg, n=NF)
img = img[0] if NF == 1 else img
if len(sys.argv) > 3:  # crop HxW
    hh, ww = (int(v) for v in sys.argv[3].split("x"))
    img = np.ascontiguousarray(img[..., :hh, :ww, :])
p = configs.params(cfg)
s = Seeds(img.shape[-2], img.shape[-3], img.shape[-1], *[p[k] for k in (
    "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
s.set_mode(mode)
if os.environ.get("MEANS_ITERS"):
    s.set_means_iters(int(os.environ["MEANS_ITERS"]))
s.debug_trace(True)
d = torch.from_numpy(img).cuda()
for _ in range(3):
    out = s.iterate(d) if NF == 1 else s.batch(d)
torch.cuda.synchronize()
tr = s.debug_trace(True)
S = s.info.subsweeps
L, I, P = s.info.levels_eff, p["iters_per_level"], s.info.colour_period
ncta = tr.shape[0]
active = tr[:, S, 1] != 0
tr = tr[active].astype(np.float64)
print(f"{cfg} {mode}: CTAs {ncta} (active {int(active.sum())}), S {S}")
prev1 = tr[:, 0:S, 1]
cur = tr[:, 1:S + 1, :]
work = cur[:, :, 0] - prev1          # (cta, S)
bar = cur[:, :, 1] - cur[:, :, 0]
parts = {"replay": cur[:, :, 2] - prev1, "stage": cur[:, :, 3] - cur[:, :, 2],
         "filter": cur[:, :, 4] - cur[:, :, 3], "decide": cur[:, :, 5] - cur[:, :, 4],
         "tail": cur[:, :, 0] - cur[:, :, 5]}
if (cur[:, :, 6] != 0).any():
    parts.update({"sum.wait": cur[:, :, 6], "sum.filter": cur[:, :, 7], "sum.decide": cur[:, :, 15]})
if (cur[:, :, 8] != 0).any():
    parts.update({"d.pre": cur[:, :, 13], "d.xy": cur[:, :, 14], "d.ring": cur[:, :, 11], "d.bin": cur[:, :, 12], "d.gath": cur[:, :, 8], "d.dec": cur[:, :, 9],
                  "d.emit": cur[:, :, 10]})
have_parts = mode == "grid"
seed = tr[:, 0, 1] - tr[:, 0, 2]
if (tr[:, 0, 2] != 0).all():
    print(f"    seed: max {seed.max():7.0f} mean {seed.mean():7.0f} cycles (launch start to the first barrier passed)")
groups = [(f"level {l}", 4 * I) for l in range(L - 1, -1, -1)] + [("pixel", P * P * I)]
i = 0
for name, n in groups:
    sl = slice(i, i + n)
    w = work[:, sl]
    line = (f"{name:>8}: work max {w.max(0).mean():7.0f} mean {w.mean():7.0f} min {w.min(0).mean():7.0f} | "
            f"barrier min {bar[:, sl].min(0).mean():6.0f} max {bar[:, sl].max(0).mean():6.0f} | "
            f"work+barrier {(w + bar[:, sl]).mean():7.0f}")
    if have_parts:
        line += " | " + " ".join(f"{k} {v[:, sl].mean():5.0f}/{v[:, sl].max(0).mean():5.0f}" for k, v in parts.items())
    print(line)
    i += n
if os.environ.get("TRACE_S"):  # phases of chosen sub-sweeps (mean / max over CTAs)
    for si in (int(v) for v in os.environ["TRACE_S"].split(",")):
        print(f"sub-sweep {si}: work {work[:, si].mean():.0f}/{work[:, si].max():.0f} barrier {bar[:, si].mean():.0f} | "
              + " ".join(f"{k} {v[:, si].mean():.0f}/{v[:, si].max():.0f}" for k, v in parts.items()))
