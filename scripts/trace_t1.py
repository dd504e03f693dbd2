"""Chain trace of k_tile1 (tracing build, SEEDS_LIB=scripts/alt_trace.so):
per sub-sweep, mean over CTAs, the steps of thread 0's CTA from the grid
barrier of the previous sub-sweep: replay issued, own work done (phase B), all
warps done (arrival), neighbour flags seen, phase A of the next sub-sweep done,
grid barrier passed.
Usage: [GAMMA=g] [TRACE_S=i,j,...] trace_t1.py [cfg]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1309_3848_b200 import configs  # noqa: E402
from paper_1309_3848_b200.seeds import Seeds  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
img = configs.frames(cfg, n=1)[0]
p = dict(configs.params(cfg))
if os.environ.get("GAMMA") is not None:  # override the smoothness prior (timing experiments)
    p["smoothness_prior"] = int(os.environ["GAMMA"])
s = Seeds(img.shape[1], img.shape[0], img.shape[2], *[p[k] for k in (
    "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
s.set_mode("grid")
s.debug_trace(True)
d = torch.from_numpy(img).cuda()
for _ in range(3):
    s.iterate(d)
torch.cuda.synchronize()
tr = s.debug_trace(True).astype(np.float64)
S = s.info.subsweeps
L, I, P = s.info.levels_eff, p["iters_per_level"], s.info.colour_period
act = tr[:, S, 1] != 0
tr = tr[act]
print(f"{cfg}: CTAs {tr.shape[0]}, S {S}; launch -> prologue done {np.mean(tr[:, 0, 1] - tr[:, 0, 2]):.0f} cycles")
start = tr[:, 0:S, 1]                # grid barrier passed (sub-sweep start)
cur = tr[:, 1:S + 1, :]
steps = [("replay", 3), ("phaseB", 2), ("arrive", 0), ("nbrs", 5), ("phaseA", 4), ("grid", 1)]


def chain(sl):
    prev = start[:, sl]
    out = []
    for nm, k in steps:
        x = cur[:, sl, k] - prev
        ok = (cur[:, sl, k] != 0) & (x >= 0) & (x < 1e6)
        out.append(f"{nm} {np.mean(x[ok]) if ok.any() else float('nan'):5.0f}")
        prev = np.where(ok, cur[:, sl, k], prev)
    return out


groups = [(f"level {l}", 4 * I) for l in range(L - 1, -1, -1)] + [("pixel", P * P * I)]
i = 0
tot = 0.0
for name, n in groups:
    sl = slice(i, i + n)
    sub = (cur[:, sl, 1] - start[:, sl]).mean()
    tot += sub * n
    print(f"{name:>8} x{n:3d}: sub-sweep {sub:6.0f} | " + " ".join(chain(sl)))
    i += n
print(f"total {tot:.0f} cycles = {tot / 1.965e3:.1f} us at 1965 MHz")
if os.environ.get("TRACE_S"):
    for si in (int(v) for v in os.environ["TRACE_S"].split(",")):
        print(f"sub-sweep {si:3d}: {(cur[:, si, 1] - start[:, si]).mean():6.0f} | " + " ".join(chain(slice(si, si + 1))))

# globaltimer stamps (ns, common clock): arrival (6), fence done (7), neighbour
# flags seen (8), grid counter seen (9)
g = tr[:, 1:S + 1, :]
if (g[:, :, 6] != 0).any():
    arr = g[:, :, 6]
    print("globaltimer (ns), mean over sub-sweeps:")
    print(f"  arrival skew (max - min over CTAs) {np.mean(arr.max(0) - arr.min(0)):7.0f}")
    print(f"  fence: {np.mean(g[:, :, 7] - arr):7.0f}")
    lastarr = arr.max(0)
    ok = g[:, :-1, 8] != 0
    print(f"  neighbour flags seen - own arrival {np.mean((g[:, :-1, 8] - arr[:, :-1])[ok]):7.0f}, - last arrival {np.mean((g[:, :-1, 8] - lastarr[None, :-1])[ok]):7.0f}")
    print(f"  grid seen - last arrival {np.mean(g[:, :, 9] - lastarr[None, :]):7.0f} (min {np.min(g[:, :, 9] - lastarr[None, :]):.0f})")
    for si in (0, 48, 64, 99):
        print(f"  sub-sweep {si}: skew {arr[:, si].max() - arr[:, si].min():.0f}, fence mean {np.mean(g[:, si, 7] - arr[:, si]):.0f} max {np.max(g[:, si, 7] - arr[:, si]):.0f}")
