"""Arrival / exit spread of k_tile1's CTAs per sub-sweep (tracing build,
globaltimer stamps: [s][6] barrier passed, [s][7] arrival).  Which CTAs arrive
last, and how much of a sub-sweep is the spread.  Usage: trace_skew.py [cfg]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1309_3848_b200 import configs  # noqa: E402
from paper_1309_3848_b200.seeds import Seeds  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
img = configs.frames(cfg, n=1)[0]
p = configs.params(cfg)
s = Seeds(img.shape[1], img.shape[0], img.shape[2], *[p[k] for k in (
    "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
s.set_mode("grid")
s.debug_trace(True)
d = torch.from_numpy(img).cuda()
runs = []
for r in range(6):
    s.iterate(d)
    torch.cuda.synchronize()
    runs.append(s.debug_trace(True).astype(np.float64))
S = s.info.subsweeps
for tr in runs[-3:]:
    act = tr[:, S, 1] != 0
    t = tr[act]
    ex = t[:, 0:S, 6]  # exit of the previous barrier (start of sub-sweep i); row 0 unset
    ar = t[:, 1:S + 1, 7]
    ex2 = t[:, 1:S + 1, 6]
    ok = slice(1, S)
    chain = ar[:, ok] - ex[:, ok]                       # per CTA: start -> arrival
    sub = ex2[:, ok].max(0) - ex[:, ok].max(0)          # last exit to last exit
    print(f"{cfg}: sub-sweep (last exit to last exit) {sub.mean():.0f} ns; chain start->arrival mean {chain.mean():.0f}, "
          f"max-over-CTAs {chain.max(0).mean():.0f}; exit spread {np.mean(ex[:, ok].max(0) - ex[:, ok].min(0)):.0f}; "
          f"arrival spread {np.mean(ar[:, ok].max(0) - ar[:, ok].min(0)):.0f}; last arrival -> last exit "
          f"{np.mean(ex2[:, ok].max(0) - ar[:, ok].max(0)):.0f}, -> first exit {np.mean(ex2[:, ok].min(0) - ar[:, ok].max(0)):.0f}")
    last = np.argmax(ar, axis=0)
    cnt = np.bincount(last, minlength=t.shape[0])
    top = np.argsort(cnt)[::-1][:8]
    print("  CTAs arriving last most often:", ", ".join(f"{c} ({cnt[c]}x)" for c in top))
    lastx = np.argmax(ex2, axis=0)
    cx = np.bincount(lastx, minlength=t.shape[0])
    print("  CTAs leaving last most often:", ", ".join(f"{c} ({cx[c]}x)" for c in np.argsort(cx)[::-1][:8]))
    # mean chain per CTA, the slowest ones
    mc = chain.mean(1)
    print("  mean chain per CTA: min %.0f median %.0f max %.0f; slowest CTAs %s" % (
        mc.min(), np.median(mc), mc.max(), list(np.argsort(mc)[::-1][:8])))
