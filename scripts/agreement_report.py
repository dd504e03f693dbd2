"""P6 report (report only): how often Proposition 1's test (R1,
PAPER.md:553-590) agrees with the sign of the exact change of the normalised
colour energy H = sum_k sum_b (h_kb / A_k)^2 that the proposed
move alone would cause -- over all proposals (removable units with a candidate)
and over the accepted ones, per level, on the COL schedule.  The paper quotes
97% (pixel) and 89% (block) on BSD in LAB.

Runs the CPU oracle (whose labels the GPU reproduces bit for bit) to every
sub-sweep's starting state and evaluates the next colour class's proposals;
writes profiles/r01/prop1_agreement.json.  Usage: agreement_report.py [c1|c2]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1309_3848_b200 import configs  # noqa: E402

RING = [(0, -1), (1, -1), (1, 0), (1, 1), (0, 1), (-1, 1), (-1, 0), (-1, -1)]


def dH(hk, hn, Ak, An, l, a):
    """Exact-in-float64 change of sum_b (h/A)^2 over k and n when l (a pixels) moves k -> n."""
    before = ((hk / Ak) ** 2).sum() + ((hn / An) ** 2).sum()
    after = (((hk - l) / (Ak - a)) ** 2).sum() + (((hn + l) / (An + a)) ** 2).sum()
    return after - before


def proposals(M, x, y, k):
    """W, E, N, S candidates (distinct, != k) and the ring mask of unit (x, y) on map M."""
    h, w = M.shape
    cand = []
    for dx, dy in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        xx, yy = x + dx, y + dy
        if 0 <= xx < w and 0 <= yy < h and M[yy, xx] != k and int(M[yy, xx]) not in cand:
            cand.append(int(M[yy, xx]))
    m = 0
    for r, (dx, dy) in enumerate(RING):
        xx, yy = x + dx, y + dy
        if 0 <= xx < w and 0 <= yy < h and M[yy, xx] == k:
            m |= 1 << r
    return cand, m


def main(cfg):
    img = configs.frames(cfg, 1)[0]
    p = configs.params(cfg)
    H, W = img.shape[:2]
    nx, ny, L = oracle.geometry(W, H, p["n_superpixels"], p["n_levels"])
    GX, GY = nx << L, ny << L
    x0 = [(i * W) // GX for i in range(GX + 1)]
    y0 = [(j * H) // GY for j in range(GY + 1)]
    B = p["bins_per_channel"] ** img.shape[2]
    bins = oracle.quantise(img, p["bins_per_channel"])
    I, P = p["iters_per_level"], 3 if p["smoothness_prior"] else 2
    stats = {}
    s = 0
    sched = [(l, c) for l in range(L - 1, -1, -1) for _ in range(I) for c in range(4)] + \
            [(-1, c) for _ in range(I) for c in range(P * P)]
    for level, colour in sched:
        r = oracle.run(img, **p, max_subsweeps=s)
        lab, K = r.labels, r.k_act
        hist = r.hist.astype(np.float64)
        A = r.sizes.astype(np.float64)
        st = stats.setdefault(level, {"proposals": 0, "agree": 0, "accepted": 0, "accepted_increase": 0})
        if level >= 0:
            bw, bh = GX >> level, GY >> level
            M = np.array([[lab[y0[j << level], x0[i << level]] for i in range(bw)] for j in range(bh)])
            units = [(i, j) for j in range(bh) for i in range(bw) if 2 * (j % 2) + (i % 2) == colour]
        else:
            M = lab
            units = [(x, y) for y in range(H) for x in range(W) if P * (y % P) + (x % P) == colour]
        for (ux, uy) in units:
            k = int(M[uy, ux])
            cand, m = proposals(M, ux, uy, k)
            if not cand or not oracle.removable(m):
                continue
            if level >= 0:
                xa, xb = x0[ux << level], x0[(ux + 1) << level]
                ya, yb = y0[uy << level], y0[(uy + 1) << level]
                lb = np.bincount(bins[ya:yb, xa:xb].ravel(), minlength=B).astype(np.float64)
                a = (xb - xa) * (yb - ya)
            else:
                lb = np.zeros(B)
                lb[bins[uy, ux]] = 1
                a = 1
            for n in cand:
                acc = oracle.colour_test(hist[n], hist[k], lb, int(A[n]), int(A[k]), a)
                inc = dH(hist[k], hist[n], A[k], A[n], lb, a) > 0
                st["proposals"] += 1
                st["agree"] += int(acc == inc)
                st["accepted"] += int(acc)
                st["accepted_increase"] += int(acc and inc)
        s += 1
    out = {}
    for level, st in sorted(stats.items()):
        out["pixel" if level < 0 else f"block level {level}"] = dict(
            st, agreement_all=st["agree"] / max(1, st["proposals"]),
            agreement_accepted=st["accepted_increase"] / max(1, st["accepted"]))
    return out


if __name__ == "__main__":
    cfgs = sys.argv[1:] or ["c1", "c2"]
    res = {"_about": "P6: Prop. 1 (R1) decision vs sign of the exact dH of the move alone, COL schedule; paper: "
                     "97% pixel / 89% block on BSD LAB (PAPER.md:796)"}
    for c in cfgs:
        res[c] = main(c)
        print(c, json.dumps({k: (round(v["agreement_all"], 3), round(v["agreement_accepted"], 3), v["proposals"])
                             for k, v in res[c].items()}))
    with open(os.path.join(ROOT, "profiles", "r01", "prop1_agreement.json"), "w") as f:
        json.dump(res, f, indent=1)
