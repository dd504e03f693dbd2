"""Pins of the oracle's compactness prior (PAPER.md:
867-868; reading M5 in DESIGN.md): at the pixel level a move k -> n also needs
the pixel strictly nearer to n's centre of gravity than to k's, the centres
(rounded to the nearest pixel) taken at the start of each pixel iteration.
Whole sub-sweeps are predicted from the definitions: histograms recounted with
numpy, Prop. 1 through the rule pinned in test_oracle_pins.py, Prop. 2 through
the pinned sum, centres recomputed from the labels.  No GPU needed."""
import numpy as np
import pytest
from scipy import ndimage

from paper_1309_3848_b200 import configs, mosaic

RING = [(0, -1), (1, -1), (1, 0), (1, 1), (0, 1), (-1, 1), (-1, 0), (-1, -1)]
FOUR = np.array([[0, 1, 0], [1, 1, 1], [0, 1, 0]])


def centres(lab, K):
    H, W = lab.shape
    ys, xs = np.mgrid[0:H, 0:W]
    A = np.bincount(lab.ravel(), minlength=K).astype(np.int64)
    sx = np.bincount(lab.ravel(), weights=xs.ravel(), minlength=K).astype(np.int64)
    sy = np.bincount(lab.ravel(), weights=ys.ravel(), minlength=K).astype(np.int64)
    a = np.maximum(A, 1)
    return (2 * sx + a) // (2 * a), (2 * sy + a) // (2 * a)


def predict(orc, lab, bins, B, colour, P, gamma, cx, cy):
    H, W = lab.shape
    K = len(cx)
    hist = np.bincount((lab.astype(np.int64) * B + bins).ravel(), minlength=K * B).reshape(K, B)
    A = hist.sum(1)
    out = lab.copy()
    for y in range(H):
        for x in range(W):
            if P * (y % P) + (x % P) != colour:
                continue
            k = int(lab[y, x])
            cand = []
            for dx, dy in ((-1, 0), (1, 0), (0, -1), (0, 1)):
                xx, yy = x + dx, y + dy
                if 0 <= xx < W and 0 <= yy < H and lab[yy, xx] != k and int(lab[yy, xx]) not in cand:
                    cand.append(int(lab[yy, xx]))
            m = sum(1 << r for r, (dx, dy) in enumerate(RING)
                    if 0 <= x + dx < W and 0 <= y + dy < H and lab[y + dy, x + dx] == k)
            if not cand or not orc.removable(m):
                continue
            l = np.zeros(B, np.int64)
            l[bins[y, x]] = 1
            for n in cand:
                if not orc.colour_test(hist[n], hist[k], l, int(A[n]), int(A[k]), 1):
                    continue
                if gamma and orc.smooth_sum(lab, x, y, k, n) < 0:
                    continue
                if not (x - cx[n]) ** 2 + (y - cy[n]) ** 2 < (x - cx[k]) ** 2 + (y - cy[k]) ** 2:
                    continue
                out[y, x] = n
                break
    return out


@pytest.mark.parametrize("gamma,L", [(0, 1), (1, 2), (1, 1)])
def test_compact_subsweeps_brute_force(orc, gamma, L):
    img = mosaic.mosaic(40, 30, 6, sigma=12.0, seed=31, grad=20.0)
    p = dict(n_superpixels=12, n_levels=L, bins_per_channel=4, smoothness_prior=gamma, iters_per_level=2)
    nx, ny, Le = orc.geometry(40, 30, 12, L)
    K, B, P = nx * ny, 4 ** 3, 3 if gamma else 2
    bins = orc.quantise(img, 4)
    s0 = 4 * Le * 2
    moved = 0
    for it in range(2):
        start = orc.run(img, **p, compact=True, max_subsweeps=s0 + it * P * P).labels
        cx, cy = centres(start, K)
        prev = start
        for c in range(P * P):
            nxt = orc.run(img, **p, compact=True, max_subsweeps=s0 + it * P * P + c + 1).labels
            np.testing.assert_array_equal(nxt, predict(orc, prev, bins, B, c, P, gamma, cx, cy),
                                          err_msg=f"iteration {it} colour {c}")
            moved += int((nxt != prev).sum())
            prev = nxt
    assert moved > 0


def test_compact_off_is_the_default(orc):
    img = configs.frames("c1")[0]
    p = configs.params("c1")
    np.testing.assert_array_equal(orc.run(img, **p).labels, orc.run(img, **p, compact=False).labels)


@pytest.mark.parametrize("schedule", [0, 1])
def test_compact_invariants(orc, schedule):
    img = configs.frames("c2")[0]
    p = configs.params("c2")
    r = orc.run(img, **p, compact=True, schedule=schedule)
    K, B = r.k_act, 125
    bins = orc.quantise(img, 5)
    h = np.bincount((r.labels.astype(np.int64) * B + bins).ravel(), minlength=K * B).reshape(K, B)
    np.testing.assert_array_equal(h, r.hist)
    assert (r.sizes > 0).all()
    for k in range(K):
        assert ndimage.label(r.labels == k, structure=FOUR)[1] == 1
    plain = orc.run(img, **p, schedule=schedule)
    px = lambda t: sum(x["moves"] for x in t if x["level"] == -1)
    assert 0 < px(r.trace) < px(plain.trace)  # the prior only removes pixel moves


@pytest.mark.parametrize("gamma", [0, 1])
def test_equal_grid_is_a_fixed_point_without_blocks(orc, gamma):
    """SPH (no block levels) with the prior on a grid of equal cells: every pixel
    is at least as near its own cell's centre as any neighbour's (ties reject),
    so no pixel can move whatever the colours."""
    img = mosaic.mosaic(40, 30, 9, sigma=12.0, seed=5, grad=30.0)   # nx = 4, ny = 3: 10 x 10 cells
    p = dict(n_superpixels=12, n_levels=0, bins_per_channel=4, smoothness_prior=gamma, iters_per_level=3)
    r = orc.run(img, **p, compact=True)
    assert sum(t["moves"] for t in r.trace) == 0
    np.testing.assert_array_equal(r.labels, orc.run(img, **dict(p, iters_per_level=0)).labels)
    if gamma == 0:  # (with gamma = 1 straight seams cannot move at all, reading Q7)
        assert sum(t["moves"] for t in orc.run(img, **p).trace) > 0  # the colours alone would move pixels
