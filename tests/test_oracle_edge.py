"""Pins of the oracle's edge prior (
reading M6 in DESIGN.md): at the pixel level a pixel whose differently labelled
4-neighbour lies across a colour edge (channel L1 difference > tau) does not
move.  Whole pixel sub-sweeps are predicted from the definitions (histograms
recounted with numpy, Prop. 1 / Prop. 2 through their pinned forms, the edge
test written out here), plus special cases.  No GPU needed."""
import numpy as np
import pytest

from paper_1309_3848_b200 import configs, mosaic

RING = [(0, -1), (1, -1), (1, 0), (1, 1), (0, 1), (-1, 1), (-1, 0), (-1, -1)]


def frozen(img, lab, x, y, tau):
    H, W = lab.shape
    for dx, dy in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        qx, qy = x + dx, y + dy
        if 0 <= qx < W and 0 <= qy < H and lab[qy, qx] != lab[y, x]:
            if np.abs(img[y, x].astype(int) - img[qy, qx].astype(int)).sum() > tau:
                return True
    return False


def predict(orc, img, lab, bins, B, colour, P, gamma, tau):
    H, W = lab.shape
    K = int(lab.max()) + 1
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
            if not cand or not orc.removable(m) or frozen(img, lab, x, y, tau):
                continue
            l = np.zeros(B, np.int64)
            l[bins[y, x]] = 1
            for n in cand:
                if not orc.colour_test(hist[n], hist[k], l, int(A[n]), int(A[k]), 1):
                    continue
                if gamma and orc.smooth_sum(lab, x, y, k, n) < 0:
                    continue
                out[y, x] = n
                break
    return out


@pytest.mark.parametrize("gamma,tau", [(0, 40), (1, 60), (0, 25)])
def test_edge_subsweeps_brute_force(orc, gamma, tau):
    img = mosaic.mosaic(40, 30, 6, sigma=12.0, seed=33, grad=20.0)
    p = dict(n_superpixels=12, n_levels=1, bins_per_channel=4, smoothness_prior=gamma, iters_per_level=2)
    nx, ny, Le = orc.geometry(40, 30, 12, 1)
    B, P = 4 ** 3, 3 if gamma else 2
    bins = orc.quantise(img, 4)
    s0 = 4 * Le * 2
    prev = orc.run(img, **p, edge_tau=tau, max_subsweeps=s0).labels
    moved = 0
    for i in range(2 * P * P):
        nxt = orc.run(img, **p, edge_tau=tau, max_subsweeps=s0 + i + 1).labels
        np.testing.assert_array_equal(nxt, predict(orc, img, prev, bins, B, i % (P * P), P, gamma, tau),
                                      err_msg=f"pixel sub-sweep {i}")
        moved += int((nxt != prev).sum())
        prev = nxt
    assert moved > 0


def test_edge_prior_limits(orc):
    """tau above any colour difference (3 x 255) finds no edge: the plain run;
    tau = 0 is off."""
    img = configs.frames("c1")[0]
    p = configs.params("c1")
    plain = orc.run(img, **p).labels
    np.testing.assert_array_equal(orc.run(img, **p, edge_tau=3 * 255).labels, plain)
    np.testing.assert_array_equal(orc.run(img, **p, edge_tau=0).labels, plain)


def test_edge_prior_freezes_pixels(orc):
    """On the noisy c2 mosaic a low threshold puts most boundaries on "edges":
    the prior removes pixel moves (and never block moves)."""
    img = configs.frames("c2")[0]
    p = configs.params("c2")
    a, b = orc.run(img, **p), orc.run(img, **p, edge_tau=20)
    px = lambda r: sum(t["moves"] for t in r.trace if t["level"] == -1)
    blk = lambda r: [t["moves"] for t in r.trace if t["level"] >= 0]
    assert px(b) < px(a) / 4
    assert blk(a) == blk(b)
