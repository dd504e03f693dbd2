"""More pins of the CPU oracle (DESIGN.md
section 2).  No GPU needed.

* EXACT mode (``oracle/exact.py``, SURVEY 8(c) modes list): the hill climbing of
  PAPER.md:437-440 with E recomputed exactly.  Every accepted move raises E by
  exactly the locally computed dE (checked against a full recompute of Eqs. 4-9
  on rationals), the result is valid, no single-pixel move improves it (a
  local-optimality certificate) and it never beats the brute-force argmax.
* Local-optimality certificates of the COL schedule on random tiny images:
  under R1 a converged run is a fixed point of its own rule; under R2 a
  converged pixel-level run is a local maximum of H' = sum h^2 (eq:proof3).
* Whole block and pixel sub-sweeps of plain runs (rule R1, gamma 0 and 1)
  predicted from scratch: histograms recounted with numpy, Proposition 1 as the
  intersection inequality on exact rationals, Proposition 2
  as its sum, the ring rule by flood fill, candidates
  W, E, N, S (reading Q5).
* The R2 block rule (raw-count intersection, eq:proof3 PAPER.md:1010-1013): on
  a block concentrated in one bin (the proposition's assumption,
  PAPER.md:967-968) it accepts only moves that raise H'.
"""
from fractions import Fraction

import numpy as np
import pytest
from scipy import ndimage

from paper_1309_3848_b200 import mosaic

FOUR = np.array([[0, 1, 0], [1, 1, 1], [0, 1, 0]])
RING = [(0, -1), (1, -1), (1, 0), (1, 1), (0, 1), (-1, 1), (-1, 0), (-1, -1)]  # (dx, dy): N NE E SE S SW W NW


def bins_of(img, bpc):
    img = img.astype(np.int64)
    b = np.zeros(img.shape[:2], np.int64)
    for c in range(img.shape[2]):
        b = b * bpc + (img[:, :, c] * bpc) // 256
    return b


def flood_removable(cells):
    """The 3x3 ring rule restated by flood fill: the unit's own-label ring cells
    (a set of (dx, dy)) contain a 4-neighbour, and all of its 4-neighbours stay
    4-connected to each other through the ring (reading Q8)."""
    edges = [c for c in cells if abs(c[0]) + abs(c[1]) == 1]
    if not edges:
        return False
    seen, stack = {edges[0]}, [edges[0]]
    while stack:
        x, y = stack.pop()
        for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
            q = (x + dx, y + dy)
            if q in cells and q not in seen:
                seen.add(q)
                stack.append(q)
    return all(e in seen for e in edges)


def intersection(a, Za, b, Zb):
    """int(c_a, c_b) = sum_j min(c_a(j), c_b(j)) on rationals."""
    return sum((min(Fraction(int(x), Za), Fraction(int(y), Zb)) for x, y in zip(a, b) if y), Fraction(0))


def prop1(hist, A, k, n, l, alpha):
    """Proposition 1, strict (reading Q6): int(c_n, c_l) > int(c_{k minus l}, c_l)."""
    return intersection(hist[n], int(A[n]), l, alpha) > intersection(hist[k] - l, int(A[k]) - alpha, l, alpha)


def smooth_S(lab, x, y, k, n):
    """Proposition 2's sum S = sum_{i in W3(p)} (b_i(n) + 1 - b_i(k)) over the
    in-image patch centres i around p, b_i(x) counted in the clamped 3x3 patch
    of i (reading Q15)."""
    H, W = lab.shape
    S = 0
    for iy in range(y - 1, y + 2):
        for ix in range(x - 1, x + 2):
            if 0 <= ix < W and 0 <= iy < H:
                patch = lab[max(0, iy - 1):iy + 2, max(0, ix - 1):ix + 2]
                S += int((patch == n).sum()) + 1 - int((patch == k).sum())
    return S


def g_raw(lab):
    H, W = lab.shape
    g = 0
    for y in range(H):
        for x in range(W):
            _, c = np.unique(lab[max(0, y - 1):y + 2, max(0, x - 1):x + 2], return_counts=True)
            g += int((c.astype(np.int64) ** 2).sum())
    return g


# ----------------------------------------------------------------------------
# EXACT mode
# ----------------------------------------------------------------------------
def _tiny_cases(orc, n, seed):
    rng = np.random.default_rng(seed)
    for t in range(n):
        W, H = int(rng.integers(4, 7)), int(rng.integers(4, 7))
        C = 1
        bpc = int(rng.integers(2, 5))
        img = rng.integers(0, 256, size=(H, W, C)).astype(np.uint8)
        K = int(rng.integers(2, 5))
        yield img, bpc, K


@pytest.mark.parametrize("gamma", [0, 1])
def test_exact_moves_raise_energy_by_their_delta(orc, gamma):
    """P7(iii): replaying the EXACT climber's log from the grid, every accepted
    move changes E (energy_exact, the whole image on rationals) by exactly its
    logged dE, dE > 0, and every intermediate partition is valid."""
    from oracle import exact
    moves = 0
    for img, bpc, K in _tiny_cases(orc, 25, 40 + gamma):
        H, W, _ = img.shape
        bins = bins_of(img, bpc)
        nx, ny, L = orc.geometry(W, H, K, 2)
        lab, log = exact.exact_climb(bins, nx, ny, L, 2, gamma)
        cur = orc.run(img, K, 2, bpc, gamma, 0).labels.astype(np.int64)  # the grid (I = 0)
        e = exact.energy_exact(cur, bins, gamma)
        for level, pixels, k, n, d in log:
            assert all(cur[p] == k for p in pixels)
            for p in pixels:
                cur[p] = n
            e2 = exact.energy_exact(cur, bins, gamma)
            assert d > 0 and e2 - e == d, (level, pixels, k, n)
            for q in (k, n):
                assert ndimage.label(cur == q, structure=FOUR)[1] == 1
            e = e2
            moves += 1
        np.testing.assert_array_equal(cur, lab)
    assert moves > (20 if gamma == 0 else 0)


@pytest.mark.parametrize("gamma", [0, 1])
def test_exact_local_optimum_certificate(orc, gamma):
    """A converged EXACT run is a local maximum: no valid single-pixel move
    raises E (full recompute), and E(result) >= E(grid)."""
    from oracle import exact
    for img, bpc, K in _tiny_cases(orc, 12, 60 + gamma):
        H, W, _ = img.shape
        bins = bins_of(img, bpc)
        nx, ny, L = orc.geometry(W, H, K, 1)
        lab, log = exact.exact_climb(bins, nx, ny, L, 2, gamma, until_stable=True)
        assert exact.improving_pixel_moves(bins, lab, gamma) == []
        grid = orc.run(img, K, 1, bpc, gamma, 0).labels
        assert exact.energy_exact(lab, bins, gamma) >= exact.energy_exact(grid, bins, gamma)


def test_exact_vs_brute_force(orc):
    """P8: EXACT never beats the global argmax over all valid 2-superpixel
    partitions (Eq. 3) and never ends below the grid; where the grid already
    is the argmax (colour seam on the grid seam) it makes no move.  Its hit
    rate on two-tone straight seams is reported, not gated: with the normalised
    colour term a greedy climber can shrink one superpixel towards a single
    uniform pixel (E -> 1 for it) and stop there (e.g. 4x4, seam at row 3:
    E = 1.609 < 2), a true local optimum (certified above)."""
    from oracle import exact
    rng = np.random.default_rng(3)
    for _ in range(10):
        img = rng.integers(0, 256, size=(4, 4, 1)).astype(np.uint8)
        bins = bins_of(img, 2)
        best, _, _ = exact.brute_force_argmax(bins, 0)
        nx, ny, L = orc.geometry(4, 4, 2, 1)
        lab, _ = exact.exact_climb(bins, nx, ny, L, 4, 0, until_stable=True)
        assert exact.energy_exact(lab, bins, 0) <= best
    hits = total = seams_on_grid = 0
    for W, H in ((4, 4), (5, 4), (4, 5), (5, 3), (3, 5), (6, 3)):
        nx, ny, L = orc.geometry(W, H, 2, 1)
        horizontal = ny == 2
        for r in range(1, H if horizontal else W):
            for top, bot in ((30, 200), (200, 30)):
                img = np.full((H, W, 1), bot, np.uint8)
                if horizontal:
                    img[:r] = top
                else:
                    img[:, :r] = top
                bins = bins_of(img, 2)
                best, arg, _ = exact.brute_force_argmax(bins, 0)
                lab, log = exact.exact_climb(bins, nx, ny, L, 4, 0, until_stable=True)
                e = exact.energy_exact(lab, bins, 0)
                grid = orc.run(img, 2, 1, 2, 0, 0).labels
                eg = exact.energy_exact(grid, bins, 0)
                assert eg <= e <= best
                if eg == best:
                    assert log == []
                    seams_on_grid += 1
                lab = lab if lab[0, 0] == 0 else 1 - lab
                hits += any(np.array_equal(lab, a) for a in arg)
                total += 1
    print(f"EXACT climber reaches the brute-force argmax on {hits}/{total} two-tone seams")
    assert total >= 30 and seams_on_grid >= 4 and hits >= seams_on_grid


# ----------------------------------------------------------------------------
# Local-optimality certificates of the coloured schedule (the P8 report)
# ----------------------------------------------------------------------------
def _ring_cells(lab, x, y, k):
    H, W = lab.shape
    return {(dx, dy) for dx, dy in RING if 0 <= x + dx < W and 0 <= y + dy < H and lab[y + dy, x + dx] == k}


def _pixel_proposals(lab):
    """(x, y, k, [candidates]) for every ring-valid boundary pixel."""
    H, W = lab.shape
    for y in range(H):
        for x in range(W):
            k = int(lab[y, x])
            cand = []
            for dx, dy in ((-1, 0), (1, 0), (0, -1), (0, 1)):
                xx, yy = x + dx, y + dy
                if 0 <= xx < W and 0 <= yy < H and lab[yy, xx] != k and int(lab[yy, xx]) not in cand:
                    cand.append(int(lab[yy, xx]))
            if cand and flood_removable(_ring_cells(lab, x, y, k)):
                yield x, y, k, cand


def test_col_r1_converged_is_a_fixed_point(orc):
    """R1 / COL run until its last pixel iteration moves nothing: no ring-valid
    single-pixel proposal passes Proposition 1 (exact rationals) -- the result
    is a local optimum of the rule that produced it."""
    rng = np.random.default_rng(2)
    checked = 0
    for t in range(20):
        img = rng.integers(0, 256, size=(6, 6, 1)).astype(np.uint8)
        bins = bins_of(img, 3)
        r = orc.run(img, 2, 1, 3, 0, 40)
        if r.trace[-1]["moves"] or sum(x["moves"] for x in r.trace if x["level"] == -1 and x["iter"] == 39):
            continue
        K, B = r.k_act, 3
        hist = np.bincount((r.labels.astype(np.int64) * B + bins).ravel(), minlength=K * B).reshape(K, B)
        A = hist.sum(1)
        for x, y, k, cand in _pixel_proposals(r.labels):
            l = np.zeros(B, np.int64)
            l[bins[y, x]] = 1
            assert not any(prop1(hist, A, k, n, l, 1) for n in cand), (t, x, y)
        checked += 1
    assert checked >= 15


def test_col_r2_converged_is_a_local_maximum_of_hprime(orc):
    """R2 / COL on the pixel level (n_levels = 0, gamma = 0) until no move: no
    ring-valid single-pixel move raises H' = sum_k sum_b h_k[b]^2 (recomputed),
    H'(result) >= H'(grid) (every R2 pixel sub-sweep raises H', P7(ii)), and
    the normalised H of the result never exceeds the brute-force optimum."""
    from oracle import exact
    rng = np.random.default_rng(12)
    checked = 0
    for t in range(20):
        img = rng.integers(0, 256, size=(4, 4, 1)).astype(np.uint8)
        bins = bins_of(img, 2)
        r = orc.run(img, 2, 0, 2, 0, 40, rule=orc.R2)
        if r.trace[-1]["moves"]:
            continue

        def hp(lab):
            h = np.bincount((lab.astype(np.int64) * 2 + bins).ravel(), minlength=4)
            return int((h ** 2).sum())
        e = hp(r.labels)
        for x, y, k, cand in _pixel_proposals(r.labels):
            for n in cand:
                after = r.labels.copy()
                after[y, x] = n
                assert hp(after) <= e, (t, x, y, n)
        grid = orc.run(img, 2, 0, 2, 0, 0).labels
        assert e >= hp(grid)
        best, _, _ = exact.brute_force_argmax(bins, 0)
        assert exact.energy_exact(r.labels, bins, 0) <= best
        checked += 1
    assert checked >= 15


# ----------------------------------------------------------------------------
# From-scratch predictions of plain R1 sub-sweeps (blocks and pixels)
# ----------------------------------------------------------------------------
def predict_block(lab, bins, B, K, level, colour, rect, GXl, GYl):
    """One block sub-sweep (reading O7: snapshot histograms, colour class
    2 (j mod 2) + (i mod 2)) of level `level` on the pixel label map."""
    hist = np.bincount((lab.astype(np.int64) * B + bins).ravel(), minlength=K * B).reshape(K, B)
    A = hist.sum(1)
    out = lab.copy()

    def blab(i, j):
        if 0 <= i < GXl and 0 <= j < GYl:
            y0, _, x0, _ = rect(level, i, j)
            return int(lab[y0, x0])
        return None
    for j in range(GYl):
        for i in range(GXl):
            if 2 * (j % 2) + (i % 2) != colour:
                continue
            y0, y1, x0, x1 = rect(level, i, j)
            k = int(lab[y0, x0])
            assert (lab[y0:y1, x0:x1] == k).all()  # one label per block during its level
            cand = []
            for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
                v = blab(i + di, j + dj)
                if v is not None and v != k and v not in cand:
                    cand.append(v)
            cells = {(dx, dy) for dx, dy in RING if blab(i + dx, j + dy) == k}
            if not cand or not flood_removable(cells):
                continue
            l = np.bincount(bins[y0:y1, x0:x1].ravel(), minlength=B).astype(np.int64)
            alpha = int(l.sum())
            for n in cand:
                if prop1(hist, A, k, n, l, alpha):
                    out[y0:y1, x0:x1] = n
                    break
    return out


def predict_pixel(lab, bins, B, K, colour, P, gamma):
    hist = np.bincount((lab.astype(np.int64) * B + bins).ravel(), minlength=K * B).reshape(K, B)
    A = hist.sum(1)
    out = lab.copy()
    for x, y, k, cand in _pixel_proposals(lab):
        if P * (y % P) + (x % P) != colour:
            continue
        l = np.zeros(B, np.int64)
        l[bins[y, x]] = 1
        for n in cand:
            if prop1(hist, A, k, n, l, 1) and (not gamma or smooth_S(lab, x, y, k, n) >= 0):
                out[y, x] = n
                break
    return out


@pytest.mark.parametrize("gamma,L,seed", [(0, 2, 31), (1, 2, 32), (1, 3, 33)])
def test_plain_subsweeps_predicted_from_scratch(orc, gamma, L, seed):
    """Every block and pixel sub-sweep of a plain R1 / COL run on a small mosaic
    equals the prediction from the labels before it (the oracle's
    max_subsweeps gives the labels after each sub-sweep)."""
    from oracle import exact
    W, H, Kreq, bpc, I = 48, 36, 12, 4, 2
    img = mosaic.mosaic(W, H, 7, sigma=14.0, seed=seed, grad=25.0)
    p = dict(n_superpixels=Kreq, n_levels=L, bins_per_channel=bpc, smoothness_prior=gamma, iters_per_level=I)
    nx, ny, Le = orc.geometry(W, H, Kreq, L)
    K, B, P = nx * ny, bpc ** 3, 3 if gamma else 2
    bins = bins_of(img, bpc)
    GX, GY, rect = exact.grid_blocks(W, H, nx, ny, Le)
    s = 0
    prev = orc.run(img, **p, max_subsweeps=0).labels
    moved_blocks = moved_pixels = 0
    for level in range(Le - 1, -1, -1):
        for it in range(I):
            for c in range(4):
                nxt = orc.run(img, **p, max_subsweeps=s + 1).labels
                want = predict_block(prev, bins, B, K, level, c, rect, GX >> level, GY >> level)
                np.testing.assert_array_equal(nxt, want, err_msg=f"level {level} iteration {it} colour {c}")
                moved_blocks += int((nxt != prev).any())
                prev, s = nxt, s + 1
    for it in range(I):
        for c in range(P * P):
            nxt = orc.run(img, **p, max_subsweeps=s + 1).labels
            want = predict_pixel(prev, bins, B, K, c, P, gamma)
            np.testing.assert_array_equal(nxt, want, err_msg=f"pixel iteration {it} colour {c}")
            moved_pixels += int((nxt != prev).sum())
            prev, s = nxt, s + 1
    full = orc.run(img, **p)
    np.testing.assert_array_equal(prev, full.labels)
    assert moved_blocks > 4 and moved_pixels > 0


# ----------------------------------------------------------------------------
# The R2 block rule (test switch; Q18)
# ----------------------------------------------------------------------------
def test_r2_block_single_bin_accepts_only_hprime_increases(orc):
    """eq:proof3 under the proposition's single-bin
    assumption: a block of alpha pixels all in bin j.  R2 (raw-count
    intersections, sum_b min(h_n, l) > sum_b min(h_k - l, l)) accepts only
    moves with dH' = 2 alpha (h_n[j] - (h_k[j] - alpha)) > 0, and accepts every
    such move whose counts are below alpha (no min clipping)."""
    rng = np.random.default_rng(21)
    acc = 0
    for _ in range(3000):
        B = int(rng.integers(1, 7))
        j = int(rng.integers(0, B))
        alpha = int(rng.integers(1, 9))
        l = np.zeros(B, np.int64)
        l[j] = alpha
        hk = rng.integers(0, 2 * alpha + 2, size=B)
        hk[j] += alpha
        hn = rng.integers(0, 2 * alpha + 2, size=B)
        if hn.sum() == 0:
            hn[0] = 1
        if hk.sum() == alpha:
            hk[(j + 1) % B] += 1
            if B == 1:
                hk[j] += 1
        before = int((hn ** 2).sum() + (hk ** 2).sum())
        after = int(((hn + l) ** 2).sum() + ((hk - l) ** 2).sum())
        got = orc.colour_test(hn, hk, l, int(hn.sum()), int(hk.sum()), alpha, rule=orc.R2, force_block=True)
        if got:
            assert after > before
            acc += 1
        if hn[j] < alpha and hk[j] - alpha < alpha:
            assert got == (after > before)
    assert acc > 300


def test_r2_block_equals_raw_intersections(orc):
    """R2 on general blocks is the unnormalised intersection inequality
    int(h_n, l) > int(h_k - l, l), both sides counted pixel by pixel: a block
    pixel in bin b is matched to one of n's (k's other) pixels of bin b while
    any are left."""
    rng = np.random.default_rng(22)
    for _ in range(1500):
        B = int(rng.integers(1, 8))
        l = rng.integers(0, 4, size=B)
        if l.sum() == 0:
            l[0] = 1
        hk = l + rng.integers(0, 5, size=B)
        if hk.sum() == l.sum():
            hk[-1] += 1
        hn = rng.integers(0, 5, size=B)
        if hn.sum() == 0:
            hn[0] = 1

        def matched(h):  # greedy pixel matching per bin
            m = 0
            for b in range(B):
                left = int(h[b])
                for _ in range(int(l[b])):
                    if left:
                        left -= 1
                        m += 1
            return m
        want = matched(hn) > matched(hk - l)
        got = orc.colour_test(hn, hk, l, int(hn.sum()), int(hk.sum()), int(l.sum()), rule=orc.R2, force_block=True)
        assert got == want
