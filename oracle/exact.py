"""Tiny exact oracle pieces (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

* ``energy_exact``: E = H + gamma G with ``fractions.Fraction`` (Eqs. 4-9,
  PAPER.md:289-419; Z = |A_k| for c, Z = patch size for b,
  reading Q2).
* ``enumerate_two_label``: every labelling of a tiny image into 2 non-empty
  4-connected superpixels (the valid set S of PAPER.md:261-266), by
  bit-parallel flood fill over all 2^N masks.
* ``brute_force_argmax``: s* = argmax_{s in S} E(s) (Eq. 3).
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np


def energy_exact(labels: np.ndarray, bins: np.ndarray, gamma: int = 0):
    labels = np.asarray(labels)
    bins = np.asarray(bins)
    H, W = labels.shape
    hsum = Fraction(0)
    for k in np.unique(labels):
        sel = bins[labels == k]
        A = sel.size
        _, cnt = np.unique(sel, return_counts=True)
        hsum += sum(Fraction(int(c), A) ** 2 for c in cnt)
    if not gamma:
        return hsum
    g = Fraction(0)
    for y in range(H):
        for x in range(W):
            patch = labels[max(0, y - 1):y + 2, max(0, x - 1):x + 2]
            _, cnt = np.unique(patch, return_counts=True)
            g += sum(Fraction(int(c), patch.size) ** 2 for c in cnt)
    return hsum + gamma * g


def _connected(masks: np.ndarray, W: int, H: int) -> np.ndarray:
    """4-connectivity of the set bits of each mask (uint64 arrays, bit y*W+x)."""
    N = W * H
    full = np.uint64((1 << N) - 1)
    notleft = np.uint64(sum(1 << (y * W + x) for y in range(H) for x in range(W) if x > 0))
    notright = np.uint64(sum(1 << (y * W + x) for y in range(H) for x in range(W) if x < W - 1))
    seed = masks & (~masks + np.uint64(1))  # lowest set bit
    comp = seed
    while True:
        grow = comp | ((comp << np.uint64(1)) & notleft) | ((comp >> np.uint64(1)) & notright) \
            | ((comp << np.uint64(W)) & full) | (comp >> np.uint64(W))
        grow &= masks
        if np.array_equal(grow, comp):
            return comp == masks
        comp = grow


def enumerate_two_label(W: int, H: int) -> np.ndarray:
    """All valid 2-superpixel labellings as (M, H, W) uint8 arrays with pixel 0 in label 0."""
    N = W * H
    assert N <= 24
    full = (1 << N) - 1
    m = np.arange(1, 1 << N, dtype=np.uint64)
    m = m[(m & np.uint64(1)) == 0]  # pixel 0 not in the set -> labelled 0 (label swap removed)
    comp = (~m) & np.uint64(full)
    ok = _connected(m, W, H) & _connected(comp, W, H)
    good = m[ok]
    bits = ((good[:, None] >> np.arange(N, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(np.uint8)
    return bits.reshape(-1, H, W)


def brute_force_argmax(bins: np.ndarray, gamma: int = 0):
    """(best energy, list of argmax labellings) over all valid 2-label partitions."""
    H, W = bins.shape
    labs = enumerate_two_label(W, H)
    best, arg = None, []
    for lab in labs:
        e = energy_exact(lab, bins, gamma)
        if best is None or e > best:
            best, arg = e, [lab]
        elif e == best:
            arg.append(lab)
    return best, arg, len(labs)


# ----------------------------------------------------------------------------
# EXACT mode (SURVEY.md 8(c) modes list): the hill climbing of PAPER.md:437-440
# ("if the energy function of the proposed partitioning increases, the solution
# is updated") with the energy recomputed exactly instead of Proposition 1/2.
# Same proposals as the paper's S5.2: blocks of the levels
# L_eff-1 .. 0, then pixels, each unit proposing the labels of its 4-neighbour
# units (W, E, N, S; reading Q5) and taking the first proposal that keeps the
# partition valid (every superpixel non-empty and 4-connected)
# and raises E = H + gamma G (Eqs. 4-9).  Sequential (raster order, each move
# applied at once, the paper's Gauss-Seidel sweep).  Tiny images only.
# ----------------------------------------------------------------------------
def _valid(labels: np.ndarray, k: int) -> bool:
    """Superpixel k non-empty and one 4-connected component (the only label a
    move can break: the receiving label gains 4-adjacent pixels)."""
    from scipy import ndimage
    m = labels == k
    if not m.any():
        return False
    return ndimage.label(m, structure=[[0, 1, 0], [1, 1, 1], [0, 1, 0]])[1] == 1


def _h_terms(bins: np.ndarray, labels: np.ndarray, ks):
    """sum over superpixels ks of sum_b (h_k[b] / |A_k|)^2 (Eq. 6 + Eq. 5)."""
    out = Fraction(0)
    for k in ks:
        sel = bins[labels == k]
        if sel.size:
            _, cnt = np.unique(sel, return_counts=True)
            out += sum(Fraction(int(c), sel.size) ** 2 for c in cnt)
    return out


def _g_terms(labels: np.ndarray, centres):
    """sum over patch centres of sum_x (b_i(x) / |patch|)^2 (Eq. 9)."""
    H, W = labels.shape
    out = Fraction(0)
    for y, x in centres:
        patch = labels[max(0, y - 1):y + 2, max(0, x - 1):x + 2]
        _, cnt = np.unique(patch, return_counts=True)
        out += sum(Fraction(int(c), patch.size) ** 2 for c in cnt)
    return out


def delta_energy(bins, labels, pixels, n, gamma=0):
    """Exact E(s') - E(s) for moving `pixels` (list of (y, x), all labelled k)
    to n, computed locally: only superpixels k and n change their colour term,
    and only patches centred within one pixel of a moved pixel change their
    boundary term."""
    k = int(labels[pixels[0]])
    after = labels.copy()
    for p in pixels:
        after[p] = n
    d = _h_terms(bins, after, (k, n)) - _h_terms(bins, labels, (k, n))
    if gamma:
        H, W = labels.shape
        cs = sorted({(y + dy, x + dx) for y, x in pixels for dy in (-1, 0, 1) for dx in (-1, 0, 1)
                     if 0 <= y + dy < H and 0 <= x + dx < W})
        d += gamma * (_g_terms(after, cs) - _g_terms(labels, cs))
    return d, after


def grid_blocks(W: int, H: int, nx: int, ny: int, L: int):
    """Level-0 block column i spans [floor(iW/GX), floor((i+1)W/GX)) with
    GX = nx 2^L (reading O2, restated); level l block (i, j) spans level-0
    columns [i 2^l, (i+1) 2^l) and rows likewise."""
    GX, GY = nx << L, ny << L
    cs = [i * W // GX for i in range(GX + 1)]
    rs = [j * H // GY for j in range(GY + 1)]

    def rect(l, i, j):
        return rs[j << l], rs[(j + 1) << l], cs[i << l], cs[(i + 1) << l]
    return GX, GY, rect


def exact_climb(bins: np.ndarray, nx: int, ny: int, L: int, iters: int, gamma: int = 0, max_moves: int = 10 ** 6,
                until_stable: bool = False):
    """EXACT-mode refinement from the grid.  Returns (labels, log) where log
    lists every accepted move as (level, pixels, k, n, dE) with the locally
    computed exact dE.  until_stable: after the I pixel iterations, keep
    sweeping the pixel level until a whole sweep accepts nothing (a local
    optimum for single-pixel moves; at most 200 extra sweeps)."""
    H, W = bins.shape
    GX, GY, rect = grid_blocks(W, H, nx, ny, L)
    lab = np.empty((H, W), np.int64)
    for j in range(GY):
        for i in range(GX):
            y0, y1, x0, x1 = rect(0, i, j)
            lab[y0:y1, x0:x1] = (j >> L) * nx + (i >> L)
    log = []

    def try_unit(level, pixels, neigh):
        nonlocal lab
        k = int(lab[pixels[0]])
        cand = []
        for q in neigh:  # W, E, N, S
            if q is not None and int(lab[q]) != k and int(lab[q]) not in cand:
                cand.append(int(lab[q]))
        for n in cand:
            d, after = delta_energy(bins, lab, pixels, n, gamma)
            if d > 0 and _valid(after, k):
                log.append((level, list(pixels), k, n, d))
                lab = after
                return

    for l in range(L - 1, -1, -1):
        bw, bh = GX >> l, GY >> l
        for _ in range(iters):
            for j in range(bh):
                for i in range(bw):
                    y0, y1, x0, x1 = rect(l, i, j)
                    px = [(y, x) for y in range(y0, y1) for x in range(x0, x1)]
                    nb = [rect(l, i - 1, j) if i > 0 else None, rect(l, i + 1, j) if i + 1 < bw else None,
                          rect(l, i, j - 1) if j > 0 else None, rect(l, i, j + 1) if j + 1 < bh else None]
                    try_unit(l, px, [None if r is None else (r[0], r[2]) for r in nb])
                    if len(log) >= max_moves:
                        return lab, log
    sweeps = 0
    while sweeps < iters or until_stable:
        before = len(log)
        for y in range(H):
            for x in range(W):
                nb = [(y, x - 1) if x > 0 else None, (y, x + 1) if x + 1 < W else None,
                      (y - 1, x) if y > 0 else None, (y + 1, x) if y + 1 < H else None]
                try_unit(-1, [(y, x)], nb)
                if len(log) >= max_moves:
                    return lab, log
        sweeps += 1
        if sweeps >= iters and (len(log) == before or sweeps >= iters + 200):
            break
    return lab, log


def improving_pixel_moves(bins: np.ndarray, labels: np.ndarray, gamma: int = 0):
    """Every valid single-pixel move k -> n (n a 4-neighbour's label) with
    E(s') > E(s), E recomputed over the whole image with energy_exact (the
    local-optimality certificate of SURVEY.md P8 when the list is empty)."""
    H, W = labels.shape
    e0 = energy_exact(labels, bins, gamma)
    out = []
    for y in range(H):
        for x in range(W):
            k = int(labels[y, x])
            seen = set()
            for yy, xx in ((y, x - 1), (y, x + 1), (y - 1, x), (y + 1, x)):
                if 0 <= yy < H and 0 <= xx < W and int(labels[yy, xx]) != k and int(labels[yy, xx]) not in seen:
                    n = int(labels[yy, xx])
                    seen.add(n)
                    after = labels.copy()
                    after[y, x] = n
                    if _valid(after, k) and energy_exact(after, bins, gamma) > e0:
                        out.append((y, x, k, n))
    return out
