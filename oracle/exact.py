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
