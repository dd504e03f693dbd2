"""Pins of the oracle's means post-processing (reading
M1 in DESIGN.md section 3): the last pixel iterations accept a move k -> n iff
the pixel's colour is strictly nearer to the mean colour of n than to that of
k (SPM, "the mean-based distance measure from SLIC", used as
post-processing).

Independent of the oracle's arithmetic: exact rationals for the nearest-mean
rule, numpy recounts for the channel sums, a from-scratch prediction of whole
sub-sweeps (means recomputed from the labels, the ring rule through the LUT
that test_oracle_pins.py pins against a flood fill, Prop. 2 through the sum
pinned by P4), and closed-form special cases.  No GPU needed.
"""
from fractions import Fraction

import numpy as np
import pytest

from paper_1309_3848_b200 import mosaic

RING = [(0, -1), (1, -1), (1, 0), (1, 1), (0, 1), (-1, 1), (-1, 0), (-1, -1)]


def sqdist_to_mean(v, S, A):
    """||v - S/A||^2 on exact rationals."""
    return sum((Fraction(int(vc)) - Fraction(int(sc), int(A))) ** 2 for vc, sc in zip(v, S))


def channel_sums(labels, img, K):
    C = img.shape[2]
    out = np.zeros((K, 4), np.int64)
    for c in range(C):
        out[:, c] = np.bincount(labels.ravel(), weights=img[:, :, c].ravel().astype(np.float64),
                                minlength=K).astype(np.int64)
    return out


def test_means_test_is_nearest_mean(orc):
    """One proposal: accept iff ||v - mu_n||^2 < ||v - mu_k||^2 exactly (ties
    reject), for random sums and sizes including near-ties."""
    rng = np.random.default_rng(11)
    n_acc = n_rej = 0
    for i in range(4000):
        C = int(rng.integers(1, 5))
        v = rng.integers(0, 256, C)
        Ak, An = int(rng.integers(2, 5000)), int(rng.integers(1, 5000))
        Sk = rng.integers(0, 256 * Ak, C)
        Sn = rng.integers(0, 256 * An, C)
        if i % 4 == 0:  # a tie: mu_n as far from v as mu_k (mirror through v)
            An = Ak
            Sn = 2 * v * Ak - Sk
            if (Sn < 0).any():
                continue
        want = sqdist_to_mean(v, Sn, An) < sqdist_to_mean(v, Sk, Ak)
        got = orc.means_test(v, Sk, Ak, Sn, An)
        assert got == want, (v, Sk, Ak, Sn, An)
        n_acc += want
        n_rej += not want
    assert n_acc > 500 and n_rej > 500


def test_means_test_extreme_sizes(orc):
    """Sizes near the N < 2^27 bound: the cross-multiplied comparison still
    equals the rational one (no overflow)."""
    A = (1 << 27) - 1
    for v, sk, sn in (([255, 0, 255], [0, 255 * A, 0], [255 * A, 0, 255 * A - 1]),
                      ([0, 0, 0], [A, A, A], [A - 1, A, A]),
                      ([128, 128, 128], [128 * A + 1] * 3, [128 * (A - 5)] * 3)):
        for An in (A, A - 5, 1):
            Sn = [min(x, 255 * An) for x in sn]
            want = sqdist_to_mean(v, Sn, An) < sqdist_to_mean(v, sk, A)
            assert orc.means_test(v, sk, A, Sn, An) == want


def _ring_mask(lab, x, y, k):
    H, W = lab.shape
    m = 0
    for r, (dx, dy) in enumerate(RING):
        xx, yy = x + dx, y + dy
        if 0 <= xx < W and 0 <= yy < H and lab[yy, xx] == k:
            m |= 1 << r
    return m


def predict_means_subsweep(orc, lab, img, colour, P, gamma, K):
    """One COL means sub-sweep written from the definitions: every pixel of
    `colour` against the snapshot `lab` (W, E, N, S candidates, first accepted)."""
    H, W = lab.shape
    S = channel_sums(lab, img, K)
    A = np.bincount(lab.ravel(), minlength=K)
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
            if not cand or not orc.removable(_ring_mask(lab, x, y, k)):
                continue
            v = img[y, x]
            dk = sqdist_to_mean(v, S[k], A[k])
            for n in cand:
                if not sqdist_to_mean(v, S[n], A[n]) < dk:
                    continue
                if gamma and orc.smooth_sum(lab, x, y, k, n) < 0:
                    continue
                out[y, x] = n
                break
    return out


@pytest.mark.parametrize("gamma,L", [(0, 1), (1, 1), (0, 0), (1, 2)])
def test_means_subsweeps_brute_force(orc, gamma, L):
    """Every means sub-sweep of a small mosaic equals its from-scratch
    prediction (means recomputed from the labels each time), which pins the
    oracle's incremental channel sums and its snapshot schedule."""
    img = mosaic.mosaic(40, 30, 6, sigma=12.0, seed=21, grad=20.0)
    I, m = 3, 2
    nx, ny, Le = orc.geometry(40, 30, 12, L)
    K = nx * ny
    P = 3 if gamma else 2
    s0 = 4 * Le * I + (I - m) * P * P
    prev = orc.run(img, 12, L, 4, gamma, I, means_iters=m, max_subsweeps=s0).labels
    moved = 0
    for i in range(m * P * P):
        nxt = orc.run(img, 12, L, 4, gamma, I, means_iters=m, max_subsweeps=s0 + i + 1).labels
        want = predict_means_subsweep(orc, prev, img, i % (P * P), P, gamma, K)
        np.testing.assert_array_equal(nxt, want, err_msg=f"means sub-sweep {i}")
        moved += int((nxt != prev).sum())
        prev = nxt
    assert moved > 0


@pytest.mark.parametrize("schedule", [0, 1])
@pytest.mark.parametrize("gamma", [0, 1])
def test_means_state_recount(orc, schedule, gamma):
    """P1 with the channel sums: after a run with means iterations, H, A and S
    equal recounts from the labels, and every superpixel is non-empty."""
    img = mosaic.mosaic(64, 48, 9, sigma=10.0, seed=5, grad=30.0)
    r = orc.run(img, 20, 2, 5, gamma, 4, schedule=schedule, means_iters=2, want_sums=True)
    K = r.k_act
    np.testing.assert_array_equal(r.sums, channel_sums(r.labels, img, K))
    np.testing.assert_array_equal(r.sizes, np.bincount(r.labels.ravel(), minlength=K))
    assert (r.sizes > 0).all()
    assert r.hist.sum(1).tolist() == r.sizes.tolist()


def test_means_off_is_the_histogram_run(orc):
    """means_iters = 0 is the plain refinement (same labels / state)."""
    img = mosaic.mosaic(48, 40, 7, sigma=8.0, seed=3, grad=10.0)
    a = orc.run(img, 16, 2, 5, 1, 3)
    b = orc.run(img, 16, 2, 5, 1, 3, means_iters=0, want_sums=True)
    np.testing.assert_array_equal(a.labels, b.labels)
    np.testing.assert_array_equal(a.hist, b.hist)


@pytest.mark.parametrize("gamma", [0, 1])
def test_means_constant_image_fixed_point(orc, gamma):
    """Every mean equals the pixel colour: no strict improvement, no move."""
    img = np.full((30, 44, 3), 77, np.uint8)
    grid = orc.run(img, 12, 2, 5, gamma, 0)
    r = orc.run(img, 12, 2, 5, gamma, 3, means_iters=3)
    np.testing.assert_array_equal(r.labels, grid.labels)
    assert sum(t["moves"] for t in r.trace) == 0


@pytest.mark.parametrize("offset", [-3, -1, 1, 3])
def test_spm_two_tone_seam_recovered(orc, offset):
    """SPM (n_levels = 0, every pixel iteration on means, gamma = 0) on a
    two-tone image whose colour seam is `offset` rows from the K = 2 grid seam:
    each boundary pixel of the wrong tone is nearer to the other superpixel's
    mean, so the seam is recovered exactly."""
    img = np.zeros((32, 32, 3), np.uint8)
    img[: 16 + offset] = (40, 90, 10)
    img[16 + offset:] = (220, 30, 160)
    want = (np.arange(32)[:, None] >= 16 + offset).astype(np.int32) * np.ones((1, 32), np.int32)
    for schedule in (0, 1):
        r = orc.run(img, 2, 0, 2, 0, 6, schedule=schedule, means_iters=6)
        np.testing.assert_array_equal(r.labels, want)


def test_means_rejects_bad_arguments(orc):
    img = np.zeros((8, 8, 3), np.uint8)
    with pytest.raises(ValueError):
        orc.run(img, 4, 1, 4, 0, 2, means_iters=3)  # more means iterations than iterations
    with pytest.raises(ValueError):
        orc.run(img, 4, 1, 4, 0, 2, means_iters=-1)
