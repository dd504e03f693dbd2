"""Unit test of the block colour test K5 as the grid kernel runs it
(include/seeds.h seeds_debug_k5, seeds_grid.cuh k5_segment): G-lane warp
segments, __match_any_sync bin merging (two pixels per lane on 128-thread
plans), segmented shuffle reductions on 32-bit halves ("narrow", the kernel's
choice for N < 2^27) or 64-bit values, and the 128-bit cross-multiplied
comparison of Proposition 1 (rule R1).

Expected decisions come from the CPU oracle's colour test (oracle/
seeds_oracle.c, __int128) on the same histograms, and, for the extreme cases,
from the intersection inequality on exact rationals.  Random and extreme int32
histograms: sizes near 2^27 (the narrow branch's limit) and near 2^31 (only the
64-bit branch is exact there).  Needs a B200: every test is marked gpu."""
from fractions import Fraction

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1309_3848_b200 import build
    build.build()
    return torch


def make_cases(rng, n, B, amax, size_hi, dense=False):
    """n proposals: a block of alpha <= amax pixels leaving superpixel 0 (size
    A_0 > alpha, histogram covering the block), four candidate slots (labels
    1..4 or empty), superpixel sizes up to size_hi."""
    H = np.zeros((n, 5, B), np.int64)
    A = np.zeros((n, 5), np.int64)
    bins = np.full((n, 64), -1, np.int64)
    alpha = rng.integers(1, amax + 1, size=n)
    cand = np.full((n, 4), -1, np.int64)
    for e in range(n):
        nb = int(rng.integers(1, min(B, 12) + 1))
        support = rng.choice(B, size=nb, replace=False)
        bins[e, :alpha[e]] = rng.choice(support, size=alpha[e])
        l = np.bincount(bins[e, :alpha[e]], minlength=B)
        for s in range(5):
            tot = int(rng.integers(max(2, alpha[e] + 1 if s == 0 else 1), size_hi - 128))
            # spread tot pixels over a few bins, biased to the block's support
            k = int(rng.integers(1, 6))
            bsel = np.concatenate([rng.choice(support, size=min(k, nb)), rng.integers(0, B, size=2)])
            w = rng.random(bsel.size) + (0.0 if dense else 0.05)
            w = w / w.sum()
            h = np.zeros(B, np.int64)
            np.add.at(h, bsel, np.floor(w * tot).astype(np.int64))
            h[bsel[0]] += tot - h.sum()
            if s == 0:
                short = np.maximum(l - h, 0)
                h += short
                if h.sum() <= alpha[e]:
                    h[bsel[0]] += alpha[e] + 1 - h.sum()
            H[e, s] = h
            A[e, s] = h.sum()
        slots = rng.permutation(4)[: int(rng.integers(1, 5))]
        labs = rng.permutation(np.arange(1, 5))
        for i, d in enumerate(slots):
            cand[e, d] = labs[i]
    return H, A, bins, alpha, cand


def oracle_decisions(orc, H, A, bins, alpha, cand):
    out = []
    for e in range(H.shape[0]):
        l = np.bincount(bins[e, :alpha[e]], minlength=H.shape[2])
        acc = -1
        for d in range(4):
            n = cand[e, d]
            if n < 0:
                continue
            if orc.colour_test(H[e, n], H[e, 0], l, int(A[e, n]), int(A[e, 0]), int(alpha[e]), force_block=True):
                acc = int(n)
                break
        out.append(acc)
    return np.array(out)


def exact_decision(H, A, l, alpha, n):
    """int(c_n, c_l) > int(c_{k minus l}, c_l) on rationals."""
    i_n = sum((min(Fraction(int(H[n][b]), int(A[n])), Fraction(int(l[b]), alpha)) for b in range(len(l)) if l[b]),
              Fraction(0))
    i_k = sum((min(Fraction(int(H[0][b] - l[b]), int(A[0]) - alpha), Fraction(int(l[b]), alpha))
               for b in range(len(l)) if l[b]), Fraction(0))
    return i_n > i_k


def run_gpu(torch, H, A, bins, alpha, cand, threads, gs, narrow):
    from paper_1309_3848_b200.seeds import debug_k5
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.int32)).cuda()
    out = debug_k5(t(H), t(A), t(bins), t(alpha), t(cand), threads, gs, narrow)
    return out.cpu().numpy()


@pytest.mark.parametrize("threads,gs", [(512, 1), (512, 3), (512, 5), (128, 2), (128, 4), (128, 5)])
@pytest.mark.parametrize("narrow", [True, False])
def test_k5_random_histograms(torch_cuda, orc, threads, gs, narrow):
    """Random proposals with sizes below 2^27 / 64: both reduction widths give
    the oracle's decisions; on 128-thread plans blocks use both pixel slots."""
    rng = np.random.default_rng(100 * gs + threads + narrow)
    G = 1 << gs
    amax = G if threads == 512 else min(2 * G, 64)
    H, A, bins, alpha, cand = make_cases(rng, 600, 125, amax, 5000)
    got = run_gpu(torch_cuda, H, A, bins, alpha, cand, threads, gs, narrow)
    want = oracle_decisions(orc, H, A, bins, alpha, cand)
    np.testing.assert_array_equal(got, want)
    assert (want >= 0).sum() > 50 and (want < 0).sum() > 50


@pytest.mark.parametrize("threads,gs", [(512, 5), (128, 5), (128, 3)])
def test_k5_extreme_sizes_64bit(torch_cuda, orc, threads, gs):
    """Sizes up to 2^31 - 1 (int32 H and A at their limit): the 64-bit
    reductions and the 128-bit products are exact -- the decisions equal the
    oracle's __int128 ones and the exact-rational definition."""
    rng = np.random.default_rng(7 + gs + threads)
    G = 1 << gs
    amax = G if threads == 512 else 2 * G
    H, A, bins, alpha, cand = make_cases(rng, 300, 512, amax, 2 ** 31 - 1)
    assert A.max() > 2 ** 30 and A.max() < 2 ** 31
    got = run_gpu(torch_cuda, H, A, bins, alpha, cand, threads, gs, False)
    want = oracle_decisions(orc, H, A, bins, alpha, cand)
    np.testing.assert_array_equal(got, want)
    for e in range(0, 300, 10):  # spot-check the oracle itself on rationals
        l = np.bincount(bins[e, :alpha[e]], minlength=512)
        first = next((int(n) for n in cand[e] if n >= 0 and exact_decision(H[e], A[e], l, int(alpha[e]), n)), -1)
        assert first == want[e]


def test_k5_narrow_branch_limit(torch_cuda, orc):
    """At the narrow branch's limit (N < 2^27, so every size < 2^27 and, with
    alpha <= 32, every sum < 2^32) the 32-bit reductions are still exact."""
    rng = np.random.default_rng(99)
    H, A, bins, alpha, cand = make_cases(rng, 400, 64, 32, 2 ** 27 - 1)
    assert A.max() > 2 ** 26 and A.max() < 2 ** 27
    got = run_gpu(torch_cuda, H, A, bins, alpha, cand, 512, 5, True)
    want = oracle_decisions(orc, H, A, bins, alpha, cand)
    np.testing.assert_array_equal(got, want)


def test_k5_ties_and_single_bins(torch_cuda, orc):
    """Hand-made edge cases: equal intersections reject (strict >, reading
    Q6); a block concentrated in one bin; every pixel its own bin; a candidate
    slot order other than W first."""
    B = 8
    H = np.zeros((4, 5, B), np.int64)
    A = np.zeros((4, 5), np.int64)
    bins = np.full((4, 64), -1, np.int64)
    alpha = np.array([2, 4, 4, 3])
    cand = np.full((4, 4), -1, np.int64)
    # 0: tie -- n has the same normalised mass in the block's bin as k minus l
    bins[0, :2] = [3, 3]
    H[0, 0, 3], H[0, 0, 5] = 6, 4          # k: 10 px, 6 in bin 3; k minus l: 4/8 in bin 3
    H[0, 1, 3], H[0, 1, 6] = 4, 4          # n: 4/8 in bin 3
    cand[0, 1] = 1
    # 1: one bin, n clearly better
    bins[1, :4] = [2, 2, 2, 2]
    H[1, 0, 2], H[1, 0, 0] = 5, 20
    H[1, 2, 2], H[1, 2, 1] = 30, 2
    cand[1, 2] = 2
    # 2: four distinct bins, candidates in slots E and S
    bins[2, :4] = [0, 1, 2, 3]
    H[2, 0, :4] = [1, 1, 1, 1]
    H[2, 0, 4] = 30
    H[2, 3, :4] = [9, 9, 9, 9]
    H[2, 4, 7] = 10
    cand[2, 1], cand[2, 3] = 4, 3
    # 3: the first candidate fails, the second passes
    bins[3, :3] = [6, 6, 7]
    H[3, 0, 6], H[3, 0, 7], H[3, 0, 0] = 2, 1, 40
    H[3, 1, 0] = 10
    H[3, 2, 6], H[3, 2, 7] = 5, 5
    cand[3, 0], cand[3, 2] = 1, 2
    for e in range(4):
        A[e] = H[e].sum(1)
        for s in range(5):
            if A[e, s] == 0:
                H[e, s, 0] = A[e, s] = 1
    want = oracle_decisions(orc, H, A, bins, alpha, cand)
    assert list(want) == [-1, 2, 3, 2]
    for threads, gs in ((512, 2), (128, 1), (128, 2)):
        for narrow in (True, False):
            np.testing.assert_array_equal(run_gpu(torch_cuda, H, A, bins, alpha, cand, threads, gs, narrow), want)
