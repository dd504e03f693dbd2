"""Pins of the oracle's block-level range (the single-
block-size variant of the authors' earlier SEEDS; reading M4
in DESIGN.md): only block levels lo..hi run, the others push their map down
untouched.  No GPU needed."""
import numpy as np
import pytest
from scipy import ndimage

from paper_1309_3848_b200 import configs

FOUR = np.array([[0, 1, 0], [1, 1, 1], [0, 1, 0]])


def test_full_range_is_the_default(orc):
    img = configs.frames("c1")[0]
    p = configs.params("c1")
    a, b = orc.run(img, **p), orc.run(img, **p, block_levels=(0, p["n_levels"] - 1))
    np.testing.assert_array_equal(a.labels, b.labels)
    np.testing.assert_array_equal(a.hist, b.hist)
    assert len(a.trace) == len(b.trace)


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_empty_range_is_sph(orc, cfg):
    """No block level runs: the grid's maps are pushed down unchanged, so the
    result is the pixel-level-only baseline SPH (n_levels = 0)
    -- the superpixel grid does not depend on n_levels (reading O2)."""
    img = configs.frames(cfg)[0]
    p = configs.params(cfg)
    a = orc.run(img, **p, block_levels=(p["n_levels"], p["n_levels"] - 1))
    b = orc.run(img, **dict(p, n_levels=0))
    np.testing.assert_array_equal(a.labels, b.labels)
    np.testing.assert_array_equal(a.hist, b.hist)
    assert [t["level"] for t in a.trace] == [-1] * len(b.trace)


@pytest.mark.parametrize("level", [0, 1, 3])
def test_single_level_invariants(orc, level):
    """One block size (reading M4): only that level's sub-sweeps run (4 I of
    them), and H, A and connectivity hold as in P1 / P2."""
    img = configs.frames("c2")[0]
    p = configs.params("c2")
    r = orc.run(img, **p, block_levels=(level, level))
    lv = [t["level"] for t in r.trace]
    assert lv.count(level) == 4 * p["iters_per_level"] and set(lv) == {level, -1}
    K, B = r.k_act, p["bins_per_channel"] ** 3
    bins = orc.quantise(img, p["bins_per_channel"])
    h = np.bincount((r.labels.astype(np.int64) * B + bins).ravel(), minlength=K * B).reshape(K, B)
    np.testing.assert_array_equal(h, r.hist)
    assert (r.sizes > 0).all()
    for k in range(K):
        assert ndimage.label(r.labels == k, structure=FOUR)[1] == 1


@pytest.mark.parametrize("offset", [-3, 3])
def test_single_level_two_tone_seam(orc, offset):
    """P9 with one block size: the finest block level alone (then the pixel
    level, gamma = 0) recovers a straight two-tone seam exactly."""
    img = np.zeros((32, 32, 1), np.uint8)
    img[: 16 + offset] = 40
    img[16 + offset:] = 220
    want = (np.arange(32)[:, None] >= 16 + offset).astype(np.int32) * np.ones((1, 32), np.int32)
    r = orc.run(img, 2, 3, 2, 0, 4, block_levels=(0, 0))
    np.testing.assert_array_equal(r.labels, want)
