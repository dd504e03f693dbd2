"""GPU parity of the block-level range (reading M4;
include/seeds.h seeds_set_block_levels): single block sizes, partial ranges, the
empty range (= SPH) and its combination with the means post-processing, bit for
bit against the oracle, with the per-sub-sweep move counts.  Needs a B200."""
import numpy as np
import pytest

from paper_1309_3848_b200 import configs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1309_3848_b200 import build
    build.build()
    return torch


def run(torch, orc, cfg, lo, hi, means=0, n=1):
    from paper_1309_3848_b200.seeds import Seeds
    f = configs.frames(cfg, n=n)
    p = configs.params(cfg)
    s = Seeds(f.shape[2], f.shape[1], f.shape[3], p["n_superpixels"], p["n_levels"], p["bins_per_channel"],
              p["smoothness_prior"], p["iters_per_level"])
    s.set_block_levels(lo, hi)
    if means:
        s.set_means_iters(means)
    lab = s.batch(torch.from_numpy(f).cuda()).cpu().numpy()
    for i in range(n):
        r = orc.run(f[i], **p, block_levels=(lo, hi if hi >= 0 else 99), means_iters=means, want_sums=bool(means))
        h, a = s.read_state(i)
        np.testing.assert_array_equal(lab[i], r.labels)
        np.testing.assert_array_equal(h.cpu().numpy(), r.hist)
        np.testing.assert_array_equal(a.cpu().numpy(), r.sizes)
        mv = s.stats(i)
        assert [int(m) for m in mv[:len(r.trace)]] == [t["moves"] for t in r.trace]
        if means:
            np.testing.assert_array_equal(s.read_sums(i).cpu().numpy(), r.sums)
    s.close()


@pytest.mark.parametrize("lo,hi", [(0, 0), (1, 1), (3, 3), (1, 2), (0, -1), (4, 3)])
def test_c2_block_ranges(torch_cuda, orc, lo, hi):
    run(torch_cuda, orc, "c2", lo, hi)


def test_c1_single_level_and_means(torch_cuda, orc):
    run(torch_cuda, orc, "c1", 1, 1, means=1)


def test_c3_batch_single_level(torch_cuda, orc):
    run(torch_cuda, orc, "c3", 2, 2, n=12)


def test_range_needs_grid_mode(torch_cuda):
    from paper_1309_3848_b200.seeds import Seeds, SeedsError
    s = Seeds(64, 48, 3, 12, 2, 4, 1, 2)
    s.set_block_levels(1, 1)
    with pytest.raises(SeedsError):
        s.set_mode("graph")
    s.set_block_levels(0, -1)
    s.set_mode("graph")
    with pytest.raises(SeedsError):
        s.set_block_levels(0, 0)
    with pytest.raises(SeedsError):
        s.set_block_levels(-1, 0)
    s.close()
