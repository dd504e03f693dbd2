"""GPU parity of the priors: the compactness prior
(reading M5, seeds_set_compactness), the edge prior (reading M6,
seeds_set_edge_prior) and their combination with the 3x3 smoothing (the
paper's combined prior).  Labels, histograms, sizes and the
per-sub-sweep move counts equal the oracle's with the prior on -- c1, c2 (both
gamma), a c3 batch on the 128-thread multi-tile plans, warm starts, and with
the means post-processing, the LAB pre-pass and block-level ranges.  Needs a
B200."""
import numpy as np
import pytest

from paper_1309_3848_b200 import configs, mosaic

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1309_3848_b200 import build
    build.build()
    return torch


def check(torch, orc, imgs, p, init=None, means=0, lab=False, levels=None, compact=True, edge=0):
    from paper_1309_3848_b200.seeds import Seeds
    n, H, W, C = imgs.shape
    s = Seeds(W, H, C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"], p["smoothness_prior"],
              p["iters_per_level"])
    s.set_compactness(compact)
    s.set_edge_prior(edge)
    if means:
        s.set_means_iters(means)
    if lab:
        s.set_colour_space("lab")
    if levels:
        s.set_block_levels(*levels)
    d = torch.from_numpy(np.ascontiguousarray(imgs)).cuda()
    di = None if init is None else torch.from_numpy(np.ascontiguousarray(init, np.int32)).cuda()
    out = s.batch(d, init_labels=di).cpu().numpy()
    opts = dict(compact=compact, edge_tau=edge, means_iters=means, colour="lab" if lab else "rgb",
                block_levels=None if levels is None else (levels[0], levels[1] if levels[1] >= 0 else 99))
    for f in range(n):
        r = orc.run(imgs[f], **p, **opts, init_labels=None if init is None else init[f])
        h, a = s.read_state(f)
        np.testing.assert_array_equal(out[f], r.labels, err_msg=f"labels frame {f}")
        np.testing.assert_array_equal(h.cpu().numpy(), r.hist)
        np.testing.assert_array_equal(a.cpu().numpy(), r.sizes)
        mv = s.stats(f)
        assert [int(m) for m in mv[:len(r.trace)]] == [t["moves"] for t in r.trace]
    s.close()
    return out


@pytest.mark.parametrize("cfg,gamma", [("c1", 1), ("c2", 1), ("c2", 0)])
def test_compact_configs(torch_cuda, orc, cfg, gamma):
    p = dict(configs.params(cfg), smoothness_prior=gamma)
    check(torch_cuda, orc, configs.frames(cfg, n=1), p)


def test_compact_c3_batch(torch_cuda, orc):
    check(torch_cuda, orc, configs.frames("c3", n=24), configs.params("c3"))


def test_compact_with_means_lab_levels(torch_cuda, orc):
    p = configs.params("c2")
    f = configs.frames("c2", n=1)
    check(torch_cuda, orc, f, p, means=2)
    check(torch_cuda, orc, f, p, lab=True, levels=(1, 2))


def test_compact_warm_start(torch_cuda, orc):
    f, _ = mosaic.moving_mosaic(3, 160, 96, 15, 8.0, seed=43)
    p = dict(n_superpixels=40, n_levels=3, bins_per_channel=5, smoothness_prior=0, iters_per_level=3)
    r0 = orc.run(f[0], **p, compact=True)
    check(torch_cuda, orc, f[1:], p, init=np.stack([r0.labels, r0.labels]))


def test_compact_equal_grid_fixed_point(torch_cuda, orc):
    img = mosaic.mosaic(40, 30, 9, sigma=12.0, seed=5, grad=30.0)[None]
    p = dict(n_superpixels=12, n_levels=0, bins_per_channel=4, smoothness_prior=0, iters_per_level=3)
    out = check(torch_cuda, orc, img, p)
    grid = orc.run(img[0], **dict(p, iters_per_level=0)).labels
    np.testing.assert_array_equal(out[0], grid)


@pytest.mark.parametrize("cfg,gamma,tau", [("c1", 1, 40), ("c2", 0, 40), ("c2", 1, 25)])
def test_edge_prior(torch_cuda, orc, cfg, gamma, tau):
    p = dict(configs.params(cfg), smoothness_prior=gamma)
    check(torch_cuda, orc, configs.frames(cfg, n=1), p, compact=False, edge=tau)


def test_combined_prior(torch_cuda, orc):
    """3x3 smoothing + compactness + edge snapping, on a c3
    batch (multi-tile plans) and with the LAB pre-pass."""
    p = configs.params("c3")
    check(torch_cuda, orc, configs.frames("c3", n=12), p, compact=True, edge=60)
    check(torch_cuda, orc, configs.frames("c2", n=1), configs.params("c2"), compact=True, edge=30, lab=True)
