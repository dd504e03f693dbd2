"""Row-band mode (include/seeds.h): any number of bands gives the one-GPU
result bit for bit.  The bands run as virtual ranks in this
process on one GPU (bands.local_run), exchanging records and halos exactly as
the ranks of a multi-GPU run do (bands.dist_run).  Needs a B200."""
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


def band_run(torch, img, p, n_bands, init=None, colour="rgb"):
    from paper_1309_3848_b200 import bands
    from paper_1309_3848_b200.seeds import SeedsBand
    H, W, C = img.shape
    bs = [SeedsBand(W, H, C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"],
                    p["smoothness_prior"], p["iters_per_level"], b, n_bands) for b in range(n_bands)]
    for b in bs:
        b.set_colour_space(colour)
    d = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    di = None if init is None else torch.from_numpy(np.ascontiguousarray(init, np.int32)).cuda()
    lab = bands.local_run(bs, d, di)
    torch.cuda.synchronize()
    hs = [b.read_state(0) for b in bs]
    rows = [(b.row0, b.row1) for b in bs]
    for b in bs:
        b.close()
    return lab.cpu().numpy(), hs, rows


@pytest.mark.parametrize("n_bands", [1, 2, 3, 6])
def test_c1_bands_equal_oracle(torch_cuda, orc, n_bands):
    img = configs.frames("c1")[0]
    p = configs.params("c1")
    lab, hs, rows = band_run(torch_cuda, img, p, n_bands)
    r = orc.run(img, **p)
    assert rows[0][0] == 0 and rows[-1][1] == img.shape[0]
    assert all(rows[i][1] == rows[i + 1][0] for i in range(len(rows) - 1))
    np.testing.assert_array_equal(lab, r.labels)
    for h, a in hs:  # every replica equals the one-GPU histograms
        np.testing.assert_array_equal(h.cpu().numpy(), r.hist)
        np.testing.assert_array_equal(a.cpu().numpy(), r.sizes)


@pytest.mark.parametrize("n_bands", [2, 5])
def test_c2_bands_equal_oracle(torch_cuda, orc, n_bands):
    img = configs.frames("c2")[0]
    p = configs.params("c2")
    lab, hs, _ = band_run(torch_cuda, img, p, n_bands)
    r = orc.run(img, **p)
    np.testing.assert_array_equal(lab, r.labels)
    np.testing.assert_array_equal(hs[-1][0].cpu().numpy(), r.hist)


def test_bands_gamma0_warm_start(torch_cuda, orc):
    f, _ = mosaic.moving_mosaic(2, 200, 120, 15, 8.0, seed=7)
    p = dict(n_superpixels=40, n_levels=3, bins_per_channel=5, smoothness_prior=0, iters_per_level=3)
    r0 = orc.run(f[0], **p)
    lab, hs, _ = band_run(torch_cuda, f[1], p, 3, init=r0.labels)
    r1 = orc.run(f[1], **p, init_labels=r0.labels)
    np.testing.assert_array_equal(lab, r1.labels)
    np.testing.assert_array_equal(hs[0][0].cpu().numpy(), r1.hist)


def test_c5_crop_bands_equal_single(torch_cuda, orc):
    """512 bins (uint16 bin plane), 5 block levels: 4 bands == the oracle."""
    f = np.ascontiguousarray(configs.frames("c5", n=1)[0, :768, :1024])
    p = dict(configs.params("c5"))
    p["n_superpixels"] = 20000 * 768 * 1024 // (8192 * 8192)
    lab, hs, _ = band_run(torch_cuda, f, p, 4)
    r = orc.run(f, **p)
    np.testing.assert_array_equal(lab, r.labels)
    np.testing.assert_array_equal(hs[1][0].cpu().numpy(), r.hist)


@pytest.mark.parametrize("n_bands", [1, 3])
def test_c2_bands_lab(torch_cuda, orc, n_bands):
    """The LAB pre-pass (reading M3) in row-band mode: every band converts the
    replicated frame and the result equals the oracle's LAB run."""
    img = configs.frames("c2")[0]
    p = configs.params("c2")
    lab, hs, _ = band_run(torch_cuda, img, p, n_bands, colour="lab")
    r = orc.run(img, **p, colour="lab")
    np.testing.assert_array_equal(lab, r.labels)
    np.testing.assert_array_equal(hs[0][0].cpu().numpy(), r.hist)


def test_bands_reject_means(torch_cuda):
    from paper_1309_3848_b200.seeds import SeedsBand, SeedsError
    b = SeedsBand(64, 48, 3, 12, 2, 4, 1, 3, 0, 2)
    with pytest.raises(SeedsError):
        b.set_means_iters(1)
    b.close()
