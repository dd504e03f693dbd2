"""GPU parity of the means post-processing (reading M1;
include/seeds.h seeds_set_means_iters): labels, histograms, sizes and the
per-superpixel channel sums equal the oracle's bit for bit -- the paper's
configs with the last iterations on means, the SPM baseline (n_levels = 0, all
pixel iterations on means), batches that need the multi-tile plans, warm
starts, the 512-bin (uint16 bin plane) path, and seeded random shapes.
Needs a B200."""
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


def make(img_shape, p, m):
    from paper_1309_3848_b200.seeds import Seeds
    H, W, C = img_shape
    s = Seeds(W, H, C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"],
              p["smoothness_prior"], p["iters_per_level"])
    s.set_means_iters(m)
    return s


def check_frame(s, f, lab, r):
    h, a = s.read_state(f)
    np.testing.assert_array_equal(lab, r.labels, err_msg=f"labels frame {f}")
    np.testing.assert_array_equal(h.cpu().numpy(), r.hist, err_msg=f"hist frame {f}")
    np.testing.assert_array_equal(a.cpu().numpy(), r.sizes, err_msg=f"sizes frame {f}")
    np.testing.assert_array_equal(s.read_sums(f).cpu().numpy(), r.sums, err_msg=f"sums frame {f}")


@pytest.mark.parametrize("cfg", ["c1", "c2"])
@pytest.mark.parametrize("m", [1, 2, 4])
def test_means_configs(torch_cuda, orc, cfg, m):
    torch = torch_cuda
    img = configs.frames(cfg, n=1)[0]
    p = dict(configs.params(cfg))
    m = min(m, p["iters_per_level"])
    s = make(img.shape, p, m)
    lab = s.iterate(torch.from_numpy(img).cuda()).cpu().numpy()
    r = orc.run(img, **p, means_iters=m, want_sums=True)
    check_frame(s, 0, lab, r)
    s.close()


@pytest.mark.parametrize("gamma", [0, 1])
def test_spm_baseline(torch_cuda, orc, gamma):
    """SPM: no block levels, every pixel iteration on means."""
    torch = torch_cuda
    img = configs.frames("c2", n=1)[0]
    p = dict(configs.params("c2"), n_levels=0, smoothness_prior=gamma)
    s = make(img.shape, p, p["iters_per_level"])
    lab = s.iterate(torch.from_numpy(img).cuda()).cpu().numpy()
    check_frame(s, 0, lab, orc.run(img, **p, means_iters=p["iters_per_level"], want_sums=True))
    s.close()


def test_means_batch_multi_tile(torch_cuda, orc):
    """48 c3 frames (CTAs own several tiles): every frame equals the oracle."""
    torch = torch_cuda
    f = configs.frames("c3", n=48)
    p = configs.params("c3")
    s = make(f.shape[1:], p, 2)
    lab = s.batch(torch.from_numpy(f).cuda()).cpu().numpy()
    for i in range(0, 48, 5):
        check_frame(s, i, lab[i], orc.run(f[i], **p, means_iters=2, want_sums=True))
    s.close()


def test_means_warm_start(torch_cuda, orc):
    """Warm start (reading O9) followed by means iterations, two video frames."""
    torch = torch_cuda
    f, _ = mosaic.moving_mosaic(3, 320, 180, 30, 8.0, seed=77)
    p = dict(n_superpixels=60, n_levels=3, bins_per_channel=5, smoothness_prior=0, iters_per_level=3)
    s = make(f.shape[1:], p, 1)
    prev_g = s.iterate(torch.from_numpy(f[0]).cuda())[None]
    prev_r = orc.run(f[0], **p, means_iters=1).labels
    for t in (1, 2):
        lab = s.batch(torch.from_numpy(f[t:t + 1]).cuda(), init_labels=prev_g)
        r = orc.run(f[t], **p, means_iters=1, init_labels=prev_r, want_sums=True)
        check_frame(s, 0, lab[0].cpu().numpy(), r)
        prev_g, prev_r = lab, r.labels
    s.close()


def test_means_512_bins_crop(torch_cuda, orc):
    """c5's 512 bins (uint16 bin plane) on a 512x512 crop, K scaled."""
    torch = torch_cuda
    img = np.ascontiguousarray(configs.frames("c5", n=1)[0, :512, :512])
    p = dict(configs.params("c5"))
    p["n_superpixels"] = p["n_superpixels"] * 512 * 512 // (8192 * 8192)
    s = make(img.shape, p, 2)
    lab = s.iterate(torch.from_numpy(img).cuda()).cpu().numpy()
    check_frame(s, 0, lab, orc.run(img, **p, means_iters=2, want_sums=True))
    s.close()


RNG = np.random.default_rng(1309)
CASES = []
for i in range(24):
    W, H = int(RNG.integers(8, 260)), int(RNG.integers(8, 180))
    C = int(RNG.integers(1, 5))
    bpc = int(RNG.choice([2, 3, 4, 5]))
    iters = int(RNG.integers(1, 5))
    CASES.append((i, W, H, C, bpc, int(RNG.integers(1, max(2, W * H // 25))), int(RNG.integers(0, 5)),
                  int(RNG.integers(0, 2)), iters, int(RNG.integers(1, iters + 1)), int(RNG.choice([1, 2]))))


@pytest.mark.parametrize("case", CASES, ids=[f"case{c[0]}" for c in CASES])
def test_means_random(torch_cuda, orc, case):
    from paper_1309_3848_b200.seeds import SeedsError
    torch = torch_cuda
    i, W, H, C, bpc, K, L, gamma, iters, m, nf = case
    p = dict(n_superpixels=K, n_levels=L, bins_per_channel=bpc, smoothness_prior=gamma, iters_per_level=iters)
    imgs = np.stack([mosaic.mosaic(W, H, 12, 9.0, seed=500 * i + f, C=C, grad=25.0) for f in range(nf)])
    try:
        s = make(imgs.shape[1:], p, m)
    except SeedsError:
        pytest.skip("geometry rejected")
    lab = s.batch(torch.from_numpy(imgs).cuda()).cpu().numpy()
    for f in range(nf):
        check_frame(s, f, lab[f], orc.run(imgs[f], **p, means_iters=m, want_sums=True))
    s.close()


def test_means_argument_checks(torch_cuda):
    from paper_1309_3848_b200.seeds import Seeds, SeedsError
    s = Seeds(64, 48, 3, 12, 2, 4, 1, 3)
    with pytest.raises(SeedsError):
        s.set_means_iters(4)          # more than iters_per_level
    with pytest.raises(SeedsError):
        s.read_sums(0)                # no run yet
    s.set_means_iters(2)
    with pytest.raises(SeedsError):
        s.set_mode("graph")           # grid mode only
    s.set_means_iters(0)
    s.set_mode("graph")
    with pytest.raises(SeedsError):
        s.set_means_iters(1)          # forced graph mode
    s.close()
