"""GPU parity of the 8-bit CIELAB pre-pass (reading M3;
include/seeds.h seeds_set_colour_space / seeds_rgb_to_lab): the conversion
equals the oracle's on all 2^24 sRGB colours, and LAB-mode runs equal the
oracle's LAB runs bit for bit in every execution mode, on batches, warm
starts, the 512-bin path and with the means post-processing.  Needs a B200."""
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


def make(shape, p, mode="auto"):
    from paper_1309_3848_b200.seeds import Seeds
    H, W, C = shape
    s = Seeds(W, H, C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"], p["smoothness_prior"],
              p["iters_per_level"])
    s.set_mode(mode)
    s.set_colour_space("lab")
    return s


def check(s, f, lab, r, sums=False):
    h, a = s.read_state(f)
    np.testing.assert_array_equal(lab, r.labels)
    np.testing.assert_array_equal(h.cpu().numpy(), r.hist)
    np.testing.assert_array_equal(a.cpu().numpy(), r.sizes)
    if sums:
        np.testing.assert_array_equal(s.read_sums(f).cpu().numpy(), r.sums)


def test_conversion_every_colour(torch_cuda, orc):
    torch = torch_cuda
    v = np.arange(1 << 24, dtype=np.uint32)
    rgb = np.stack([(v >> 16) & 255, (v >> 8) & 255, v & 255], -1).astype(np.uint8)
    s = make((8, 8, 3), dict(n_superpixels=1, n_levels=0, bins_per_channel=4, smoothness_prior=0, iters_per_level=1))
    got = s.rgb_to_lab(torch.from_numpy(rgb).cuda()).cpu().numpy()
    np.testing.assert_array_equal(got, orc.rgb_to_lab(rgb))
    s.close()


@pytest.mark.parametrize("mode", ["grid", "graph"])
@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_lab_runs(torch_cuda, orc, cfg, mode):
    from paper_1309_3848_b200.seeds import SeedsError
    torch = torch_cuda
    img = configs.frames(cfg, n=1)[0]
    p = configs.params(cfg)
    try:
        s = make(img.shape, p, mode)
    except SeedsError:
        pytest.skip(f"{mode} mode does not fit")
    lab = s.iterate(torch.from_numpy(img).cuda()).cpu().numpy()
    check(s, 0, lab, orc.run(img, **p, colour="lab"))
    s.close()


def test_lab_batch_and_means(torch_cuda, orc):
    torch = torch_cuda
    f = configs.frames("c3", n=24)
    p = configs.params("c3")
    s = make(f.shape[1:], p)
    s.set_means_iters(1)
    lab = s.batch(torch.from_numpy(f).cuda()).cpu().numpy()
    for i in (0, 7, 23):
        check(s, i, lab[i], orc.run(f[i], **p, colour="lab", means_iters=1, want_sums=True), sums=True)
    s.close()


def test_lab_warm_and_host_entry(torch_cuda, orc):
    torch = torch_cuda
    clip = configs.clips("c4")[0, :2]
    p = configs.params("c4")
    s = make(clip.shape[1:], p)
    g0 = s.iterate(torch.from_numpy(clip[0]).cuda())
    r0 = orc.run(clip[0], **p, colour="lab")
    np.testing.assert_array_equal(g0.cpu().numpy(), r0.labels)
    out = np.empty((1,) + clip.shape[1:3], np.int32)
    s.batch_host(np.ascontiguousarray(clip[1:2]), out, init_labels=g0.cpu().numpy()[None])
    np.testing.assert_array_equal(out[0], orc.run(clip[1], **p, colour="lab", init_labels=r0.labels).labels)
    s.close()


def test_lab_512_bins_crop(torch_cuda, orc):
    torch = torch_cuda
    img = np.ascontiguousarray(configs.frames("c5", n=1)[0, :768, :768])
    p = dict(configs.params("c5"))
    p["n_superpixels"] = p["n_superpixels"] * 768 * 768 // (8192 * 8192)
    s = make(img.shape, p)
    lab = s.iterate(torch.from_numpy(img).cuda()).cpu().numpy()
    check(s, 0, lab, orc.run(img, **p, colour="lab"))
    s.close()


def test_lab_needs_three_channels(torch_cuda):
    from paper_1309_3848_b200.seeds import Seeds, SeedsError
    s = Seeds(32, 32, 1, 4, 1, 4, 0, 1)
    with pytest.raises(SeedsError):
        s.set_colour_space("lab")
    s.close()
