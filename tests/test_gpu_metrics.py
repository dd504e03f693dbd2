"""GPU parity of the quality metrics (include/seeds.h
seeds_metrics): UE / CUE / ASA / BR numerators equal the oracle's exactly --
refined partitions of c1-c4 frames against their mosaics' region maps, a c5
crop, random label maps, several tolerances -- and the error paths.  Needs a
B200."""
import numpy as np
import pytest

from paper_1309_3848_b200 import configs

pytestmark = pytest.mark.gpu

KEYS = ("n", "ue_num", "cue_num", "asa_num", "gt_boundary", "br_hits", "max_segments")


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1309_3848_b200 import build
    build.build()
    return torch


def ctx_for(shape, p):
    from paper_1309_3848_b200.seeds import Seeds
    H, W, C = shape
    return Seeds(W, H, C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"], p["smoothness_prior"],
                 p["iters_per_level"])


def same(got, want):
    for k in KEYS:
        assert got[k] == want[k], (k, got[k], want[k])
    for k in ("ue", "cue", "asa", "br"):
        assert got[k] == pytest.approx(want[k], rel=1e-12, abs=1e-15)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c4"])
@pytest.mark.parametrize("eps", [1, 2, 3])
def test_metrics_of_refined_frames(torch_cuda, orc, cfg, eps):
    torch = torch_cuda
    img = configs.frames(cfg, n=1)[0]
    gt = configs.regions(cfg, n=1)[0]
    R = int(gt.max()) + 1
    p = configs.params(cfg)
    s = ctx_for(img.shape, p)
    lab = s.iterate(torch.from_numpy(img).cuda())
    got = s.metrics(lab, torch.from_numpy(gt).cuda(), R, eps)
    same(got, orc.metrics(lab.cpu().numpy(), gt, s.info.k_actual, R, eps))
    s.close()


def test_metrics_c3_frames(torch_cuda, orc):
    torch = torch_cuda
    f, g = configs.frames("c3", n=4), configs.regions("c3", n=4)
    p = configs.params("c3")
    s = ctx_for(f.shape[1:], p)
    lab = s.batch(torch.from_numpy(f).cuda())
    for i in range(4):
        R = int(g[i].max()) + 1
        same(s.metrics(lab[i], torch.from_numpy(g[i]).cuda(), R),
             orc.metrics(lab[i].cpu().numpy(), g[i], s.info.k_actual, R))
    s.close()


def test_metrics_c5_crop(torch_cuda, orc):
    torch = torch_cuda
    img = np.ascontiguousarray(configs.frames("c5", n=1)[0, :2048, :2048])
    gt = np.ascontiguousarray(configs.regions("c5", n=1)[0, :2048, :2048])
    R = int(gt.max()) + 1
    p = dict(configs.params("c5"))
    p["n_superpixels"] = p["n_superpixels"] * 2048 * 2048 // (8192 * 8192)
    s = ctx_for(img.shape, p)
    lab = s.iterate(torch.from_numpy(img).cuda())
    same(s.metrics(lab, torch.from_numpy(gt).cuda(), R), orc.metrics(lab.cpu().numpy(), gt, s.info.k_actual, R))
    s.close()


def test_metrics_random_maps(torch_cuda, orc):
    """Label maps that are not partitions of the refinement (blocky random
    maps, ragged sizes), random segment maps."""
    torch = torch_cuda
    rng = np.random.default_rng(99)
    for t in range(12):
        H, W = int(rng.integers(5, 200)), int(rng.integers(5, 300))
        s = ctx_for((H, W, 3), dict(n_superpixels=int(rng.integers(1, 60)), n_levels=1, bins_per_channel=4,
                                    smoothness_prior=0, iters_per_level=1))
        K = s.info.k_actual
        b = int(rng.integers(1, 9))
        lab = np.repeat(np.repeat(rng.integers(0, K, ((H + b - 1) // b, (W + b - 1) // b)), b, 0), b, 1)[:H, :W]
        R = int(rng.integers(1, 12))
        gb = int(rng.integers(1, 12))
        gt = np.repeat(np.repeat(rng.integers(0, R, ((H + gb - 1) // gb, (W + gb - 1) // gb)), gb, 0), gb, 1)[:H, :W]
        lab, gt = np.ascontiguousarray(lab, np.int32), np.ascontiguousarray(gt, np.int32)
        eps = int(rng.integers(1, 5))
        same(s.metrics(torch.from_numpy(lab).cuda(), torch.from_numpy(gt).cuda(), R, eps),
             orc.metrics(lab, gt, K, R, eps))
        s.close()


def test_metrics_errors(torch_cuda):
    from paper_1309_3848_b200.seeds import SeedsError
    torch = torch_cuda
    s = ctx_for((64, 64, 3), dict(n_superpixels=1, n_levels=0, bins_per_channel=4, smoothness_prior=0,
                                  iters_per_level=1))
    lab = torch.zeros((64, 64), dtype=torch.int32, device="cuda")
    gt = torch.arange(64 * 64, dtype=torch.int32, device="cuda").view(64, 64) % 40
    with pytest.raises(SeedsError):   # one superpixel meets 40 segments: more than its 32 slots
        s.metrics(lab, gt, 40)
    with pytest.raises(SeedsError):   # segment id out of range
        s.metrics(lab, gt, 10)
    s.close()
