"""Randomised shapes and parameters (seeded): every execution mode against the
oracle, bit for bit -- odd sizes, ragged tiles, deep or no block levels, 1-4
channels, up to 4096 bins, batches of several frames, warm starts.  Needs a
B200."""
import numpy as np
import pytest

from paper_1309_3848_b200 import mosaic

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(20261019)
CASES = []
for i in range(64):
    W = int(RNG.integers(8, 300))
    H = int(RNG.integers(8, 200))
    C = int(RNG.integers(1, 5))
    bpc = int(RNG.choice([1, 2, 3, 4, 5, 8, 16] if C <= 3 else [2, 4, 8]))
    while bpc ** C > 4096:
        bpc //= 2
    K = int(RNG.integers(1, max(2, W * H // 20)))
    L = int(RNG.integers(0, 6))
    gamma = int(RNG.integers(0, 2))
    iters = int(RNG.integers(0, 5))
    nf = int(RNG.choice([1, 1, 2, 3]))
    warm = bool(RNG.integers(0, 4) == 0)
    CASES.append((i, W, H, C, bpc, K, L, gamma, iters, nf, warm))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1309_3848_b200 import build
    build.build()
    return torch


@pytest.mark.parametrize("case", CASES, ids=[f"case{c[0]}" for c in CASES])
@pytest.mark.parametrize("mode", ["grid", "graph", "resident"])
def test_random_case(torch_cuda, orc, case, mode):
    from paper_1309_3848_b200.seeds import Seeds, SeedsError
    torch = torch_cuda
    i, W, H, C, bpc, K, L, gamma, iters, nf, warm = case
    p = dict(n_superpixels=K, n_levels=L, bins_per_channel=bpc, smoothness_prior=gamma, iters_per_level=iters)
    imgs = np.stack([mosaic.mosaic(W, H, int(RNG.integers(1, 30)), 10.0, seed=1000 * i + f, C=C, grad=20.0)
                     for f in range(nf)])
    try:
        s = Seeds(W, H, C, K, L, bpc, gamma, iters)
    except SeedsError:
        pytest.skip("geometry rejected (K_act or block area out of range)")
    try:
        s.set_mode(mode)
    except SeedsError:
        pytest.skip(f"{mode} mode does not fit this frame")
    init = None
    if warm:
        prev = [orc.run(im, **p).labels for im in imgs]
        init = np.stack(prev)
    d = torch.from_numpy(np.ascontiguousarray(imgs)).cuda()
    di = None if init is None else torch.from_numpy(np.ascontiguousarray(init, np.int32)).cuda()
    lab = s.batch(d, init_labels=di).cpu().numpy()
    for f in range(nf):
        r = orc.run(imgs[f], **p, init_labels=None if init is None else init[f])
        h, a = s.read_state(f)
        np.testing.assert_array_equal(lab[f], r.labels, err_msg=f"labels frame {f}")
        np.testing.assert_array_equal(h.cpu().numpy(), r.hist, err_msg=f"hist frame {f}")
        np.testing.assert_array_equal(a.cpu().numpy(), r.sizes, err_msg=f"sizes frame {f}")
    s.close()
