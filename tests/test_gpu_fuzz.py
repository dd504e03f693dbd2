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
@pytest.mark.parametrize("mode", ["grid", "grid128", "graph"])
def test_random_case(torch_cuda, orc, monkeypatch, case, mode):
    """grid128: grid mode on the 128-thread plans with two pixels per lane in
    the segment path (SEEDS_GRID_NT=128, SEEDS_SEG2=1)."""
    from paper_1309_3848_b200.seeds import Seeds, SeedsError
    torch = torch_cuda
    if mode == "grid128":
        monkeypatch.setenv("SEEDS_GRID_NT", "128")
        monkeypatch.setenv("SEEDS_SEG2", "1")
        mode = "grid"
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


FEATURE_CASES = []
for i in range(40):
    W = int(RNG.integers(8, 260))
    H = int(RNG.integers(8, 180))
    C = int(RNG.choice([1, 3, 3, 4]))
    bpc = int(RNG.choice([2, 3, 4, 5]))
    K = int(RNG.integers(1, max(2, W * H // 30)))
    L = int(RNG.integers(0, 5))
    gamma = int(RNG.integers(0, 2))
    iters = int(RNG.integers(1, 5))
    nf = int(RNG.choice([1, 2, 4]))
    lab = bool(C == 3 and RNG.integers(0, 2))
    means = int(RNG.integers(0, iters + 1)) if RNG.integers(0, 2) else 0
    lo = int(RNG.integers(0, 3))
    hi = int(RNG.integers(-1, 4))
    warm = bool(RNG.integers(0, 4) == 0)
    host = bool(RNG.integers(0, 2))
    compact = bool(RNG.integers(0, 2))
    edge = int(RNG.choice([0, 0, 20, 60]))
    FEATURE_CASES.append((i, W, H, C, bpc, K, L, gamma, iters, nf, lab, means, lo, hi, warm, host, compact, edge))


@pytest.mark.parametrize("case", FEATURE_CASES, ids=[f"feat{c[0]}" for c in FEATURE_CASES])
def test_random_feature_combination(torch_cuda, orc, case):
    """Grid mode with the SURVEY 8(f) options combined at random (LAB pre-pass,
    means post-processing, compactness prior, block-level range, warm starts,
    the chunked host entry point): labels equal the oracle's with the same
    options."""
    from paper_1309_3848_b200.seeds import Seeds, SeedsError
    torch = torch_cuda
    i, W, H, C, bpc, K, L, gamma, iters, nf, lab, means, lo, hi, warm, host, compact, edge = case
    p = dict(n_superpixels=K, n_levels=L, bins_per_channel=bpc, smoothness_prior=gamma, iters_per_level=iters)
    imgs = np.stack([mosaic.mosaic(W, H, int(RNG.integers(1, 30)), 10.0, seed=7000 + 10 * i + f, C=C, grad=20.0)
                     for f in range(nf)])
    try:
        s = Seeds(W, H, C, K, L, bpc, gamma, iters)
    except SeedsError:
        pytest.skip("geometry rejected")
    if lab:
        s.set_colour_space("lab")
    s.set_means_iters(means)
    s.set_block_levels(lo, hi)
    s.set_compactness(compact)
    s.set_edge_prior(edge)
    opts = dict(colour="lab" if lab else "rgb", means_iters=means, block_levels=(lo, hi if hi >= 0 else 99),
                compact=compact, edge_tau=edge)
    init = np.stack([orc.run(im, **p, **opts).labels for im in imgs]) if warm else None
    if host:
        out = np.empty((nf, H, W), np.int32)
        s.batch_host(np.ascontiguousarray(imgs), out, init_labels=None if init is None else np.ascontiguousarray(init))
    else:
        d = torch.from_numpy(np.ascontiguousarray(imgs)).cuda()
        di = None if init is None else torch.from_numpy(np.ascontiguousarray(init, np.int32)).cuda()
        out = s.batch(d, init_labels=di).cpu().numpy()
    for f in range(nf):
        r = orc.run(imgs[f], **p, **opts, init_labels=None if init is None else init[f])
        np.testing.assert_array_equal(out[f], r.labels, err_msg=f"labels frame {f}")
        if not host:
            h, a = s.read_state(f)
            np.testing.assert_array_equal(h.cpu().numpy(), r.hist, err_msg=f"hist frame {f}")
    s.close()


# ----------------------------------------------------------------------------
# Round 2 features under random shapes: row bands in one launch (1-8 bands,
# cold and warm, 1-4 channels, u8 and u16 bins) and the anytime budget replay.
# ----------------------------------------------------------------------------
BRNG = np.random.default_rng(20261020)
BAND_CASES = []
for i in range(24):
    W = int(BRNG.integers(24, 320))
    H = int(BRNG.integers(24, 240))
    C = int(BRNG.integers(1, 4))
    bpc = int(BRNG.choice([2, 3, 4, 5, 8] if C <= 2 else [2, 4, 5, 8]))
    K = int(BRNG.integers(4, max(5, W * H // 150)))
    L = int(BRNG.integers(0, 5))
    gamma = int(BRNG.integers(0, 2))
    iters = int(BRNG.integers(1, 4))
    nb = int(BRNG.integers(1, 9))
    warm = bool(BRNG.integers(0, 3) == 0)
    BAND_CASES.append((i, W, H, C, bpc, K, L, gamma, iters, nb, warm))


@pytest.mark.parametrize("case", BAND_CASES, ids=[f"band{c[0]}" for c in BAND_CASES])
def test_random_bands(torch_cuda, orc, case):
    """seeds_create_bands with a random band count: labels, histograms and
    sizes equal the oracle's one-GPU run (warm cases start from the oracle's
    cold result of the previous frame)."""
    from paper_1309_3848_b200.seeds import SeedsBands, SeedsError
    torch = torch_cuda
    i, W, H, C, bpc, K, L, gamma, iters, nb, warm = case
    p = dict(n_superpixels=K, n_levels=L, bins_per_channel=bpc, smoothness_prior=gamma, iters_per_level=iters)
    f = [mosaic.mosaic(W, H, int(BRNG.integers(2, 25)), 9.0, seed=5000 + 10 * i + t, C=C, grad=20.0)
         for t in range(2)]
    nb = max(1, min(nb, orc.geometry(W, H, K, L)[1]))  # at most one band per superpixel row
    try:
        s = SeedsBands(W, H, C, K, L, bpc, gamma, iters, nb)
    except SeedsError:
        pytest.skip("band count or geometry rejected (bands of < 2 rows, more bands than superpixel rows)")
    init = orc.run(f[0], **p).labels if warm else None
    img = f[1]
    lab = s.run(torch.from_numpy(np.ascontiguousarray(img)).cuda(),
                None if init is None else torch.from_numpy(init).cuda()).cpu().numpy()
    h, a = s.read_state(0)
    r = orc.run(img, **p, init_labels=init)
    np.testing.assert_array_equal(lab, r.labels)
    np.testing.assert_array_equal(h.cpu().numpy(), r.hist)
    np.testing.assert_array_equal(a.cpu().numpy(), r.sizes)
    s.close()


@pytest.mark.parametrize("case", CASES[:16], ids=[f"budget{c[0]}" for c in CASES[:16]])
def test_random_budget_replay(torch_cuda, orc, case):
    """Random budgets (5-60% of a measured run): the run stops at some
    sub-sweep r and equals the oracle's run with max_subsweeps = r."""
    from paper_1309_3848_b200.seeds import Seeds, SeedsError
    torch = torch_cuda
    i, W, H, C, bpc, K, L, gamma, iters, nf, warm = case
    if iters == 0:
        pytest.skip("no sub-sweeps to stop in")
    p = dict(n_superpixels=K, n_levels=L, bins_per_channel=bpc, smoothness_prior=gamma, iters_per_level=iters)
    img = mosaic.mosaic(W, H, 12, 10.0, seed=7000 + i, C=C, grad=20.0)
    try:
        s = Seeds(W, H, C, K, L, bpc, gamma, iters)
        s.set_mode("grid")
    except SeedsError:
        pytest.skip("no grid plan / geometry rejected")
    d = torch.from_numpy(img).cuda()
    for _ in range(2):
        s.iterate(d)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s.iterate(d)
    b.record()
    torch.cuda.synchronize()
    frac = float(BRNG.uniform(0.05, 0.6))
    s.set_time_budget(max(1, int(a.elapsed_time(b) * 1000 * frac)))
    lab = s.iterate(d).cpu().numpy()
    rr = s.last_subsweeps()
    ref = orc.run(img, **p, max_subsweeps=rr)
    np.testing.assert_array_equal(lab, ref.labels)
    np.testing.assert_array_equal(s.read_state(0)[0].cpu().numpy(), ref.hist)
    s.close()
