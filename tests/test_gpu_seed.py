"""GPU checks of the seeding kernel (grid mode): quantisation, grid labels and
the superpixel histograms built from shared-memory privatised block
histograms (include/seeds.h seeds_debug_block_hist; seeds_grid.cuh seed).

P1b on the GPU ("summing the histograms of the composing
blocks"): the top-level block histograms the seed counted equal numpy counts
over the block rectangles of reading O2, equal the level-0 block histograms
summed 2x2 level by level, and every superpixel's H row equals the sum of its
four top-level blocks.  Warm starts (hashed label slots, and tiles with more
labels than slots, which fall back to global atomics) recount H exactly.
Needs a B200: every test is marked gpu."""
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


def bins_of(img, bpc):
    img = img.astype(np.int64)
    b = np.zeros(img.shape[:2], np.int64)
    for c in range(img.shape[2]):
        b = b * bpc + (img[:, :, c] * bpc) // 256
    return b


def mk(shape, p, iters=None):
    from paper_1309_3848_b200.seeds import Seeds
    H, W, C = shape
    return Seeds(W, H, C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"], p["smoothness_prior"],
                 p["iters_per_level"] if iters is None else iters)


@pytest.mark.parametrize("cfg,nf", [("c1", 1), ("c2", 1), ("c3", 3)])
def test_top_block_histograms_sum_to_superpixels(torch_cuda, orc, cfg, nf):
    torch = torch_cuda
    f = configs.frames(cfg, n=nf)
    p = configs.params(cfg)
    s = mk(f.shape[1:], p, iters=0)  # I = 0: the seed alone (the grid, A30)
    g = s.info
    L, GX, GY, B = g.levels_eff, g.grid_x, g.grid_y, g.bins_total
    tx, ty = GX >> (L - 1), GY >> (L - 1)
    out = torch.zeros((nf, ty * tx, B), dtype=torch.int32, device="cuda")
    s.debug_block_hist(out)
    s.batch(torch.from_numpy(f).cuda())
    torch.cuda.synchronize()
    got = out.cpu().numpy().reshape(nf, ty, tx, B)
    H, W = f.shape[1:3]
    cs = [i * W // GX for i in range(GX + 1)]   # reading O2, restated
    rs = [j * H // GY for j in range(GY + 1)]
    for fi in range(nf):
        bins = bins_of(f[fi], p["bins_per_channel"])
        lvl = np.zeros((GY, GX, B), np.int64)  # level-0 block histograms
        for j in range(GY):
            for i in range(GX):
                lvl[j, i] = np.bincount(bins[rs[j]:rs[j + 1], cs[i]:cs[i + 1]].ravel(), minlength=B)
        for _ in range(L - 1):  # parent = sum of its 2 x 2 children
            lvl = lvl.reshape(lvl.shape[0] // 2, 2, lvl.shape[1] // 2, 2, B).sum(axis=(1, 3))
        np.testing.assert_array_equal(got[fi], lvl)
        # the superpixel rows: sums of the four top-level blocks
        sp = got[fi].reshape(ty // 2, 2, tx // 2, 2, B).sum(axis=(1, 3)).reshape(-1, B)
        h, a = s.read_state(fi)
        np.testing.assert_array_equal(h.cpu().numpy(), sp)
        np.testing.assert_array_equal(a.cpu().numpy(), sp.sum(1))
    s.close()


@pytest.mark.parametrize("pattern", ["previous", "stripes"])
def test_warm_seed_recounts_exactly(torch_cuda, orc, pattern):
    """Warm-start seed (hashed label slots per tile): H and A equal a recount of
    (init labels, bins).  'stripes' gives every tile far more labels than
    slots (2-pixel stripes of all K labels), exercising the global fallback."""
    torch = torch_cuda
    f = configs.frames("c4", n=2)
    p = configs.params("c4")
    s = mk(f.shape[1:], p, iters=0)
    K, B = s.info.k_actual, s.info.bins_total
    H, W = f.shape[1:3]
    if pattern == "previous":
        init = np.stack([orc.run(f[0], **p).labels] * 2)
    else:
        init = np.broadcast_to(((np.arange(W)[None, :] // 2 + np.arange(H)[:, None]) % K).astype(np.int32),
                               (2, H, W)).copy()
    lab = s.batch(torch.from_numpy(f).cuda(), init_labels=torch.from_numpy(init).cuda())
    for fi in range(2):
        bins = bins_of(f[fi], p["bins_per_channel"])
        want = np.bincount((init[fi].astype(np.int64) * B + bins).ravel(), minlength=K * B).reshape(K, B)
        h, a = s.read_state(fi)
        np.testing.assert_array_equal(h.cpu().numpy(), want)
        np.testing.assert_array_equal(a.cpu().numpy(), want.sum(1))
        np.testing.assert_array_equal(lab[fi].cpu().numpy(), init[fi])
    s.close()


@pytest.mark.parametrize("bpc", [5, 8])
@pytest.mark.parametrize("aligned", [True, False])
def test_warm_seed_word_path_and_fallback(torch_cuda, orc, bpc, aligned):
    """Warm seed of rows of a multiple of four pixels: k_seed_warm (word loads
    of four pixels, uint8 bins for bpc=5 / uint16 for bpc=8) when the label
    buffer is 16-byte aligned, k_seed_cells when it is not (a view one int32
    into its allocation).  Both: H and A equal a recount of (init labels, bins),
    the refined labels equal the oracle's warm run (PAPER.md:259-262 validity,
    reading Q13/O9)."""
    torch = torch_cuda
    f = configs.frames("c1", n=2)
    p = dict(configs.params("c1"), bins_per_channel=bpc)
    H, W = f.shape[1:3]
    assert W % 4 == 0
    init = np.stack([orc.run(f[0], **p).labels, orc.run(f[1], **p).labels]).astype(np.int32)
    s = mk(f.shape[1:], p, iters=0)
    K, B = s.info.k_actual, s.info.bins_total
    buf = torch.zeros(init.size + 4, dtype=torch.int32, device="cuda")
    off = 0 if aligned else 1
    buf[off:off + init.size] = torch.from_numpy(init.ravel()).cuda()
    d_init = buf[off:off + init.size].view(init.shape)
    lab = s.batch(torch.from_numpy(f).cuda(), init_labels=d_init)
    for fi in range(2):
        bins = bins_of(f[fi], bpc)
        want = np.bincount((init[fi].astype(np.int64) * B + bins).ravel(), minlength=K * B).reshape(K, B)
        h, a = s.read_state(fi)
        np.testing.assert_array_equal(h.cpu().numpy(), want)
        np.testing.assert_array_equal(a.cpu().numpy(), want.sum(1))
        np.testing.assert_array_equal(lab[fi].cpu().numpy(), init[fi])
    s.close()
    # the whole warm run (pixel level) against the oracle
    s = mk(f.shape[1:], p)
    lab = s.batch(torch.from_numpy(f).cuda(), init_labels=d_init)
    for fi in range(2):
        r = orc.run(f[fi], **p, init_labels=init[fi])
        h, a = s.read_state(fi)
        np.testing.assert_array_equal(lab[fi].cpu().numpy(), r.labels)
        np.testing.assert_array_equal(h.cpu().numpy(), r.hist)
        np.testing.assert_array_equal(a.cpu().numpy(), r.sizes)
    s.close()
