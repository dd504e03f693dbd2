"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle's
coloured schedule (COL, rule R1), element by element.  Labels, histograms
and sizes are integers, so the bar is bit-exactness (BASELINE.json
north_star).  Needs a B200: every test is marked gpu."""
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


MODES = ["graph", "grid"]


@pytest.fixture(params=MODES)
def mode(request):
    return request.param


def gpu_run(torch, img, p, init=None, limit=-1, mode="auto"):
    from paper_1309_3848_b200.seeds import Seeds
    imgs = img if img.ndim == 4 else img[None]
    n, H, W, C = imgs.shape
    s = Seeds(W, H, C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"],
              p["smoothness_prior"], p["iters_per_level"])
    s.set_mode(mode)
    if limit >= 0:
        s.debug_limit(limit)
    d = torch.from_numpy(np.ascontiguousarray(imgs)).cuda()
    di = None if init is None else torch.from_numpy(np.ascontiguousarray(init, np.int32)).cuda()
    lab = s.batch(d, init_labels=di)
    torch.cuda.synchronize()
    hs, as_ = [], []
    for f in range(n):
        h, a = s.read_state(f)
        hs.append(h.cpu().numpy())
        as_.append(a.cpu().numpy())
    out = lab.cpu().numpy(), np.stack(hs), np.stack(as_), s
    return out


def assert_parity(torch, orc, img, p, init=None, limit=-1, mode="auto"):
    lab, h, a, s = gpu_run(torch, img, p, init=init, limit=limit, mode=mode)
    imgs = img if img.ndim == 4 else img[None]
    for f in range(imgs.shape[0]):
        r = orc.run(imgs[f], **p, init_labels=None if init is None else init[f], max_subsweeps=limit)
        assert s.info.k_actual == r.k_act
        np.testing.assert_array_equal(lab[f], r.labels, err_msg=f"labels frame {f}")
        np.testing.assert_array_equal(h[f], r.hist, err_msg=f"hist frame {f}")
        np.testing.assert_array_equal(a[f], r.sizes, err_msg=f"sizes frame {f}")
        # accepted moves per pixel sub-sweep equal the oracle's
        mv = s.stats(f)
        for i, t in enumerate(r.trace):
            if t["level"] == -1:
                assert mv[i] == t["moves"], (f, i)
    return lab, s


def test_c1_full(torch_cuda, orc, mode):
    assert_parity(torch_cuda, orc, configs.frames("c1")[0], configs.params("c1"), mode=mode)


@pytest.mark.parametrize("gamma", [0, 1])
def test_c2_full(torch_cuda, orc, gamma, mode):
    p = configs.params("c2")
    p["smoothness_prior"] = gamma
    assert_parity(torch_cuda, orc, configs.frames("c2")[0], p, mode=mode)


def test_c1_every_subsweep(torch_cuda, orc, mode):
    """Bisection hook: the state after s sub-sweeps matches for every s."""
    img = configs.frames("c1")[0]
    p = configs.params("c1")
    for s in range(0, 35):
        assert_parity(torch_cuda, orc, img, p, limit=s, mode=mode)


def test_c2_subsweeps(torch_cuda, orc, mode):
    img = configs.frames("c2")[0]
    p = configs.params("c2")
    for s in (1, 4, 17, 63, 64, 65, 80):
        assert_parity(torch_cuda, orc, img, p, limit=s, mode=mode)


@pytest.mark.parametrize("W,H,K,L,bpc,C,gamma,iters", [
    (37, 23, 7, 3, 5, 3, 1, 3),     # ragged: blocks of unequal size, odd grid
    (37, 23, 7, 3, 5, 3, 0, 3),
    (64, 48, 12, 0, 5, 3, 1, 4),    # n_levels = 0: pixel level only (SPH)
    (64, 48, 12, 2, 5, 3, 1, 0),    # iters = 0: the grid (GRID baseline)
    (1, 1, 1, 2, 5, 3, 1, 2),       # one pixel
    (1, 40, 3, 2, 4, 1, 1, 3),      # one column
    (50, 1, 4, 2, 4, 1, 0, 3),      # one row
    (3, 2, 6, 1, 2, 1, 0, 2),       # K_act = N (every superpixel one pixel)
    (90, 70, 30, 2, 1, 3, 1, 2),    # bpc = 1: one bin, no move can pass (strict test)
    (80, 60, 20, 2, 8, 3, 1, 3),    # B = 512: uint16 bin plane
    (80, 60, 20, 2, 4, 4, 0, 3),    # 4 channels, B = 256
    (64, 64, 4, 5, 16, 2, 1, 2),    # deep levels (clamped), B = 256
    (200, 150, 2000, 3, 5, 3, 1, 2),  # many tiny superpixels, L clamped
])
def test_shapes_and_degenerate_cases(torch_cuda, orc, W, H, K, L, bpc, C, gamma, iters, mode):
    img = mosaic.mosaic(W, H, max(1, min(20, W * H // 30)), 9.0, seed=W * 1000 + H, C=C, grad=20.0)
    p = dict(n_superpixels=K, n_levels=L, bins_per_channel=bpc, smoothness_prior=gamma,
             iters_per_level=iters)
    assert_parity(torch_cuda, orc, img, p, mode=mode)


def test_constant_image(torch_cuda, orc, mode):
    img = np.full((61, 47, 3), 99, np.uint8)
    p = dict(n_superpixels=12, n_levels=2, bins_per_channel=5, smoothness_prior=1, iters_per_level=3)
    lab, s = assert_parity(torch_cuda, orc, img, p, mode=mode)
    assert s.stats(0).sum() == 0


def test_batch_independent_frames(torch_cuda, orc, mode):
    """c3-shaped batch (K=400): every frame equals its own oracle run."""
    imgs = configs.frames("c3", n=6)
    assert_parity(torch_cuda, orc, imgs, configs.params("c3"), mode=mode)


def test_warm_start(torch_cuda, orc, mode):
    """Warm start (reading O9): labels of frame t seed frame t+1."""
    f, _ = mosaic.moving_mosaic(3, 160, 96, 15, 8.0, seed=42)
    p = dict(n_superpixels=40, n_levels=3, bins_per_channel=5, smoothness_prior=0, iters_per_level=3)
    r0 = orc.run(f[0], **p)
    init = np.stack([r0.labels, r0.labels])
    assert_parity(torch_cuda, orc, f[1:], p, init=init, mode=mode)


def test_c3_sampled_full_batch(torch_cuda, orc, mode):
    """The full 256-frame c3 batch in one launch; frames 0, 85, 170, 255 checked
    against the oracle, every frame checked for histogram/size invariants."""
    imgs = configs.frames("c3")
    p = configs.params("c3")
    lab, h, a, s = gpu_run(torch_cuda, imgs, p, mode=mode)
    N = imgs.shape[1] * imgs.shape[2]
    assert (a.sum(1) == N).all()
    assert (h.sum(2) == a).all()
    for f in (0, 85, 170, 255):
        r = orc.run(imgs[f], **p)
        np.testing.assert_array_equal(lab[f], r.labels)
        np.testing.assert_array_equal(h[f], r.hist)


def test_repeat_launch_is_deterministic(torch_cuda, mode):
    """Graph replays give identical output (no order dependence on the GPU)."""
    from paper_1309_3848_b200.seeds import Seeds
    img = configs.frames("c2")[0]
    p = configs.params("c2")
    s = Seeds(img.shape[1], img.shape[0], 3, *[p[k] for k in (
        "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
    s.set_mode(mode)
    d = torch_cuda.from_numpy(img).cuda()
    out = torch_cuda.empty(img.shape[:2], dtype=torch_cuda.int32, device="cuda")
    ref = s.iterate(d, out).clone()
    for _ in range(5):
        s.iterate(d, out)
        assert torch_cuda.equal(out, ref)


def test_host_entry_point(torch_cuda, orc):
    from paper_1309_3848_b200.seeds import Seeds
    img = configs.frames("c1")[0]
    p = configs.params("c1")
    s = Seeds(img.shape[1], img.shape[0], 3, *[p[k] for k in (
        "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
    out = np.empty(img.shape[:2], np.int32)
    s.batch_host(np.ascontiguousarray(img), out)
    np.testing.assert_array_equal(out, orc.run(img, **p).labels)


def test_modes_resolved(torch_cuda):
    """A c2 frame fits a grid tile plan (grid mode, the AUTO choice) with one
    tile per CTA, so a cold run is one k_tile1 launch (seed and int32 output
    inside it); every mode reports its launch count; the removed resident mode
    (2) is rejected."""
    from paper_1309_3848_b200.seeds import Seeds
    s = Seeds(481, 321, 3, 200, 4, 5, 1, 4)
    assert s.info.exec_mode == 3 and s.info.kernels_per_run == 1  # k_tile1
    assert s._lib.seeds_set_mode(s._ctx, 2) == -1
    s.set_mode("graph")
    assert s.info.exec_mode == 1 and s.info.kernels_per_run == 107
    s.set_mode("grid")
    assert s.info.exec_mode == 3 and s.info.kernels_per_run == 1


def test_two_contexts_on_two_streams(torch_cuda, orc):
    """Two contexts of different frame sizes enqueue on two streams at once
    (their persistent launches each span every SM; the runtime serialises
    them): both results equal the oracle's and neither run deadlocks."""
    from paper_1309_3848_b200.seeds import Seeds
    torch = torch_cuda
    f1, f2 = configs.frames("c1")[0], configs.frames("c2")[0]
    p1, p2 = configs.params("c1"), configs.params("c2")
    mk = lambda f, p: Seeds(f.shape[1], f.shape[0], 3, *[p[k] for k in (
        "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
    s1, s2 = mk(f1, p1), mk(f2, p2)
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    d1, d2 = torch.from_numpy(f1).cuda(), torch.from_numpy(f2).cuda()
    torch.cuda.synchronize()
    outs = []
    for _ in range(3):
        with torch.cuda.stream(a):
            l1 = s1.iterate(d1, stream=a)
        with torch.cuda.stream(b):
            l2 = s2.iterate(d2, stream=b)
        outs.append((l1, l2))
    torch.cuda.synchronize()
    r1, r2 = orc.run(f1, **p1).labels, orc.run(f2, **p2).labels
    for l1, l2 in outs:
        np.testing.assert_array_equal(l1.cpu().numpy(), r1)
        np.testing.assert_array_equal(l2.cpu().numpy(), r2)
    s1.close()
    s2.close()


def test_alternating_batch_sizes(torch_cuda, orc):
    """One context alternating batch sizes (24, 1, 8, 24, 1, query, 8): the
    cached tile plans (plan_grid's PlanSlot) are switched without re-planning
    and every result still equals the oracle's, including batches run after a
    fifth batch size evicted the oldest plan."""
    from paper_1309_3848_b200.seeds import Seeds
    torch = torch_cuda
    f = configs.frames("c3", n=24)
    p = configs.params("c3")
    s = Seeds(f.shape[2], f.shape[1], 3, *[p[k] for k in (
        "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
    d = torch.from_numpy(f).cuda()
    ref = {i: orc.run(f[i], **p).labels for i in (0, 3, 5, 23)}
    for n in (24, 1, 8, 24, 1, 5, 3, 2, 24, 8):
        lab = s.batch(d[:n]).cpu().numpy()
        s._refresh()  # seeds_query plans nf = 1
        for i in ref:
            if i < n:
                np.testing.assert_array_equal(lab[i], ref[i])
    s.close()


@pytest.mark.parametrize("mode", ["auto"])
@pytest.mark.parametrize("big_first", [True, False])
def test_interleaved_contexts_same_kernel(torch_cuda, orc, big_first, mode):
    """Two contexts with the same parameters (so the same k_grid
    instantiation) but different frame sizes, hence different dynamic shared
    memory per CTA: creating the second must not lower the first one's
    opt-in, whichever is larger."""
    from paper_1309_3848_b200.seeds import Seeds, SeedsError
    torch = torch_cuda
    p = configs.params("c3")
    big = configs.frames("c3", n=1)[0]
    small = np.ascontiguousarray(big[:96, :128])
    ps = dict(p, n_superpixels=max(4, p["n_superpixels"] * 96 * 128 // (big.shape[0] * big.shape[1])))
    mk = lambda f, q: Seeds(f.shape[1], f.shape[0], 3, *[q[k] for k in (
        "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
    order = [(big, p), (small, ps)] if big_first else [(small, ps), (big, p)]
    ctx = [mk(f, q) for f, q in order]
    try:
        for s in ctx:
            s.set_mode(mode)
    except SeedsError:
        pytest.skip(f"{mode} mode does not fit")
    for _ in range(2):
        for s, (f, q) in zip(ctx, order):
            lab = s.iterate(torch.from_numpy(f).cuda()).cpu().numpy()
            np.testing.assert_array_equal(lab, orc.run(f, **q).labels)
    for s in ctx:
        s.close()


@pytest.mark.parametrize("chunks", [0, 1])
def test_batch_host_warm_chain(torch_cuda, orc, chunks):
    """seeds_batch_host_warm: four streams of three frames each from host
    memory, every frame warm-started from the previous call's labels left on
    the device; equals the oracle's warm chain (reading O9) frame by frame, with
    and without the chunked copy pipeline.  A different frame count than the
    previous host call, or no previous call, is SEEDS_ESTATE (and leaves the
    chain as it was)."""
    from paper_1309_3848_b200.seeds import Seeds, SeedsError
    f = configs.frames("c2", n=12)
    p = configs.params("c2")
    streams = f.reshape(3, 4, *f.shape[1:])  # time x stream
    s = Seeds(f.shape[2], f.shape[1], 3, *[p[k] for k in (
        "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
    s.set_host_chunks(chunks)
    out = np.empty((4,) + f.shape[1:3], np.int32)
    with pytest.raises(SeedsError):
        s.batch_host_warm(np.ascontiguousarray(streams[0]), out)
    prev = [None] * 4
    for t in range(3):
        if t == 0:
            s.batch_host(np.ascontiguousarray(streams[0]), out)
        else:
            s.batch_host_warm(np.ascontiguousarray(streams[t]), out)
        for i in range(4):
            r = orc.run(streams[t, i], **p, init_labels=prev[i]).labels
            np.testing.assert_array_equal(out[i], r)
            prev[i] = r
    with pytest.raises(SeedsError):
        s.batch_host_warm(np.ascontiguousarray(streams[0, :2]), np.empty((2,) + f.shape[1:3], np.int32))
    s.batch_host_warm(np.ascontiguousarray(streams[0]), out)  # the rejected call left the chain intact
    for i in range(4):
        np.testing.assert_array_equal(out[i], orc.run(streams[0, i], **p, init_labels=prev[i]).labels)
    s.close()


def test_batch_host_pinned_single_frames(torch_cuda, orc):
    """seeds_batch_host / _warm on single frames in page-locked host buffers,
    then from pageable ones: a warm chain equal to the oracle's frame by frame."""
    torch = torch_cuda
    from paper_1309_3848_b200.seeds import Seeds
    f = configs.frames("c2", n=3)
    p = configs.params("c2")
    s = Seeds(f.shape[2], f.shape[1], 3, *[p[k] for k in (
        "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
    hin = torch.from_numpy(np.ascontiguousarray(f[:1])).pin_memory()
    hout = torch.full((1,) + f.shape[1:3], -1, dtype=torch.int32).pin_memory()
    s.batch_host(hin.numpy(), hout.numpy())
    r0 = orc.run(f[0], **p).labels
    np.testing.assert_array_equal(hout[0].numpy(), r0)
    hin.copy_(torch.from_numpy(f[1:2]))
    s.batch_host_warm(hin.numpy(), hout.numpy())
    r1 = orc.run(f[1], **p, init_labels=r0).labels
    np.testing.assert_array_equal(hout[0].numpy(), r1)
    out = np.empty((1,) + f.shape[1:3], np.int32)  # pageable buffers, the same chain
    s.batch_host_warm(np.ascontiguousarray(f[2:3]), out)
    np.testing.assert_array_equal(out[0], orc.run(f[2], **p, init_labels=r1).labels)
    s.close()


def test_video_host_chain(torch_cuda, orc):
    """seeds_video_host: three time steps of four streams from host memory in
    one call (copies of neighbouring steps overlapping each step's run), every
    step after the first warm-started from the previous one (reading O9); equals
    the oracle's warm chain frame by frame.  A second call with continue_prev
    continues the chain, as does a following seeds_batch_host_warm; continuing
    with another stream count, or without a previous host call, is SEEDS_ESTATE."""
    from paper_1309_3848_b200.seeds import Seeds, SeedsError
    f = configs.frames("c2", n=16)
    p = configs.params("c2")
    video = np.ascontiguousarray(f[:12].reshape(3, 4, *f.shape[1:]))  # time x stream
    s = Seeds(f.shape[2], f.shape[1], 3, *[p[k] for k in (
        "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
    out = np.empty(video.shape[:4], np.int32)
    with pytest.raises(SeedsError):
        s.video_host(video, out, continue_prev=True)
    s.video_host(video, out)
    prev = [None] * 4
    for t in range(3):
        for i in range(4):
            r = orc.run(video[t, i], **p, init_labels=prev[i]).labels
            np.testing.assert_array_equal(out[t, i], r)
            prev[i] = r
    # continue the chain: three more steps (their labels end in the second buffer and are carried back
    # for the next call), then one host_warm step
    more = np.ascontiguousarray(np.stack([video[1], video[0], video[2]]))
    out2 = np.empty(more.shape[:4], np.int32)
    s.video_host(more, out2, continue_prev=True)
    for t in range(3):
        for i in range(4):
            r = orc.run(more[t, i], **p, init_labels=prev[i]).labels
            np.testing.assert_array_equal(out2[t, i], r)
            prev[i] = r
    one = np.empty((4,) + f.shape[1:3], np.int32)
    s.batch_host_warm(np.ascontiguousarray(video[2]), one)
    for i in range(4):
        np.testing.assert_array_equal(one[i], orc.run(video[2, i], **p, init_labels=prev[i]).labels)
    with pytest.raises(SeedsError):  # another stream count cannot continue this chain
        s.video_host(np.ascontiguousarray(f[:2].reshape(1, 2, *f.shape[1:])), np.empty((1, 2) + f.shape[1:3], np.int32),
                     continue_prev=True)
    with pytest.raises(ValueError):
        s.video_host(video, np.empty((3, 4, 2, 2), np.int32))
    s.close()


@pytest.mark.parametrize("nt", ["512", "128"])
@pytest.mark.parametrize("seg2", ["0", "1"])
@pytest.mark.parametrize("cfg", ["c1", "c2", "c4"])
def test_segment_path_layouts(torch_cuda, orc, monkeypatch, cfg, seg2, nt):
    """The G-lane segment path of the small block levels with one pixel per
    lane (SEEDS_SEG2=0) and with two (SEEDS_SEG2=1: G >= area / 2, a cross
    count between the two slots of a lane; 128-thread plans only) -- AUTO
    picks per level and plan -- in both plan shapes (SEEDS_GRID_NT) equal the
    oracle bit for bit (labels, histograms, sizes)."""
    monkeypatch.setenv("SEEDS_SEG2", seg2)
    monkeypatch.setenv("SEEDS_GRID_NT", nt)
    torch = torch_cuda
    img = configs.frames(cfg, n=1)[0]
    p = configs.params(cfg)
    assert_parity(torch, orc, img, p, mode="grid")
