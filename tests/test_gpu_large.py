"""GPU checks at BASELINE.json's large sizes (c4 video, c5 8192x8192, 512 bins).

c4: one clip of the 1920x1080 video (frame 0 cold, frames 1..7 warm-started
from the previous output, reading Q14/O9) is compared with the oracle's own
chain element by element, and a two-clip batch likewise.

c5: the full-size run is checked by properties that hold at any size -- labels in
range, every superpixel non-empty and one 4-connected component,
H equal to a recount from (labels, bins) and summing to A (Eq. 6), the sizes
summing to N -- and by bit-equality of two independent execution modes (grid
and graph).  A 1024x1024 crop with the same superpixel size and 512 bins is
compared with the oracle bit for bit, and so is the full frame (labels,
histograms, sizes; about a minute of one host core for the oracle).  Needs a B200: every test is marked gpu."""
import os

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


def ctx(img_shape, p, mode):
    from paper_1309_3848_b200.seeds import Seeds
    H, W, C = img_shape
    s = Seeds(W, H, C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"],
              p["smoothness_prior"], p["iters_per_level"])
    s.set_mode(mode)
    return s


@pytest.mark.parametrize("mode", ["grid", "graph"])
def test_c4_clip_warm_chain(torch_cuda, orc, mode):
    """Clip 0 of c4: frame 0 cold, frames 1..7 warm from the previous labels;
    every frame's labels, histograms and sizes equal the oracle's chain."""
    torch = torch_cuda
    f = configs.frames("c4", n=8)
    p = configs.params("c4")
    s = ctx(f.shape[1:], p, mode)
    prev_gpu, prev_ref = None, None
    for t in range(8):
        d = torch.from_numpy(np.ascontiguousarray(f[t:t + 1])).cuda()
        lab = s.batch(d, init_labels=prev_gpu)
        h, a = s.read_state(0)
        r = orc.run(f[t], **p, init_labels=prev_ref)
        np.testing.assert_array_equal(lab[0].cpu().numpy(), r.labels, err_msg=f"labels t={t}")
        np.testing.assert_array_equal(h.cpu().numpy(), r.hist, err_msg=f"hist t={t}")
        np.testing.assert_array_equal(a.cpu().numpy(), r.sizes, err_msg=f"sizes t={t}")
        prev_gpu, prev_ref = lab, r.labels


def test_c4_two_clips_batched(torch_cuda, orc):
    """Two clips advanced together (one batch of 2 frames per time step, the
    bench's layout): frames t = 0, 1, 2 of both clips equal the oracle's chains."""
    torch = torch_cuda
    c = configs.CONFIGS["c4"]
    f = configs.frames("c4", n=c["clip"] + 3)
    p = configs.params("c4")
    clips = [f[0:3], f[c["clip"]:c["clip"] + 3]]
    s = ctx(f.shape[1:], p, "auto")
    prev, refs = None, [None, None]
    for t in range(3):
        d = torch.from_numpy(np.ascontiguousarray(np.stack([clips[0][t], clips[1][t]]))).cuda()
        lab = s.batch(d, init_labels=prev)
        for i in range(2):
            r = orc.run(clips[i][t], **p, init_labels=refs[i])
            np.testing.assert_array_equal(lab[i].cpu().numpy(), r.labels, err_msg=f"clip {i} t={t}")
            refs[i] = r.labels
        prev = lab


def test_c5_crop_oracle_parity(torch_cuda, orc):
    """1024x1024 crop of c5 with K scaled to keep the superpixel size (512 bins,
    uint16 bin plane, 5 block levels): bit-exact against the oracle."""
    torch = torch_cuda
    f = np.ascontiguousarray(configs.frames("c5", n=1)[0, :1024, :1024])
    p = dict(configs.params("c5"))
    p["n_superpixels"] = 20000 * 1024 * 1024 // (8192 * 8192)
    s = ctx(f.shape, p, "auto")
    lab = s.iterate(torch.from_numpy(f).cuda())
    h, a = s.read_state(0)
    r = orc.run(f, **p)
    np.testing.assert_array_equal(lab.cpu().numpy(), r.labels)
    np.testing.assert_array_equal(h.cpu().numpy(), r.hist)
    np.testing.assert_array_equal(a.cpu().numpy(), r.sizes)


def _bins(torch, img, bpc):
    """Uniform bins of the test's own (reading Q1: q_c = v_c bpc >> 8, channel 0
    most significant) -- restated here, not shared with either implementation."""
    v = img.to(torch.int64)
    b = torch.zeros(v.shape[:2], dtype=torch.int64, device=v.device)
    for ch in range(v.shape[2]):
        b = b * bpc + ((v[..., ch] * bpc) >> 8)
    return b


def test_c5_full_frame_properties_and_modes(torch_cuda, orc):
    torch = torch_cuda
    from scipy import sparse
    from scipy.sparse.csgraph import connected_components
    f = configs.frames("c5", n=1)[0]
    p = configs.params("c5")
    d = torch.from_numpy(f).cuda()
    outs = {}
    for mode in ("grid", "graph"):
        s = ctx(f.shape, p, mode)
        lab = s.iterate(d)
        h, a = s.read_state(0)
        outs[mode] = (lab, h, a, s.info)
        s.close()
    lab, h, a, info = outs["grid"]
    assert torch.equal(lab, outs["graph"][0]) and torch.equal(h, outs["graph"][1])
    K, B = info.k_actual, info.bins_total
    N = f.shape[0] * f.shape[1]
    assert int(lab.min()) >= 0 and int(lab.max()) < K
    # H is the recount of (labels, bins) and sums to A; sizes sum to N
    bins = _bins(torch, d, p["bins_per_channel"])
    recount = torch.bincount((lab.to(torch.int64) * B + bins).flatten(), minlength=K * B).view(K, B)
    assert torch.equal(recount.to(torch.int32), h)
    assert torch.equal(h.sum(1), a) and int(a.sum()) == N and bool((a > 0).all())
    # every superpixel is one 4-connected component
    L = lab.cpu().numpy()
    Hh, Ww = L.shape
    idx = np.arange(Hh * Ww, dtype=np.int64).reshape(Hh, Ww)
    eh = L[:, 1:] == L[:, :-1]
    ev = L[1:, :] == L[:-1, :]
    rows = np.concatenate([idx[:, 1:][eh], idx[1:, :][ev]])
    cols = np.concatenate([idx[:, :-1][eh], idx[:-1, :][ev]])
    g = sparse.coo_matrix((np.ones(rows.size, np.int8), (rows, cols)), shape=(Hh * Ww, Hh * Ww))
    ncomp, _ = connected_components(g, directed=False)
    assert ncomp == K
    # the full frame against the oracle (about a minute of one host core)
    r = orc.run(f, **p)
    np.testing.assert_array_equal(L, r.labels)
    np.testing.assert_array_equal(h.cpu().numpy(), r.hist)
    np.testing.assert_array_equal(a.cpu().numpy(), r.sizes)


def test_multi_tile_plans_are_deterministic(torch_cuda):
    """Plans whose CTAs own several tiles (TMA prefetch of the next tile while
    the current one is decided): repeated runs through the device and the host
    entry points give identical labels and histograms (c4 batch of 8 frames,
    and the c5 frame)."""
    torch = torch_cuda
    for cfg, n in (("c4", 8), ("c5", 1)):
        f = configs.frames(cfg, n=n)
        p = configs.params(cfg)
        s = ctx(f.shape[1:], p, "auto")
        d = torch.from_numpy(f).cuda()
        ref = s.batch(d).clone()
        ref_h = s.read_state(n - 1)[0].clone()
        for _ in range(3):
            assert torch.equal(s.batch(d), ref)
            assert torch.equal(s.read_state(n - 1)[0], ref_h)
        out = np.empty((n,) + f.shape[1:3], np.int32)
        s.batch_host(np.ascontiguousarray(f), out)
        np.testing.assert_array_equal(out, ref.cpu().numpy())
        s.close()


def test_c4_video_host_matches_device(torch_cuda):
    """The c4 video (8 clips x 4 frames) through one seeds_video_host call
    (pinned buffers, copies overlapping the runs): identical to the device
    entry point chained frame by frame with explicit previous labels."""
    torch = torch_cuda
    cl = configs.clips("c4")[:, :4]
    p = configs.params("c4")
    s = ctx(cl.shape[2:], p, "auto")
    video = torch.from_numpy(np.ascontiguousarray(cl.transpose(1, 0, 2, 3, 4))).pin_memory()  # time x clip
    out = torch.empty(video.shape[:4], dtype=torch.int32).pin_memory()
    s.video_host(video.numpy(), out.numpy())
    prev = None
    for t in range(video.shape[0]):
        ref = s.batch(video[t].cuda(), init_labels=prev)
        np.testing.assert_array_equal(out[t].numpy(), ref.cpu().numpy())
        prev = ref.clone()
    s.close()


def test_c4_host_warm_chain_matches_device(torch_cuda):
    """The c4 video (8 clips) through seeds_batch_host_warm, frame 0 cold, then
    frames 1-3 warm from the labels the previous host call left on the device
    (device-entry runs in between do not disturb them): identical to the device entry point given the previous labels explicitly."""
    torch = torch_cuda
    cl = configs.clips("c4")[:, :4]
    p = configs.params("c4")
    s = ctx(cl.shape[2:], p, "auto")
    out = np.empty((cl.shape[0],) + cl.shape[2:4], np.int32)
    prev = None
    for t in range(cl.shape[1]):
        x = np.ascontiguousarray(cl[:, t])
        if t == 0:
            s.batch_host(x, out)
        else:
            s.batch_host_warm(x, out)
        ref = s.batch(torch.from_numpy(x).cuda(), init_labels=prev)
        np.testing.assert_array_equal(out, ref.cpu().numpy())
        prev = ref.clone()
    s.close()
