"""Row-band mode (include/seeds.h): any number of bands gives the one-GPU
result bit for bit.

* seeds_create_bands: every band in one launch on this GPU -- each band with
  its own label plane and the histograms of the superpixels it owns, halo rows
  written into the neighbours' planes and histogram updates sent to the owner
  band inside the kernel, exactly the exchange of a multi-GPU run with peer
  memory replaced by other buffers of the same device;
* seeds_create_banded with world = 1: the cross-device code path (sys-scope
  counter barrier after the local one, IPC bootstrap) on one rank;
* two processes on one GPU map each other's buffers through CUDA IPC (the
  bootstrap of a multi-GPU run; their kernels are not run together -- they
  would wait on each other on one device).
Needs a B200."""
import os
import socket

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


def band_run(torch, img, p, n_bands, init=None, colour="rgb", repeat=1):
    from paper_1309_3848_b200.seeds import SeedsBands
    H, W, C = img.shape
    s = SeedsBands(W, H, C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"], p["smoothness_prior"],
                   p["iters_per_level"], n_bands)
    s.set_colour_space(colour)
    d = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    di = None if init is None else torch.from_numpy(np.ascontiguousarray(init, np.int32)).cuda()
    for _ in range(repeat):
        lab = s.run(d, di)
    torch.cuda.synchronize()
    h, a = s.read_state(0)
    out = lab.cpu().numpy(), h.cpu().numpy(), a.cpu().numpy(), (s.row0, s.row1, s.n_bands, s.band)
    s.close()
    return out


@pytest.mark.parametrize("n_bands", [1, 2, 3, 6])
def test_c1_bands_equal_oracle(torch_cuda, orc, n_bands):
    img = configs.frames("c1")[0]
    p = configs.params("c1")
    lab, h, a, info = band_run(torch_cuda, img, p, n_bands)
    r = orc.run(img, **p)
    assert info == (0, img.shape[0], n_bands, -1)
    np.testing.assert_array_equal(lab, r.labels)
    np.testing.assert_array_equal(h, r.hist)
    np.testing.assert_array_equal(a, r.sizes)


@pytest.mark.parametrize("n_bands", [2, 5, 8])
def test_c2_bands_equal_oracle(torch_cuda, orc, n_bands):
    img = configs.frames("c2")[0]
    p = configs.params("c2")
    lab, h, a, _ = band_run(torch_cuda, img, p, n_bands, repeat=2)
    r = orc.run(img, **p)
    np.testing.assert_array_equal(lab, r.labels)
    np.testing.assert_array_equal(h, r.hist)
    np.testing.assert_array_equal(a, r.sizes)


def test_bands_gamma0_warm_start(torch_cuda, orc):
    f, _ = mosaic.moving_mosaic(2, 200, 120, 15, 8.0, seed=7)
    p = dict(n_superpixels=40, n_levels=3, bins_per_channel=5, smoothness_prior=0, iters_per_level=3)
    r0 = orc.run(f[0], **p)
    lab, h, _, _ = band_run(torch_cuda, f[1], p, 3, init=r0.labels)
    r1 = orc.run(f[1], **p, init_labels=r0.labels)
    np.testing.assert_array_equal(lab, r1.labels)
    np.testing.assert_array_equal(h, r1.hist)


@pytest.mark.parametrize("n_bands", [4, 7])
def test_c5_crop_bands_equal_oracle(torch_cuda, orc, n_bands):
    """512 bins (uint16 bin plane), 5 block levels, multi-tile 128-thread plans."""
    f = np.ascontiguousarray(configs.frames("c5", n=1)[0, :768, :1024])
    p = dict(configs.params("c5"))
    p["n_superpixels"] = 20000 * 768 * 1024 // (8192 * 8192)
    lab, h, a, _ = band_run(torch_cuda, f, p, n_bands)
    r = orc.run(f, **p)
    np.testing.assert_array_equal(lab, r.labels)
    np.testing.assert_array_equal(h, r.hist)
    np.testing.assert_array_equal(a, r.sizes)


@pytest.mark.parametrize("n_bands", [1, 3])
def test_c2_bands_lab(torch_cuda, orc, n_bands):
    img = configs.frames("c2")[0]
    p = configs.params("c2")
    lab, h, _, _ = band_run(torch_cuda, img, p, n_bands, colour="lab")
    r = orc.run(img, **p, colour="lab")
    np.testing.assert_array_equal(lab, r.labels)
    np.testing.assert_array_equal(h, r.hist)


def test_bands_reject_single_gpu_features(torch_cuda):
    from paper_1309_3848_b200.seeds import SeedsBands, SeedsError
    b = SeedsBands(64, 48, 3, 12, 2, 4, 1, 3, 2)
    for call in (lambda: b.set_means_iters(1), lambda: b.set_time_budget(10), lambda: b.set_compactness(True)):
        with pytest.raises(SeedsError):
            call()
    b.close()
    with pytest.raises(SeedsError):  # more bands than superpixel rows
        SeedsBands(64, 48, 3, 12, 2, 4, 1, 3, 9)


@pytest.mark.parametrize("cfg", ["c2", "c1"])
def test_cross_device_path_world1(torch_cuda, orc, cfg):
    """seeds_create_banded(rank 0, world 1): the sys-scope band barrier (its
    counters carried from run to run) gives the oracle's result, three runs in
    a row."""
    torch = torch_cuda
    from paper_1309_3848_b200.seeds import SeedsBand
    img = configs.frames(cfg)[0]
    p = configs.params(cfg)
    H, W, C = img.shape
    s = SeedsBand(W, H, C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"], p["smoothness_prior"],
                  p["iters_per_level"], 0, 1)
    assert (s.row0, s.row1, s.n_bands, s.band) == (0, H, 1, 0)
    d = torch.from_numpy(img).cuda()
    r = orc.run(img, **p)
    for _ in range(3):
        lab = s.run(d)
        np.testing.assert_array_equal(lab.cpu().numpy(), r.labels)
    np.testing.assert_array_equal(s.read_state(0)[0].cpu().numpy(), r.hist)
    s.close()


def _free_port():
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def _ipc_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1309_3848_b200 import bands
        p = configs.params("c2")
        b = bands.make_band(481, 321, 3, p["n_superpixels"], p["n_levels"], p["bins_per_channel"],
                            p["smoothness_prior"], p["iters_per_level"], bootstrap="caller")
        q.put((rank, b.row0, b.row1, b.n_bands, b.band, len(b.export())))
        dist.barrier()
        b.close()
    except Exception as e:  # report, do not hang the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_process_ipc_bootstrap(torch_cuda):
    """Two ranks (both on GPU 0) create their bands, exchange export() blobs
    over gloo and map each other's buffers (seeds_band_connect); the band
    rows tile the frame."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=300)
        res[r[0]] = r
    for pr in procs:
        pr.join(timeout=120)
    assert all(len(v) == 6 for v in res.values()), res
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == 321
    assert res[0][3:5] == (2, 0) and res[1][3:5] == (2, 1)
    for pr in procs:
        assert pr.exitcode == 0
