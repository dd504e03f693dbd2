"""GPU checks of the C-ABI boundary's error behaviour and of the anytime
budget (include/seeds.h):

* warm-start labels outside [0, K_act) never index out of bounds: the run is
  flagged and the next synchronising call returns SEEDS_ESTATE (-5)
  (seeds_batch contract; PAPER.md:259-262 defines the valid set S);
* seeds_validate_labels finds out-of-range, missing and non-4-connected
  superpixels, and seeds_set_validate rejects such warm starts before the run;
* seeds_set_time_budget stops at a sub-sweep boundary; the count reached,
  replayed through seeds_debug_limit and the oracle's max_subsweeps, gives the
  same labels and histograms bit for bit.

Needs a B200: every test is marked gpu."""
import numpy as np
import pytest

from paper_1309_3848_b200 import configs

pytestmark = pytest.mark.gpu

ESTATE = -5


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1309_3848_b200 import build
    build.build()
    return torch


def mk(img_shape, p, mode="auto"):
    from paper_1309_3848_b200.seeds import Seeds
    H, W, C = img_shape
    s = Seeds(W, H, C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"], p["smoothness_prior"],
              p["iters_per_level"])
    s.set_mode(mode)
    return s


@pytest.mark.parametrize("mode", ["grid", "graph"])
@pytest.mark.parametrize("bad", [-1, "K", 65535, -2 ** 31])
def test_out_of_range_init_labels_flag_estate(torch_cuda, orc, mode, bad):
    from paper_1309_3848_b200.seeds import SeedsError
    torch = torch_cuda
    img = configs.frames("c1")[0]
    p = configs.params("c1")
    s = mk(img.shape, p, mode)
    good = orc.run(img, **p).labels
    init = good.copy()
    init[7, 11] = s.info.k_actual if bad == "K" else bad
    d = torch.from_numpy(img).cuda()[None]
    s.batch(d, init_labels=torch.from_numpy(init).cuda()[None])
    with pytest.raises(SeedsError) as e:
        s.read_state(0)
    assert e.value.status == ESTATE
    # the flag is reported once; a valid warm start afterwards is clean and exact
    lab = s.batch(d, init_labels=torch.from_numpy(good).cuda()[None])
    h, a = s.read_state(0)
    r = orc.run(img, **p, init_labels=good)
    np.testing.assert_array_equal(lab[0].cpu().numpy(), r.labels)
    np.testing.assert_array_equal(h.cpu().numpy(), r.hist)
    s.close()


def test_out_of_range_init_labels_host_entry(torch_cuda, orc):
    from paper_1309_3848_b200.seeds import SeedsError
    img = configs.frames("c1", n=2)
    p = configs.params("c1")
    s = mk(img.shape[1:], p)
    init = np.stack([orc.run(f, **p).labels for f in img]).astype(np.int32)
    init[1, 0, 0] = 999
    out = np.empty(init.shape, np.int32)
    with pytest.raises(SeedsError) as e:
        s.batch_host(np.ascontiguousarray(img), out, init_labels=init)
    assert e.value.status == ESTATE
    s.close()


def test_validate_labels(torch_cuda, orc):
    from paper_1309_3848_b200.seeds import SeedsError
    torch = torch_cuda
    img = configs.frames("c2")[0]
    p = configs.params("c2")
    s = mk(img.shape, p)
    K = s.info.k_actual
    good = orc.run(img, **p).labels
    assert s.validate_labels(torch.from_numpy(good).cuda()) == (0, -1, -1)
    grid = orc.run(img, **dict(p, iters_per_level=0)).labels
    assert s.validate_labels(torch.from_numpy(np.stack([grid, good])).cuda()) == (0, -1, -1)
    # a missing superpixel: k merged into the label of its first 4-neighbour
    k = 37
    ys, xs = np.nonzero(good == k)
    n = good[ys[0] - 1, xs[0]] if ys[0] > 0 else good[ys[0], xs[0] - 1]
    miss = good.copy()
    miss[good == k] = n
    with pytest.raises(SeedsError) as e:
        s.validate_labels(torch.from_numpy(miss).cuda())
    assert e.value.status == ESTATE and "no pixel" in str(e.value)
    # a split superpixel: one far pixel of another superpixel relabelled k
    split = good.copy()
    Hh, Ww = good.shape
    corners = [(0, 0, 1, 0, 0, 1), (0, Ww - 1, 1, Ww - 1, 0, Ww - 2), (Hh - 1, 0, Hh - 2, 0, Hh - 1, 1),
               (Hh - 1, Ww - 1, Hh - 2, Ww - 1, Hh - 1, Ww - 2)]
    # a corner pixel whose two neighbours share its label: relabelling it keeps its own superpixel connected
    y0, x0 = next((y, x) for y, x, ya, xa, yb, xb in corners
                  if good[y, x] != k and good[ya, xa] == good[yb, xb] == good[y, x])
    split[y0, x0] = k
    with pytest.raises(SeedsError) as e:
        s.validate_labels(torch.from_numpy(np.stack([good, split])).cuda())
    assert e.value.status == ESTATE and "frame 1" in str(e.value) and "4-connected" in str(e.value)
    # out of range
    oor = good.copy()
    oor[3, 3] = K
    oor[4, 4] = -7
    with pytest.raises(SeedsError) as e:
        s.validate_labels(torch.from_numpy(oor).cuda())
    assert "2 labels outside" in str(e.value)
    s.close()


def test_validating_warm_start(torch_cuda, orc):
    """seeds_set_validate(1): an invalid warm start is rejected before the run
    (nothing enqueued), a valid one runs exactly as without validation."""
    from paper_1309_3848_b200.seeds import SeedsError
    torch = torch_cuda
    f = configs.frames("c4", n=2)
    p = configs.params("c4")
    s = mk(f.shape[1:], p)
    s.set_validate(True)
    prev = orc.run(f[0], **p).labels
    bad = prev.copy()
    bad[100, 100] = bad[500, 900] if bad[500, 900] != bad[100, 100] else bad[0, 0]
    d = torch.from_numpy(f[1:2]).cuda()
    try:
        s.validate_labels(torch.from_numpy(bad).cuda())
        pytest.skip("the relabelled pixel happened to keep the partition valid")
    except SeedsError:
        pass
    with pytest.raises(SeedsError) as e:
        s.batch(d, init_labels=torch.from_numpy(bad).cuda()[None])
    assert e.value.status == ESTATE
    lab = s.batch(d, init_labels=torch.from_numpy(prev).cuda()[None])
    r = orc.run(f[1], **p, init_labels=prev)
    np.testing.assert_array_equal(lab[0].cpu().numpy(), r.labels)
    s.close()


@pytest.mark.parametrize("cfg,frac", [("c2", 0.5), ("c2", 0.15), ("c1", 0.6)])
def test_time_budget_replays_exactly(torch_cuda, orc, cfg, frac):
    """Anytime termination: measure a full run, give a budget of a fraction of
    it; the run stops after r sub-sweeps (0 < r < total), its labels and
    histograms equal the oracle's run with max_subsweeps = r and the GPU's
    own run with seeds_debug_limit(r)."""
    torch = torch_cuda
    img = configs.frames(cfg)[0]
    p = configs.params(cfg)
    s = mk(img.shape, p)
    d = torch.from_numpy(img).cuda()
    total = s.info.subsweeps
    s.iterate(d)
    assert s.last_subsweeps() == total
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    times = []
    for _ in range(5):
        ev[0].record()
        s.iterate(d)
        ev[1].record()
        torch.cuda.synchronize()
        times.append(ev[0].elapsed_time(ev[1]))
    budget_us = max(1, int(min(times) * 1000 * frac))
    s.set_time_budget(budget_us)
    lab = s.iterate(d).cpu().numpy()
    r = s.last_subsweeps()
    h, a = s.read_state(0)
    print(f"{cfg}: full run {min(times) * 1000:.0f} us, budget {budget_us} us -> {r}/{total} sub-sweeps")
    assert 0 < r < total
    ref = orc.run(img, **p, max_subsweeps=r)
    np.testing.assert_array_equal(lab, ref.labels)
    np.testing.assert_array_equal(h.cpu().numpy(), ref.hist)
    np.testing.assert_array_equal(a.cpu().numpy(), ref.sizes)
    s.set_time_budget(0)
    s.debug_limit(r)
    np.testing.assert_array_equal(s.iterate(d).cpu().numpy(), lab)
    assert s.last_subsweeps() == r
    s.close()


def test_time_budget_edges(torch_cuda, orc):
    """A budget above the run time changes nothing; a 1 us budget stops at the
    first boundaries with a valid partition equal to the oracle's prefix; a
    batch stops all frames after the same sub-sweep."""
    torch = torch_cuda
    f = configs.frames("c3", n=4)
    p = configs.params("c3")
    s = mk(f.shape[1:], p)
    d = torch.from_numpy(f).cuda()
    full = s.batch(d).clone()
    s.set_time_budget(10 ** 7)
    assert torch.equal(s.batch(d), full) and s.last_subsweeps() == s.info.subsweeps
    s.set_time_budget(1)
    lab = s.batch(d).cpu().numpy()
    r = s.last_subsweeps()
    assert 0 <= r <= 2
    for i in range(4):
        ref = orc.run(f[i], **p, max_subsweeps=r)
        np.testing.assert_array_equal(lab[i], ref.labels)
        np.testing.assert_array_equal(s.read_state(i)[0].cpu().numpy(), ref.hist)
    s.close()


def test_time_budget_rejected_in_graph_mode(torch_cuda):
    from paper_1309_3848_b200.seeds import SeedsError
    s = mk((120, 160, 3), configs.params("c1"), "graph")
    with pytest.raises(SeedsError):
        s.set_time_budget(100)
    s.close()
