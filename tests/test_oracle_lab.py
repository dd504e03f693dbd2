"""Pins of the oracle's 8-bit CIELAB pre-pass (the paper
bins LAB; reading M3 in DESIGN.md: an integer fixed-point
conversion).  Checked against the CIE definitions evaluated in float64 with
numpy (written independently here), exact anchors and invariants.  No GPU."""
import numpy as np
import pytest


def lab_float(rgb):
    """CIELAB (D65) of 8-bit sRGB from the definitions, float64, then the 8-bit
    encoding L*255/100, a+128, b+128 rounded half up and clamped."""
    c = rgb.astype(np.float64) / 255.0
    lin = np.where(c <= 0.04045, c / 12.92, ((c + 0.055) / 1.055) ** 2.4)
    M = np.array([[0.412453, 0.357580, 0.180423], [0.212671, 0.715160, 0.072169],
                  [0.019334, 0.119193, 0.950227]])
    xyz = lin @ M.T / M.sum(1)          # X/Xn, Y/Yn, Z/Zn
    d = 6.0 / 29.0
    f = np.where(xyz > d ** 3, np.cbrt(xyz), xyz / (3 * d * d) + 4.0 / 29.0)
    L = 116 * f[..., 1] - 16
    a = 500 * (f[..., 0] - f[..., 1])
    b = 200 * (f[..., 1] - f[..., 2])
    out = np.stack([np.floor(L * 255 / 100 + 0.5), np.floor(a + 0.5) + 128, np.floor(b + 0.5) + 128], -1)
    return np.clip(out, 0, 255)


def test_lab_within_one_level_of_the_definition(orc):
    rng = np.random.default_rng(31)
    rgb = rng.integers(0, 256, (200000, 3)).astype(np.uint8)
    rgb[:256] = np.arange(256, dtype=np.uint8)[:, None]     # the grey axis
    got = orc.rgb_to_lab(rgb).astype(np.int64)
    want = lab_float(rgb)
    err = np.abs(got - want)
    assert err.max() <= 1
    assert (err == 0).mean() > 0.95


def test_lab_anchors_and_greys(orc):
    anchors = np.array([[255, 255, 255], [0, 0, 0]], np.uint8)
    np.testing.assert_array_equal(orc.rgb_to_lab(anchors), [[255, 128, 128], [0, 128, 128]])
    grey = np.repeat(np.arange(256, dtype=np.uint8)[:, None], 3, 1)
    lab = orc.rgb_to_lab(grey).astype(np.int64)
    assert (lab[:, 1] == 128).all() and (lab[:, 2] == 128).all()   # X = Y = Z on the grey axis
    assert (np.diff(lab[:, 0]) >= 0).all()                          # L monotone in the grey level


def test_lab_run_invariants(orc):
    """A LAB run: H equals the recount of the LAB bins, sizes sum to N."""
    from paper_1309_3848_b200 import configs
    img = configs.frames("c1", 1)[0]
    p = configs.params("c1")
    r = orc.run(img, **p, colour="lab")
    lab = orc.rgb_to_lab(img)
    bins = orc.quantise(lab, p["bins_per_channel"])
    B = p["bins_per_channel"] ** 3
    h = np.bincount((r.labels.astype(np.int64) * B + bins).ravel(), minlength=r.k_act * B).reshape(r.k_act, B)
    np.testing.assert_array_equal(h, r.hist)
    assert r.sizes.sum() == img.shape[0] * img.shape[1] and (r.sizes > 0).all()
    assert not np.array_equal(r.labels, orc.run(img, **p).labels)  # the colour space matters


def test_lab_needs_three_channels(orc):
    with pytest.raises(ValueError):
        orc.rgb_to_lab(np.zeros((4, 4, 1), np.uint8))
