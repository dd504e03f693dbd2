"""BASELINE.json's five workloads as parameter sets.

Pure data: no method arithmetic.  ``frames(cfg)`` draws the synthetic input of
a config with the seeded generator in ``mosaic.py`` (seed = 1000 * index).
Readings Q4 (n_levels counts block levels), Q12 (I = 4 where unstated) and Q13
(gamma: 1 for c1-c3 and c5, 0 for the warm-started video c4) are DESIGN.md's.
"""
from __future__ import annotations

import os

import numpy as np

from . import mosaic

CONFIGS = {
    "c1": dict(index=0, W=160, H=120, C=3, K=48, L=2, bpc=5, gamma=1, iters=2,
               R=12, sigma=8.0, grad=0.0, frames=1),
    "c2": dict(index=1, W=481, H=321, C=3, K=200, L=4, bpc=5, gamma=1, iters=4,
               R=40, sigma=10.0, grad=30.0, frames=1),
    "c3": dict(index=2, W=481, H=321, C=3, K=400, L=4, bpc=5, gamma=1, iters=4,
               R=(40, 80), sigma=(5.0, 15.0), grad=30.0, frames=256),
    "c4": dict(index=3, W=1920, H=1080, C=3, K=1000, L=5, bpc=5, gamma=0, iters=4,
               R=150, sigma=8.0, grad=30.0, frames=64, clip=8),
    "c5": dict(index=4, W=8192, H=8192, C=3, K=20000, L=6, bpc=8, gamma=1, iters=4,
               R=5000, sigma=10.0, grad=30.0, frames=1),
}


def params(cfg: str) -> dict:
    c = CONFIGS[cfg]
    return dict(n_superpixels=c["K"], n_levels=c["L"], bins_per_channel=c["bpc"],
                smoothness_prior=c["gamma"], iters_per_level=c["iters"])


CACHE_DIR = os.environ.get("SEEDS_INPUT_CACHE", "/tmp/seeds_inputs")


def frames(cfg: str, n: int | None = None):
    """(n, H, W, C) uint8 frames of config ``cfg``.  Large inputs are cached as
    .npy under CACHE_DIR (a speed-up only: a missing or unreadable cache file
    is regenerated from the seed)."""
    c = CONFIGS[cfg]
    n_ = c["frames"] if n is None else n
    if c["W"] * c["H"] * n_ >= 4_000_000:
        path = os.path.join(CACHE_DIR, f"{cfg}_{c['index']}_{n_}.npy")
        try:
            out = np.load(path)
            if out.shape == (n_, c["H"], c["W"], c["C"]) and out.dtype == np.uint8:
                return out
        except Exception:
            pass
        out = _frames(cfg, n_)
        try:
            os.makedirs(CACHE_DIR, exist_ok=True)
            tmp = f"{path}.{os.getpid()}.npy"
            np.save(tmp, out)
            os.replace(tmp, path)
        except Exception:
            pass
        return out
    return _frames(cfg, n_)


def clips(cfg: str = "c4"):
    """The video of ``cfg`` as (n_clips, clip_len, H, W, C): clip c is frames
    [c * clip_len, (c + 1) * clip_len) (reading Q14: clips of 8 frames; frame 0
    of a clip starts cold, the others from the previous frame's labels)."""
    c = CONFIGS[cfg]
    f = frames(cfg)
    L = c["clip"]
    return f.reshape(c["frames"] // L, L, c["H"], c["W"], c["C"])


def _frames(cfg: str, n: int):
    c = CONFIGS[cfg]
    seed = 1000 * c["index"]
    if cfg == "c3":
        return mosaic.mosaic_batch(n, c["W"], c["H"], c["R"][0], c["R"][1], c["sigma"][0],
                                   c["sigma"][1], seed=seed, grad=c["grad"], C=c["C"])
    if cfg == "c4":
        f, _ = mosaic.moving_mosaic(n, c["W"], c["H"], c["R"], c["sigma"], seed=seed,
                                    grad=c["grad"], C=c["C"])
        return f
    out = np.empty((n, c["H"], c["W"], c["C"]), np.uint8)
    for i in range(n):
        out[i] = mosaic.mosaic(c["W"], c["H"], c["R"], c["sigma"], seed=seed + i, C=c["C"],
                               grad=c["grad"])
    return out


def regions(cfg: str, n: int | None = None) -> np.ndarray:
    """(n, H, W) int32 ground-truth region maps of ``frames(cfg, n)``: the
    Voronoi region of every pixel (the mosaic's objects), for the quality
    metrics of SURVEY 8(f) rank 2.  Large maps are cached like the frames."""
    c = CONFIGS[cfg]
    n_ = c["frames"] if n is None else n
    path = os.path.join(CACHE_DIR, f"{cfg}_{c['index']}_{n_}_regions.npy")
    big = c["W"] * c["H"] * n_ >= 4_000_000
    if big:
        try:
            out = np.load(path)
            if out.shape == (n_, c["H"], c["W"]) and out.dtype == np.int32:
                return out
        except Exception:
            pass
    seed = 1000 * c["index"]
    if cfg == "c3":
        _, out = mosaic.mosaic_batch(n_, c["W"], c["H"], c["R"][0], c["R"][1], c["sigma"][0], c["sigma"][1],
                                     seed=seed, grad=c["grad"], C=c["C"], return_regions=True)
    elif cfg == "c4":
        _, out = mosaic.moving_mosaic(n_, c["W"], c["H"], c["R"], c["sigma"], seed=seed, grad=c["grad"], C=c["C"])
    else:
        out = np.stack([mosaic.mosaic(c["W"], c["H"], c["R"], c["sigma"], seed=seed + i, C=c["C"], grad=c["grad"],
                                      return_regions=True)[1] for i in range(n_)])
    if big:
        try:
            os.makedirs(CACHE_DIR, exist_ok=True)
            tmp = f"{path}.{os.getpid()}.npy"
            np.save(tmp, out)
            os.replace(tmp, path)
        except Exception:
            pass
    return out


def n_regions(cfg: str, frame: int = 0) -> int:
    """Number of ground-truth regions of frame ``frame`` (ids are 0..R-1)."""
    return int(regions(cfg, frame + 1)[frame].max()) + 1
