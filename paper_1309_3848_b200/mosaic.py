"""Seeded synthetic Voronoi-mosaic frames: the inputs shared by the oracle and
the CUDA path (recipe G1).

This module holds none of the method's arithmetic -- only random input
generation.  The paper measures on BSD natural images (PAPER.md:671-676,
S6); the dataset is not available, so these mosaics stand in for it with the
frame shape, superpixel counts and bin counts of BASELINE.json's configs.

Recipe (numpy PCG64, seed = 1000 * cfg_index + frame_index by convention):
  * R sites uniform-real in [0, W) x [0, H); a pixel belongs to the site
    nearest to its centre (x + .5, y + .5) (scipy cKDTree);
  * region mean colour uniform integers in [0, 255]^C;
  * optional linear gradient: direction theta ~ U[0, 2 pi), per-channel
    amplitude a_c ~ U[-grad, grad]; value += a_c * ((t - t_min)/(t_max - t_min) - 1/2)
    with t the projection of the pixel centre on theta over the region;
  * i.i.d. Gaussian noise N(0, sigma^2) per pixel and channel, np.rint, clip
    to [0, 255] -> uint8 HWC.
"""
from __future__ import annotations

import numpy as np
from scipy.spatial import cKDTree


def _regions(sites: np.ndarray, W: int, H: int) -> np.ndarray:
    ys, xs = np.mgrid[0:H, 0:W]
    pts = np.stack([xs.ravel() + 0.5, ys.ravel() + 0.5], axis=1)
    _, idx = cKDTree(sites).query(pts, k=1)
    return idx.reshape(H, W).astype(np.int32)


def _paint(rng, region, R, W, H, C, grad, colours=None, grad_params=None):
    if colours is None:
        colours = rng.integers(0, 256, size=(R, C)).astype(np.float64)
    img = colours[region]  # (H, W, C)
    if grad > 0:
        if grad_params is None:
            theta = rng.uniform(0.0, 2 * np.pi, size=R)
            amp = rng.uniform(-grad, grad, size=(R, C))
        else:
            theta, amp = grad_params
        ys, xs = np.mgrid[0:H, 0:W]
        t = (xs + 0.5) * np.cos(theta)[region] + (ys + 0.5) * np.sin(theta)[region]
        flat_r = region.ravel()
        tmin = np.full(R, np.inf)
        tmax = np.full(R, -np.inf)
        np.minimum.at(tmin, flat_r, t.ravel())
        np.maximum.at(tmax, flat_r, t.ravel())
        span = np.where(tmax > tmin, tmax - tmin, 1.0)
        u = (t - tmin[region]) / span[region] - 0.5
        img = img + amp[region] * u[..., None]
    return img, colours


def _finish(rng, img, sigma):
    img = img + rng.normal(0.0, sigma, size=img.shape)
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def mosaic(W: int, H: int, R: int, sigma: float, seed: int, C: int = 3, grad: float = 0.0,
           return_regions: bool = False):
    """One (H, W, C) uint8 Voronoi mosaic frame."""
    rng = np.random.Generator(np.random.PCG64(seed))
    sites = np.stack([rng.uniform(0, W, R), rng.uniform(0, H, R)], axis=1)
    region = _regions(sites, W, H)
    img, _ = _paint(rng, region, R, W, H, C, grad)
    out = _finish(rng, img, sigma)
    return (out, region) if return_regions else out


def mosaic_batch(n: int, W: int, H: int, r_lo: int, r_hi: int, s_lo: float, s_hi: float,
                 seed: int, grad: float = 30.0, C: int = 3, return_regions: bool = False):
    """n independent frames (c3): R ~ U{r_lo..r_hi}, sigma ~ U[s_lo, s_hi] per frame."""
    out = np.empty((n, H, W, C), np.uint8)
    regions = np.empty((n, H, W), np.int32) if return_regions else None
    for f in range(n):
        rng = np.random.Generator(np.random.PCG64(seed * 100003 + f))
        R = int(rng.integers(r_lo, r_hi + 1))
        sigma = float(rng.uniform(s_lo, s_hi))
        r = mosaic(W, H, R, sigma, seed=seed * 100003 + f + 7, C=C, grad=grad, return_regions=return_regions)
        if return_regions:
            out[f], regions[f] = r
        else:
            out[f] = r
    return (out, regions) if return_regions else out


def moving_mosaic(n_frames: int, W: int, H: int, R: int, sigma: float, seed: int,
                  vmax: float = 3.0, grad: float = 30.0, C: int = 3):
    """Video (c4): sites move at constant velocity |v| ~ U[0, vmax] px/frame,
    reflecting at the borders; colours and gradients fixed per site; noise
    redrawn per frame.  Returns (frames (n, H, W, C) uint8, regions (n, H, W))."""
    rng = np.random.Generator(np.random.PCG64(seed))
    pos = np.stack([rng.uniform(0, W, R), rng.uniform(0, H, R)], axis=1)
    speed = rng.uniform(0, vmax, R)
    ang = rng.uniform(0, 2 * np.pi, R)
    vel = np.stack([speed * np.cos(ang), speed * np.sin(ang)], axis=1)
    colours = rng.integers(0, 256, size=(R, C)).astype(np.float64)
    theta = rng.uniform(0.0, 2 * np.pi, size=R)
    amp = rng.uniform(-grad, grad, size=(R, C))
    frames = np.empty((n_frames, H, W, C), np.uint8)
    regions = np.empty((n_frames, H, W), np.int32)
    for f in range(n_frames):
        region = _regions(pos, W, H)
        img, _ = _paint(rng, region, R, W, H, C, grad, colours=colours, grad_params=(theta, amp))
        frames[f] = _finish(rng, img, sigma)
        regions[f] = region
        pos = pos + vel
        for d, lim in ((0, W), (1, H)):
            lo = pos[:, d] < 0
            pos[lo, d] = -pos[lo, d]
            vel[lo, d] = -vel[lo, d]
            hi = pos[:, d] >= lim
            pos[hi, d] = 2 * lim - pos[hi, d] - 1e-9
            vel[hi, d] = -vel[hi, d]
    return frames, regions
