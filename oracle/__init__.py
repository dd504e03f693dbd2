"""CPU oracle for the SEEDS hill-climbing refinement (arXiv 1309.3848).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
package.  The product path (``paper_1309_3848_b200``) never imports it and
shares no code with it.

``oracle/seeds_oracle.c`` is the oracle proper (plain C, one thread); this
module compiles it with gcc and wraps it with ctypes.  ``oracle/exact.py``
holds the tiny exact (``fractions``) energies and brute-force enumeration.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "seeds_oracle.c")
_LIB = os.path.join(_HERE, "libseeds_oracle.so")

COL, SEQ = 0, 1
R1, R2 = 0, 1


class Trace(ctypes.Structure):
    _fields_ = [
        ("level", ctypes.c_int32),
        ("iter", ctypes.c_int32),
        ("colour", ctypes.c_int32),
        ("moves", ctypes.c_int32),
        ("visits", ctypes.c_int64),
        ("boundary", ctypes.c_int64),
        ("removable", ctypes.c_int64),
        ("h_norm", ctypes.c_double),
        ("h_raw", ctypes.c_double),
        ("g_raw", ctypes.c_double),
        ("g_norm", ctypes.c_double),
    ]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc -O2 (plain C, no vectorisation flags)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        _lib.oracle_run.restype = ctypes.c_int
        _lib.oracle_run.argtypes = [
            ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            P(Trace), ctypes.c_int, P(ctypes.c_int), ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
            ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
        ]
        _lib.oracle_rgb_to_lab.restype = None
        _lib.oracle_rgb_to_lab.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        _lib.oracle_metrics.restype = ctypes.c_int
        _lib.oracle_metrics.argtypes = [ctypes.c_void_p, ctypes.c_void_p] + [ctypes.c_int] * 5 + [ctypes.c_void_p]
        _lib.oracle_means_test.restype = ctypes.c_int
        _lib.oracle_means_test.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                           ctypes.c_void_p, ctypes.c_int64]
        _lib.oracle_geometry.restype = ctypes.c_int
        _lib.oracle_geometry.argtypes = [ctypes.c_int] * 4 + [P(ctypes.c_int)] * 3
        _lib.oracle_removable.restype = ctypes.c_int
        _lib.oracle_removable.argtypes = [ctypes.c_int]
        _lib.oracle_quantise.restype = None
        _lib.oracle_quantise.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 4 + [ctypes.c_void_p]
        _lib.oracle_energy.restype = None
        _lib.oracle_energy.argtypes = [ctypes.c_void_p, ctypes.c_void_p] + [ctypes.c_int] * 5 + [
            ctypes.c_void_p]
        i64p = ctypes.c_void_p
        for name in ("oracle_colour_test", "oracle_colour_test_block"):
            f = getattr(_lib, name)
            f.restype = ctypes.c_int
            f.argtypes = [i64p, i64p, i64p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                          ctypes.c_int64, ctypes.c_int]
        _lib.oracle_smooth_sum.restype = ctypes.c_int
        _lib.oracle_smooth_sum.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 6
    return _lib


def colour_test(hn, hk, l, An, Ak, alpha, rule=R1, force_block=False) -> bool:
    """Proposition 1 on one proposal (see oracle_colour_test in seeds_oracle.c)."""
    hn = np.ascontiguousarray(hn, np.int64)
    hk = np.ascontiguousarray(hk, np.int64)
    l = np.ascontiguousarray(l, np.int64)
    f = lib().oracle_colour_test_block if force_block else lib().oracle_colour_test
    r = f(hn.ctypes.data, hk.ctypes.data, l.ctypes.data, hn.size, int(An), int(Ak), int(alpha), rule)
    if r < 0:
        raise ValueError("bad arguments")
    return bool(r)


def smooth_sum(lab: np.ndarray, x: int, y: int, k: int, n: int) -> int:
    """Proposition 2 sum S for moving pixel (x, y) from k to n."""
    lab = np.ascontiguousarray(lab, np.int32)
    H, W = lab.shape
    return int(lib().oracle_smooth_sum(lab.ctypes.data, W, H, x, y, k, n))


def geometry(W: int, H: int, K: int, L: int):
    """(nx, ny, L_eff) of the initial grid (reading O2)."""
    nx, ny, le = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    if lib().oracle_geometry(W, H, K, L, ctypes.byref(nx), ctypes.byref(ny), ctypes.byref(le)) != 0:
        raise ValueError("invalid geometry arguments")
    return nx.value, ny.value, le.value


def removable(mask: int) -> bool:
    return bool(lib().oracle_removable(mask))


def quantise(img: np.ndarray, bpc: int) -> np.ndarray:
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W, C = img.shape
    out = np.empty((H, W), np.int32)
    lib().oracle_quantise(img.ctypes.data, W, H, C, bpc, out.ctypes.data)
    return out


def energy(labels: np.ndarray, img: np.ndarray, bpc: int, K: int):
    """(H, H', G', G) of a labelling (reading O10)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    H, W, C = img.shape
    out = np.zeros(4, np.float64)
    lib().oracle_energy(labels.ctypes.data, img.ctypes.data, W, H, C, bpc, K, out.ctypes.data)
    return tuple(float(v) for v in out)


@dataclass
class Result:
    labels: np.ndarray      # (H, W) int32
    hist: np.ndarray        # (K_act, B) int32
    sizes: np.ndarray       # (K_act,) int32
    trace: list             # per sub-sweep dicts
    k_act: int
    sums: np.ndarray | None = None  # (K_act, 4) int64 channel sums (reading M1), if asked for


def run(img: np.ndarray, n_superpixels: int, n_levels: int, bins_per_channel: int,
        smoothness_prior: int, iters_per_level: int, schedule: int = COL, rule: int = R1,
        init_labels: np.ndarray | None = None, want_energy: bool = False,
        shuffle_seed: int = 0, max_subsweeps: int = -1, trace_cap: int = 4096,
        means_iters: int = 0, want_sums: bool = False, colour: str = "rgb",
        block_levels: tuple | None = None, compact: bool = False, edge_tau: int = 0) -> Result:
    """Refine `img` (H, W, C uint8).  means_iters > 0: the last means_iters
    pixel iterations use the SPM nearest-mean test (reading M1).  colour =
    "lab": the 8-bit CIELAB pre-pass (reading M3) first; every later step
    (bins, means) sees the converted image.  block_levels = (lo, hi): only
    block levels lo..hi run (reading M4; (l, l) = one block size).  compact:
    the compactness prior at the pixel level (reading M5).  edge_tau > 0: the
    edge prior with that colour-difference threshold (reading M6)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    if colour == "lab":
        img = rgb_to_lab(img)
    elif colour != "rgb":
        raise ValueError(f"unknown colour space {colour!r}")
    if img.ndim == 2:
        img = img[:, :, None]
    H, W, C = img.shape
    nx, ny, _ = geometry(W, H, n_superpixels, n_levels)
    K = nx * ny
    B = bins_per_channel ** C
    labels = np.empty((H, W), np.int32)
    hist = np.empty((K, B), np.int32)
    sizes = np.empty((K,), np.int32)
    tr = (Trace * trace_cap)()
    tlen = ctypes.c_int(0)
    init_ptr = None
    if init_labels is not None:
        init_labels = np.ascontiguousarray(init_labels, dtype=np.int32)
        init_ptr = init_labels.ctypes.data
    sums = np.empty((K, 4), np.int64) if want_sums else None
    k = lib().oracle_run(img.ctypes.data, W, H, C, n_superpixels, n_levels, bins_per_channel,
                         int(smoothness_prior), iters_per_level, schedule, rule, init_ptr,
                         labels.ctypes.data, hist.ctypes.data, sizes.ctypes.data, tr, trace_cap,
                         ctypes.byref(tlen), int(want_energy), shuffle_seed, max_subsweeps,
                         int(means_iters), None if sums is None else sums.ctypes.data,
                         -1 if block_levels is None else int(block_levels[0]),
                         -1 if block_levels is None else int(block_levels[1]), int(bool(compact)),
                         int(edge_tau))
    if k < 0:
        raise ValueError("oracle_run rejected its arguments")
    trace = []
    for i in range(min(tlen.value, trace_cap)):
        t = tr[i]
        trace.append({f: getattr(t, f) for f, _ in Trace._fields_})
    return Result(labels, hist, sizes, trace, k, sums)


def means_test(v, Sk, Ak: int, Sn, An: int) -> bool:
    """The means test (reading M1) on one proposal: pixel colour v (C values),
    channel sums and sizes of k (the pixel counted in k) and of n."""
    v = np.ascontiguousarray(v, dtype=np.uint8)
    C = v.shape[0]
    Sk = np.zeros(4, np.int64) + np.pad(np.asarray(Sk, np.int64), (0, 4 - C))
    Sn = np.zeros(4, np.int64) + np.pad(np.asarray(Sn, np.int64), (0, 4 - C))
    return bool(lib().oracle_means_test(v.ctypes.data, C, Sk.ctypes.data, int(Ak), Sn.ctypes.data, int(An)))


def metrics(labels, gt, K: int, R: int, eps: int = 2) -> dict:
    """Quality metrics of a partition against ground-truth segments (SURVEY
    8(f) rank 2): integer numerators and the ratios."""
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    gt = np.ascontiguousarray(gt, dtype=np.int32)
    H, W = labels.shape
    out = np.zeros(7, np.int64)
    if lib().oracle_metrics(labels.ctypes.data, gt.ctypes.data, W, H, int(K), int(R), int(eps), out.ctypes.data):
        raise ValueError("oracle_metrics rejected its arguments")
    n, ue, cue, asa, nb, hits, most = (int(v) for v in out)
    return dict(n=n, ue_num=ue, cue_num=cue, asa_num=asa, gt_boundary=nb, br_hits=hits, max_segments=most,
                ue=ue / n, cue=cue / n, asa=asa / n, br=hits / nb if nb else 1.0)


def rgb_to_lab(img: np.ndarray) -> np.ndarray:
    """8-bit sRGB (..., 3) -> 8-bit CIELAB (L 255/100, a + 128, b + 128), the
    integer fixed-point conversion of reading M3."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    if img.shape[-1] != 3:
        raise ValueError("the LAB pre-pass needs 3 channels")
    out = np.empty_like(img)
    lib().oracle_rgb_to_lab(img.ctypes.data, img.size // 3, out.ctypes.data)
    return out