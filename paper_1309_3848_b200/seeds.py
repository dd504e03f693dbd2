"""Python binding of libseeds.so (include/seeds.h): argument marshalling only.

Every step of the refinement runs in the CUDA kernels behind the C ABI; this
module converts torch tensors / numpy arrays to pointers and streams.  There
is no CPU fallback: if the library is missing or no CUDA device is present,
the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# SEEDS_LIB: another build of the same library (A/B measurements, the tracing
# build of scripts/build_trace.sh); the default is the in-tree libseeds.so
LIB_PATH = os.environ.get("SEEDS_LIB") or os.path.join(_PKG, "libseeds.so")

_STATUS = {0: "ok", -1: "invalid argument", -2: "out of memory", -3: "CUDA error",
           -4: "NCCL error", -5: "invalid state", -6: "problem exceeds an integer width"}

EXPORTS = ["seeds_create", "seeds_iterate", "seeds_batch", "seeds_batch_host", "seeds_query",
           "seeds_read_state", "seeds_debug_limit", "seeds_stats", "seeds_sync", "seeds_destroy",
           "seeds_profile", "seeds_profile_collect", "seeds_set_mode", "seeds_debug_trace",
           "seeds_status_string", "seeds_last_error", "seeds_create_banded", "seeds_band_info",
           "seeds_create_bands", "seeds_nccl_unique_id", "seeds_band_export", "seeds_band_connect", "seeds_band_run",
           "seeds_set_means_iters", "seeds_read_sums", "seeds_metrics", "seeds_set_colour_space",
           "seeds_rgb_to_lab", "seeds_set_block_levels", "seeds_set_host_chunks", "seeds_set_compactness",
           "seeds_set_edge_prior", "seeds_batch_host_warm", "seeds_validate_labels", "seeds_set_validate",
           "seeds_set_time_budget", "seeds_last_subsweeps", "seeds_debug_k5",
           "seeds_debug_block_hist", "seeds_video_host"]


class _Metrics(ctypes.Structure):
    _fields_ = [("n", ctypes.c_longlong), ("ue_num", ctypes.c_longlong), ("cue_num", ctypes.c_longlong),
                ("asa_num", ctypes.c_longlong), ("gt_boundary", ctypes.c_longlong), ("br_hits", ctypes.c_longlong),
                ("max_segments", ctypes.c_int), ("ue", ctypes.c_double), ("cue", ctypes.c_double),
                ("asa", ctypes.c_double), ("br", ctypes.c_double)]


class SeedsError(RuntimeError):
    def __init__(self, status: int, detail: str = ""):
        super().__init__(f"{_STATUS.get(status, status)}" + (f": {detail}" if detail else ""))
        self.status = status


class Info(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "width", "height", "channels", "nx", "ny", "k_actual", "levels_eff", "grid_x", "grid_y",
        "colour_period", "bins_total", "bin_bytes", "subsweeps", "max_block_area",
        "kernels_per_run", "exec_mode", "grid_ctas", "grid_tiles")] + [
        ("workspace_bytes_per_frame", ctypes.c_size_t)]


_lib = None


def load(path: str = LIB_PATH):
    """Load libseeds.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built: run `python -m paper_1309_3848_b200.build`")
    lib = ctypes.CDLL(path)
    vp, i = ctypes.c_void_p, ctypes.c_int
    sig = {
        "seeds_create": ([i] * 8 + [ctypes.POINTER(vp)], i),
        "seeds_iterate": ([vp, vp, vp, vp], i),
        "seeds_batch": ([vp, vp, i, vp, vp, vp], i),
        "seeds_batch_host": ([vp, vp, i, vp, vp, vp], i),
        "seeds_batch_host_warm": ([vp, vp, i, vp, vp], i),
        "seeds_video_host": ([vp, vp, i, i, i, vp, vp], i),
        "seeds_query": ([vp, ctypes.POINTER(Info)], i),
        "seeds_read_state": ([vp, i, vp, vp, vp], i),
        "seeds_debug_limit": ([vp, i], i),
        "seeds_set_means_iters": ([vp, i], i),
        "seeds_read_sums": ([vp, i, vp, vp], i),
        "seeds_metrics": ([vp, vp, vp, i, i, vp, vp], i),
        "seeds_set_colour_space": ([vp, i], i),
        "seeds_set_block_levels": ([vp, i, i], i),
        "seeds_set_host_chunks": ([vp, i], i),
        "seeds_set_compactness": ([vp, i], i),
        "seeds_set_edge_prior": ([vp, i], i),
        "seeds_validate_labels": ([vp, vp, i, vp, vp], i),
        "seeds_set_validate": ([vp, i], i),
        "seeds_set_time_budget": ([vp, ctypes.c_longlong], i),
        "seeds_last_subsweeps": ([vp, vp, vp], i),
        "seeds_debug_k5": ([vp, vp, i, vp, vp, vp, i, i, i, i, vp, vp], i),
        "seeds_debug_block_hist": ([vp, vp], i),
        "seeds_rgb_to_lab": ([vp, vp, ctypes.c_longlong, vp, vp], i),
        "seeds_stats": ([vp, i, vp, i, vp], i),
        "seeds_sync": ([vp, vp], i),
        "seeds_profile": ([vp, i], i),
        "seeds_set_mode": ([vp, i], i),
        "seeds_debug_trace": ([vp, i, vp, i], i),
        "seeds_profile_collect": ([vp, vp, vp, vp], i),
        "seeds_destroy": ([vp], None),
        "seeds_create_banded": ([i] * 10 + [vp, ctypes.POINTER(vp)], i),
        "seeds_create_bands": ([i] * 9 + [ctypes.POINTER(vp)], i),
        "seeds_nccl_unique_id": ([vp], i),
        "seeds_band_export": ([vp, vp, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)], i),
        "seeds_band_connect": ([vp, vp, i], i),
        "seeds_band_info": ([vp, vp, vp, vp, vp], i),
        "seeds_band_run": ([vp, vp, vp, vp, vp], i),
        "seeds_status_string": ([i], ctypes.c_char_p),
        "seeds_last_error": ([vp], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        if path != os.path.join(_PKG, "libseeds.so") and not hasattr(lib, name):
            continue  # an older A/B build (SEEDS_LIB) may lack newer entry points
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _stream_ptr(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def debug_k5(H, A, bins, alpha, cand, threads: int, gshift: int, narrow: bool, stream=None):
    """Unit test entry of the block colour test K5 (include/seeds.h
    seeds_debug_k5): int32 CUDA tensors H (n, 5, B), A (n, 5), bins (n, 64),
    alpha (n,), cand (n, 4) -> int32 CUDA tensor (n,) of accepted labels / -1."""
    import torch
    lib = load()
    ts = (H, A, bins, alpha, cand)
    if not all(isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.int32 and t.is_contiguous() for t in ts):
        raise TypeError("every table must be a contiguous int32 CUDA tensor")
    n, _, B = H.shape
    if A.shape != (n, 5) or bins.shape != (n, 64) or alpha.shape != (n,) or cand.shape != (n, 4):
        raise ValueError("table shapes")
    out = torch.full((n,), -2, dtype=torch.int32, device=H.device)
    st = lib.seeds_debug_k5(H.data_ptr(), A.data_ptr(), B, bins.data_ptr(), alpha.data_ptr(), cand.data_ptr(), n,
                            threads, gshift, int(bool(narrow)), out.data_ptr(), _stream_ptr(stream))
    if st != 0:
        raise SeedsError(st)
    return out


@dataclass
class Geometry:
    nx: int
    ny: int
    k_actual: int
    levels_eff: int
    grid_x: int
    grid_y: int
    colour_period: int
    bins_total: int
    bin_bytes: int
    subsweeps: int
    max_block_area: int
    kernels_per_run: int
    exec_mode: int
    grid_ctas: int
    grid_tiles: int
    workspace_bytes_per_frame: int


class Seeds:
    """One refinement context (seeds_create ... seeds_destroy)."""

    def __init__(self, width: int, height: int, channels: int, n_superpixels: int, n_levels: int,
                 bins_per_channel: int, smoothness_prior: int, iters_per_level: int):
        self._lib = load()
        self._ctx = ctypes.c_void_p()
        st = self._lib.seeds_create(width, height, channels, n_superpixels, n_levels,
                                    bins_per_channel, int(smoothness_prior), iters_per_level,
                                    ctypes.byref(self._ctx))
        if st != 0:
            raise SeedsError(st)
        self.width, self.height, self.channels = width, height, channels
        info = Info()
        self._check(self._lib.seeds_query(self._ctx, ctypes.byref(info)))
        self.info = Geometry(**{f: getattr(info, f) for f in Geometry.__dataclass_fields__})

    def _check(self, st: int):
        if st != 0:
            raise SeedsError(st, self._lib.seeds_last_error(self._ctx).decode())

    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            self._lib.seeds_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- device entry points (torch tensors on the current CUDA device) -------
    def _frames(self, images):
        import torch
        if not (isinstance(images, torch.Tensor) and images.is_cuda and images.dtype == torch.uint8
                and images.is_contiguous()):
            raise TypeError("images must be a contiguous uint8 CUDA tensor")
        n = images.numel() // (self.width * self.height * self.channels)
        if n * self.width * self.height * self.channels != images.numel() or n < 1:
            raise ValueError("images do not hold whole frames of the context's size")
        return n

    def iterate(self, image, labels_out=None, stream=None):
        """Cold refinement of one frame: (H, W, C) uint8 CUDA tensor -> (H, W) int32."""
        import torch
        self._frames(image)
        if labels_out is None:
            labels_out = torch.empty((self.height, self.width), dtype=torch.int32, device=image.device)
        self._check(self._lib.seeds_iterate(self._ctx, image.data_ptr(), labels_out.data_ptr(),
                                            _stream_ptr(stream)))
        return labels_out

    def batch(self, images, init_labels=None, labels_out=None, stream=None):
        """(n, H, W, C) uint8 CUDA tensor [+ (n, H, W) int32 warm-start labels] -> (n, H, W) int32."""
        import torch
        n = self._frames(images)
        if labels_out is None:
            labels_out = torch.empty((n, self.height, self.width), dtype=torch.int32,
                                     device=images.device)
        init_ptr = None
        if init_labels is not None:
            if not (init_labels.is_cuda and init_labels.dtype == torch.int32
                    and init_labels.is_contiguous() and init_labels.numel() == labels_out.numel()):
                raise TypeError("init_labels must be a contiguous int32 CUDA tensor of n*H*W")
            init_ptr = init_labels.data_ptr()
        self._check(self._lib.seeds_batch(self._ctx, images.data_ptr(), n, init_ptr,
                                          labels_out.data_ptr(), _stream_ptr(stream)))
        return labels_out

    def _host_frames(self, images, labels_out) -> int:
        """Frames of a host call; the buffers must match exactly (the C side
        copies n*H*W*C bytes in and n*H*W int32 out)."""
        if not (isinstance(images, np.ndarray) and images.dtype == np.uint8 and images.flags.c_contiguous):
            raise TypeError("images must be a C-contiguous uint8 numpy array")
        fr = self.width * self.height * self.channels
        n = images.size // fr
        if n < 1 or n * fr != images.size:
            raise ValueError("images do not hold whole frames of the context's size")
        if not (isinstance(labels_out, np.ndarray) and labels_out.dtype == np.int32
                and labels_out.flags.c_contiguous and labels_out.flags.writeable):
            raise TypeError("labels_out must be a writeable C-contiguous int32 numpy array")
        if labels_out.size != n * self.width * self.height:
            raise ValueError(f"labels_out holds {labels_out.size} values, the call writes {n * self.width * self.height}")
        return n

    def batch_host(self, images: np.ndarray, labels_out: np.ndarray, init_labels=None, stream=None):
        """Host-memory entry point (copies in, runs, copies out, synchronises)."""
        n = self._host_frames(images, labels_out)
        init_ptr = None
        if init_labels is not None:
            if not (isinstance(init_labels, np.ndarray) and init_labels.dtype == np.int32
                    and init_labels.flags.c_contiguous and init_labels.size == labels_out.size):
                raise TypeError("init_labels must be a C-contiguous int32 numpy array of n*H*W values")
            init_ptr = init_labels.ctypes.data
        self._check(self._lib.seeds_batch_host(self._ctx, images.ctypes.data, n, init_ptr,
                                               labels_out.ctypes.data, _stream_ptr(stream)))
        return labels_out

    def batch_host_warm(self, images: np.ndarray, labels_out: np.ndarray, stream=None):
        """Next frames of n video streams from host memory, each warm-started
        from the previous host call's labels still on the device
        (seeds_batch_host_warm)."""
        n = self._host_frames(images, labels_out)
        self._check(self._lib.seeds_batch_host_warm(self._ctx, images.ctypes.data, n, labels_out.ctypes.data,
                                                    _stream_ptr(stream)))
        return labels_out

    def video_host(self, images: np.ndarray, labels_out: np.ndarray, continue_prev: bool = False, stream=None):
        """n_steps x n_streams video frames (time-major, uint8 (T, n, H, W, C))
        from host memory in one call, each step warm-started from the previous
        one's labels (seeds_video_host); labels_out int32 (T, n, H, W)."""
        if not (isinstance(images, np.ndarray) and images.ndim >= 4):
            raise TypeError("images must be a (T, n, H, W[, C]) uint8 numpy array")
        T, n = images.shape[0], images.shape[1]
        if self._host_frames(images, labels_out) != T * n:
            raise ValueError("images must hold T x n whole frames")
        self._check(self._lib.seeds_video_host(self._ctx, images.ctypes.data, n, T, int(bool(continue_prev)),
                                               labels_out.ctypes.data, _stream_ptr(stream)))
        return labels_out

    def read_state(self, frame: int = 0, stream=None):
        """(hist (K_act, B) int32, sizes (K_act,) int32) CUDA tensors after the last run."""
        import torch
        K, B = self.info.k_actual, self.info.bins_total
        h = torch.empty((K, B), dtype=torch.int32, device="cuda")
        a = torch.empty((K,), dtype=torch.int32, device="cuda")
        self._check(self._lib.seeds_read_state(self._ctx, frame, h.data_ptr(), a.data_ptr(),
                                               _stream_ptr(stream)))
        return h, a

    def stats(self, frame: int = 0, stream=None) -> np.ndarray:
        out = np.zeros(self.info.subsweeps, np.int32)
        self._check(self._lib.seeds_stats(self._ctx, frame, out.ctypes.data, out.size,
                                          _stream_ptr(stream)))
        return out

    KINDS = ("seed", "block", "pixel", "emit", "frame")
    MODES = {"auto": 0, "graph": 1, "grid": 3}

    def set_mode(self, mode: str):
        self._check(self._lib.seeds_set_mode(self._ctx, self.MODES[mode]))
        self._refresh()

    def _refresh(self):
        info = Info()
        self._check(self._lib.seeds_query(self._ctx, ctypes.byref(info)))
        self.info = Geometry(**{f: getattr(info, f) for f in Geometry.__dataclass_fields__})

    def profile(self, enable: bool = True):
        self._check(self._lib.seeds_profile(self._ctx, int(enable)))

    def profile_collect(self, stream=None):
        """{kind: (total ms, launches)} accumulated over profiled runs."""
        ms = np.zeros(5, np.float64)
        n = np.zeros(5, np.int64)
        self._check(self._lib.seeds_profile_collect(self._ctx, _stream_ptr(stream), ms.ctypes.data,
                                                    n.ctypes.data))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(self.KINDS)}

    def debug_trace(self, enable: bool = True, n_sm: int | None = None):
        """Grid mode: per-CTA clock64 stamps [cta, phase, slot] (include/seeds.h)."""
        if n_sm is None:
            import torch
            n_sm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        cs = 4 * n_sm
        n = cs * (self.info.subsweeps + 4) * 16
        out = np.zeros(n, np.int64)
        self._check(self._lib.seeds_debug_trace(self._ctx, int(enable), out.ctypes.data if enable else None, n))
        return out.reshape(cs, self.info.subsweeps + 4, 16)

    def set_means_iters(self, means_iters: int):
        """The last means_iters pixel iterations use the means test (SPM
        post-processing, include/seeds.h seeds_set_means_iters)."""
        self._check(self._lib.seeds_set_means_iters(self._ctx, int(means_iters)))

    def set_compactness(self, on: bool = True):
        """The compactness prior at the pixel level (include/seeds.h seeds_set_compactness)."""
        self._check(self._lib.seeds_set_compactness(self._ctx, int(bool(on))))

    def set_edge_prior(self, tau: int):
        """The edge prior with colour-difference threshold tau (0 = off;
        include/seeds.h seeds_set_edge_prior)."""
        self._check(self._lib.seeds_set_edge_prior(self._ctx, int(tau)))

    def set_block_levels(self, lo: int, hi: int = -1):
        """Only block levels lo..hi run (include/seeds.h seeds_set_block_levels)."""
        self._check(self._lib.seeds_set_block_levels(self._ctx, int(lo), int(hi)))

    def set_host_chunks(self, chunks: int):
        """Chunks of the batch_host copy / compute pipeline (0 = automatic, 1 = off)."""
        self._check(self._lib.seeds_set_host_chunks(self._ctx, int(chunks)))

    COLOURS = {"rgb": 0, "lab": 1}

    def set_colour_space(self, space: str):
        """"rgb" (default) or "lab": the 8-bit CIELAB pre-pass of reading M3
        (include/seeds.h seeds_set_colour_space)."""
        self._check(self._lib.seeds_set_colour_space(self._ctx, self.COLOURS[space]))

    def rgb_to_lab(self, rgb, stream=None):
        """(..., 3) uint8 CUDA tensor of sRGB -> the same shape of 8-bit CIELAB."""
        import torch
        out = torch.empty_like(rgb)
        self._check(self._lib.seeds_rgb_to_lab(self._ctx, rgb.data_ptr(), rgb.numel() // 3, out.data_ptr(),
                                               _stream_ptr(stream)))
        return out

    def read_sums(self, frame: int = 0, stream=None):
        """(K_act, 4) int64 CUDA tensor: channel sums S[k][c] after the last run
        (means post-processing only)."""
        import torch
        out = torch.empty((self.info.k_actual, 4), dtype=torch.int64, device="cuda")
        self._check(self._lib.seeds_read_sums(self._ctx, frame, out.data_ptr(), _stream_ptr(stream)))
        return out

    def metrics(self, labels, gt, n_segments: int, eps: int = 2, stream=None) -> dict:
        """UE / CUE / ASA / BR of (H, W) int32 CUDA labels against (H, W) int32
        CUDA ground-truth segment ids (include/seeds.h seeds_metrics)."""
        out = _Metrics()
        self._check(self._lib.seeds_metrics(self._ctx, labels.data_ptr(), gt.data_ptr(), int(n_segments), int(eps),
                                            ctypes.byref(out), _stream_ptr(stream)))
        return {f: getattr(out, f) for f, _ in _Metrics._fields_}

    def validate_labels(self, labels, stream=None) -> tuple:
        """Check (n, H, W) / (H, W) int32 CUDA labels form valid partitions
        (include/seeds.h seeds_validate_labels): returns (out_of_range,
        first_missing, first_split); raises SeedsError(SEEDS_ESTATE) if invalid."""
        import torch
        if not (isinstance(labels, torch.Tensor) and labels.is_cuda and labels.dtype == torch.int32
                and labels.is_contiguous()):
            raise TypeError("labels must be a contiguous int32 CUDA tensor")
        n = labels.numel() // (self.width * self.height)
        if n < 1 or n * self.width * self.height != labels.numel():
            raise ValueError("labels do not hold whole frames of the context's size")
        rep = np.zeros(3, np.int64)
        st = self._lib.seeds_validate_labels(self._ctx, labels.data_ptr(), n, rep.ctypes.data, _stream_ptr(stream))
        if st not in (0, -5):
            self._check(st)
        out = tuple(int(v) for v in rep)
        if st == -5:
            raise SeedsError(st, self._lib.seeds_last_error(self._ctx).decode())
        return out

    def set_validate(self, on: bool = True):
        """Validate warm-start labels before every run (include/seeds.h seeds_set_validate)."""
        self._check(self._lib.seeds_set_validate(self._ctx, int(bool(on))))

    def debug_block_hist(self, out=None):
        """out: a zeroed (n, n_top_blocks, B) int32 CUDA tensor that later cold
        runs fill with the seed's top-level block histograms (None: off;
        include/seeds.h seeds_debug_block_hist)."""
        self._check(self._lib.seeds_debug_block_hist(self._ctx, None if out is None else out.data_ptr()))

    def set_time_budget(self, budget_us: int):
        """Anytime termination after budget_us microseconds (0 = off;
        include/seeds.h seeds_set_time_budget)."""
        self._check(self._lib.seeds_set_time_budget(self._ctx, int(budget_us)))

    def last_subsweeps(self, stream=None) -> int:
        """Sub-sweeps the last run performed (include/seeds.h seeds_last_subsweeps)."""
        out = ctypes.c_int()
        self._check(self._lib.seeds_last_subsweeps(self._ctx, ctypes.byref(out), _stream_ptr(stream)))
        return out.value

    def debug_limit(self, max_subsweeps: int):
        self._check(self._lib.seeds_debug_limit(self._ctx, max_subsweeps))

    def sync(self, stream=None):
        self._check(self._lib.seeds_sync(self._ctx, _stream_ptr(stream)))


def nccl_unique_id() -> bytes:
    """A new NCCL unique id (128 bytes) for SeedsBand's bootstrap (rank 0
    creates it, the caller distributes it; include/seeds.h seeds_nccl_unique_id)."""
    lib = load()
    buf = ctypes.create_string_buffer(128)
    st = lib.seeds_nccl_unique_id(buf)
    if st != 0:
        raise SeedsError(st)
    return buf.raw


class _BandMixin:
    """Row-band run of one frame (include/seeds.h "Row-band mode")."""

    def _band_init(self):
        r0, r1, nb, b = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        self._check(self._lib.seeds_band_info(self._ctx, ctypes.byref(r0), ctypes.byref(r1), ctypes.byref(nb),
                                              ctypes.byref(b)))
        self.row0, self.row1, self.n_bands, self.band = r0.value, r1.value, nb.value, b.value

    def run(self, image, init_labels=None, labels_out=None, stream=None):
        """(H, W, C) uint8 CUDA tensor (the whole frame) [+ (H, W) int32 warm-start
        labels] -> (H, W) int32 CUDA tensor; this context's rows are written."""
        import torch
        self._frames(image)
        if labels_out is None:
            labels_out = torch.zeros((self.height, self.width), dtype=torch.int32, device=image.device)
        self._check(self._lib.seeds_band_run(self._ctx, image.data_ptr(),
                                             None if init_labels is None else init_labels.data_ptr(),
                                             labels_out.data_ptr(), _stream_ptr(stream)))
        return labels_out


class SeedsBands(_BandMixin, Seeds):
    """Every band of a row-band run in this process, one launch on the current
    device (seeds_create_bands)."""

    def __init__(self, width: int, height: int, channels: int, n_superpixels: int, n_levels: int,
                 bins_per_channel: int, smoothness_prior: int, iters_per_level: int, n_bands: int):
        self._lib = load()
        self._ctx = ctypes.c_void_p()
        st = self._lib.seeds_create_bands(width, height, channels, n_superpixels, n_levels, bins_per_channel,
                                          int(smoothness_prior), iters_per_level, n_bands, ctypes.byref(self._ctx))
        if st != 0:
            raise SeedsError(st)
        self.width, self.height, self.channels = width, height, channels
        self._refresh()
        self._band_init()


class SeedsBand(_BandMixin, Seeds):
    """Band `rank` of a `world`-rank row-band run, one device per rank
    (seeds_create_banded).  nccl_id (bytes from nccl_unique_id(), the same on
    every rank): the library exchanges the ranks' CUDA IPC handles itself;
    None with world > 1: call connect() with every rank's export() blob."""

    def __init__(self, width: int, height: int, channels: int, n_superpixels: int, n_levels: int,
                 bins_per_channel: int, smoothness_prior: int, iters_per_level: int, rank: int, world: int,
                 nccl_id: bytes | None = None):
        self._lib = load()
        self._ctx = ctypes.c_void_p()
        idbuf = None if nccl_id is None else ctypes.create_string_buffer(bytes(nccl_id), 128)
        st = self._lib.seeds_create_banded(width, height, channels, n_superpixels, n_levels, bins_per_channel,
                                           int(smoothness_prior), iters_per_level, rank, world, idbuf,
                                           ctypes.byref(self._ctx))
        if st != 0:
            raise SeedsError(st)
        self.width, self.height, self.channels = width, height, channels
        self._refresh()
        self._band_init()

    def export(self) -> bytes:
        n = ctypes.c_size_t()
        self._check(self._lib.seeds_band_export(self._ctx, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        self._check(self._lib.seeds_band_export(self._ctx, buf, n.value, ctypes.byref(n)))
        return buf.raw

    def connect(self, blobs):
        """blobs: every rank's export(), in rank order."""
        data = b"".join(blobs)
        self._check(self._lib.seeds_band_connect(self._ctx, data, len(blobs)))
