#!/usr/bin/env python
"""Benchmark of the SEEDS refinement hot path on B200 (BASELINE.json metric:
"Mpixels/s SEEDS refinement (481x321 frames/s, 200 SP); % of B200 HBM peak").

One step = one whole refinement (seed, every block and pixel sub-sweep, emit)
of one batch of synthetic frames already resident in HBM.  Default workload:
c2 = one 481x321 RGB Voronoi-mosaic frame, K=200, 4 block levels, I=4, 125
bins, gamma=1 (BASELINE.json configs[1]).  The other configs:
  c1  160x120 single frame (the oracle's small case)
  c3  256 independent 481x321 frames, K=400 -- sharded by frame over ranks
  c4  64 frames of 1920x1080 video, K=1000, L=5, gamma=0, as 8 clips of 8:
      frame 0 of a clip cold, frames 1..7 warm-started from the previous
      frame's labels (reading Q14/O9) -- clips sharded over ranks
  c5  one 8192x8192 frame, K=20000, L=6 (-> 5), 512 bins
A c2 (c1) frame is not partitioned: N GPUs run N independent replicas
("scaling": "weak").  c3 and c4 shard a fixed job ("strong"); c5 at N > 1 (or
with --bands) is refined as N row bands, one per rank, exchanging sparse
histogram-delta records (all-gather) and two-row label halos (send/recv) over
torch.distributed after every sub-sweep ("strong", include/seeds.h row-band mode).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5] [--mode auto|grid|graph]
  python bench.py --impl reference ...   # the CPU oracle, timed as it stands

L2: a 512 MiB buffer (> 126 MB L2) is rewritten between timed steps, outside
the CUDA-event brackets of each step.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1309_3848_b200 import configs  # noqa: E402

METRIC = "Mpixels/s SEEDS refinement (481x321 frames/s, 200 SP); % of B200 HBM peak"
UNIT = "Mpixels/s"
MODE_NAMES = {1: "graph", 3: "grid"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def frame_bytes(info, C, N, iters, warm=False):
    """Algorithmic bytes of one frame: image in, bin plane out,
    int32 labels out, per block iteration one pass over the bin plane, per
    pixel iteration one pass over labels + bins.  Cold: N [C + bb + 4 + I L bb
    + I (2 + bb)]; warm (no block levels, int32 labels in): N [C + bb + 8 + I (2 + bb)]."""
    bb, L = info.bin_bytes, info.levels_eff
    if warm:
        return N * (C + bb + 8 + iters * (2 + bb))
    return N * (C + bb + 4 + iters * L * bb + iters * (2 + bb))


def algorithmic_bytes(info, C, nf, N, iters):
    """Per-launch algorithmic bytes of each kernel class."""
    bb, P = info.bin_bytes, info.colour_period
    return {
        "seed": nf * N * (C + bb + (0 if info.levels_eff > 0 else 2)),
        "block": nf * N * bb / 4.0,
        "pixel": nf * N * (2 + bb) / float(P * P),
        "emit": nf * N * (2 + 4),
        "frame": nf * frame_bytes(info, C, N, iters),
    }


class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line): an in-process NVML thread polling every
    2 ms between start() and stop(); nvidia-smi (-lms 20, only the samples taken
    between start and stop kept) when NVML is not importable."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.max_mhz = 0.0
        self.thread = None
        self.proc = None
        self.run = False

    def start(self):
        import threading
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = None
            try:  # the CUDA device's own PCI address (CUDA and NVML orders can differ)
                import torch
                pr = torch.cuda.get_device_properties(self.index)
                h = nv.nvmlDeviceGetHandleByPciBusId(
                    f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0")
            except Exception:
                h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            bits = {n: getattr(nv, a, 0) for n, a in self.REASONS.items()}
        except Exception:
            return self._start_smi()
        self.run = True

        def poll():
            while self.run:
                try:
                    mhz = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((mhz, sorted(n for n, b in bits.items() if b and r & b)))
                except Exception:
                    pass
                time.sleep(0.002)
        self.thread = threading.Thread(target=poll, daemon=True)
        self.thread.start()
        t0 = time.perf_counter()
        while not self.samples and time.perf_counter() - t0 < 1.0:  # the sampler is live before timing starts
            time.sleep(0.001)
        self.samples.clear()

    def _start_smi(self):
        if not shutil.which("nvidia-smi"):
            return
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits", "-lms", "20"],
                                     stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        time.sleep(0.5)  # let it start before timing

    def stop(self):
        if self.thread is not None:
            self.run = False
            self.thread.join()
            data = list(self.samples)
        elif self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            data = []
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                try:
                    self.max_mhz = max(self.max_mhz, float(f[1]))
                    data.append((float(f[0]), sorted(n for n, v in zip(self.REASONS, f[2:6]) if v.lower() == "active")))
                except (ValueError, IndexError):
                    continue
            os.unlink(self.path)
        else:
            return None
        if not data:
            return None
        sm = sorted(d[0] for d in data)
        reasons = sorted({r for d in data for r in d[1]})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(sm),
                "sampler": "nvml" if self.thread is not None else "nvidia-smi"}


class BandWorkload:
    """c5 in row-band mode (include/seeds.h): across ranks, this rank refines
    band `rank` of `world` (one GPU each; the exchange runs inside the kernel
    over peer memory, bootstrapped once through NCCL); on one rank with
    --bands K, all K bands in one launch on this GPU."""

    def __init__(self, name, rank, world, local_bands=1):
        self.name = name
        c = self.c = configs.CONFIGS[name]
        self.p = configs.params(name)
        self.W, self.H, self.C = c["W"], c["H"], c["C"]
        self.N = self.W * self.H
        self.img = configs.frames(name, n=1)[0]
        self.rank, self.world = rank, world
        self.local_bands = local_bands
        self.frames_per_step = 1
        self.scaling = "strong"
        self.parallelism = f"row bands/{world}" if world > 1 else f"{local_bands} row bands in one launch"
        self.nf = 1
        self.groups = [None]  # one run per step

    def make_context(self):
        p = self.p
        args = (self.W, self.H, self.C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"],
                p["smoothness_prior"], p["iters_per_level"])
        if self.world > 1:
            from paper_1309_3848_b200 import bands
            return bands.make_band(*args, bootstrap="nccl")
        from paper_1309_3848_b200.seeds import SeedsBands
        return SeedsBands(*args, self.local_bands)

    def describe(self, info):
        p = self.p
        return (f"{self.name}: one {self.W}x{self.H} RGB Voronoi mosaic as {self.s.n_bands} row bands (this rank: rows "
                f"{self.s.row0}..{self.s.row1}), K={p['n_superpixels']} (K_act={info.k_actual}), "
                f"L={info.levels_eff}, I={p['iters_per_level']}, B={info.bins_total}, gamma={p['smoothness_prior']}")

    def setup(self, torch, s):
        self.s = s
        self.d_in = torch.from_numpy(self.img).cuda()
        self.d_out = torch.zeros((self.H, self.W), dtype=torch.int32, device="cuda")
        self.h_in = torch.from_numpy(self.img).pin_memory()
        self.h_out = torch.zeros((self.H, self.W), dtype=torch.int32).pin_memory()
        self.d_tmp_in = torch.empty_like(self.d_in)
        self.d_tmp_out = torch.zeros_like(self.d_out)

    def step(self, s, stream):
        s.run(self.d_in, labels_out=self.d_out, stream=stream)

    def host_step(self, s, stream):
        self.d_tmp_in.copy_(self.h_in, non_blocking=True)
        s.run(self.d_tmp_in, labels_out=self.d_tmp_out, stream=stream)
        self.h_out[s.row0:s.row1].copy_(self.d_tmp_out[s.row0:s.row1], non_blocking=True)
        stream.synchronize()

    def check(self, torch):
        s = self.s
        assert torch.equal(self.h_out[s.row0:s.row1], self.d_out[s.row0:s.row1].cpu())

    def h2d_bytes(self):
        return self.img.nbytes

    def d2h_bytes(self):
        return (self.s.row1 - self.s.row0) * self.W * 4

    def algorithmic_bytes(self, info):
        return frame_bytes(info, self.C, self.N, self.p["iters_per_level"]) * (self.s.row1 - self.s.row0) / self.H


class Workload:
    """The frames one rank refines per step, on the device and from the host."""

    def __init__(self, name, rank, world):
        import numpy as np
        self.name = name
        c = self.c = configs.CONFIGS[name]
        self.p = configs.params(name)
        self.W, self.H, self.C = c["W"], c["H"], c["C"]
        self.N = self.W * self.H
        if name == "c3":
            per = c["frames"] // world
            self.groups = [configs.frames(name)[rank * per:(rank + 1) * per]]
            self.warm = [False]
            self.scaling = "strong"
            self.parallelism = f"frames/{world}"
        elif name == "c4":
            clips = configs.clips(name)
            mine = clips[rank::world]  # clips round-robin to ranks
            self.groups = [np.ascontiguousarray(mine[:, t]) for t in range(c["clip"])]
            self.warm = [t > 0 for t in range(c["clip"])]
            self.scaling = "strong"
            self.parallelism = f"clips/{world}"
        else:
            self.groups = [configs.frames(name, n=1)]
            self.warm = [False]
            self.scaling = "weak"
            self.parallelism = "replicas"
        self.nf = self.groups[0].shape[0]
        self.frames_per_step = self.nf * len(self.groups)

    def describe(self, info):
        c, p = self.c, self.p
        extra = ""
        if self.name == "c4":
            extra = f", {len(self.groups)}-frame clips x {self.nf} per rank (frame 0 cold, 1..7 warm)"
        return (f"{self.name}: {self.frames_per_step} x {self.W}x{self.H} RGB Voronoi mosaic per rank, "
                f"K={p['n_superpixels']} (K_act={info.k_actual}), L={info.levels_eff}, "
                f"I={p['iters_per_level']}, B={info.bins_total}, gamma={p['smoothness_prior']}{extra}")

    def make_context(self):
        from paper_1309_3848_b200.seeds import Seeds
        p = self.p
        return Seeds(self.W, self.H, self.C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"],
                     p["smoothness_prior"], p["iters_per_level"])

    def video(self):
        """A warm chain (group 0 cold, every later group warm): the host path is one
        seeds_video_host call over all groups."""
        return len(self.groups) > 1 and not self.warm[0] and all(self.warm[1:])

    def check(self, torch):
        for h, d in zip(self.h_out, self.d_out):
            assert torch.equal(h, d.cpu()), "host and device entry points disagree"

    def setup(self, torch, s=None):
        self.d_in = [torch.from_numpy(g).cuda() for g in self.groups]
        self.d_out = [torch.empty((self.nf, self.H, self.W), dtype=torch.int32, device="cuda")
                      for _ in self.groups]
        if self.video():  # time-major (T, n, H, W, C) / (T, n, H, W) pinned buffers
            import numpy as np
            self.h_video = torch.from_numpy(np.stack(self.groups)).pin_memory()
            self.h_vout = torch.empty((len(self.groups), self.nf, self.H, self.W), dtype=torch.int32).pin_memory()
            self.h_in = list(self.h_video.unbind(0))
            self.h_out = list(self.h_vout.unbind(0))
        else:
            self.h_in = [torch.from_numpy(g).pin_memory() for g in self.groups]
            self.h_out = [torch.empty((self.nf, self.H, self.W), dtype=torch.int32).pin_memory()
                          for _ in self.groups]

    def step(self, s, stream):
        for i, d in enumerate(self.d_in):
            init = self.d_out[i - 1] if self.warm[i] else None
            s.batch(d, init_labels=init, labels_out=self.d_out[i], stream=stream)

    def host_step(self, s, stream):
        """Through the host-memory C-ABI entry point: copies in, runs, copies out."""
        if self.video():  # one call: step t + 1's copy in and t - 1's copy out overlap step t
            s.video_host(self.h_video.numpy(), self.h_vout.numpy(), stream=stream)
            return
        for i, h in enumerate(self.h_in):
            # a warm group continues each clip from the previous group's labels,
            # which the previous host call left on the device (seeds_batch_host_warm)
            if self.warm[i]:
                s.batch_host_warm(h.numpy(), self.h_out[i].numpy(), stream=stream)
            else:
                s.batch_host(h.numpy(), self.h_out[i].numpy(), stream=stream)

    def h2d_bytes(self):
        return sum(g.nbytes for g in self.groups)

    def d2h_bytes(self):
        return len(self.groups) * self.nf * self.N * 4

    def algorithmic_bytes(self, info):
        return sum(self.nf * frame_bytes(info, self.C, self.N, self.p["iters_per_level"], warm=w)
                   for w in self.warm)


def reference_sample(name):
    """A bounded sample of config `name` for the CPU oracle: (frames, params, note)."""
    import numpy as np
    p = configs.params(name)
    if name == "c3":
        return configs.frames(name, n=2), p, "2 frames of c3 (481x321, K=400)"
    if name == "c4":
        return configs.clips(name)[0, :1], p, "frame 0 of clip 0 of c4 (1920x1080, K=1000, cold)"
    if name == "c5":
        # a 1024x1024 crop with the same superpixel size and bins (K scaled by area)
        f = configs.frames(name, n=1)[:, :1024, :1024]
        q = dict(p)
        q["n_superpixels"] = max(1, p["n_superpixels"] * 1024 * 1024 // (8192 * 8192))
        return np.ascontiguousarray(f), q, "1024x1024 crop of c5, K scaled to 312 (same superpixel size, 512 bins)"
    return configs.frames(name, n=1), p, f"1 frame of {name}"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def parallel_sample(name, workers, clip_len=None):
    """Batch configs (c3, c4): frame- / clip-parallel on the host
    cores.  c3: min(cores, 256) independent frames.  c4: the whole video -- its
    8 clips in parallel, each a warm-started chain (frame 0 cold, frames 1..7
    from the previous labels, reading Q14/O9): shape (8, 8, H, W, C)."""
    p = configs.params(name)
    if name == "c3":
        f = configs.frames(name, n=min(workers, 256))
        return f, p, f"{len(f)} frames of c3"
    f = configs.clips(name)
    if clip_len:
        f = f[:, :clip_len]
    return f, p, f"the {f.shape[0]} clips x {f.shape[1]} warm-chained frames of c4"


def oracle_frames(imgs, p, workers):
    """Run the oracle on every frame of `imgs` with `workers` threads (ctypes
    releases the GIL; the oracle keeps no global state).  A 5-D `imgs` is a
    set of clips: each thread runs one clip's warm-started chain."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor

    def one(img):
        if img.ndim == 4:  # a clip: frame t warm-started from frame t - 1's labels
            prev = None
            for fr in img:
                prev = oracle.run(fr, **p, init_labels=prev).labels
        else:
            oracle.run(img, **p)
    if workers <= 1:
        for img in imgs:
            one(img)
        return
    with ThreadPoolExecutor(max_workers=workers) as ex:
        list(ex.map(one, list(imgs)))


def sample_pixels(imgs):
    """Pixels of a sample of frames (4-D) or clips (5-D)."""
    n = 1
    for d in imgs.shape[:-3]:
        n *= d
    return n * imgs.shape[-3] * imgs.shape[-2]


def cpu_baseline(name, budget_s=10.0, means_iters=0, colour="rgb", compact=False, edge=0):
    """The oracle as it stands (COL schedule) on a bounded sample: one thread
    on single-frame configs (the paper's setting); frame-parallel on all host
    cores for the batch configs c3 and c4, with the one-thread figure beside it."""
    import oracle
    imgs, p, note = reference_sample(name)
    if means_iters:
        p = dict(p, means_iters=means_iters)
        note += f", last {means_iters} pixel iterations on means"
    if colour != "rgb":
        p = dict(p, colour=colour)
        note += f", {colour} pre-pass"
    if compact:
        p = dict(p, compact=True)
        note += ", compactness prior"
    if edge:
        p = dict(p, edge_tau=edge)
        note += f", edge prior tau {edge}"
    oracle.build()
    n, px, t0 = 0, 0, time.perf_counter()
    while True:
        img = imgs[n % len(imgs)]
        oracle.run(img, **p)
        n += 1
        px += img.shape[0] * img.shape[1]
        el = time.perf_counter() - t0
        if el >= budget_s or n >= 200:
            break
    single = {"value": px / el / 1e6, "unit": UNIT, "cores": 1, "kind": "oracle",
              "sample": f"{n} runs of {note}, single thread, COL schedule, {el:.1f} s"}
    # the paper's sequential sweep (SEQ) on the same sample, beside it
    t0 = time.perf_counter()
    oracle.run(imgs[0], **p, schedule=oracle.SEQ)
    single["seq_value"] = imgs[0].shape[0] * imgs[0].shape[1] / (time.perf_counter() - t0) / 1e6
    if name not in ("c3", "c4"):
        return single
    imgs, p, note = parallel_sample(name, host_cores())
    workers = min(host_cores(), len(imgs))  # threads actually used
    if means_iters:
        p = dict(p, means_iters=means_iters)
    if colour != "rgb":
        p = dict(p, colour=colour)
    if compact:
        p = dict(p, compact=True)
    if edge:
        p = dict(p, edge_tau=edge)
    t0 = time.perf_counter()
    oracle_frames(imgs, p, workers)
    el = time.perf_counter() - t0
    px = sample_pixels(imgs)
    return {"value": px / el / 1e6, "unit": UNIT, "cores": workers, "kind": "oracle",
            "sample": f"{note}, in parallel on {workers} host threads, COL schedule, {el:.1f} s",
            "single_thread": single}


def cpu_info():
    """Host CPU model and core count (the cpu_baseline
    states the host it ran on)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "affinity_cores": host_cores()}


def measure_extra(name, steps, flush, stream, torch):
    """One more config measured in the same process (the `extra` map of the
    bench line): device-resident steps timed with CUDA
    events on the launching stream, L2 flushed between steps, per-launch
    profile events for the roofline, traffic from the committed ncu capture."""
    wl = Workload(name, 0, 1)
    s = wl.make_context()
    info = s.info
    wl.setup(torch, s)
    for _ in range(3):
        wl.step(s, stream)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.fill_(i & 0xFF)
        ev[i][0].record(stream)
        wl.step(s, stream)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / steps
    s.profile(True)
    prof = None
    for i in range(min(steps, 5)):
        flush.fill_(i & 0xFF)
        wl.step(s, stream)
        prof = s.profile_collect(stream=stream)
    s.profile(False)
    ms_launch, nl = prof["frame"]
    avg_us = 1e3 * ms_launch / max(1, nl)
    ab = wl.algorithmic_bytes(info) / len(wl.groups)
    hbm, hbm_src = peaks()
    achieved = ab / (avg_us / 1e6) / 1e9
    traffic = None
    try:
        ent = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(f"{name}/grid", {}).get("frame")
        traffic = ent.get("dram_bytes") if isinstance(ent, dict) else ent
    except Exception:
        pass
    out = {"workload": wl.describe(info), "value": wl.frames_per_step * wl.N / (ms / 1e3) / 1e6, "unit": UNIT,
           "ms_per_step": ms, "steps": steps,
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                        "traffic": traffic, "kernel": "frame", "avg_launch_us": avg_us,
                        "algorithmic_bytes_per_launch": ab, "peak_source": hbm_src},
           "gpu_launches": info.kernels_per_run * len(wl.groups) * steps}
    s.close()
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    name = args.config
    oracle.build()
    workers = host_cores() if name in ("c3", "c4") else 1
    if workers > 1:  # batch configs: each step is one parallel batch on the host cores
        imgs, p, note = parallel_sample(name, workers, clip_len=2)  # c4: each step 8 clips x 2 frames
        workers = min(workers, len(imgs))
        batches = [imgs[i:i + workers] for i in range(0, len(imgs), workers)]
        note = f"{note}, in parallel on {workers} host threads"
    else:
        imgs, p, note = reference_sample(name)
        batches = [imgs[i:i + 1] for i in range(len(imgs))]
    if args.means_iters:
        p = dict(p, means_iters=args.means_iters)
        note += f", last {args.means_iters} pixel iterations on means"
    if args.colour != "rgb":
        p = dict(p, colour=args.colour)
        note += f", {args.colour} pre-pass"
    if args.compact:
        p = dict(p, compact=True)
        note += ", compactness prior"
    if args.edge:
        p = dict(p, edge_tau=args.edge)
        note += f", edge prior tau {args.edge}"
    for i in range(args.warmup):
        b0 = batches[i % len(batches)][:1]
        oracle_frames(b0[:, :1] if b0.ndim == 5 else b0, p, 1)
    t, px = [], 0
    for i in range(args.steps):
        bt = batches[i % len(batches)]
        t0 = time.perf_counter()
        oracle_frames(bt, p, workers)
        t.append(time.perf_counter() - t0)
        px += sample_pixels(bt)
    tot = sum(t)
    v = px / tot / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic",
            "config": {"workload": f"{name}: {note} per step, oracle COL schedule"},
            "cpu_baseline": dict({"value": v, "unit": UNIT, "cores": workers, "kind": "oracle",
                                  "sample": f"{args.steps} steps, each {note}"}, **cpu_info()),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="auto", choices=["auto", "graph", "grid"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--bands", type=int, default=0,
                    help="c5 on one rank: row-band mode with this many bands in one launch (multi-rank c5 always bands)")
    ap.add_argument("--colour", default="rgb", choices=["rgb", "lab"],
                    help="lab: the 8-bit CIELAB pre-pass inside the timed run (reading M3)")
    ap.add_argument("--compact", action="store_true", help="the compactness prior at the pixel level (reading M5)")
    ap.add_argument("--edge", type=int, default=0, help="the edge prior with this colour threshold (reading M6)")
    ap.add_argument("--extra", default="auto",
                    help="comma-separated configs measured in the same run into the line's `extra` map "
                         "(auto: c3,c5 on a default one-GPU c2 run; none: off)")
    ap.add_argument("--means-iters", type=int, default=0,
                    help="SPM means post-processing: the last M pixel iterations use the means test (reading M1)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1309_3848_b200.seeds import Seeds

    name = args.config
    banded = name == "c5" and (world > 1 or args.bands > 0)
    wl = BandWorkload(name, rank, world, max(1, args.bands)) if banded else Workload(name, rank, world)
    p = wl.p
    s = wl.make_context()
    if not banded:
        s.set_mode(args.mode)
        if args.means_iters:
            s.set_means_iters(args.means_iters)
        if args.compact:
            s.set_compactness(True)
        if args.edge:
            s.set_edge_prior(args.edge)
    if args.colour != "rgb":
        s.set_colour_space(args.colour)
    info = s.info
    stream = torch.cuda.current_stream()
    wl.setup(torch, s)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    for _ in range(max(3, args.warmup)):
        wl.step(s, stream)
    torch.cuda.synchronize()
    info = s.info
    mode_name = "grid-bands" if banded else MODE_NAMES.get(info.exec_mode, str(info.exec_mode))

    # ---- timed region: K steps, CUDA events on the launching stream -------
    clocks = Clocks(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i & 0xFF)  # evict L2 between steps (outside the events)
        ev[i][0].record(stream)
        wl.step(s, stream)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    tot_ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([tot_ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms_max = float(t.item())
    # pixels refined by the whole job per step: a banded c5 frame is one frame over all ranks
    px_all = (wl.N if banded else wl.frames_per_step * wl.N * world) * args.steps
    value = px_all / (tot_ms_max / 1e3) / 1e6
    runs_per_step = len(wl.groups)
    launches = info.kernels_per_run * runs_per_step * args.steps
    if banded:  # seed + k_grid + one emit per band of this process
        launches = (2 + (s.n_bands if s.band < 0 else 1)) * args.steps

    # ---- per-kernel timing pass (event pairs inside the graph) ------------
    kp = min(args.steps, 20)
    s.profile(True)
    prof = None
    for i in range(kp):
        flush.fill_(i & 0xFF)
        wl.step(s, stream)
        prof = s.profile_collect(stream=stream)
    s.profile(False)
    torch.cuda.synchronize()
    ab = algorithmic_bytes(info, wl.C, wl.nf, wl.N, p["iters_per_level"])
    ab["frame"] = wl.algorithmic_bytes(info) / runs_per_step  # per launch (a warm run has no block levels)
    kinds = {k: {"ms_total": v[0] / kp, "launches": v[1] // kp,
                 "avg_launch_us": 1e3 * v[0] / max(1, v[1]),
                 "gbps": (ab[k] / (v[0] / max(1, v[1]) / 1e3) / 1e9) if v[1] else None}
             for k, v in prof.items() if v[1]}
    dom = max(kinds, key=lambda k: kinds[k]["ms_total"])
    hbm, hbm_src = peaks()
    traffic, inst, ncu_us = None, None, None
    default_path = not (args.means_iters or args.compact or args.edge or args.colour != "rgb")
    try:  # ncu evidence of the same launch (profiles/ncu_traffic.json, scripts/gpu_final_profiles.sh)
        if not default_path:
            raise KeyError("the ncu captures are of the default path")
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        ent = tr.get(f"{name}/{mode_name}", {}).get(dom)
        if isinstance(ent, dict):
            traffic, inst, ncu_us = ent.get("dram_bytes"), ent.get("warp_inst"), ent.get("launch_us")
        else:
            traffic = ent
    except Exception:
        pass
    achieved = kinds[dom]["gbps"]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm if achieved else None, "traffic": traffic,
                "kernel": dom, "peak_source": hbm_src,
                "algorithmic_bytes_per_launch": ab[dom],
                "note": "latency-bound: one grid barrier per sub-sweep dominates a single frame"
                        if wl.frames_per_step * wl.N < 4_000_000 else "per-launch algorithmic bytes / launch time"}

    # Issue-rate roofline: the kernel is latency / issue bound, not HBM bound
    # (DESIGN.md section 6): warp instructions of one launch (ncu) over the
    # live launch time, against 4 issue slots x #SM x the sampled SM clock.
    # SURVEY 8(d) fraction (1): the DRAM bandwidth ncu measured for the launch
    if traffic and ncu_us:
        roofline["ncu_dram_gbs"] = traffic / (ncu_us * 1e3)
        roofline["ncu_dram_frac"] = roofline["ncu_dram_gbs"] / hbm
    # The instruction count and its time come from the same ncu capture (for
    # c4 that capture is a cold 8-frame launch while the bench averages cold
    # and warm launches, so the live average would not pair with it).
    issue = None
    if inst and ncu_us:
        sm_mhz = (clk or {}).get("sm_mhz") or 1965.0
        peak_gis = 4 * torch.cuda.get_device_properties(local).multi_processor_count * sm_mhz / 1e3
        ach = inst / (ncu_us * 1e3)
        issue = {"bound": "issue", "achieved": ach, "peak": peak_gis, "unit": "Gwarp-inst/s",
                 "frac": ach / peak_gis, "warp_inst_per_launch": inst, "ncu_launch_us": ncu_us,
                 "live_avg_launch_us": kinds[dom]["avg_launch_us"],
                 "inst_source": "ncu smsp__inst_executed.sum and gpu__time_duration.sum of one launch"}
        if name == "c4":
            issue["note"] = "ncu capture: a cold 8-frame launch (block levels + pixel level); warm launches are cheaper"
            roofline["traffic_note"] = "ncu traffic of a cold 8-frame launch"

    # ---- end to end through the host-memory C-ABI entry point --------------
    for _ in range(3):
        wl.host_step(s, stream)
    e2e_ms = 0.0
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        wl.host_step(s, stream)
        b.record(stream)
        b.synchronize()
        e2e_ms += a.elapsed_time(b)
    t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = px_all / (float(t.item()) / 1e3) / 1e6
    wl.check(torch)

    if rank == 0:
        fb = wl.algorithmic_bytes(info)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms_max / args.steps, "higher_is_better": True,
            "scaling": wl.scaling, "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": wl.describe(info),
                       "frames_per_step_per_rank": wl.frames_per_step,
                       "exec_mode": mode_name,
                       "means_iters": args.means_iters,
                       "colour": args.colour,
                       "compact": args.compact,
                       "edge_tau": args.edge,
                       "grid_ctas": info.grid_ctas, "grid_tiles_per_frame": info.grid_tiles,
                       # the refinement kernel the roofline's "frame" launch is: one k_tile1 launch per
                       # cold run when every CTA owns one tile, else seed + k_grid + emit
                       "refine_kernel": ("k_tile1" if mode_name == "grid" and info.kernels_per_run == 1 else
                                         "k_grid" if mode_name.startswith("grid") else "graph kernels"),
                       "parallelism": wl.parallelism,
                       "exchange": ("inside the persistent kernel: owner-band histogram updates and halo label rows "
                                    "through peer memory, one counter barrier per sub-sweep") if banded else None,
                       "l2": "512 MiB buffer rewritten between timed steps (outside events)"},
            "frames_per_s": wl.frames_per_step * world * args.steps / (tot_ms_max / 1e3),
            "e2e_hbm_frac": (fb * args.steps / (tot_ms_max / 1e3) / 1e9) / hbm,
            "roofline": roofline,
            "issue_roofline": issue,
            "kernels": kinds,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(wl.h2d_bytes()),
                    "d2h_bytes_per_step": int(wl.d2h_bytes())},
            "gpu_launches": launches,
            "clocks": clk,
        }
        extra = args.extra
        if extra == "auto":
            extra = "c3,c5" if (name == "c2" and world == 1 and default_path and args.mode == "auto") else "none"
        if extra != "none":
            line["extra"] = {}
            for x in extra.split(","):
                line["extra"][x] = measure_extra(x, min(args.steps, 10), flush, stream, torch)
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(name, args.cpu_budget, args.means_iters, args.colour, args.compact,
                                                args.edge)
            line["cpu_baseline"].update(cpu_info())
        out = json.dumps(line)
        print(out)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(out + "\n")
    s.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
