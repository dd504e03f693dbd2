#!/usr/bin/env python
"""Benchmark of the SEEDS refinement hot path on B200 (BASELINE.json metric:
"Mpixels/s SEEDS refinement (481x321 frames/s, 200 SP); % of B200 HBM peak").

One step = one whole refinement (seed, every block and pixel sub-sweep, emit)
of one batch of synthetic frames already resident in HBM.  Default workload:
c2 = one 481x321 RGB Voronoi-mosaic frame, K=200, 4 block levels, I=4, 125
bins, gamma=1 (BASELINE.json configs[1]).  A c2 frame does not shard, so N
GPUs run N independent replicas ("scaling": "weak"); --config c3 runs the
256-frame batch sharded by frame ("strong").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c1]
  python bench.py --impl reference ...   # the CPU oracle, timed as it stands

L2: a 512 MiB buffer (> 126 MB L2) is rewritten between timed steps, outside
the CUDA-event brackets of each step; the inputs themselves fit in L2.
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


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def algorithmic_bytes(info, C, nf, N):
    """Per-launch algorithmic bytes of each kernel class."""
    bb, P, L = info.bin_bytes, info.colour_period, info.levels_eff
    return {
        "seed": nf * N * (C + bb + (0 if L > 0 else 2)),   # image in, bins (+ labels) out
        "block": nf * N * bb / 4.0,                         # bin plane once per 4 sub-sweeps
        "pixel": nf * N * (2 + bb) / float(P * P),          # labels + bins once per P^2 sub-sweeps
        "emit": nf * N * (2 + 4),                           # uint16 in, int32 out
    }


def frame_bytes(info, C, N, iters):
    """Algorithmic bytes of one cold frame: N [C + bb + 4 + I L bb + I (2 + bb)]."""
    bb, L = info.bin_bytes, info.levels_eff
    return N * (C + bb + 4 + iters * L * bb + iters * (2 + bb))


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        if not shutil.which("nvidia-smi"):
            return
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits", "-lms", "100"],
                                     stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def workload(name, rank, world):
    c = configs.CONFIGS[name]
    if name == "c3":
        per = c["frames"] // world
        lo = rank * per
        imgs = configs.frames(name)[lo:lo + per]
        scaling = "strong"
    else:
        imgs = configs.frames(name, n=1)
        scaling = "weak"
    return c, imgs, scaling


def cpu_baseline(name, budget_s=10.0):
    """The oracle as it stands (one thread, COL schedule) on a bounded sample."""
    import oracle
    c = configs.CONFIGS[name]
    p = configs.params(name)
    imgs = configs.frames(name, n=1 if name != "c3" else 4)
    oracle.build()
    n, t0 = 0, time.perf_counter()
    while True:
        oracle.run(imgs[n % len(imgs)], **p)
        n += 1
        el = time.perf_counter() - t0
        if el >= budget_s or n >= 200:
            break
    px = n * c["W"] * c["H"]
    return {"value": px / el / 1e6, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{n} {c['W']}x{c['H']} frames of {name}, single thread, COL schedule, "
                      f"{el:.1f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    name = args.config
    c = configs.CONFIGS[name]
    p = configs.params(name)
    imgs = configs.frames(name, n=1 if name != "c3" else 2)
    oracle.build()
    for i in range(args.warmup):
        oracle.run(imgs[i % len(imgs)], **p)
    t = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        oracle.run(imgs[i % len(imgs)], **p)
        t.append(time.perf_counter() - t0)
    tot = sum(t)
    px = args.steps * c["W"] * c["H"]
    v = px / tot / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": {"workload": f"{name}: {c['W']}x{c['H']} RGB mosaic, "
                                                        f"1 frame/step, oracle COL schedule"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{args.steps} frames of {name}, one frame per step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="auto", choices=["auto", "graph", "resident", "grid"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--json-out", default=None)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
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
    c, imgs, scaling = workload(name, rank, world)
    nf, H, W, C = imgs.shape
    N = H * W
    p = configs.params(name)
    s = Seeds(W, H, C, p["n_superpixels"], p["n_levels"], p["bins_per_channel"],
              p["smoothness_prior"], p["iters_per_level"])
    s.set_mode(args.mode)
    info = s.info
    stream = torch.cuda.current_stream()
    d_img = torch.from_numpy(np.ascontiguousarray(imgs)).cuda()
    d_out = torch.empty((nf, H, W), dtype=torch.int32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def step():
        s.batch(d_img, labels_out=d_out, stream=stream)

    for i in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

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
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = sum(step_ms)
    t = torch.tensor([tot_ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms_max = float(t.item())
    px_all = nf * N * world * args.steps
    value = px_all / (tot_ms_max / 1e3) / 1e6
    launches = info.kernels_per_run * args.steps

    # ---- per-kernel timing pass (event pairs inside the graph) ------------
    s.profile(True)
    kp = min(args.steps, 20)
    for i in range(kp):
        flush.fill_(i & 0xFF)
        step()
        prof = s.profile_collect(stream=stream)
    s.profile(False)
    torch.cuda.synchronize()
    ab = algorithmic_bytes(info, C, nf, N)
    ab["frame"] = frame_bytes(info, C, N, p["iters_per_level"]) * nf
    kinds = {k: {"ms_total": v[0] / kp, "launches": v[1] // kp,
                 "avg_launch_us": 1e3 * v[0] / max(1, v[1]),
                 "gbps": (ab[k] / (v[0] / max(1, v[1]) / 1e3) / 1e9) if v[1] else None}
             for k, v in prof.items()}
    dom = max(kinds, key=lambda k: kinds[k]["ms_total"])
    hbm, hbm_src = peaks()
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get(name, {}).get(dom)
    except Exception:
        pass
    achieved = kinds[dom]["gbps"]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm if achieved else None, "traffic": traffic,
                "kernel": dom, "peak_source": hbm_src,
                "algorithmic_bytes_per_launch": ab[dom]}

    # ---- end to end through the host-memory C-ABI entry point --------------
    h_img = torch.from_numpy(np.ascontiguousarray(imgs)).pin_memory()
    h_out = torch.empty((nf, H, W), dtype=torch.int32).pin_memory()
    h_img_np, h_out_np = h_img.numpy(), h_out.numpy()
    for _ in range(3):
        s.batch_host(h_img_np, h_out_np, stream=stream)
    e2e_ms = 0.0
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        s.batch_host(h_img_np, h_out_np, stream=stream)
        b.record(stream)
        b.synchronize()
        e2e_ms += a.elapsed_time(b)
    t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = px_all / (float(t.item()) / 1e3) / 1e6
    assert (h_out == d_out.cpu()).all(), "host and device entry points disagree"

    if rank == 0:
        fb = frame_bytes(info, C, N, p["iters_per_level"])
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms_max / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": f"{name}: {nf} x {W}x{H} RGB Voronoi mosaic per rank, "
                                   f"K={p['n_superpixels']} (K_act={info.k_actual}), "
                                   f"L={info.levels_eff}, I={p['iters_per_level']}, "
                                   f"B={info.bins_total}, gamma={p['smoothness_prior']}",
                       "frames_per_step_per_rank": nf,
                       "exec_mode": {1: "graph", 2: "resident", 3: "grid"}[info.exec_mode],
                       "cluster_size": info.cluster_size,
                       "parallelism": "replicas" if scaling == "weak" else f"frames/{world}",
                       "l2": "512 MiB buffer rewritten between timed steps (outside events)"},
            "frames_per_s": nf * world * args.steps / (tot_ms_max / 1e3),
            "e2e_hbm_frac": (fb * nf * args.steps / (tot_ms_max / 1e3) / 1e9) / hbm,
            "roofline": roofline,
            "kernels": kinds,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(nf * N * C),
                    "d2h_bytes_per_step": int(nf * N * 4)},
            "gpu_launches": launches,
            "clocks": clk,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(name, args.cpu_budget)
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
