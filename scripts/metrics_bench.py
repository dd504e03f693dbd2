"""Time seeds_metrics (UE / CUE / ASA / BR) on refined
frames of c2, c4 and c5 against their mosaic region maps; prints one JSON line
per config with the per-call time, Mpx/s and the HBM fraction of its
algorithmic bytes (labels + ground truth read once: 8 B/px)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1309_3848_b200 import configs  # noqa: E402
from paper_1309_3848_b200.seeds import Seeds  # noqa: E402

hbm = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 6650.0
for cfg in (sys.argv[1:] or ["c2", "c4", "c5"]):
    img, gt = configs.frames(cfg, n=1)[0], configs.regions(cfg, n=1)[0]
    p = configs.params(cfg)
    s = Seeds(img.shape[1], img.shape[0], img.shape[2], *[p[k] for k in (
        "n_superpixels", "n_levels", "bins_per_channel", "smoothness_prior", "iters_per_level")])
    lab = s.iterate(torch.from_numpy(img).cuda())
    g = torch.from_numpy(gt).cuda()
    R = int(gt.max()) + 1
    for _ in range(3):
        m = s.metrics(lab, g, R)
    torch.cuda.synchronize()
    n = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        m = s.metrics(lab, g, R)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / n
    dev = e0.elapsed_time(e1) / 1e3 / n
    N = img.shape[0] * img.shape[1]
    print(json.dumps({"config": cfg, "pixels": N, "segments": R, "call_ms": wall * 1e3, "device_ms": dev * 1e3,
                      "mpx_s": N / wall / 1e6, "hbm_frac": 8 * N / dev / 1e9 / hbm,
                      "metrics": {k: m[k] for k in ("ue", "cue", "asa", "br", "max_segments")}}))
    s.close()
