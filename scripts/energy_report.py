"""P14 report (north star: "the final energy of the coloured schedule is
reported next to the sequential sweep's"): final H (normalised colour term,
PAPER.md:977), G' (raw boundary term) and E = H + gamma G of the coloured
snapshot schedule (COL, what the GPU computes bit for bit) and of the paper's
sequential raster sweep (SEQ), per config, plus the grid's energy.  Runs the
CPU oracle only; writes profiles/r01/energies.json."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1309_3848_b200 import configs  # noqa: E402

out = {}
cases = [("c1", None), ("c2", None), ("c3", None), ("c4", None), ("c5", (1024, 1024))]
for cfg, crop in cases:
    p = dict(configs.params(cfg))
    if cfg == "c4":
        img = configs.frames(cfg, n=1)[0]
    else:
        img = configs.frames(cfg, n=1)[0]
    note = "full frame"
    if crop:
        img = np.ascontiguousarray(img[:crop[0], :crop[1]])
        p["n_superpixels"] = p["n_superpixels"] * crop[0] * crop[1] // (8192 * 8192)
        note = f"{crop[0]}x{crop[1]} crop, K scaled"
    row = {"note": note, "params": p}
    g = orc_grid = oracle.run(img, **dict(p, iters_per_level=0))
    Hn, Hr, Gr, Gn = oracle.energy(g.labels, img, p["bins_per_channel"], g.k_act)
    row["grid"] = {"H": Hn, "Graw": Gr}
    for name, sch in (("COL", oracle.COL), ("SEQ", oracle.SEQ)):
        r = oracle.run(img, **p, schedule=sch)
        Hn, Hr, Gr, Gn = oracle.energy(r.labels, img, p["bins_per_channel"], r.k_act)
        row[name] = {"H": Hn, "Graw": Gr, "E": Hn + p["smoothness_prior"] * Gn}
    out[cfg] = row
    print(cfg, note, "grid H %.3f | COL H %.3f G' %.0f | SEQ H %.3f G' %.0f" % (
        row["grid"]["H"], row["COL"]["H"], row["COL"]["Graw"], row["SEQ"]["H"], row["SEQ"]["Graw"]))
with open(os.path.join(ROOT, "profiles", "r01", "energies.json"), "w") as f:
    json.dump(out, f, indent=1)
