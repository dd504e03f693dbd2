"""profiles/ncu_traffic.json from ncu --set full captures of one refinement launch (k_tile1 for
the single-tile c2 plan, k_grid for c3-c5):
DRAM bytes (read + write) and warp instructions per launch, per config."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    get = lambda n: (float(v[h.index(n)].replace(",", "")), u[h.index(n)])
    rb, ru = get("dram__bytes_read.sum")
    wb, wu = get("dram__bytes_write.sum")
    inst, _ = get("smsp__inst_executed.sum")
    t, tu = get("gpu__time_duration.sum")
    return {"dram_bytes": int(rb * UNITS[ru] + wb * UNITS[wu]), "warp_inst": int(inst),
            "launch_us": t * (1e3 if tu == "ms" else 1.0)}


res = {"_source": "ncu --set full --clock-control none of one refinement launch (scripts/make_traffic.py): "
                  "c2 k_tile1 (seed, refinement and int32 labels in one launch), c3-c5 k_grid; "
                  "c3 and c4 are cold batch launches (c4: one 8-frame time step)"}
for arg in sys.argv[1:]:
    key, path = arg.split("=")
    res[key] = {"frame": raw(path)}
    print(key, res[key])
with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
    json.dump(res, f, indent=1)
