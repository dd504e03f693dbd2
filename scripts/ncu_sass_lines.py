"""Warp-stall samples of an ncu report by CUDA source line, EXCLUDING the
stall_barrier samples (warps parked at a CTA barrier), with the dominant stall
reasons per line: the critical path of the busy warps.
usage: ncu_sass_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, cur, fname = None, None, ""
agg = collections.defaultdict(collections.Counter)
src = {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0] not in ("", "Function Name"):
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()[:80]
    elif hdr and r and r[0] == "" and cur and len(r) == len(hdr):
        d = dict(zip(["ln", "s1", "addr", "sass"] + hdr[4:], r))
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k and k != "stall_barrier" and v not in ("", "0", "-"):
                agg[cur][k[6:]] += int(v)
tot = sum(sum(c.values()) for c in agg.values()) or 1
print(f"non-barrier stall samples {tot}")
for key, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    n = sum(c.values())
    why = " ".join(f"{k}:{v}" for k, v in c.most_common(3))
    print(f"{100 * n / tot:5.1f}% {n:6d} {key[0]}:{key[1]:<5d} {src.get(key, '')[:70]:70s} {why}")
