"""Aggregate an ncu source page (cuda,sass) by CUDA source line: warp-stall
samples, instructions executed; usage: ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
lines = []
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0] not in ("", "Function Name"):
        d = dict(zip(hdr[:2] + ["addr", "sass"] + hdr[4:], r))
        try:
            lines.append((int(d["Warp Stall Sampling (All Samples)"]), int(d["Instructions Executed"] or 0),
                          fname, int(r[0]), r[1].strip()[:90]))
        except (ValueError, KeyError):
            pass
tot = sum(x[0] for x in lines) or 1
lines.sort(reverse=True)
print(f"total samples {tot}")
for s, ins, f, ln, src in lines[:top]:
    print(f"{100 * s / tot:5.1f}% {s:7d} {ins:10d} {f}:{ln:<5d} {src}")
