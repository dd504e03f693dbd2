"""Aggregate an ncu 'source --print-source cuda,sass' CSV per CUDA source line."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None; cur = None; out = []
for r in rows:
    if len(r) == 2 and r[0] in ('File Path', 'File Name'): cur = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': hdr = r; continue
    if hdr is None or len(r) < len(hdr) or r[2] != '-': continue
    d = dict(zip(hdr[4:], r[4:]))
    stalls = {h: int(v) for h, v in zip(hdr[32:49], r[32:49]) if v.isdigit() and int(v) > 0}
    try: out.append((int(r[4]), int(r[7]), cur, r[0], r[1].strip()[:90], stalls))
    except ValueError: pass
ts = sum(o[0] for o in out); ti = sum(o[1] for o in out)
print("samples", ts, "warp-instructions", ti)
for o in sorted(out, key=lambda o: -o[0])[:top]:
    st = ' '.join(f"{k[6:]}={v}" for k, v in sorted(o[5].items(), key=lambda kv: -kv[1])[:3])
    print(f"{o[0]:>6} {100*o[0]/ts:5.1f}% inst {o[1]:>9} {o[2]}:{o[3]} {o[4]} | {st}")
