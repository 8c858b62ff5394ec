"""Aggregate an ncu --page source --csv --print-source=cuda,sass dump per source line.
usage: python tools/ncu_lines.py dump.csv [topN]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur = None
out = []
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0]:
        continue
    d = dict(zip(hdr, r))
    try:
        samp = int(d["Warp Stall Sampling (All Samples)"])
        inst = int(d["Instructions Executed"])
    except (KeyError, ValueError):
        continue
    out.append((samp, inst, cur, r[0], r[1][:90]))
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print(f"total samples {ts}  total warp instructions {ti:.3e}")
for s, i, f, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{100*s/ts:5.1f}% smp {100*i/ti:5.1f}% inst  {f}:{ln}  {src.strip()}")
