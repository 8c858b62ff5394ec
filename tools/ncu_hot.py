"""Top source lines of an ncu report by warp-stall samples.

    python tools/ncu_hot.py <rep.ncu-rep> [n]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = None
tot = 0
for blk in out.split('"File Path"')[1:] if '"File Path"' in out else [out]:
    lines = list(csv.reader(io.StringIO('"File Path"' + blk)))
    fname = lines[0][1].split("/")[-1]
    hdr = None
    for r in lines:
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            si = hdr.index("Warp Stall Sampling (All Samples)")
            ii = hdr.index("Instructions Executed")
            continue
        if hdr and len(r) > si and r[0].isdigit():
            try:
                s = int(r[si])
            except ValueError:
                continue
            tot += s
            rows.append((s, fname, int(r[0]), r[1].strip()[:110], r[ii]))
rows.sort(reverse=True)
print(f"total samples {tot}")
for s, f, ln, src, ins in rows[:n]:
    print(f"{100*s/tot:5.1f}% {f}:{ln:<5} inst={ins:>12}  {src}")
