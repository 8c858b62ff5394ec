"""Per-region stall samples / instructions of the path kernel from an ncu report.

    python tools/ncu_regions.py <rep.ncu-rep> <kernel-mangled-substring> [cubin]

Maps every SASS instruction (ncu --page source --print-source sass) to the
nearest preceding trace.cu source line in `nvdisasm -gi` of the same kernel
(inlined dmath / rng / physics code is attributed to the trace.cu line that
called it), then sums samples and executed instructions per trace.cu region.
"""
import csv
import io
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, kern = sys.argv[1], sys.argv[2]
cubin = sys.argv[3] if len(sys.argv) > 3 and sys.argv[3] != "-" else None
if cubin is None:
    os.makedirs("/tmp/ncu_regions", exist_ok=True)
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2511_07586_b200/csrc/trace.o")],
                   cwd="/tmp/ncu_regions", capture_output=True)
    cubin = "/tmp/ncu_regions/trace.sm_100a.cubin"
sass = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout
# the kernel's text section
start = None
lines = sass.splitlines()
for i, l in enumerate(lines):
    if l.startswith(".text.") and kern in l and l.endswith(":"):
        start = i
        break
assert start is not None, "kernel not found"
ctx_line = {}  # offset -> (file, line, trace_line)
cur_file, cur_line, trace_line = None, None, 0
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//---------------------"):
        break
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
    if m:
        cur_file, cur_line = os.path.basename(m.group(1)), int(m.group(2))
        if cur_file == "trace.cu":
            trace_line = cur_line
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        ctx_line[int(m.group(1), 16)] = (cur_file, cur_line, trace_line)

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows_all = list(csv.reader(io.StringIO(out)))
# one block per profiled kernel: a "Kernel Name" row, a header row, then SASS rows
rows, take = [], False
for r in rows_all:
    if r and r[0] == "Kernel Name":
        base_name = kern.split("ILi")[0]
        take = (base_name + "<") in r[1] or (base_name + "(") in r[1] or kern in r[1]
        if take and rows:
            break  # first matching kernel only
        continue
    if take:
        rows.append(r)
rows.insert(0, ["Kernel Name"])
hdr = rows[1]
ai, si, ii = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = [(int(r[ai], 16), int(r[si] or 0), int(r[ii] or 0)) for r in rows[2:] if len(r) > ii and r[ai].startswith("0x")]
ti_col = hdr.index("Thread Instructions Executed") if "Thread Instructions Executed" in hdr else None
loc_col = hdr.index("L2 Theoretical Sectors Local") if "L2 Theoretical Sectors Local" in hdr else None
extra_by_addr = {int(r[ai], 16): (int(r[ti_col] or 0) if ti_col is not None else 0,
                                  int(float(r[loc_col] or 0)) if loc_col is not None else 0)
                 for r in rows[2:] if len(r) > ii and r[ai].startswith("0x")}
stall_cols = [(h, hdr.index(h)) for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
stall_by_addr = {int(r[ai], 16): {h: int(r[c] or 0) for h, c in stall_cols}
                 for r in rows[2:] if len(r) > ii and r[ai].startswith("0x")}
base = min(a for a, _, _ in data)

# regions: each starts at the first trace.cu line containing its marker and
# runs to the next region's start (markers in file order)
MARKERS = [
    ("helpers", "constexpr unsigned kFull"), ("make_fray", "FRay make_fray("), ("minmax/ffma2", "float fmin3("),
    ("tri_test", "bool tri_test("), ("traverse", "bool traverse("), ("fill_hit", "HitInfo<NT> fill_hit("),
    ("slot/state", "struct Path {"), ("locate", "Entry locate("), ("cover", "bool covered("),
    ("init_path", "void init_path("), ("project", "void project("), ("det helpers", "det_at("),
    ("flush_sums", "void flush_sums("), ("freq_phasor", "Cx freq_phasor("), ("kernel setup", "path_kernel(TraceParams P)"),
    ("next sub-range", "// ---- next sub-range"), ("regen", "// ---- regenerate dead lanes"),
    ("query", "double t = 0.0;"), ("pend/visible", "bool visible = false;"), ("shading", "load_em<L>(sl, s, S.ambient_n);"),
    ("chi/queue", "// ---- chi visibility"), ("accumulate/records", "// ---- bistatic fan"),
    ("counters", "// ---- counters ----"), ("accumulate_kernel", "accumulate_kernel(TraceParams P"),
]
src = open(os.environ.get("MCSBR_TRACE_SRC", os.path.join(ROOT, "paper_2511_07586_b200/csrc/trace.cu"))).read().splitlines()
REGIONS = []
starts = []
for name, mk in MARKERS:
    ln = next((i + 1 for i, l in enumerate(src) if mk in l), None)
    if ln is not None:
        starts.append((ln, name))
starts.sort()
for k, (ln, name) in enumerate(starts):
    REGIONS.append((name, ln, starts[k + 1][0] - 1 if k + 1 < len(starts) else 10**9))


def region(tl):
    for n, a, b in REGIONS:
        if a <= tl <= b:
            return n
    return f"other:{tl}"


agg = {}
for a, s, i in data:
    f, ln, tl = ctx_line.get(a - base, (None, None, 0))
    r = region(tl)
    x = agg.setdefault(r, [0, 0, 0])
    x[0] += s
    x[1] += i
    x[2] += 1
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"{len(data)} SASS instructions ({len(data) * 16 / 1024:.0f} KB), {ts} samples, {ti:.3e} warp inst")
stall_reg = {}
for a, s_, i in data:
    r = region(ctx_line.get(a - base, (None, None, 0))[2])
    d = stall_reg.setdefault(r, {})
    for h, v in stall_by_addr.get(a, {}).items():
        d[h] = d.get(h, 0) + v
thr_reg, loc_reg = {}, {}
for a, s_, i in data:
    r = region(ctx_line.get(a - base, (None, None, 0))[2])
    t_, l_ = extra_by_addr.get(a, (0, 0))
    thr_reg[r] = thr_reg.get(r, 0) + t_
    loc_reg[r] = loc_reg.get(r, 0) + l_
for r, (s, i, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    simt = thr_reg.get(r, 0) / i if i else 0.0
    print(f"{r:22s} {100 * s / ts:5.1f}% samples  {100 * i / ti:5.1f}% inst  {n:5d} sass ({n * 16 / 1024:.1f} KB)"
          f"  simt {simt:4.1f}  local sectors {loc_reg.get(r, 0):.3g}")
    d = stall_reg.get(r, {})
    tot = sum(d.values()) or 1
    top = sorted(d.items(), key=lambda kv: -kv[1])[:6]
    if s / ts > 0.02:
        print("      " + "  ".join(f"{h[6:]} {100 * v / tot:.0f}%" for h, v in top))

if len(sys.argv) > 4:  # top SASS instructions of one region
    want = sys.argv[4]
    sass_text = {}
    for r in rows[2:]:
        if len(r) > ii and r[ai].startswith("0x"):
            sass_text[int(r[ai], 16)] = r[1].strip()
    top = sorted(((s, i, a) for a, s, i in data if region(ctx_line.get(a - base, (0, 0, 0))[2]) == want), reverse=True)
    for s, i, a in top[:60]:
        f, ln, tl = ctx_line.get(a - base, (None, None, 0))
        print(f"{100 * s / ts:5.2f}% {i:>11d} {a - base:6x} {f}:{ln} ({tl})  {sass_text[a][:70]}")

if len(sys.argv) > 5 and sys.argv[5] == "lines":  # samples / instructions / code bytes per trace.cu line
    per = {}
    for a, s, i in data:
        tl = ctx_line.get(a - base, (None, None, 0))[2]
        x = per.setdefault(tl, [0, 0, 0, 0])
        x[0] += s
        x[1] += i
        x[2] += 1
        x[3] += extra_by_addr.get(a, (0, 0))[1]
    key = 3 if len(sys.argv) > 6 and sys.argv[6] == "local" else 0
    print("trace.cu line: samples% inst% sass local-sectors")
    for tl, (s, i, n, lc) in sorted(per.items(), key=lambda kv: -kv[1][key])[:40]:
        txt = src[tl - 1].strip()[:70] if 0 < tl <= len(src) else ""
        print(f"{tl:5d} {100 * s / ts:5.1f} {100 * i / ti:5.1f} {n:5d} {lc:10.3g}  {txt}")
