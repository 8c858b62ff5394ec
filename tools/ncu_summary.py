"""Summarise ncu outputs into profiles/ (committed evidence).

usage: python tools/ncu_summary.py <launches.csv> <full.ncu-rep> <round-tag>
writes profiles/<tag>_launches.csv (kernel, count, total/mean ms, share),
       profiles/<tag>_path_kernel.json (key metrics of the full capture),
       profiles/path_kernel_dram.json (dram bytes per launch, read by bench.py)
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
launches, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
prof = os.path.join(ROOT, "profiles")
os.makedirs(prof, exist_ok=True)

rows = [r for r in csv.reader(l for l in open(launches) if not l.startswith("=="))]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    if len(r) > vi:
        k = r[ki].split("(")[0]
        tot[k] += float(r[vi].replace(",", ""))
        cnt[k] += 1
allns = sum(tot.values())
with open(os.path.join(prof, f"{tag}_launches.csv"), "w") as f:
    f.write("kernel,launches,total_ms,mean_ms,share\n")
    for k in sorted(tot, key=lambda k: -tot[k]):
        f.write(f"{k},{cnt[k]},{tot[k] / 1e6:.4f},{tot[k] / cnt[k] / 1e6:.4f},{tot[k] / allns:.4f}\n")

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
want = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_active_pct",
    "sm__warps_active.avg.per_cycle_active": "warps_active_per_sm",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "simt_efficiency_threads",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum": "local_ld_sectors",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum": "local_st_sectors",
    "lts__t_bytes.sum": "l2_bytes",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
}
out = {"source": os.path.basename(rep), "command": "python tools/profile_c2.py (c2 sweep, 2nd path_kernel launch)"}
for i, name in enumerate(h):
    if name in want:
        out[want[name]] = {"value": v[i], "unit": u[i]}


def to_bytes(x):
    val = float(x["value"].replace(",", ""))
    return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(x["unit"], 1)


dram = to_bytes(out["dram_read"]) + to_bytes(out["dram_write"])
out["dram_bytes_per_launch"] = dram
with open(os.path.join(prof, f"{tag}_path_kernel.json"), "w") as f:
    json.dump(out, f, indent=1)
with open(os.path.join(prof, "path_kernel_dram.json"), "w") as f:
    json.dump({"dram_bytes_per_launch": dram, "source": f"profiles/{tag}_path_kernel.json"}, f, indent=1)
print(json.dumps(out, indent=1))
