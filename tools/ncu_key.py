"""Key metrics + stall breakdown of ncu reports (one line per report).

    python tools/ncu_key.py a.ncu-rep [b.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "ms",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
    "sm__warps_active.avg.per_cycle_active": "warps/SM",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "simt",
    "l1tex__t_sector_hit_rate.pct": "L1hit%",
    "lts__t_sector_hit_rate.pct": "L2hit%",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64%",
    "dram__bytes_read.sum": "dramR",
    "sm__inst_executed.sum": "inst",
}
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u, v = r[0], r[1], r[2]
    d = dict(zip(h, v))
    units = dict(zip(h, u))
    line = {name: f"{d.get(k, '?')}{units.get(k, '')}" for k, name in KEYS.items()}
    st = {k.split("stalled_")[1]: float(x.replace(",", "")) for k, x in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k and x}
    tot = sum(st.values()) or 1
    top = sorted(st.items(), key=lambda kv: -kv[1])[:7]
    print(rep.split("/")[-1], line)
    print("   stalls:", ", ".join(f"{k} {100 * x / tot:.0f}%" for k, x in top))
