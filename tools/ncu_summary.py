"""Summarise ncu outputs into profiles/ (committed evidence).

usage: python tools/ncu_summary.py <launches.csv|-> <full.ncu-rep> <round-tag> [name] [command] [workload paths]
writes profiles/<tag>_launches.csv            (kernel, count, total/mean ms, share) unless '-'
       profiles/<tag>_<name>.json             key metrics of the full capture (name default
                                              'path_kernel' = the c2 bench workload)
       profiles/path_kernel_dram.json         dram bytes per launch (read by bench.py; c2 only)

The metrics answer the north star's question for the path kernel: achieved
L2 / HBM GB/s, SM issue and the FP32 (fma), FP64 and SFU (xu) pipe
utilisation against the B200's peaks, plus the stall mix.
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
name = sys.argv[4] if len(sys.argv) > 4 else "path_kernel"
command = sys.argv[5] if len(sys.argv) > 5 else "python tools/profile_c2.py (c2 sweep, 2nd path_kernel launch)"
prof = os.path.join(ROOT, "profiles")
os.makedirs(prof, exist_ok=True)

if launches != "-":
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
    "dram__bytes.sum.per_second": "dram_bandwidth",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "lts__t_bytes.sum.per_second": "l2_bandwidth",
    "lts__t_sectors.sum.per_second": "l2_sectors_per_second",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_bytes.sum.per_second": "l1_bandwidth",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "smsp_issue_active_pct",
    "sm__warps_active.avg.per_cycle_active": "warps_active_per_sm",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_static": "smem_static_per_block",
    "launch__shared_mem_config_size": "smem_carveout",
    "smsp__inst_executed.sum": "warp_instructions",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "simt_efficiency_threads",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fp32_fma_inst_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_inst_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "sfu_xu_inst_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_inst_pct",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum": "local_ld_sectors",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum": "local_st_sectors",
    "lts__t_sectors.sum": "l2_sectors",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed": "l1_throughput_pct",
}
out = {"source": os.path.basename(rep), "command": command}
for i, key in enumerate(h):
    base = key.split(".", 2)[-1] if key.startswith(("SM_A.", "SM_B.", "LTS.", "DRAM.")) else key
    if key in want or base in want:
        out[want.get(key, want.get(base))] = {"value": v[i], "unit": u[i]}
    elif base == "l1tex__t_sectors.sum":
        out["l1_sectors"] = {"value": v[i], "unit": u[i]}
stalls = {k.split("stalled_")[1]: float(x.replace(",", "")) for k, x in zip(h, v)
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k and x}
tot_s = sum(stalls.values()) or 1.0
out["stall_mix_pct"] = {k: round(100 * x / tot_s, 1) for k, x in sorted(stalls.items(), key=lambda kv: -kv[1])
                        if 100 * x / tot_s >= 0.5}


def to_bytes(x):
    val = float(x["value"].replace(",", ""))
    return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(x["unit"], 1)


if "l2_bandwidth" not in out and "l2_sectors_per_second" in out:  # 32-byte sectors
    x = out["l2_sectors_per_second"]
    per_ns = float(x["value"].replace(",", "")) * {"sector/ns": 1.0, "sector/us": 1e-3, "sector/s": 1e-9}.get(
        x["unit"], float("nan"))
    out["l2_bandwidth"] = {"value": f"{per_ns * 32:.3f}", "unit": "Gbyte/s"}
dram = to_bytes(out["dram_read"]) + to_bytes(out["dram_write"])
out["dram_bytes_per_launch"] = dram
with open(os.path.join(prof, f"{tag}_{name}.json"), "w") as f:
    json.dump(out, f, indent=1)
if len(sys.argv) > 7:  # the bench workload's path-kernel evidence: profiles/path_kernel_<workload>.json
    wl, paths = sys.argv[6], float(sys.argv[7])

    def num(k, scale=1.0):
        x = out.get(k)
        return None if x is None else float(str(x["value"]).replace(",", "")) * scale

    digest = {"source": f"profiles/{tag}_{name}.json", "command": command,
              "duration_ms": num("duration"), "dram_bytes_per_launch": dram,
              "l2_hit_pct": num("l2_hit_pct"), "l1_hit_pct": num("l1_hit_pct"),
              "l2_throughput_pct": num("l2_throughput_pct"),
              "l1_throughput_pct": num("l1_throughput_pct"),
              "l1_bytes_per_launch": None if num("l1_sectors") is None else 32 * num("l1_sectors"),
              "l2_bytes_per_launch": None if num("l2_sectors") is None else 32 * num("l2_sectors"),
              "issue_active_pct": num("smsp_issue_active_pct"), "warps_active_per_sm": num("warps_active_per_sm"),
              "fp64_pipe_pct": num("fp64_pipe_pct"), "fp32_fma_pipe_pct": num("fma_pipe_pct"),
              "sfu_xu_inst_pct": num("sfu_xu_inst_pct"), "simt_threads_per_warp": num("simt_efficiency_threads"),
              "stall_mix_pct": out.get("stall_mix_pct")}
    with open(os.path.join(prof, f"path_kernel_{wl}.json"), "w") as f:
        json.dump({"dram_bytes_per_path": dram / paths, "paths_per_launch": paths, "digest": digest}, f, indent=1)
print(json.dumps(out, indent=1))
