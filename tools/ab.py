"""A/B timing of library variants and scheduling knobs in ONE box session
(box-to-box variance is ~5%, so only same-box comparisons mean anything).

    python tools/ab.py [--configs c1,c4] [--c2] [--reps 2] VARIANT ...
VARIANT = tag=lib[,KEY=VAL...]   lib '' = the in-tree default library,
                                 else paper_2511_07586_b200/libmcsbr_gpu_<lib>.so
e.g.  python tools/ab.py --c2 --configs c1,c3 new= old=old gss0=,MCSBR_GSS=0,MCSBR_CHUNK_MAX=224
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c4,c5")
ap.add_argument("--c2", action="store_true")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("variants", nargs="+")
a = ap.parse_args()
res = {}
for rep in range(a.reps):
    for v in a.variants:
        tag, rest = v.split("=", 1)
        parts = rest.split(",")
        env = dict(os.environ)
        env.pop("MCSBR_GPU_LIB", None)
        if parts[0]:
            env["MCSBR_GPU_LIB"] = os.path.join(ROOT, "paper_2511_07586_b200", f"libmcsbr_gpu_{parts[0]}.so")
        for kv in parts[1:]:
            k, val = kv.split("=", 1)
            env[k] = val
        row = res.setdefault(tag, {})
        if a.c2:
            out = subprocess.run([sys.executable, "tools/profile_c2.py"], cwd=ROOT, env=env,
                                 capture_output=True, text=True).stdout.strip().splitlines()
            ms = float(out[-1].split("kernel_ms")[1].split()[0]) if out else float("nan")
            row.setdefault("c2", []).append(round(ms, 3))
        if a.configs:
            path = f"/tmp/ab_{tag}.json"
            subprocess.run([sys.executable, "tools/bench_configs.py", "--configs", a.configs, "--out", path],
                           cwd=ROOT, env=env, capture_output=True, text=True)
            try:
                d = json.load(open(path))
            except Exception as e:  # noqa: BLE001
                d = {}
                print(tag, "failed", e)
            for k, x in d.items():
                row.setdefault(k, []).append(round(x.get("gpu_ms_per_angle", x.get("gpu_ms")), 3))
        print(tag, row, flush=True)
print(json.dumps(res))
