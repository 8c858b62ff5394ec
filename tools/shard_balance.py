"""Load balance of the multi-GPU ray shards on one GPU: every rank's
mcsbr_gpu_trace_device shard of a bench workload, timed alone (CUDA events
on the launch stream); prints per-rank times, max / mean and the resulting
strong-scaling efficiency bound  T(1) / (W * max_r T_r).

    python tools/shard_balance.py [c5|c2] [--angles K] [--worlds 2,4,8]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_07586_b200 as M  # noqa: E402
from paper_2511_07586_b200 import _abi as A  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="c5")
ap.add_argument("--angles", type=int, default=16)
ap.add_argument("--worlds", default="2,4,8")
args = ap.parse_args()
W = bench.WORKLOADS[args.workload]
sd = W.scene_fn()
dev = torch.device("cuda", 0)
scene = M.Scene(sd)
lam = bench.C0 / W.freqs[-1]
excs = W.excs_fn()
idx = np.linspace(0, len(excs) - 1, min(args.angles, len(excs))).round().astype(int)
excs = [excs[i] for i in idx]
spws = [bench.spw_for(M, scene, e, lam, W.rays) for e in excs]
ccfg = W.config(M).to_c()
n, nf = len(excs), len(W.freqs)
incs = (A.Incidence * n)(*[e.incidence(s) for e, s in zip(excs, spws)])
rxs = (A.Receiver * n)(*[e.receiver() for e in excs])
freqs = np.ascontiguousarray(W.freqs)
sums = torch.zeros(n * nf * 8, dtype=torch.float64, device=dev)
cnt = torch.zeros(A.MCSBR_COUNTER_WORDS, dtype=torch.int64, device=dev)
stream = torch.cuda.current_stream(dev)
L = A.lib()


def shard(rank, world, reps=2):
    best = None
    for _ in range(reps):
        sums.zero_()
        cnt.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        A.check(L.mcsbr_gpu_trace_device(scene.handle, incs, n, rxs, 1, 1,
                                         freqs.ctypes.data_as(C.POINTER(C.c_double)), nf, C.byref(ccfg), rank,
                                         world, C.c_void_p(sums.data_ptr()), C.c_void_p(cnt.data_ptr()),
                                         C.c_void_p(stream.cuda_stream)))
        b.record(stream)
        torch.cuda.synchronize()
        t = a.elapsed_time(b)
        best = t if best is None else min(best, t)
    return best


shard(0, 1)  # warm-up (coverage bitmaps, record ratio)
t1 = shard(0, 1)
out = {"workload": args.workload, "incidences": n, "t1_ms": t1}
for w in [int(x) for x in args.worlds.split(",")]:
    ts = [shard(r, w) for r in range(w)]
    out[f"w{w}"] = {"ms": [round(x, 3) for x in ts], "max_over_mean": max(ts) / (sum(ts) / w),
                    "efficiency_bound": t1 / (w * max(ts))}
print(json.dumps(out, indent=1))
