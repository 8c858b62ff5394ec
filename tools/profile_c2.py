"""One warm-up + one timed launch of the bench workload (c2 sweep) for ncu.

    python tools/profile_c2.py [--angles N]
ncu: --set full -k regex:path_kernel -s 1 -c 1 (the second path_kernel launch).
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2511_07586_b200 as M  # noqa: E402
from paper_2511_07586_b200 import _abi as A  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--angles", type=int, default=181)
args = ap.parse_args()
W = bench.WORKLOADS["c2"]
sd, excs = W.scene_fn(), W.excs_fn()
excs = excs[:: max(1, len(excs) // args.angles)][: args.angles]
scene = M.Scene(sd)
lam = bench.C0 / W.freqs[-1]
spws = [bench.spw_for(M, scene, e, lam, W.rays) for e in excs]
cfg = W.config(M)
L = A.lib()
for it in range(3):
    L.mcsbr_gpu_kernel_timing(1)
    vals, st = M.estimate_batch(scene, [(e, s) for e, s in zip(excs, spws)], [[e] for e in excs],
                                W.freqs, cfg)
pk = C.c_double()
L.mcsbr_gpu_kernel_times(C.byref(pk), None, None, None)
L.mcsbr_gpu_kernel_timing(0)
print(f"paths {st.rays_launched} kernel_ms {st.kernel_ms:.3f} path_kernel_ms {pk.value:.3f} "
      f"Gpaths/s {st.rays_launched / st.kernel_ms / 1e6:.3f} segments {st.segments_traced} "
      f"occlusion {st.occlusion_queries}")
