"""Where the bench's e2e time goes: scene create (upload + BVH), the batch
call, destroy -- each timed separately over a few repetitions.

    python tools/e2e_breakdown.py [c2|c5]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_07586_b200 as M  # noqa: E402

W = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else 'c2']
sd, excs = W.scene_fn(), W.excs_fn()
scene = M.Scene(sd)
lam = bench.C0 / W.freqs[-1]
spws = [bench.spw_for(M, scene, e, lam, W.rays) for e in excs]
cfg = W.config(M)
inc = list(zip(excs, spws))
rx = [[e] for e in excs]
freqs = W.freqs
import ctypes as C  # noqa: E402

from paper_2511_07586_b200 import _abi as A  # noqa: E402

L = A.lib()
for k in range(int(os.environ.get("REPS", "4"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s2 = M.Scene(sd)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    L.mcsbr_gpu_kernel_timing(1)
    vals, st = M.estimate_batch(s2, inc, rx, freqs, cfg)
    t2 = time.perf_counter()
    kt = [C.c_double(), C.c_uint64(), C.c_double(), C.c_uint64()]
    L.mcsbr_gpu_kernel_times(*[C.byref(x) for x in kt])
    L.mcsbr_gpu_kernel_timing(0)
    print(f"   path kernel {kt[0].value:.2f} ms in {kt[1].value} launches, accumulate {kt[2].value:.2f} ms")
    s2.close()
    t3 = time.perf_counter()
    print(f"rep {k}: scene_create {1e3*(t1-t0):.2f} ms  estimate_batch {1e3*(t2-t1):.2f} ms "
          f"(kernel {st.kernel_ms:.2f} ms, wall {st.wall_ms:.2f} ms)  destroy {1e3*(t3-t2):.2f} ms")
for k in range(3):
    t1 = time.perf_counter()
    vals, st = M.estimate_batch(scene, inc, rx, freqs, cfg)
    t2 = time.perf_counter()
    print(f"same scene: estimate_batch {1e3*(t2-t1):.2f} ms (kernel {st.kernel_ms:.2f})")
