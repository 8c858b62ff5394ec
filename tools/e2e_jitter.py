"""Per-call timing of the bench's e2e step, repeated, to find host-side jitter."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_07586_b200 as M  # noqa: E402

W = bench.WORKLOADS['c2']
sd, excs = W.scene_fn(), W.excs_fn()
scene = M.Scene(sd)
lam = bench.C0 / W.freqs[-1]
spws = [bench.spw_for(M, scene, e, lam, W.rays) for e in excs]
cfg = W.config(M)
inc = list(zip(excs, spws))
rx = [[e] for e in excs]
freqs = W.freqs
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
gc.collect()
gc.disable()
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s2 = M.Scene(sd)
    t1 = time.perf_counter()
    vals, st = M.estimate_batch(s2, inc, rx, freqs, cfg)
    t2 = time.perf_counter()
    s2.close()
    t3 = time.perf_counter()
    print(f"{k}: create {1e3*(t1-t0):7.2f}  batch {1e3*(t2-t1):7.2f} (kernel {st.kernel_ms:6.2f})  close {1e3*(t3-t2):6.2f}  total {1e3*(t3-t0):7.2f}", flush=True)
