import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench, paper_2511_07586_b200 as M
W = bench.WORKLOADS['c2']
sd, excs = W.scene_fn(), W.excs_fn()
for k in range(10):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s = M.Scene(sd); torch.cuda.synchronize(); t1 = time.perf_counter()
    info = s.bvh_info()
    s.close(); t2 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} ms (bvh {info['build_ms']:.2f} ms) destroy {1e3*(t2-t1):.2f}")
