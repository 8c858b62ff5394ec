"""Traversal-only throughput on bench-like rays (diagnostic).

Centre-sampled first-segment launch rays of c2 sweep angles (same stratified
rectangle as the path kernel) through the standalone intersect kernel,
timed with CUDA events.  usage: python tools/trace_only.py [every_nth_angle]
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2511_07586_b200 as M  # noqa: E402
from paper_2511_07586_b200 import _abi as A  # noqa: E402

step = int(sys.argv[1]) if len(sys.argv) > 1 else 30
W = bench.WORKLOADS['c2']
sd, excs = W.scene_fn(), W.excs_fn()
scene = M.Scene(sd)
lam = bench.C0 / W.freqs[-1]
L = A.lib()
dev = torch.device("cuda", 0)
P, D = [], []
for e in excs[::step]:
    spw = bench.spw_for(M, scene, e, lam, W.rays)
    grid, n = M.launch_plan(scene, e.k_inc, 0.0, spw, lam, 1)
    r = grid.rect
    su = -1 + 2 * (np.arange(grid.nu) + 0.5) / grid.nu
    sv = -1 + 2 * (np.arange(grid.nv) + 0.5) / grid.nv
    p = (np.array(r.center) + (su[None, :, None] * r.half_u) * np.array(r.u_axis)
         + (sv[:, None, None] * r.half_v) * np.array(r.v_axis)).reshape(-1, 3)
    P.append(p)
    D.append(np.broadcast_to(np.array(e.k_inc), p.shape))
o = torch.from_numpy(np.ascontiguousarray(np.concatenate(P))).to(dev)
d = torch.from_numpy(np.ascontiguousarray(np.concatenate(D))).to(dev)
n = o.shape[0]
tmin = torch.zeros(n, dtype=torch.float64, device=dev)
t = torch.empty(n, dtype=torch.float64, device=dev)
ids = torch.empty(n, dtype=torch.int32, device=dev)
torch.cuda.synchronize()
for any_hit in (0, 1):
    for it in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = L.mcsbr_gpu_intersect_device(scene.handle, C.c_void_p(o.data_ptr()), C.c_void_p(d.data_ptr()),
                                          C.c_void_p(tmin.data_ptr()), n, any_hit, C.c_void_p(t.data_ptr()),
                                          C.c_void_p(ids.data_ptr()), None)
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0, L.mcsbr_gpu_last_error()
    ms = e0.elapsed_time(e1)
    hits = int((ids != -1).sum())
    print(f"any_hit={any_hit} rays {n} hits {hits} {ms:.3f} ms  {n / ms / 1e6:.2f} G rays/s", flush=True)
