import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, '/root/repo')
import bench, paper_2511_07586_b200 as M
ai = int(sys.argv[1]); lim = int(sys.argv[2]) if len(sys.argv) > 2 else 0
sd, excs = bench.workload(M)
scene = M.Scene(sd)
lam = bench.C0 / bench.FREQ
e = excs[ai]
spw = bench.spw_for(M, scene, e, lam)
grid, n = M.launch_plan(scene, e.k_inc, 0.0, spw, lam, 1)
r = grid.rect
su = -1 + 2 * (np.arange(grid.nu) + 0.5) / grid.nu; sv = -1 + 2 * (np.arange(grid.nv) + 0.5) / grid.nv
p = (np.array(r.center) + (su[None, :, None] * r.half_u) * np.array(r.u_axis) + (sv[:, None, None] * r.half_v) * np.array(r.v_axis)).reshape(-1, 3)
if lim: p = p[:lim]
d = np.broadcast_to(np.array(e.k_inc), p.shape).copy()
try:
    t, ids = scene.intersect_batch(p, d, 0.0)
    print("angle", ai, "k", e.k_inc, "rays", len(p), "hits", (ids != 0xFFFFFFFF).sum(), flush=True)
except Exception as ex:
    print("angle", ai, "k", e.k_inc, "FAILED", ex, flush=True)
    np.save(f"/root/repo/gpurun_out/bad_rays_{ai}.npy", np.concatenate([p, d], 1)[:: max(1, len(p)//200000)])
