"""Node visits / triangle tests per query (needs the MCSBR_TRAVERSAL_STATS
build: python tools/build_variants.py --stats 4).

    python tools/traversal_stats.py [c1|c2|c4|c5]
"""
import ctypes as C
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
os.environ.setdefault("MCSBR_GPU_LIB", os.path.join(ROOT, "paper_2511_07586_b200", "libmcsbr_gpu_stats.so"))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2511_07586_b200 as M  # noqa: E402
from paper_2511_07586_b200 import _abi as A  # noqa: E402
from paper_2511_07586_b200.geometry import airframe  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
if cfg_name == "c2":
    W = bench.WORKLOADS["c2"]
    sd, excs = W.scene_fn(), W.excs_fn()[::10]
    scene = M.Scene(sd)
    lam = bench.C0 / W.freqs[-1]
    incs = [(e, bench.spw_for(M, scene, e, lam, W.rays)) for e in excs]
    freqs, cfg = W.freqs, W.config(M)
elif cfg_name == "c1":
    sd = M.make_builtin_scene("sphere", {"subdivisions": 5})
    scene = M.Scene(sd)
    e = M.monostatic_excitation(90.0, 0.0)
    incs, excs = [(e, 0.0)], [e]
    freqs, cfg = [10e9], M.McConfig(strata_per_wavelength=30, samples_per_stratum=1, max_bounce=8, seed=1)
else:
    c4 = cfg_name == "c4"
    sd, _ = airframe(200_000, seed=4) if c4 else airframe(1_000_000, seed=5, dielectric_skin="--pec" not in sys.argv)
    scene = M.Scene(sd)
    freqs = np.linspace(9.5e9, 10.5e9, 64) if c4 else np.linspace(8e9, 12e9, 128)
    lam = 299792458.0 / freqs[-1]
    excs = [M.monostatic_excitation(90.0, a) for a in (-2.0, 0.0, 2.0)]
    rays = 2e6 if c4 else 16e6
    incs = []
    for e in excs:
        grid, _ = M.launch_plan(scene, e.k_inc, 0.0, 1.0, lam, 1)
        incs.append((e, lam * math.sqrt(rays / grid.rect.area())))
    cfg = (M.McConfig(strata_per_wavelength=10, samples_per_stratum=1, max_bounce=10, seed=4) if c4 else
           M.McConfig(strata_per_wavelength=10, samples_per_stratum=1, max_bounce=24, seed=5,
                      roulette=M.RouletteConfig(enabled=True, q=0.5, min_bounce=3)))
L = A.lib()
get = L.mcsbr_gpu_stats_visits
get.restype = None
get.argtypes = [C.POINTER(C.c_ulonglong)]
b0 = (C.c_ulonglong * 9)()
b1 = (C.c_ulonglong * 9)()
get(b0)
vals, st = M.estimate_batch(scene, incs, [[e] for e in excs], freqs, cfg)
get(b1)
d = [b1[i] - b0[i] for i in range(9)]
q = st.segments_traced + st.occlusion_queries
print(f"{cfg_name}: paths {st.rays_launched} segments {st.segments_traced} occlusion {st.occlusion_queries} "
      f"kernel {st.kernel_ms:.2f} ms bvh {scene.bvh_info()}")
for k, name in enumerate(("launch", "surface", "occlusion")):
    n = max(d[3 * k + 2], 1)
    print(f"  {name:9s} traced {d[3 * k + 2]:>11d}  node visits/query {d[3 * k] / n:6.2f}  "
          f"triangle tests/query {d[3 * k + 1] / n:6.2f}")
