"""Node visits / triangle tests per query on the c2 sweep (needs the
MCSBR_TRAVERSAL_STATS build: python tools/build_variants.py --stats 4)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("MCSBR_GPU_LIB", os.path.join(ROOT, "paper_2511_07586_b200", "libmcsbr_gpu_stats.so"))
import bench  # noqa: E402
import paper_2511_07586_b200 as M  # noqa: E402
from paper_2511_07586_b200 import _abi as A  # noqa: E402

sd, excs = bench.workload(M)
excs = excs[::10]
scene = M.Scene(sd)
lam = bench.C0 / bench.FREQ
spws = [bench.spw_for(M, scene, e, lam) for e in excs]
L = A.lib()
get = L.mcsbr_gpu_stats_visits
get.restype = None
get.argtypes = [C.POINTER(C.c_ulonglong)]
buf = (C.c_ulonglong * 2)()
get(buf)
v0, t0 = buf[0], buf[1]
vals, st = M.estimate_batch(scene, list(zip(excs, spws)), [[e] for e in excs], [bench.FREQ], bench.config(M))
get(buf)
q = st.segments_traced + st.occlusion_queries
print(f"queries {q}  node visits/query {(buf[0] - v0) / q:.2f}  triangle tests/query {(buf[1] - t0) / q:.2f}"
      f"  bvh {scene.bvh_info()}")
