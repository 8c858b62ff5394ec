"""BVH build time (event-timed, device) and scene creation wall time for the
bench scenes: python tools/build_time.py [c2|c4|c5 ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_07586_b200 as M  # noqa: E402
from paper_2511_07586_b200.geometry import airframe  # noqa: E402

for name in sys.argv[1:] or ["c2", "c4", "c5"]:
    if name == "c2":
        obj, mm = M.dihedral_grid(0.5, 64)
        sd = M.load_scene(obj, mm)
    else:
        sd, _ = airframe(200_000, seed=4) if name == "c4" else airframe(1_000_000, seed=5, dielectric_skin=True)
    for k in range(3):
        t0 = time.perf_counter()
        s = M.Scene(sd)
        info = s.bvh_info()
        t1 = time.perf_counter()
        s.close()
        print(f"{name}: create {1e3 * (t1 - t0):.1f} ms, bvh {info['build_ms']:.1f} ms, nodes {info['nodes']}, "
              f"depth {info['max_depth']}", flush=True)
