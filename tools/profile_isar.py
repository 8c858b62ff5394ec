"""One warm-up + one timed launch of an ISAR config (c4 or c5) for ncu, with
the per-path counters that explain its cost.

    python tools/profile_isar.py c4|c5 [--angles N]
ncu: --set full -k regex:path_kernel -s 1 -c 1 (the second path_kernel launch).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import bench_configs as B  # noqa: E402
import numpy as np  # noqa: E402

import paper_2511_07586_b200 as M  # noqa: E402
from paper_2511_07586_b200.geometry import airframe  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", choices=["c4", "c5"])
ap.add_argument("--angles", type=int, default=8)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--lossless", action="store_true", help="c5 skins with real permittivity (the reference's model)")
ap.add_argument("--pec", action="store_true", help="c5 airframe without the dielectric skins")
ap.add_argument("--nf", type=int, default=0, help="override the number of frequencies")
ap.add_argument("--philox", action="store_true", help="statistical mode (Philox stream)")
ap.add_argument("--fast", action="store_true", help="statistical mode with fp32 triangle tests (parity_fp64_refine off)")
a = ap.parse_args()
if a.config == "c4":
    sd, _ = airframe(200_000, seed=4)
    cfg = M.McConfig(strata_per_wavelength=10, samples_per_stratum=1, max_bounce=10, seed=4)
    freqs, n_az, half, rays = np.linspace(9.5e9, 10.5e9, 64), 64, 3.0, 2e6
else:
    sd, _ = airframe(1_000_000, seed=5, dielectric_skin=not a.pec)
    if a.lossless:
        sd.eps_imag = None
    cfg = M.McConfig(strata_per_wavelength=10, samples_per_stratum=1, max_bounce=24, seed=5,
                     roulette=M.RouletteConfig(enabled=True, q=0.5, min_bounce=3))
    freqs, n_az, half, rays = np.linspace(8e9, 12e9, 128), 128, 5.0, 16e6
if a.nf:
    freqs = np.linspace(freqs[0], freqs[-1], a.nf) if a.nf > 1 else freqs[-1:]
if a.philox or a.fast:
    cfg.rng_mode = M.RngMode.PHILOX
    cfg.parity_fp64_refine = not a.fast
s = M.Scene(sd)
lam = B.C0 / freqs[-1]
az = np.linspace(-half, half, n_az)
sel = az[np.linspace(0, n_az - 1, a.angles).round().astype(int)]
excs = [M.monostatic_excitation(90.0, float(x)) for x in sel]
spws = [B.spw_for(s, e, lam, rays) for e in excs]
import ctypes as C  # noqa: E402

from paper_2511_07586_b200 import _abi as A  # noqa: E402

L = A.lib()
for _ in range(a.reps):
    L.mcsbr_gpu_kernel_timing(1)
    vals, st = M.estimate_batch(s, list(zip(excs, spws)), [[e] for e in excs], freqs, cfg)
tm = [C.c_double(), C.c_uint64(), C.c_double(), C.c_uint64()]
L.mcsbr_gpu_kernel_times(C.byref(tm[0]), C.byref(tm[1]), C.byref(tm[2]), C.byref(tm[3]))
L.mcsbr_gpu_kernel_timing(0)
N = st.rays_launched
print(json.dumps({"config": a.config, "angles": len(excs), "paths": N, "kernel_ms": st.kernel_ms,
                  "path_kernel_ms": tm[0].value, "path_launches": tm[1].value,
                  "accumulate_ms": tm[2].value, "accumulate_launches": tm[3].value,
                  "paths_per_s": N / st.kernel_ms * 1e3,
                  "segments_per_path": st.segments_traced / N,
                  "occlusion_per_path": st.occlusion_queries / N,
                  "contributions_per_path": st.contributions / N,
                  "rays_per_bounce": list(st.rays_per_bounce[:12])}))
