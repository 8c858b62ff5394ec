"""The NUFFT accumulation (default) against the direct phasor kernel
(MCSBR_ACC=direct) on the same c4/c5 launch: max |a - b| / max |b| per
incidence, and both accumulation times.

    python tools/acc_compare.py c5 [--angles 16] [--lossless]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import ctypes as C  # noqa: E402

import bench_configs as B  # noqa: E402
import numpy as np  # noqa: E402

import paper_2511_07586_b200 as M  # noqa: E402
from paper_2511_07586_b200 import _abi as A  # noqa: E402
from paper_2511_07586_b200.geometry import airframe  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", choices=["c4", "c5"])
ap.add_argument("--angles", type=int, default=16)
ap.add_argument("--lossless", action="store_true")
a = ap.parse_args()
if a.config == "c4":
    sd, _ = airframe(200_000, seed=4)
    cfg = M.McConfig(strata_per_wavelength=10, samples_per_stratum=1, max_bounce=10, seed=4)
    freqs, n_az, half, rays = np.linspace(9.5e9, 10.5e9, 64), 64, 3.0, 2e6
else:
    sd, _ = airframe(1_000_000, seed=5, dielectric_skin=True)
    if a.lossless:
        sd.eps_imag = None
    cfg = M.McConfig(strata_per_wavelength=10, samples_per_stratum=1, max_bounce=24, seed=5,
                     roulette=M.RouletteConfig(enabled=True, q=0.5, min_bounce=3))
    freqs, n_az, half, rays = np.linspace(8e9, 12e9, 128), 128, 5.0, 16e6
s = M.Scene(sd)
lam = B.C0 / freqs[-1]
az = np.linspace(-half, half, n_az)
sel = az[np.linspace(0, n_az - 1, a.angles).round().astype(int)]
excs = [M.monostatic_excitation(90.0, float(x)) for x in sel]
spws = [B.spw_for(s, e, lam, rays) for e in excs]
L = A.lib()
out = {}
for mode in ("direct", "nufft", "direct", "nufft"):
    if mode == "direct":
        os.environ["MCSBR_ACC"] = "direct"
    else:
        os.environ.pop("MCSBR_ACC", None)
    L.mcsbr_gpu_kernel_timing(1)
    vals, st = M.estimate_batch(s, list(zip(excs, spws)), [[e] for e in excs], freqs, cfg)
    tm = [C.c_double(), C.c_uint64(), C.c_double(), C.c_uint64()]
    L.mcsbr_gpu_kernel_times(C.byref(tm[0]), C.byref(tm[1]), C.byref(tm[2]), C.byref(tm[3]))
    L.mcsbr_gpu_kernel_timing(0)
    out[mode] = (vals, tm[0].value, tm[2].value, st.kernel_ms)
d, n = out["direct"][0], out["nufft"][0]
err = [float(np.max(np.abs(n[i] - d[i])) / np.max(np.abs(d[i]))) for i in range(len(excs))]
print(json.dumps({"config": a.config, "lossless": a.lossless, "angles": len(excs),
                  "max_rel_err": max(err), "median_rel_err": float(np.median(err)),
                  "direct_ms": {"path": out["direct"][1], "acc": out["direct"][2], "total": out["direct"][3]},
                  "nufft_ms": {"path": out["nufft"][1], "acc": out["nufft"][2], "total": out["nufft"][3]}}))
