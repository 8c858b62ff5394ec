"""Multi-frequency bistatic fan vs one trace per receiver (MCSBR_FAN=0):
c3's coated sphere (lossy shells, level 5), one incidence, R receivers in
theta, F uniform frequencies around 3 GHz, ~8 M paths.

    python tools/fan_time.py [--rx 32] [--nf 16]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402

import ctypes as C  # noqa: E402

import bench_configs as B  # noqa: E402
import paper_2511_07586_b200 as M  # noqa: E402
from paper_2511_07586_b200 import _abi as A  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rx", type=int, default=32)
ap.add_argument("--nf", type=int, default=16)
a = ap.parse_args()
obj, mm = M.coated_sphere(subdivisions=5)
s = M.Scene(M.load_scene(obj, mm))
freqs = np.linspace(2.9e9, 3.1e9, a.nf)
cfg = M.McConfig(strata_per_wavelength=10, samples_per_stratum=1, seed=3, max_bounce=16,
                 roulette=M.RouletteConfig(enabled=True, min_bounce=3))
inc = M.monostatic_excitation(90.0, 0.0)
spw = B.spw_for(s, inc, B.C0 / freqs[-1], 8e6)
rxs = [M.bistatic_excitation(90.0, 0.0, float(th), 0.0) for th in np.linspace(0.0, 180.0, a.rx)]
out = {}
for tag, fan in (("fan", "1"), ("per_receiver", "0")):
    os.environ["MCSBR_FAN"] = fan
    ms = []
    L = A.lib()
    for _ in range(3):
        L.mcsbr_gpu_kernel_timing(1)
        vals, st = M.estimate_batch(s, [(inc, spw)], [rxs], freqs, cfg)
        ms.append(st.kernel_ms)
    tm = [C.c_double(), C.c_uint64(), C.c_double(), C.c_uint64()]
    L.mcsbr_gpu_kernel_times(C.byref(tm[0]), C.byref(tm[1]), C.byref(tm[2]), C.byref(tm[3]))
    L.mcsbr_gpu_kernel_timing(0)
    out[tag] = {"kernel_ms": min(ms), "path_kernel_ms": tm[0].value, "path_launches": tm[1].value,
                "accumulate_ms": tm[2].value, "accumulate_launches": tm[3].value,
                "paths": st.rays_launched, "contributions": st.contributions}
    out[tag + "_vals"] = vals
d = np.max(np.abs(out["fan_vals"] - out["per_receiver_vals"])) / np.max(np.abs(out["per_receiver_vals"]))
print(json.dumps({"rx": a.rx, "nf": a.nf, "fan": out["fan"], "per_receiver": out["per_receiver"],
                  "speedup": out["per_receiver"]["kernel_ms"] / out["fan"]["kernel_ms"], "max_rel_diff": float(d)}))
