"""All five BASELINE.json configs on one B200 against the reference CPU solver.

    python tools/bench_configs.py [--configs c1,c3,c4,c5] [--cpu] [--out profiles/r02_configs.json]

For each config, on the GPU:

* device: CUDA-event time of the whole sweep (`estimate_batch`, every
  incidence and receiver of the config, after one warm-up);
* e2e: the public API from host buffers per repetition -- `Scene(...)`
  (upload + BVH build), `estimate_batch`, `close()` -- wall clock, median
  of 3 (the same definition as bench.py's `e2e`);
* clocks: nvidia-smi sampled during the GPU runs (bench.Clocks).

With --cpu, the reference (`oracle/_ref`, the reference compiled from its
sources, `estimate()` with workers = all host cores) on a sample of the same
sweep at the full ray count: c1 the whole config; c3 4 of the 361
receivers (the reference traces one receiver per call); c4 / c5 4 of the
azimuths spread over the sweep.  The reference has real permittivity only,
so for c3 / c5 the comparison runs the GPU on the lossless twin of the scene
too (same geometry and real parts), and the speed-up is stated against
that; the lossy GPU numbers are reported beside it.  `gpu_vs_ref` compares
the GPU and the reference on the sampled incidences (same RNG stream, parity
mode: summation order only, except c5's reference-BVH quirk).

Inputs are synthetic (generated meshes, counter-RNG launch jitter), with the
shapes / sizes / settings of BASELINE.json and SURVEY.md §8d.  c2 is
bench.py's secondary line and is measured there.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2511_07586_b200 as M  # noqa: E402
from paper_2511_07586_b200 import _abi as A  # noqa: E402
from paper_2511_07586_b200.geometry import airframe  # noqa: E402

C0 = 299792458.0


def spw_for(scene, exc, lam, rays):
    grid, _ = M.launch_plan(scene, exc.k_inc, 0.0, 1.0, lam, 1)
    return lam * math.sqrt(rays / grid.rect.area())


def gpu_sweep(sd, incs, rxs, freqs, cfg, reps=3):
    """device time of the sweep (kernel timing API, warm scene) and e2e
    (scene create + batch + close per repetition, median)"""
    L = A.lib()
    scene = M.Scene(sd)
    M.estimate_batch(scene, incs, rxs, freqs, cfg)  # warm-up
    L.mcsbr_gpu_kernel_timing(1)
    t0 = time.perf_counter()
    vals, st = M.estimate_batch(scene, incs, rxs, freqs, cfg)
    wall = time.perf_counter() - t0
    kt = [C.c_double(), C.c_uint64(), C.c_double(), C.c_uint64()]
    L.mcsbr_gpu_kernel_times(*[C.byref(x) for x in kt])
    L.mcsbr_gpu_kernel_timing(0)
    scene.close()
    e2e = []
    for _ in range(reps):
        t0 = time.perf_counter()
        s2 = M.Scene(sd)
        M.estimate_batch(s2, incs, rxs, freqs, cfg)
        s2.close()
        e2e.append(time.perf_counter() - t0)
    return vals, st, {"device_ms": st.kernel_ms, "path_kernel_ms": kt[0].value, "accumulate_ms": kt[2].value,
                      "batch_wall_ms": wall * 1e3, "e2e_ms": [round(1e3 * x, 2) for x in e2e],
                      "e2e_median_ms": 1e3 * statistics.median(e2e)}


def cpu_ref(sd, excs_spws, rx_list, freqs, cfg):
    """reference estimate() on all host cores, one call per (incidence,
    receiver) of the sample; returns (paths, seconds, values per call, cores)"""
    import oracle

    rs = oracle.ref_scene(sd)
    cores = os.cpu_count() or 1
    paths, secs, values = 0, 0.0, []
    for (exc, spw), rx in zip(excs_spws, rx_list):
        c = M.McConfig(**{**cfg.__dict__, "strata_per_wavelength": spw}).to_c()
        r = oracle.ref_estimate(rs, rx.to_c(), np.asarray(freqs, float), c, cores)
        values.append(r["values"])
        paths += r["stats"].rays_launched
        secs += r["stats"].wall_ms / 1e3
    return paths, secs, values, cores


def agreement(gpu, ref):
    gpu, ref = np.asarray(gpu), np.asarray(ref)
    rel = float(np.max(np.abs(gpu - ref)) / max(np.max(np.abs(ref)), 1e-300))
    db = []
    for ch in (M.VV, M.HH):
        a, b = np.abs(gpu[ch]), np.abs(ref[ch])
        ok = (a > 0) & (b > 0)
        if ok.any():
            db.append(20 * np.log10(a[ok] / b[ok]))
    rms = float(np.sqrt(np.mean(np.concatenate(db) ** 2))) if db else 0.0
    return {"max_rel_diff": rel, "rms_db_diff": rms}


def report(name, gpu, paths, cpu_part=None):
    out = {"config": name, "paths_per_sweep": int(paths), **gpu,
           "device_paths_per_s": paths / (gpu["device_ms"] / 1e3),
           "e2e_paths_per_s": paths / (gpu["e2e_median_ms"] / 1e3)}
    if cpu_part:
        out["cpu_ref"] = cpu_part
    return out


def c1(cpu):
    sd = M.make_builtin_scene("sphere", {"subdivisions": 5})
    exc = M.monostatic_excitation(90.0, 0.0)
    cfg = M.McConfig(strata_per_wavelength=30, samples_per_stratum=1, max_bounce=8, seed=1)
    vals, st, g = gpu_sweep(sd, [(exc, 0.0)], [[exc]], [10e9], cfg)
    sig = abs(vals[0, 0, M.HH, 0]) ** 2
    out = report("c1 PEC sphere L5 (20,480 tris), theta 90 phi 0, 10 GHz, HH, spw 30 spp 1, max 8", g,
                 st.rays_launched)
    out.update({"sigma_hh_m2": sig, "db_vs_pi_r2": 10 * math.log10(sig / math.pi)})
    if cpu:
        p, t, v, cores = cpu_ref(sd, [(exc, 30.0)], [exc], [10e9], cfg)
        out["cpu_ref"] = {"paths_per_s": p / t, "cores": cores, "sample": "the whole config",
                          "gpu_vs_ref": agreement(vals[0, 0], v[0])}
        out["speedup_e2e"] = out["e2e_paths_per_s"] / (p / t)
    return out


def c3(cpu):
    inc = M.monostatic_excitation(90.0, 0.0)
    rx = [M.bistatic_excitation(90.0, 0.0, float(th), 0.0) for th in np.linspace(0.0, 180.0, 361)]
    cfg = M.McConfig(strata_per_wavelength=275, samples_per_stratum=1, max_bounce=16, seed=3,
                     roulette=M.RouletteConfig(enabled=True, q=0.5, min_bounce=3))
    out = {}
    for lossy in (True, False):
        obj, mm = M.coated_sphere(subdivisions=5, lossless=not lossy)
        sd = M.load_scene(obj, mm)
        vals, st, g = gpu_sweep(sd, [(inc, 0.0)], [rx], [3e9], cfg)
        paths = st.rays_launched // math.ceil(361 / 32)  # the fan traces 32 receivers per launch
        key = "lossy" if lossy else "lossless_twin"
        r = report("c3 coated PEC sphere (61,440 tris, eps 4.0-0.1j / 2.2-0.01j" + ("" if lossy else ", real parts")
                   + "), 3 GHz, 361 bistatic receivers, spw 275 (8.04M paths), Fresnel, RR q0.5 >= 3, max 16",
                   g, paths * 361)
        r["unit_note"] = "paths = path-receiver pairs (8.04M paths x 361 receivers), as the reference counts them"
        out[key] = r
        if cpu and not lossy:
            pick = [0, 120, 240, 360]
            p, t, v, cores = cpu_ref(sd, [(inc, 275.0)] * len(pick), [rx[i] for i in pick], [3e9], cfg)
            agr = [agreement(vals[0, i], v[k]) for k, i in enumerate(pick)]
            r["cpu_ref"] = {"paths_per_s": p / t, "cores": cores,
                            "sample": f"receivers {pick} of 361 at the full 8.04M paths (one reference call each)",
                            "gpu_vs_ref": {"max_rel_diff": max(a["max_rel_diff"] for a in agr),
                                           "rms_db_diff": max(a["rms_db_diff"] for a in agr)}}
            r["speedup_e2e"] = r["e2e_paths_per_s"] / (p / t)
    return out


def isar(name, sd, n_az, az_half, freqs, rays, cfg, cpu, twin=None):
    scene = M.Scene(sd)
    lam = C0 / freqs[-1]
    excs = [M.monostatic_excitation(90.0, float(a)) for a in np.linspace(-az_half, az_half, n_az)]
    spws = [spw_for(scene, e, lam, rays) for e in excs]
    scene.close()
    incs, rxs = list(zip(excs, spws)), [[e] for e in excs]
    vals, st, g = gpu_sweep(sd, incs, rxs, freqs, cfg)
    out = {"config": report(name, g, st.rays_launched)}
    if twin is not None:
        tv, tst, tg = gpu_sweep(twin, incs, rxs, freqs, cfg)
        out["lossless_twin"] = report(name + " -- lossless twin (real parts)", tg, tst.rays_launched)
    if cpu:
        ref_sd = twin if twin is not None else sd
        cmp_vals = tv if twin is not None else vals
        pick = list(np.linspace(0, n_az - 1, 4).round().astype(int))
        p, t, v, cores = cpu_ref(ref_sd, [incs[i] for i in pick], [excs[i] for i in pick], freqs, cfg)
        agr = [agreement(cmp_vals[i, 0], v[k]) for k, i in enumerate(pick)]
        part = {"paths_per_s": p / t, "cores": cores,
                "sample": f"azimuths {pick} of {n_az} at the full ray count"
                          + ("; the lossless twin (the reference has real permittivity only)" if twin else ""),
                "gpu_vs_ref": {"max_rel_diff": max(a["max_rel_diff"] for a in agr),
                               "rms_db_diff": max(a["rms_db_diff"] for a in agr)}}
        tgt = out["lossless_twin"] if twin is not None else out["config"]
        tgt["cpu_ref"] = part
        tgt["speedup_e2e"] = tgt["e2e_paths_per_s"] / (p / t)
    return out


def c4(cpu):
    sd, _ = airframe(200_000, seed=4)
    cfg = M.McConfig(strata_per_wavelength=10, samples_per_stratum=1, max_bounce=10, seed=4)
    return isar("c4 PEC airframe (~200k tris, seed 4), ISAR 64 f (9.5-10.5 GHz) x 64 az (+-3 deg nose-on), "
                "2M paths/angle, max 10, VV", sd, 64, 3.0, np.linspace(9.5e9, 10.5e9, 64), 2e6, cfg, cpu)


def c5(cpu):
    W = bench.WORKLOADS["c5"]
    return isar("c5 airframe (~1M tris, seed 5), lossy 2-layer skins on wings/fin, ISAR 128 f (8-12 GHz) x "
                "128 az (+-5 deg), 16M paths/angle, RR, max 24", W.scene_fn(), 128, 5.0, W.freqs, W.rays,
                W.config(M), cpu, W.ref_scene_fn())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c3,c4,c5")
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_configs.json"))
    a = ap.parse_args()
    res = {}
    clk = bench.Clocks(0)
    for c in a.configs.split(","):
        t0 = time.time()
        res[c] = {"c1": c1, "c3": c3, "c4": c4, "c5": c5}[c](a.cpu)
        res[c]["wall_s"] = time.time() - t0
        print(c, json.dumps(res[c]), flush=True)
    res["clocks"] = clk.stop()
    res["cpu_model"] = bench.cpu_model()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
