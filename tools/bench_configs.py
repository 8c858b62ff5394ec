"""All five BASELINE.json configs on one B200 + the reference CPU solver on bounded samples.

    python tools/bench_configs.py [--configs c1,c3,c4,c5] [--cpu] [--out profiles/r01_configs.json]

For each config: the GPU sweep (device time of the batch call, after one
warm-up), ray paths/s, the sweep wall time (extrapolated from a subset of
angles where the full sweep is impractically long: stated per entry), and
optionally the reference estimate() (oracle/_ref, all host cores) timed on a
bounded sample of the same workload with its own extrapolation.  c2 is the
headline of bench.py and is not repeated here.

Inputs are synthetic (generated meshes, counter-RNG launch jitter), with the
shapes / sizes / settings of BASELINE.json and SURVEY.md §8d.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_07586_b200 as M  # noqa: E402
from paper_2511_07586_b200.geometry import airframe  # noqa: E402

C0 = 299792458.0


def spw_for(scene, exc, lam, rays):
    grid, _ = M.launch_plan(scene, exc.k_inc, 0.0, 1.0, lam, 1)
    return lam * math.sqrt(rays / grid.rect.area())


def run_gpu(scene, incs, rxs, freqs, cfg, reps=2):
    vals, st = None, None
    for _ in range(reps):
        vals, st = M.estimate_batch(scene, incs, rxs, freqs, cfg)
    return vals, st


def cpu_ref(sd, excs_spws, freqs, cfg, max_s=20.0):
    """reference estimate() on all host cores over the given (excitation, spw)
    list (stops early after max_s seconds); returns (paths, seconds, n_done)."""
    import oracle

    rs = oracle.ref_scene(sd)
    cores = os.cpu_count() or 1
    paths, secs, n = 0, 0.0, 0
    cpu_ref.values = []
    for exc, spw in excs_spws:
        c = M.McConfig(**{**cfg.__dict__, "strata_per_wavelength": spw}).to_c()
        r = oracle.ref_estimate(rs, exc.to_c(), np.asarray(freqs, float), c, cores)
        cpu_ref.values.append(r["values"])
        paths += r["stats"].rays_launched
        secs += r["stats"].wall_ms / 1e3
        n += 1
        if secs > max_s:
            break
    return paths, secs, n, cores


def agreement(gpu, ref):
    """GPU vs reference complex sweep values [4][nf] of one incidence: the
    largest relative difference and the RMS dB difference of the co-pol
    channels over the frequencies (same RNG stream: summation order only)."""
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


def c1(cpu):
    sd = M.make_builtin_scene("sphere", {"subdivisions": 5})
    s = M.Scene(sd)
    exc = M.monostatic_excitation(90.0, 0.0)
    cfg = M.McConfig(strata_per_wavelength=30, samples_per_stratum=1, max_bounce=8, seed=1)
    vals, st = run_gpu(s, [(exc, 0.0)], [[exc]], [10e9], cfg)
    sig = abs(vals[0, 0, M.HH, 0]) ** 2
    out = {"config": "c1 PEC sphere L5 (20,480 tris), theta 90 phi 0, 10 GHz, HH, spw 30 spp 1, max 8",
           "paths": st.rays_launched, "gpu_ms": st.kernel_ms,
           "gpu_paths_per_s": st.rays_launched / (st.kernel_ms / 1e3),
           "sigma_hh_m2": sig, "db_vs_pi_r2": 10 * math.log10(sig / math.pi),
           "segments_per_path": st.segments_traced / st.rays_launched}
    if cpu:
        p, t, n, cores = cpu_ref(sd, [(exc, 30.0)], [10e9], cfg)
        out["cpu_ref"] = {"paths_per_s": p / t, "cores": cores, "sample": "full config",
                          "gpu_vs_ref": agreement(vals[0, 0], cpu_ref.values[0])}
        out["speedup_kernel"] = out["gpu_paths_per_s"] / (p / t)
    return out


def c3(cpu, lossy=True):
    obj, mm = M.coated_sphere(subdivisions=5, lossless=not lossy)
    sd = M.load_scene(obj, mm)
    s = M.Scene(sd)
    inc = M.monostatic_excitation(90.0, 0.0)
    rx = [M.bistatic_excitation(90.0, 0.0, float(th), 0.0) for th in np.linspace(0.0, 180.0, 361)]
    cfg = M.McConfig(strata_per_wavelength=275, samples_per_stratum=1, max_bounce=16, seed=3,
                     roulette=M.RouletteConfig(enabled=True, q=0.5, min_bounce=3))
    vals, st = run_gpu(s, [(inc, 0.0)], [rx], [3e9], cfg, reps=1)
    launches = math.ceil(361 / 32)
    paths = st.rays_launched // launches
    out = {"config": "c3 coated PEC sphere (61,440 tris, eps 4.0-0.1j / 2.2-0.01j"
                     + ("" if lossy else ", lossless") + "), 3 GHz, 361 bistatic receivers, "
                     "spw 275 (8.04M paths), Fresnel, RR q0.5 >= 3, max 16",
           "paths_per_incidence": paths, "receivers": 361, "gpu_ms": st.kernel_ms,
           "gpu_path_receivers_per_s": paths * 361 / (st.kernel_ms / 1e3),
           "occlusion_queries": st.occlusion_queries, "fan_launches": launches}
    if cpu:
        obj, mm = M.coated_sphere(subdivisions=5, lossless=True)
        sdl = M.load_scene(obj, mm)
        p, t, n, cores = cpu_ref(sdl, [(rx[180], 275.0)], [3e9], cfg)
        gl = M.estimate(M.Scene(sdl), rx[180], [3e9], M.McConfig(**{**cfg.__dict__, "strata_per_wavelength": 275.0}))
        out["cpu_ref"] = {"path_receivers_per_s": p / t, "cores": cores,
                          "sample": "1 of 361 receivers (the reference re-traces per receiver), "
                                    "lossless skins (the reference has real eps only)",
                          "sweep_s_extrapolated": t * 361,
                          "gpu_vs_ref": agreement(gl.sweep.values, cpu_ref.values[0])}
        out["speedup_sweep"] = out["cpu_ref"]["sweep_s_extrapolated"] / (st.kernel_ms / 1e3)
    return out


def isar(name, sd, n_az, az_half, freqs, rays, cfg, gpu_angles, cpu, cpu_sd=None):
    s = M.Scene(sd)
    lam = C0 / freqs[-1]
    az = np.linspace(-az_half, az_half, n_az)
    sel = az[np.linspace(0, n_az - 1, gpu_angles).round().astype(int)]
    excs = [M.monostatic_excitation(90.0, float(a)) for a in sel]
    spws = [spw_for(s, e, lam, rays) for e in excs]
    vals, st = run_gpu(s, list(zip(excs, spws)), [[e] for e in excs], freqs, cfg, reps=2)
    per_angle_ms = st.kernel_ms / len(excs)
    out = {"config": name, "triangles": int(sd.n_triangles), "frequencies": len(freqs),
           "azimuths": n_az, "paths_per_angle": st.rays_launched / len(excs),
           "gpu_angles_run": len(excs), "gpu_ms_per_angle": per_angle_ms,
           "gpu_paths_per_s": st.rays_launched / (st.kernel_ms / 1e3),
           "gpu_sweep_s": per_angle_ms * n_az / 1e3 if len(excs) < n_az else st.kernel_ms / 1e3,
           "sweep_extrapolated": len(excs) < n_az}
    if cpu:
        p, t, n, cores = cpu_ref(cpu_sd if cpu_sd is not None else sd, [(excs[0], spws[0])], freqs, cfg,
                                 max_s=60.0)
        out["cpu_ref"] = {"paths_per_s": p / t, "cores": cores, "sample": f"{n} azimuth at full rays",
                          "sweep_s_extrapolated": t / n * n_az}
        if cpu_sd is None:
            out["cpu_ref"]["gpu_vs_ref"] = agreement(vals[0, 0], cpu_ref.values[0])
        else:  # the reference has real permittivity only: compare the GPU's lossless twin
            g2, _ = M.estimate_batch(M.Scene(cpu_sd), [(excs[0], spws[0])], [[excs[0]]], freqs, cfg)
            out["cpu_ref"]["gpu_vs_ref"] = agreement(g2[0, 0], cpu_ref.values[0])
            out["cpu_ref"]["gpu_vs_ref"]["note"] = "GPU run of the same scene with the reference's real permittivity"
        out["speedup_sweep"] = out["cpu_ref"]["sweep_s_extrapolated"] / out["gpu_sweep_s"]
    return out


def c4(cpu):
    sd, info = airframe(200_000, seed=4)
    cfg = M.McConfig(strata_per_wavelength=10, samples_per_stratum=1, max_bounce=10, seed=4)
    return isar("c4 PEC airframe (~200k tris, seed 4), ISAR 64 f (9.5-10.5 GHz) x 64 az (+-3 deg "
                "nose-on), 2M paths/angle, max 10, VV", sd, 64, 3.0, np.linspace(9.5e9, 10.5e9, 64),
                2e6, cfg, 64, cpu)


def c5(cpu):
    sd, info = airframe(1_000_000, seed=5, dielectric_skin=True)
    cfg = M.McConfig(strata_per_wavelength=10, samples_per_stratum=1, max_bounce=24, seed=5,
                     roulette=M.RouletteConfig(enabled=True, q=0.5, min_bounce=3))
    cpu_sd = None
    if cpu:
        cpu_sd, _ = airframe(1_000_000, seed=5, dielectric_skin=True)
        cpu_sd.eps_imag = None
    return isar("c5 airframe (~1M tris, seed 5), lossy 2-layer skins on wings/fin, ISAR 128 f "
                "(8-12 GHz) x 128 az (+-5 deg), 16M paths/angle, RR, max 24", sd, 128, 5.0,
                np.linspace(8e9, 12e9, 128), 16e6, cfg, 128, cpu, cpu_sd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c3,c4,c5")
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_configs.json"))
    a = ap.parse_args()
    res = {}
    for c in a.configs.split(","):
        t0 = time.time()
        res[c] = {"c1": c1, "c3": c3, "c4": c4, "c5": c5}[c](a.cpu)
        res[c]["wall_s"] = time.time() - t0
        print(c, json.dumps(res[c]), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
