"""Benchmark of the MC-SBR hot path (BASELINE.json metric: ray-paths/sec).

Workload (BASELINE.json configs[1], SURVEY.md §8d "c2"): PEC dihedral corner
reflector, two 0.5 m x 0.5 m plates at 90 deg, each a 64 x 64 quad grid
(16,384 triangles, generated here: the paper's meshes are not available),
monostatic azimuth sweep phi in [-45, 45] deg about the bisector in 181
steps, theta = 90 deg, 10 GHz, VV, ~1M ray paths per angle (strata per
wavelength chosen per angle so nu*nv ~ 1e6, seed 2), max 4 bounces,
occlusion on.  One step = the whole 181-angle sweep (~1.8e8 ray paths) in
ONE device launch.  Inputs are synthetic (generated geometry, counter-RNG
launch jitter); no dataset is involved.

Arms:
  default            the CUDA path.  value = ray paths of the whole job /
                     device time of the step (CUDA events on the launch
                     stream, max over ranks); e2e = the same sweep through the
                     public C ABI from HOST buffers (scene upload + GPU BVH
                     build + estimate_batch + result download) per step.
  --impl reference   the reference's own CPU implementation (oracle/_ref,
                     compiled from /root/reference sources) on all host
                     cores, on a bounded sample of the same sweep's angles.

Multi-GPU (torchrun): every rank traces a disjoint entry range of every
angle (strong scaling of one sweep) and the complex accumulators are summed
with one NCCL all-reduce.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C0 = 299792458.0
FREQ = 10e9
N_ANGLES = 181
RAYS_PER_ANGLE = 1_000_000
MAX_BOUNCE = 4
SEED = 2


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_digest(path):
    """Pipe / bandwidth utilisation of the path kernel from the committed ncu
    capture of this same workload (profiles/, tools/ncu_summary.py)."""
    with open(path) as f:
        d = json.load(f)

    def val(k):
        x = d.get(k)
        return None if x is None else float(str(x["value"]).replace(",", ""))

    def gbs(k):
        x = d.get(k)
        if x is None:
            return None
        scale = {"byte/s": 1e-9, "Kbyte/s": 1e-6, "Mbyte/s": 1e-3, "Gbyte/s": 1.0, "Tbyte/s": 1e3}
        return val(k) * scale.get(x["unit"], float("nan"))

    return {"source": "profiles/" + os.path.basename(path),
            "l2_GBps": gbs("l2_bandwidth"), "l2_throughput_pct": val("l2_throughput_pct"),
            "l2_hit_pct": val("l2_hit_pct"), "l1_hit_pct": val("l1_hit_pct"),
            "dram_GBps": gbs("dram_bandwidth"), "issue_active_pct": val("smsp_issue_active_pct"),
            "fp64_pipe_pct": val("fp64_pipe_pct"), "fp32_fma_pipe_pct": val("fma_pipe_pct"),
            "sfu_xu_inst_pct": val("sfu_xu_inst_pct"), "simt_threads_per_warp": val("simt_efficiency_threads"),
            "limiter": "instruction issue / latency (fp64 shading + dependent node fetches); "
                       "the BVH is L1/L2-resident, so neither HBM nor L2 bandwidth binds"}


def workload(M):
    obj, mm = M.dihedral_grid(0.5, 64)
    sd = M.load_scene(obj, mm)
    phis = 45.0 + np.linspace(-45.0, 45.0, N_ANGLES)
    excs = [M.monostatic_excitation(90.0, float(p)) for p in phis]
    return sd, excs


def spw_for(M, scene, exc, lam):
    """strata per wavelength giving nu*nv ~ RAYS_PER_ANGLE for this incidence."""
    grid, _ = M.launch_plan(scene, exc.k_inc, 0.0, 1.0, lam, 1)
    area = grid.rect.area()
    return lam * math.sqrt(RAYS_PER_ANGLE / area)


def config(M):
    return M.McConfig(strata_per_wavelength=50.0, samples_per_stratum=1, max_bounce=MAX_BOUNCE,
                      seed=SEED, branch_strategy=M.BranchStrategy.FRESNEL)


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, index: int):
        self.p = None
        self.path = f"/tmp/mcsbr_clocks_{os.getpid()}.csv"
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,utilization.gpu,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        rows = []
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 7:
                    rows.append(f)
        except Exception:
            return None
        if not rows:
            return None
        load = [r for r in rows if r[2] not in ("0", "[N/A]")] or rows
        sm = [float(r[0]) for r in load if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(load)}


def run_reference(args, rank, world):
    """Reference arm: the unmodified reference estimate() on the host cores."""
    if rank != 0:
        return None
    import oracle
    import paper_2511_07586_b200.geometry as G
    from paper_2511_07586_b200 import _abi as A
    import paper_2511_07586_b200.solver as S

    obj, mm = G.dihedral_grid(0.5, 64)
    sd = G.load_scene(obj, mm)
    cores = os.cpu_count() or 1
    L = oracle.ref()
    rs = oracle.ref_scene(sd)
    lam = C0 / FREQ
    phis = 45.0 + np.linspace(-45.0, 45.0, N_ANGLES)
    # bounded sample: SAMPLE angles per step, spread over the sweep
    sample_idx = np.linspace(0, N_ANGLES - 1, args.ref_angles).round().astype(int)
    def plan_spw(exc_c):
        out = np.zeros(11)
        L.ref_launch_rect(rs.h, oracle.dp(np.array(exc_c.k_inc[:])), 0.0, oracle.dp(out))
        area = 4.0 * out[9] * out[10]
        return lam * math.sqrt(RAYS_PER_ANGLE / area)

    def one_step():
        paths = 0
        t = 0.0
        for i in sample_idx:
            exc = A.Excitation()
            L.ref_monostatic_excitation(90.0, float(phis[i]), C.byref(exc))
            c = S.McConfig(strata_per_wavelength=plan_spw(exc), samples_per_stratum=1,
                           max_bounce=MAX_BOUNCE, seed=SEED).to_c()
            r = oracle.ref_estimate(rs, exc, np.array([FREQ]), c, cores)
            paths += r["stats"].rays_launched
            t += r["stats"].wall_ms / 1e3
        return paths, t

    for _ in range(args.warmup):
        one_step()
    tot_p, tot_t = 0, 0.0
    for _ in range(args.steps):
        p, t = one_step()
        tot_p += p
        tot_t += t
    v = tot_p / tot_t
    line = {
        "impl": "reference", "metric": "ray-paths/sec", "value": v, "unit": "ray-paths/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c2: PEC dihedral 2x(2x64x64) tris, 181-angle monostatic azimuth "
                               "sweep, 10 GHz VV, ~1M ray paths/angle, max 4 bounces",
                   "sample": f"{len(sample_idx)} of {N_ANGLES} angles per step"},
        "cpu_baseline": {"value": v, "unit": "ray-paths/s", "cores": cores, "kind": "reference",
                         "sample": f"{len(sample_idx)} of {N_ANGLES} sweep angles per step at the "
                                   "full ~1M ray paths per angle, reference estimate() with "
                                   f"workers={cores}"},
        "e2e": {"value": v, "unit": "ray-paths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "sweep_wall_ms_extrapolated": 1e3 * tot_t / args.steps * N_ANGLES / len(sample_idx),
    }
    return line


def cpu_baseline_quick(sd, excs, spws, gpu_values):
    """Rank-0 reference timing on a bounded sample (2 angles, all host cores);
    also returns the GPU-vs-reference RCS error on those angles."""
    import oracle
    import paper_2511_07586_b200.solver as S

    cores = os.cpu_count() or 1
    rs = oracle.ref_scene(sd)
    idx = [0, N_ANGLES // 2]
    paths, t = 0, 0.0
    errs = []
    for i in idx:
        c = S.McConfig(strata_per_wavelength=spws[i], samples_per_stratum=1, max_bounce=MAX_BOUNCE,
                       seed=SEED).to_c()
        r = oracle.ref_estimate(rs, excs[i].to_c(), np.array([FREQ]), c, cores)
        paths += r["stats"].rays_launched
        t += r["stats"].wall_ms / 1e3
        ref_vv = r["values"][0, 0]
        gpu_vv = gpu_values[i, 0, 0, 0]
        errs.append(20 * math.log10(abs(gpu_vv) / abs(ref_vv)))
    return {"value": paths / t, "unit": "ray-paths/s", "cores": cores, "kind": "reference",
            "sample": f"2 of {N_ANGLES} sweep angles (phi 0 and 45 deg) at the full ~1M paths each, "
                      f"reference estimate() with workers={cores}"}, errs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-angles", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    import torch

    import paper_2511_07586_b200 as M
    from paper_2511_07586_b200 import _abi as A

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = A.lib()

    sd, excs = workload(M)
    scene = M.Scene(sd, device=local)
    lam = C0 / FREQ
    spws = [spw_for(M, scene, e, lam) for e in excs]
    cfg = config(M)
    ccfg = cfg.to_c()
    n_inc = len(excs)
    incs = (A.Incidence * n_inc)(*[e.incidence(s) for e, s in zip(excs, spws)])
    rxs = (A.Receiver * n_inc)(*[e.receiver() for e in excs])
    freqs = np.array([FREQ])
    nf = 1
    dev = torch.device("cuda", local)
    sums = torch.zeros(n_inc * nf * 8, dtype=torch.float64, device=dev)
    counters = torch.zeros(A.MCSBR_COUNTER_WORDS, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    def step():
        sums.zero_()
        counters.zero_()
        rc = L.mcsbr_gpu_trace_device(scene.handle, incs, n_inc, rxs, 1, 1,
                                      freqs.ctypes.data_as(C.POINTER(C.c_double)), nf,
                                      C.byref(ccfg), rank, world, C.c_void_p(sums.data_ptr()),
                                      C.c_void_p(counters.data_ptr()),
                                      C.c_void_p(stream.cuda_stream))
        if rc != 0:
            raise RuntimeError(L.mcsbr_gpu_last_error().decode())
        if dist is not None:
            dist.all_reduce(sums)
            dist.all_reduce(counters)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---- timed region: K steps, L2 flushed between steps (untimed) ----
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk = Clocks(local)
    launches0 = L.mcsbr_gpu_last_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for k in range(args.steps):
        flush.fill_(float(k))
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    clocks = clk.stop()
    launches = L.mcsbr_gpu_last_launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = sum(step_ms) / len(step_ms)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    cnt = counters.cpu().numpy().astype(np.uint64)
    st = A.Stats()
    rc = L.mcsbr_gpu_decode_counters(cnt.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(st))
    if rc != 0:
        raise RuntimeError(L.mcsbr_gpu_last_error().decode())
    paths = int(st.rays_launched)
    value = paths / (ms / 1e3)

    # ---- kernel-only timing for the roofline (same stream, single launch) ----
    kev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    sums.zero_()
    counters.zero_()
    kev[0].record(stream)
    L.mcsbr_gpu_trace_device(scene.handle, incs, n_inc, rxs, 1, 1,
                             freqs.ctypes.data_as(C.POINTER(C.c_double)), nf, C.byref(ccfg), rank,
                             world, C.c_void_p(sums.data_ptr()), C.c_void_p(counters.data_ptr()),
                             C.c_void_p(stream.cuda_stream))
    kev[1].record(stream)
    torch.cuda.synchronize(dev)
    kernel_ms = kev[0].elapsed_time(kev[1])
    kcnt = counters.cpu().numpy().astype(np.uint64)
    kst = A.Stats()
    L.mcsbr_gpu_decode_counters(kcnt.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(kst))
    T = sd.n_triangles
    bq = 64 * math.ceil(math.log2(T / 4)) + 4 * 48  # SURVEY.md §8d traversal bytes per query
    queries = int(kst.segments_traced) + int(kst.occlusion_queries)
    # accumulation roofline: C * R * (160 + 32 F) FP32-equivalent
    # flops + C * R * F sincos per path against the FP32 / SFU peaks at the
    # measured max clock (the kernel computes them in fp64: a lower bound on
    # the work, so the fraction is an upper bound on the share)
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            f_clk = float(json.load(f).get("sm_max_mhz", 1965.0)) * 1e6
    except Exception:
        f_clk = 1965.0e6
    contribs = int(kst.contributions)
    acc_flops = contribs * (160 + 32 * nf)
    acc_sincos = contribs * nf
    acc = {"model": "SURVEY.md 8d: C*R*(160+32F) FP32 flops + C*R*F sincos per path (F = 1, R = 1)",
           "contributions_per_path": contribs / max(int(kst.rays_launched), 1),
           "fp32_tflops": acc_flops / (kernel_ms / 1e3) / 1e12,
           "fp32_peak_tflops": sm_count * 128 * 2 * f_clk / 1e12,
           "sincos_per_s": acc_sincos / (kernel_ms / 1e3),
           "sfu_peak_per_s": sm_count * 16 * f_clk}
    acc["fp32_frac"] = acc["fp32_tflops"] / acc["fp32_peak_tflops"]
    acc["sfu_frac"] = acc["sincos_per_s"] / acc["sfu_peak_per_s"]
    alg_bytes = queries * bq
    achieved = alg_bytes / (kernel_ms / 1e3) / 1e9
    peak, peak_kind = peaks()
    traffic = None
    ncu = None
    prof = os.path.join(ROOT, "profiles", "path_kernel_dram.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pk = json.load(f)
            traffic = pk.get("dram_bytes_per_launch")
            ncu = ncu_digest(os.path.join(ROOT, pk["source"]))
        except Exception:
            pass

    # ---- e2e: public C ABI from host buffers (scene upload + BVH + sweep + readback) ----
    # N = 1: solver.estimate_batch (the drop-in batch call); N > 1: every rank
    # runs distributed.sweep_sharded (its shard + NCCL all-reduce + finalize);
    # per step the time is the max over ranks.
    from paper_2511_07586_b200 import distributed as D

    e2e_t = []
    inc_list = [(e, s) for e, s in zip(excs, spws)]
    rx_list = [[e] for e in excs]
    import gc

    gc.collect()
    gc.disable()  # a collector pause is not part of the workload
    for k in range(max(args.steps, 1) + 2):
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        s2 = M.Scene(sd, device=local)
        if world > 1:
            vals, st2 = D.sweep_sharded(s2, inc_list, rx_list, freqs, cfg)
        else:
            vals, st2 = M.estimate_batch(s2, inc_list, rx_list, freqs, cfg)
        s2.close()
        dt = time.perf_counter() - t0
        if dist is not None:
            tt = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        if k > 1:  # two untimed warm-up steps
            e2e_t.append(dt)
    gc.enable()
    # median over the timed steps (host-side jitter of one step would
    # otherwise dominate the mean); every step's time is reported beside it
    e2e_value = st2.rays_launched / statistics.median(e2e_t)
    h2d = (sd.vertices.nbytes + sd.triangles.nbytes + sd.materials.nbytes
           + C.sizeof(incs) + C.sizeof(rxs) + freqs.nbytes)
    d2h = vals.nbytes + A.MCSBR_COUNTER_WORDS * 8

    cpu = None
    rcs_err = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle  # noqa: F401

            cpu, errs = cpu_baseline_quick(sd, excs, spws, vals)
            rcs_err = max(abs(e) for e in errs)
        except Exception as e:  # reference library missing on this box
            cpu = {"value": None, "unit": "ray-paths/s", "cores": os.cpu_count(),
                   "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": "ray-paths/sec", "value": value, "unit": "ray-paths/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "c2: PEC dihedral 2x(2x64x64)=16384 tris, 181-angle monostatic "
                                   "azimuth sweep (phi 0..90 deg abs), theta 90, 10 GHz VV, ~1M ray "
                                   "paths/angle, max 4 bounces, occlusion on, seed 2, parity RNG",
                       "paths_per_step": paths, "angles": N_ANGLES,
                       "l2": "flushed between steps (256 MB write, untimed)",
                       "parallelism": f"ray-shard x{world}"},
            "sweep_wall_ms": ms,
            "rcs_err_db_vs_cpu_ref": rcs_err,
            "e2e": {"value": e2e_value, "unit": "ray-paths/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": [round(1e3 * x, 3) for x in e2e_t],
                    "path": "Scene(...) upload + GPU BVH build, estimate_batch (plan, launch, "
                            "finalize, download), Scene.close() -- the public API a user calls; "
                            "value from the median step"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "path_kernel", "kernel_ms": kernel_ms,
                         "algorithmic_bytes": alg_bytes, "bytes_per_query": bq,
                         "queries_per_path": queries / max(int(kst.rays_launched), 1),
                         "peak_kind": peak_kind,
                         "note": "SURVEY.md 8d model: 960 B per query as if every node/triangle byte came "
                                 "from DRAM; the working set is cache-resident (see ncu), so frac > 1 "
                                 "means the kernel moves the model's bytes faster than HBM could"},
            "ncu": ncu,
            "accumulation_roofline": acc,
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
