"""MCSBR_REDUCE_EXACT (csrc/fixedpoint.cuh): byte-reproducible far-field sums.

The reference promises artifacts that are byte-identical across reruns and
worker counts (proj/include/mcsbr/runner.hpp:2-5, tests/test_cli_config.cpp:
95-123) through its fixed-order block merge (src/solver_mc.cpp:212-216).
The GPU schedules paths dynamically; the exact mode instead rounds every
term once to 192-bit fixed point and sums integers, so the bits do not
depend on scheduling, launch grouping or the number of shards / GPUs:

* three reruns give the same bytes (F = 1 and F > 1, PEC and lossy);
* shard counts 1 / 2 / 4 (mcsbr_gpu_trace_device per rank on this GPU, limbs
  summed as the integer all-reduce would) give the same bytes;
* many small launch groups and a forced record-buffer overflow give the
  same bytes;
* the exact sums agree with the fp64-atomic sums and the oracle to
  summation-order rounding.
"""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2511_07586_b200 as M
from paper_2511_07586_b200 import _abi as A
from paper_2511_07586_b200 import distributed as D
from paper_2511_07586_b200.geometry import airframe
from tests.helpers import oracle_estimate

pytestmark = pytest.mark.gpu

EXACT, FAST = M.Reduction.EXACT, M.Reduction.FAST


def _cases():
    obj, mm = M.dihedral_grid(0.5, 16)
    dih = M.load_scene(obj, mm)
    e = [M.monostatic_excitation(90.0, p) for p in (5.0, 30.0, 45.0, 85.0)]
    yield ("dihedral_f1", dih, [(x, 8.0) for x in e], [[x] for x in e], [10e9],
           dict(samples_per_stratum=2, max_bounce=4, seed=2))
    skin, _ = airframe(6_000, seed=5, dielectric_skin=True)
    e = [M.monostatic_excitation(80.0, a) for a in (-3.0, 4.0)]
    yield ("airframe_lossy_f16", skin, [(x, 0.7) for x in e], [[x] for x in e], np.linspace(8e9, 12e9, 16),
           dict(samples_per_stratum=2, max_bounce=24, seed=5, roulette=M.RouletteConfig(enabled=True, min_bounce=3)))
    obj, mm = M.coated_sphere(subdivisions=2, lossless=True)
    coat = M.load_scene(obj, mm)
    inc = M.monostatic_excitation(90.0, 0.0)
    yield ("coated_sphere_bistatic_fan", coat, [(inc, 10.0)],
           [[M.bistatic_excitation(90.0, 0.0, th, 0.0) for th in (0.0, 60.0, 120.0)]], [3e9],
           dict(samples_per_stratum=1, max_bounce=16, seed=3, roulette=M.RouletteConfig(enabled=True, min_bounce=3)))


CASES = list(_cases())


def _run(s, incs, rxs, freqs, kw, red, env=None):
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        return M.estimate_batch(s, incs, rxs, freqs, M.McConfig(reduction=red, **kw))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_exact_sums_are_byte_identical_across_reruns_and_groupings(case):
    name, sd, incs, rxs, freqs, kw = case
    s = M.Scene(sd)
    runs = [_run(s, incs, rxs, freqs, kw, EXACT)[0] for _ in range(3)]
    runs.append(_run(s, incs, rxs, freqs, kw, EXACT, {"MCSBR_GROUP_ENTRIES": "3000"})[0])
    runs.append(_run(s, incs, rxs, freqs, kw, EXACT, {"MCSBR_REC_CAP": "500"})[0])  # direct-add overflow path
    runs.append(_run(s, incs, rxs, freqs, kw, EXACT, {"MCSBR_CHUNK_MAX": "64", "MCSBR_BAND": "0"})[0])
    for r in runs[1:]:
        assert r.tobytes() == runs[0].tobytes()
    fast, _ = _run(s, incs, rxs, freqs, kw, FAST)
    scale = np.max(np.abs(fast))
    assert np.max(np.abs(fast - runs[0])) <= 1e-12 * scale


@pytest.mark.parametrize("world", [2, 4])
def test_exact_shards_are_byte_identical_to_one_launch(world):
    """The multi-GPU partition (mcsbr_gpu_trace_device rank / world) on this
    GPU, every rank's int64 limbs added as the integer all-reduce adds them:
    the same bytes as the single launch, for 1, 2 and 4 shards."""
    import torch

    _, sd, incs, rxs, freqs, kw = CASES[1]
    s = M.Scene(sd)
    cfg = M.McConfig(reduction=EXACT, **kw)
    full, st_full = M.estimate_batch(s, incs, rxs, freqs, cfg)
    n = len(incs)
    inc = (A.Incidence * n)(*[e.incidence(spw) for e, spw in incs])
    rx = (A.Receiver * n)(*[r[0].receiver() for r in rxs])
    c = cfg.to_c()
    dev = torch.device("cuda", 0)
    nf = len(freqs)
    fr = np.ascontiguousarray(freqs, dtype=np.float64)
    limbs = torch.zeros(n * nf * 8 * A.MCSBR_EXACT_LIMBS, dtype=torch.int64, device=dev)
    counters = torch.zeros(A.MCSBR_COUNTER_WORDS, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    for rank in range(world):
        A.check(A.lib().mcsbr_gpu_trace_device(
            s.handle, inc, n, rx, 1, 1, fr.ctypes.data_as(C.POINTER(C.c_double)), nf, C.byref(c), rank, world,
            C.c_void_p(limbs.data_ptr()), C.c_void_p(counters.data_ptr()), C.c_void_p(stream.cuda_stream)))
    vals, st = D.allreduce_finalize(limbs, counters, freqs, n)
    assert st.rays_launched == st_full.rays_launched and st.contributions == st_full.contributions
    assert vals.reshape(n, 1, 4, nf).tobytes() == full.tobytes()


def test_exact_shards_with_empty_ranks():
    """Incidences smaller than one stripe (1024 dispatch indices): only rank 0
    has launch units, the other ranks launch nothing for them; the limbs of
    all ranks still add up to the single launch's bytes."""
    import torch

    obj, mm = M.dihedral_grid(0.5, 16)
    sd = M.load_scene(obj, mm)
    s = M.Scene(sd)
    excs = [M.monostatic_excitation(90.0, p) for p in (10.0, 45.0)]
    incs, rxs = [(e, 1.5) for e in excs], [[e] for e in excs]  # a few hundred entries each
    freqs = np.linspace(9e9, 11e9, 3)
    cfg = M.McConfig(reduction=EXACT, samples_per_stratum=1, max_bounce=4, seed=4)
    full, st_full = M.estimate_batch(s, incs, rxs, freqs, cfg)
    assert 0 < st_full.rays_launched < 2 * 1024
    n, nf = len(incs), len(freqs)
    inc = (A.Incidence * n)(*[e.incidence(spw) for e, spw in incs])
    rx = (A.Receiver * n)(*[r[0].receiver() for r in rxs])
    c = cfg.to_c()
    dev = torch.device("cuda", 0)
    fr = np.ascontiguousarray(freqs, dtype=np.float64)
    limbs = torch.zeros(n * nf * 8 * A.MCSBR_EXACT_LIMBS, dtype=torch.int64, device=dev)
    counters = torch.zeros(A.MCSBR_COUNTER_WORDS, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    for rank in range(4):
        A.check(A.lib().mcsbr_gpu_trace_device(
            s.handle, inc, n, rx, 1, 1, fr.ctypes.data_as(C.POINTER(C.c_double)), nf, C.byref(c), rank, 4,
            C.c_void_p(limbs.data_ptr()), C.c_void_p(counters.data_ptr()), C.c_void_p(stream.cuda_stream)))
    vals, st = D.allreduce_finalize(limbs, counters, freqs, n)
    assert st.rays_launched == st_full.rays_launched and st.contributions == st_full.contributions
    assert vals.reshape(n, 1, 4, nf).tobytes() == full.tobytes()


def test_exact_matches_oracle():
    _, sd, incs, rxs, freqs, kw = CASES[0]
    exc, spw = incs[1]
    cfg = M.McConfig(reduction=EXACT, **{**kw, "strata_per_wavelength": spw})
    r = M.estimate(M.Scene(sd), exc, freqs, cfg)
    ref = oracle_estimate(sd, exc, freqs, cfg, contributions=False)
    assert r.stats.contributions == ref["stats"].contributions
    assert np.max(np.abs(r.sweep.values - ref["values"])) <= 1e-12 * np.max(np.abs(ref["values"]))
