"""The wavefront kernels (csrc/wavefront.cu: wf_shade + wf_trace over a path
pool) against the persistent megakernel and the oracle.

The wavefront runs the deferred-accumulation Monte Carlo mode (F > 1)
without parity instrumentation; it must reproduce the megakernel's sweep to
summation-order rounding and its RunStats exactly (same arithmetic, same
per-path events), on PEC, lossless-dielectric and lossy scenes, with and
without occlusion and roulette, in both RNG modes, across launch groups and
when the record buffer overflows.  MCSBR_WAVEFRONT=0 selects the megakernel
(read by the library on every call).
"""
import os

import numpy as np
import pytest

import paper_2511_07586_b200 as M
from paper_2511_07586_b200.geometry import airframe
from tests.helpers import oracle_estimate

pytestmark = pytest.mark.gpu


def _stats(st):
    return (st.rays_launched, st.segments_traced, st.contributions, st.grazing_kills, st.cap_kills,
            st.occlusion_queries, tuple(st.rays_per_bounce), tuple(st.roulette_candidates),
            tuple(st.roulette_survivors), st.culled_launch_rays)


def _both(scene, incs, rxs, freqs, cfg, occlusion=True, env=None):
    out = {}
    for wf in ("1", "0"):
        old = {k: os.environ.get(k) for k in ["MCSBR_WAVEFRONT", *(env or {})]}
        os.environ["MCSBR_WAVEFRONT"] = wf
        os.environ.update(env or {})
        try:
            out[wf] = M.estimate_batch(scene, incs, rxs, freqs, cfg, occlusion_enabled=occlusion)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    return out["1"], out["0"]


def _cases():
    cases = []
    af, _ = airframe(6_000, seed=4)
    e = [M.monostatic_excitation(90.0, a) for a in (-2.0, 0.5, 3.0)]
    cases.append(("airframe_pec", af, [(x, 1.0) for x in e], [[x] for x in e], np.linspace(9.5e9, 10.5e9, 8),
                  M.McConfig(samples_per_stratum=1, max_bounce=10, seed=4), True, None))
    skin, _ = airframe(6_000, seed=5, dielectric_skin=True)
    lossless = airframe(6_000, seed=5, dielectric_skin=True)[0]
    lossless.eps_imag = None
    e = [M.monostatic_excitation(80.0, a) for a in (-3.0, 4.0)]
    rr = M.RouletteConfig(enabled=True, min_bounce=3)
    cases.append(("airframe_skin_lossy", skin, [(x, 0.7) for x in e], [[x] for x in e], np.linspace(8e9, 12e9, 40),
                  M.McConfig(samples_per_stratum=2, max_bounce=24, seed=5, roulette=rr), True, None))
    cases.append(("airframe_skin_lossless_philox", lossless, [(x, 0.7) for x in e], [[x] for x in e],
                  np.linspace(8e9, 12e9, 7),
                  M.McConfig(samples_per_stratum=1, max_bounce=24, seed=9, roulette=rr, rng_mode=M.RngMode.PHILOX),
                  True, None))
    glass = M.make_builtin_scene("glass_cube", {"eps_r": 2.25, "size_m": 1.0})
    e = [M.bistatic_excitation(20.0, 40.0, 60.0, 10.0)]
    cases.append(("glass_no_occlusion", glass, [(x, 6.0) for x in e], [[x] for x in e], np.linspace(1e9, 3e9, 5),
                  M.McConfig(samples_per_stratum=2, seed=99, roulette=M.RouletteConfig(enabled=True)), False, None))
    sph = M.make_builtin_scene("sphere", {"subdivisions": 3})
    e = [M.monostatic_excitation(t, 10.0 * t) for t in (0.0, 30.0, 60.0, 90.0)]
    cases.append(("sphere_groups_overflow", sph, [(x, 8.0) for x in e], [[x] for x in e],
                  [2e9, 2.3e9, 3.1e9],  # non-uniform grid
                  M.McConfig(samples_per_stratum=2, max_bounce=8, seed=3), True,
                  {"MCSBR_GROUP_ENTRIES": "20000", "MCSBR_REC_CAP": "3000"}))
    return cases


CASES = _cases()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_wavefront_equals_megakernel(case):
    name, sd, incs, rxs, freqs, cfg, occl, env = case
    s = M.Scene(sd)
    (vw, sw), (vm, sm) = _both(s, incs, rxs, freqs, cfg, occl, env)
    assert _stats(sw) == _stats(sm)
    assert sw.contributions > 0
    scale = np.max(np.abs(vm))
    assert np.max(np.abs(vw - vm)) <= 1e-9 * scale


def test_wavefront_equals_oracle():
    """F > 1 estimate_batch (wavefront) == the oracle restatement of the reference."""
    af, _ = airframe(6_000, seed=4)
    exc = M.monostatic_excitation(90.0, 2.0)
    freqs = np.linspace(9.5e9, 10.5e9, 8)
    cfg = M.McConfig(strata_per_wavelength=1.0, samples_per_stratum=1, seed=4, max_bounce=10)
    v, st = M.estimate_batch(M.Scene(af), [(exc, 0.0)], [[exc]], freqs, cfg)
    ref = oracle_estimate(af, exc, freqs, cfg, contributions=False)
    assert st.rays_launched == ref["stats"].rays_launched
    assert st.contributions == ref["stats"].contributions
    assert st.segments_traced == ref["stats"].segments_traced
    scale = np.max(np.abs(ref["values"]))
    assert np.max(np.abs(v[0, 0] - ref["values"])) <= 1e-9 * scale
