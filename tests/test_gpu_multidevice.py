"""Multi-GPU inside the library (mcsbr_gpu_scene_create_multi).

Only one GPU is reachable in this environment, so the device list repeats
device 0: every replica is a full copy of the scene (arrays copied from the
primary, no second BVH build) with its own stream and buffers, driven by its
own host thread -- the same code path as distinct GPUs, minus NVLink.  The
shards' kernels never wait on one another.

* estimate_batch over 3 replicas == the single-device sweep (EXACT: the
  same bytes; FAST: to summation-order rounding), counters equal;
* estimate(workers=2) shards over 2 of them; workers=1 uses one;
* parity instrumentation on a multi-device scene runs on devices[0] and
  stays bit-exact against the oracle.
"""
import numpy as np
import pytest

import paper_2511_07586_b200 as M
from paper_2511_07586_b200.geometry import airframe
from tests.helpers import contribs_identical, oracle_estimate, sort_contribs

pytestmark = pytest.mark.gpu


def _stats(st):
    return (st.rays_launched, st.segments_traced, st.contributions, st.occlusion_queries, st.cap_kills,
            tuple(st.rays_per_bounce), st.culled_launch_rays)


@pytest.mark.parametrize("reduction", [M.Reduction.EXACT, M.Reduction.FAST])
def test_multi_device_batch_equals_single_device(reduction):
    sd, _ = airframe(6_000, seed=5, dielectric_skin=True)
    excs = [M.monostatic_excitation(80.0, a) for a in (-3.0, 0.0, 4.0)]
    incs, rxs = [(e, 0.7) for e in excs], [[e] for e in excs]
    freqs = np.linspace(8e9, 12e9, 9)
    cfg = M.McConfig(samples_per_stratum=2, max_bounce=24, seed=5, reduction=reduction,
                     roulette=M.RouletteConfig(enabled=True, min_bounce=3))
    one, st1 = M.estimate_batch(M.Scene(sd), incs, rxs, freqs, cfg)
    multi = M.Scene(sd, devices=[0, 0, 0])
    three, st3 = M.estimate_batch(multi, incs, rxs, freqs, cfg)
    assert _stats(st3) == _stats(st1)
    if reduction == M.Reduction.EXACT:
        assert three.tobytes() == one.tobytes()
    else:
        assert np.max(np.abs(three - one)) <= 1e-12 * np.max(np.abs(one))


def test_estimate_workers_select_devices_and_instrumentation_stays_exact():
    obj, mm = M.dihedral_grid(0.5, 16)
    sd = M.load_scene(obj, mm)
    exc = M.monostatic_excitation(90.0, 30.0)
    cfg = M.McConfig(strata_per_wavelength=8, samples_per_stratum=2, max_bounce=4, seed=2,
                     reduction=M.Reduction.EXACT)
    single = M.estimate(M.Scene(sd), exc, [10e9], cfg)
    multi = M.Scene(sd, devices=[0, 0])
    for workers in (1, 2, 8):
        r = M.estimate(multi, exc, [10e9], cfg, workers=workers)
        assert r.sweep.values.tobytes() == single.sweep.values.tobytes()
        assert r.stats.rays_launched == single.stats.rays_launched
    got = []
    r = M.estimate(multi, exc, [10e9], cfg, workers=2, contributions_out=got)
    ref = oracle_estimate(sd, exc, [10e9], cfg)
    assert contribs_identical(sort_contribs(ref["contributions"]), got[0])
    assert r.stats.contributions == ref["stats"].contributions
