"""GPU: the deferred accumulation on uniform frequency grids as a type-1
non-uniform DFT (csrc/spread.cu) against the direct per-frequency phasor
kernel (trace.cu accumulate_kernel, MCSBR_ACC=direct) on the same records.

Both evaluate SweepAccumulator::add (farfield.cpp:130-146); the direct kernel
is itself pinned to the oracle at 1e-9 (test_gpu_parity.py), and so is the
default path (the parity suites run through it).  Here the two accumulations
of one launch must agree to 1e-11 of the largest sum: the spreading kernel's
own error is ~2e-13 per term (tools/nufft_error.py).
"""
import numpy as np
import pytest

import paper_2511_07586_b200 as M
from tests.helpers import oracle_estimate

pytestmark = pytest.mark.gpu


def both(monkeypatch, scene, exc, freqs, cfg, **env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    a = M.estimate(scene, exc, freqs, cfg)
    monkeypatch.setenv("MCSBR_ACC", "direct")
    b = M.estimate(scene, exc, freqs, cfg)
    monkeypatch.delenv("MCSBR_ACC")
    assert a.stats.contributions == b.stats.contributions > 0
    return a.sweep.values, b.sweep.values


def rel(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


@pytest.mark.parametrize("nf", [32, 33, 64, 128, 255, 256])
def test_spread_equals_direct_pec(nf, monkeypatch):
    sd = M.make_builtin_scene("sphere", {"subdivisions": 3})
    s = M.Scene(sd)
    exc = M.monostatic_excitation(50.0, 30.0)
    cfg = M.McConfig(strata_per_wavelength=6, samples_per_stratum=1, max_bounce=8, seed=11)
    a, b = both(monkeypatch, s, exc, np.linspace(8e9, 12e9, nf), cfg)
    assert rel(a, b) <= 1e-11


def test_spread_matches_oracle_on_a_dihedral_sweep():
    """Several incidences per launch (per-incidence grids), 128 f: == oracle."""
    obj, mm = M.dihedral_grid(0.5, 8)
    sd = M.load_scene(obj, mm)
    s = M.Scene(sd)
    cfg = M.McConfig(strata_per_wavelength=3, samples_per_stratum=1, max_bounce=4, seed=2)
    excs = [M.monostatic_excitation(90.0, float(p)) for p in np.linspace(10.0, 80.0, 5)]
    freqs = np.linspace(8e9, 12e9, 128)
    vals, _ = M.estimate_batch(s, [(e, 0.0) for e in excs], [[e] for e in excs], freqs, cfg)
    for i, e in enumerate(excs):
        ref = oracle_estimate(sd, e, freqs, cfg, contributions=False)
        assert np.max(np.abs(vals[i, 0] - ref["values"])) <= 1e-9 * np.max(np.abs(ref["values"]))


def lossy_cube(eps_i):
    obj, mm = M.builtin_scene("glass_cube", {"size_m": 1.0, "center_z_m": -0.5, "eps_r": 2.25})
    sd = M.load_scene(obj, mm)
    e = np.zeros(len(sd.materials))
    e[1:] = eps_i
    sd.eps_imag = e
    return sd


@pytest.mark.parametrize("eps_i,env", [(0.001, {}), (0.01, {}), (0.3, {}),
                                       (0.01, {"MCSBR_NUFFT_ETA_POLY": "0"}),
                                       (0.01, {"MCSBR_NUFFT_ETA_MAX": "0"}), (0.3, {"MCSBR_NUFFT_ETA_MAX": "0"})],
                         ids=["tiny-loss", "weak-loss", "strong-loss", "weak-loss-exact", "weak-loss-direct",
                              "strong-loss-direct"])
def test_spread_equals_direct_lossy(eps_i, env, monkeypatch):
    """Complex path lengths: a small imaginary grid offset is spread with the
    kernel polynomial's continuation (|eta| <= 0.1 cells), a larger one with
    the kernel's own analytic continuation (MCSBR_NUFFT_ETA_POLY=0 forces it),
    a large one (and every one under MCSBR_NUFFT_ETA_MAX=0) is added directly."""
    s = M.Scene(lossy_cube(eps_i))
    exc = M.monostatic_excitation(20.0, 40.0)
    cfg = M.McConfig(strata_per_wavelength=6, samples_per_stratum=2, seed=99,
                     roulette=M.RouletteConfig(enabled=True))
    a, b = both(monkeypatch, s, exc, np.linspace(1e9, 3e9, 64), cfg, **env)
    assert rel(a, b) <= 1e-11
