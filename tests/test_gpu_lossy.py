"""GPU: the lossy-media extension (the reference has only
real permittivity, proj/include/mcsbr/em_math.hpp:99-105, so these are the
pins for the extension):

1. the complex-index transport with Im eps = 0 reproduces the reference model
   BIT-FOR-BIT (contributions) -- the extension is a strict generalisation;
2. a lossy dielectric cube at normal incidence converges to the
   transfer-matrix slab reflection with a COMPLEX index (the reference's
   slab oracle, proj/src/oracles.cpp:32-64, with n complex), i.e. the
   reference's own "MC estimator converges to the slab oracle" test
   (tests/test_solvers.cpp:480-499) extended to loss;
3. continuity: Im eps -> 0 recovers the lossless sweep.
"""
import numpy as np
import pytest

import paper_2511_07586_b200 as M
from tests.helpers import contribs_identical, oracle_estimate, sort_contribs

pytestmark = pytest.mark.gpu

C0 = 299792458.0


def slab_reflection(layers, f, pec_backed=False, n0=1.0, nt=1.0):
    """Normal-incidence chain-matrix reflection (oracles.cpp:32-64), complex n."""
    k0 = 2 * np.pi * f / C0
    m = np.eye(2, dtype=complex)
    for n, d in layers:
        delta = k0 * n * d
        lm = np.array([[np.cos(delta), -1j * np.sin(delta) / n],
                       [-1j * n * np.sin(delta), np.cos(delta)]])
        m = lm @ m
    a, b, c, d = m[0, 0], m[0, 1], m[1, 0], m[1, 1]
    if pec_backed:
        return -(a + b * n0) / (a - b * n0)
    return (c + n0 * d - nt * a - nt * n0 * b) / (nt * a - nt * n0 * b - c + n0 * d)


def cube(size, eps_r, eps_i=None):
    obj, mm = M.builtin_scene("glass_cube", {"size_m": size, "center_z_m": -0.5 * size,
                                             "eps_r": eps_r})
    sd = M.load_scene(obj, mm)
    if eps_i is not None:
        e = np.zeros(len(sd.materials))
        e[1:] = eps_i
        sd.eps_imag = e
    return sd


def test_lossy_transport_with_zero_loss_is_bit_exact():
    sd = cube(1.0, 2.25)
    sd_l = cube(1.0, 2.25, eps_i=0.0)  # eps_imag given (all zero): complex transport kernel
    exc = M.monostatic_excitation(20.0, 40.0)
    freqs = np.linspace(1e9, 3e9, 5)
    cfg = M.McConfig(strata_per_wavelength=6, samples_per_stratum=2, seed=99,
                     roulette=M.RouletteConfig(enabled=True))
    got = []
    r = M.estimate(M.Scene(sd_l), exc, freqs, cfg, contributions_out=got)
    ref = oracle_estimate(sd, exc, freqs, cfg)
    assert contribs_identical(got[0], sort_contribs(ref["contributions"]))
    assert np.max(np.abs(r.sweep.values - ref["values"])) <= 1e-9 * np.max(np.abs(ref["values"]))


@pytest.mark.parametrize("eps_i", [0.05, 0.3])
def test_lossy_cube_converges_to_complex_slab_oracle(eps_i):
    size, eps_r = 1.0, 2.25
    sd = cube(size, eps_r, eps_i)
    n = np.sqrt(eps_r - 1j * eps_i)
    assert n.imag < 0
    freqs = np.linspace(1.03e9, 2.91e9, 11)
    cfg = M.McConfig(strata_per_wavelength=10, samples_per_stratum=16,
                     branch_strategy=M.BranchStrategy.FIFTY_FIFTY, seed=11, max_bounce=15)
    r = M.estimate(M.Scene(sd), M.monostatic_excitation(0.0, 0.0), freqs, cfg)
    k0 = 2 * np.pi * freqs / C0
    want = np.array([1j * k * size * size * slab_reflection([(n, size)], f) / np.sqrt(np.pi)
                     for k, f in zip(k0, freqs)])
    got = r.sweep.values[M.VV]
    db = 20 * np.log10(np.abs(got)) - 20 * np.log10(np.abs(want))
    assert np.mean(np.abs(db)) < 0.15, db
    # phase too (the reference test only checks magnitude)
    assert np.max(np.abs(np.angle(got / want))) < 0.05


def test_lossy_continuity_to_lossless():
    sd = cube(1.0, 2.25)
    sd_l = cube(1.0, 2.25, eps_i=1e-9)
    exc = M.monostatic_excitation(10.0, 30.0)
    freqs = np.linspace(1e9, 3e9, 4)
    cfg = M.McConfig(strata_per_wavelength=5, samples_per_stratum=2, seed=5)
    a = M.estimate(M.Scene(sd), exc, freqs, cfg).sweep.values
    b = M.estimate(M.Scene(sd_l), exc, freqs, cfg).sweep.values
    assert np.max(np.abs(a - b)) <= 1e-6 * np.max(np.abs(a))


def test_lossy_coated_sphere_config3_geometry():
    """c3 materials (4.0-0.1j, 2.2-0.01j on a PEC core): runs, attenuates
    relative to the lossless coating, and stays finite."""
    obj, mm = M.coated_sphere(subdivisions=3, lossless=False)
    lossy = M.load_scene(obj, mm)
    obj, mm = M.coated_sphere(subdivisions=3, lossless=True)
    clean = M.load_scene(obj, mm)
    exc = M.bistatic_excitation(90.0, 0.0, 60.0, 0.0)
    cfg = M.McConfig(strata_per_wavelength=10, samples_per_stratum=2, seed=3, max_bounce=16,
                     roulette=M.RouletteConfig(enabled=True, min_bounce=3))
    a = M.estimate(M.Scene(clean), exc, [3e9], cfg)
    b = M.estimate(M.Scene(lossy), exc, [3e9], cfg)
    assert np.all(np.isfinite(b.sweep.values))
    assert a.stats.rays_launched == b.stats.rays_launched
    assert b.stats.contributions > 0
    assert not np.allclose(a.sweep.values, b.sweep.values)
