"""GPU: the lossy-media extension (the reference has only
real permittivity, proj/include/mcsbr/em_math.hpp:99-105, so these are the
pins for the extension):

1. the complex-index transport with Im eps = 0 reproduces the reference model
   BIT-FOR-BIT (contributions) -- the extension is a strict generalisation;
2. a lossy dielectric cube at normal incidence converges to the
   transfer-matrix slab reflection with a COMPLEX index (the reference's
   slab oracle, proj/src/oracles.cpp:32-64, with n complex), i.e. the
   reference's own "MC estimator converges to the slab oracle" test
   (tests/test_solvers.cpp:276-295) extended to loss;
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


def layered_slab(a, layers, metal=0.01):
    """A planar stack on a PEC block, lateral extent [-a, a]^2, top face at
    z = 0: layers = [(name, eps_r, eps_i, thickness), ...] from the top.
    Every interface is one horizontal quad (normal +z, front = the medium
    above); the side walls of every band close its medium against air."""
    from paper_2511_07586_b200.geometry import scene_from_arrays

    verts, faces, reg, regions = [], [], [], []

    index = {}

    def vid(q):  # shared vertices: the media boundaries must be closed manifolds
        if q not in index:
            index[q] = len(verts)
            verts.append(q)
        return index[q]

    def quad(p, region):
        if region not in regions:
            regions.append(region)
        i = [vid(q) for q in p]
        faces.extend([(i[0], i[1], i[2]), (i[0], i[2], i[3])])
        reg.extend([regions.index(region)] * 2)

    def band(z0, z1, inside):  # side walls of z in [z0, z1], outward normals
        quad([(a, -a, z0), (a, a, z0), (a, a, z1), (a, -a, z1)], ("air", inside))
        quad([(-a, a, z0), (-a, -a, z0), (-a, -a, z1), (-a, a, z1)], ("air", inside))
        quad([(a, a, z0), (-a, a, z0), (-a, a, z1), (a, a, z1)], ("air", inside))
        quad([(-a, -a, z0), (a, -a, z0), (a, -a, z1), (-a, -a, z1)], ("air", inside))

    def horiz(z, above, below):
        quad([(-a, -a, z), (a, -a, z), (a, a, z), (-a, a, z)], (above, below))

    mats = {"air": {"eps_r": 1.0}, "metal": {"pec": True}}
    z, above = 0.0, "air"
    for name, er, ei, t in layers:
        horiz(z, above, name)
        band(z - t, z, name)
        mats[name] = {"eps_r": er, "eps_i": ei}
        z, above = z - t, name
    horiz(z, above, "metal")
    band(z - metal, z, "metal")
    quad([(-a, a, z - metal), (a, a, z - metal), (a, -a, z - metal), (-a, -a, z - metal)], ("air", "metal"))
    return scene_from_arrays(np.array(verts, float), np.array(faces), np.array(reg), regions, mats)


@pytest.mark.parametrize("name,layers,f0,f1", [
    # c5's two-layer skin: 2 mm eps 3.5-0.05j over 4 mm eps 10-1.0j on PEC (8-12 GHz)
    ("c5_skin", [("outer", 3.5, 0.05, 0.002), ("inner", 10.0, 1.0, 0.004)], 8e9, 12e9),
    # the planar analogue of c3's shells: 5 mm eps 2.2-0.01j over 10 mm eps 4.0-0.1j on PEC (2.5-3.5 GHz)
    ("c3_shells", [("outer", 2.2, 0.01, 0.005), ("inner", 4.0, 0.1, 0.010)], 2.5e9, 3.5e9),
])
def test_multilayer_lossy_stack_matches_chain_matrix_oracle(name, layers, f0, f1):
    """SURVEY.md §8c lossy pin: Monte Carlo on a planar PEC-backed two-layer
    lossy slab at normal incidence against the complex chain-matrix oracle
    (oracles.cpp:32-64 generalised to complex index, incl. its pec_backed
    branch :56-59): within 0.1 dB and 0.05 rad at every frequency."""
    a = 0.15
    sd = layered_slab(a, layers)
    ns = [np.sqrt(er - 1j * ei) for _, er, ei, _ in layers]
    freqs = np.linspace(f0, f1, 9)
    cfg = M.McConfig(strata_per_wavelength=8, samples_per_stratum=64, seed=17, max_bounce=40,
                     branch_strategy=M.BranchStrategy.FRESNEL)
    r = M.estimate(M.Scene(sd), M.monostatic_excitation(0.0, 0.0), freqs, cfg)
    k0 = 2 * np.pi * freqs / C0
    area = (2 * a) ** 2
    want = np.array([1j * k * area * slab_reflection([(n, t) for n, (_, _, _, t) in zip(ns, layers)], f,
                                                     pec_backed=True) / np.sqrt(np.pi)
                     for k, f in zip(k0, freqs)])
    got = r.sweep.values[M.VV]
    db = 20 * np.log10(np.abs(got) / np.abs(want))
    ph = np.angle(got / want)
    assert np.max(np.abs(db)) < 0.1, (db, ph)
    assert np.max(np.abs(ph)) < 0.05, (db, ph)
