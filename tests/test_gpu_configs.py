"""BASELINE.json configs c1-c5 on the GPU against the oracle and the compiled reference.

One test per configuration, at the configuration's own geometry and
settings (strata reduced only where the single-threaded oracle would take
minutes), through the product's public API:

* every emitted contribution (per incidence / receiver) is BIT-IDENTICAL to
  the oracle's (tests/helpers.py contribs_identical: IEEE equality), and the
  RunStats counters are equal;
* the far-field sweep agrees with the UNMODIFIED reference (oracle/_ref,
  reference estimate() on all host cores) within the north-star bound of
  1e-4 relative (in practice ~1e-14: only the summation order differs);
* c5's lossless twin is the one case where the reference disagrees with its
  own brute-force intersection (near-coincident skin surfaces, DESIGN.md
  §2): the test proves every differing path is one whose launch ray the
  reference's BVH and the reference's brute force trace differently, and
  that the sweeps agree to 1e-9 once those paths are taken out of both.

Shapes: SURVEY.md §8d / BASELINE.json configs.  Oracle / reference are test
infrastructure only (oracle/__init__.py).
"""
import ctypes as C
import math
import os

import numpy as np
import pytest

import oracle
import paper_2511_07586_b200 as M
from paper_2511_07586_b200.geometry import airframe
from tests.helpers import contribs_identical, sort_contribs

pytestmark = pytest.mark.gpu

C0 = 299792458.0
CORES = os.cpu_count() or 1


def _spw(scene, exc, lam, rays):
    grid, _ = M.launch_plan(scene, exc.k_inc, 0.0, 1.0, lam, 1)
    return lam * math.sqrt(rays / grid.rect.area())


def _check(sd, gpu_scene, exc, freqs, cfg, ref_h=None, port_h=None, ref_tol=1e-4, capacity=1 << 23):
    """GPU estimate vs oracle (bit-exact contributions, exact counters) and
    vs the reference (sweep within ref_tol).  Returns the three results."""
    got = []
    r = M.estimate(gpu_scene, exc, freqs, cfg, contributions_out=got, contributions_capacity=capacity)
    port_h = port_h or oracle.port_scene(sd)
    p = oracle.port_estimate(port_h, exc.to_c(), np.asarray(freqs, float), cfg.to_c(), True, capacity)
    a, b = sort_contribs(p["contributions"]), got[0]
    assert p["n_contributions"] == len(a) == len(b) == r.stats.contributions > 0
    assert contribs_identical(a, b), "contributions differ from the oracle"
    st = p["stats"]
    assert (r.stats.rays_launched, r.stats.segments_traced, r.stats.cap_kills, r.stats.grazing_kills) == (
        st.rays_launched, st.segments_traced, st.cap_kills, st.grazing_kills)
    assert r.stats.rays_per_bounce == list(st.rays_per_bounce[: st.n_rounds])
    scale = np.max(np.abs(p["values"]))
    assert np.max(np.abs(p["values"] - r.sweep.values)) <= 1e-9 * scale
    ref = None
    if ref_h is not None:
        ref = oracle.ref_estimate(ref_h, exc.to_c(), np.asarray(freqs, float), cfg.to_c(), CORES)
        if ref_tol is not None:
            rel = np.max(np.abs(ref["values"] - r.sweep.values)) / np.max(np.abs(ref["values"]))
            assert rel <= ref_tol, rel
    return r, p, ref, b


def test_c1_sphere_full_config():
    """c1: PEC icosphere L5 (20,480 triangles), theta 90 phi 0, 10 GHz, spw 30
    (4,008,004 paths, the full configuration), max 8, seed 1."""
    sd = M.make_builtin_scene("sphere", {"subdivisions": 5})
    s = M.Scene(sd)
    exc = M.monostatic_excitation(90.0, 0.0)
    cfg = M.McConfig(strata_per_wavelength=30, samples_per_stratum=1, max_bounce=8, seed=1)
    r, p, ref, _ = _check(sd, s, exc, [10e9], cfg, ref_h=oracle.ref_scene(sd))
    assert r.stats.rays_launched == 4_008_004
    sigma = abs(r.sweep.values[M.HH, 0]) ** 2
    assert abs(10 * np.log10(sigma / np.pi)) < 1.0  # the reference sits ~0.5-0.7 dB below pi r^2


def test_c2_dihedral_three_sweep_angles():
    """c2: the bench's 64x64-per-plate dihedral at 3 of its 181 angles (ends
    and bisector), ~1M paths each, 10 GHz, max 4, seed 2."""
    obj, mm = M.dihedral_grid(0.5, 64)
    sd = M.load_scene(obj, mm)
    s = M.Scene(sd)
    ref_h, port_h = oracle.ref_scene(sd), oracle.port_scene(sd)
    lam = C0 / 10e9
    for phi in (0.0, 45.0, 90.0):
        exc = M.monostatic_excitation(90.0, phi)
        cfg = M.McConfig(strata_per_wavelength=_spw(s, exc, lam, 1e6), samples_per_stratum=1, max_bounce=4, seed=2)
        r, _, _, _ = _check(sd, s, exc, [10e9], cfg, ref_h=ref_h, port_h=port_h)
        assert r.stats.rays_launched > 900_000


def test_c3_coated_sphere_receivers():
    """c3 (lossless twin, the reference model): PEC core + 10 mm / 5 mm shells,
    each an L5 icosphere (61,440 triangles), 3 GHz, Fresnel sampling, RR q 0.5
    from bounce 3, max 16, seed 3, at reduced strata (spw 60).  Every receiver
    of a 4-receiver bistatic fan: contributions bit-exact vs the oracle; the
    fan (one trace for all receivers) equals the per-receiver estimates."""
    obj, mm = M.coated_sphere(subdivisions=5, lossless=True)
    sd = M.load_scene(obj, mm)
    s = M.Scene(sd)
    ref_h, port_h = oracle.ref_scene(sd), oracle.port_scene(sd)
    cfg = M.McConfig(strata_per_wavelength=60, samples_per_stratum=1, max_bounce=16, seed=3,
                     roulette=M.RouletteConfig(enabled=True, q=0.5, min_bounce=3))
    rxs = [M.bistatic_excitation(90.0, 0.0, th, 0.0) for th in (0.0, 60.0, 120.0, 180.0)]
    singles = []
    for e in rxs:
        r, _, _, _ = _check(sd, s, e, [3e9], cfg, ref_h=ref_h, port_h=port_h)
        singles.append(r.sweep.values)
    inc = M.monostatic_excitation(90.0, 0.0)
    fan, st = M.estimate_batch(s, [(inc, 0.0)], [rxs], [3e9], cfg)
    for k in range(len(rxs)):
        scale = np.max(np.abs(singles[k]))
        assert np.max(np.abs(fan[0, k] - singles[k])) <= 1e-9 * scale


def test_c4_airframe_two_azimuths():
    """c4: PEC airframe (199,996 triangles, seed 4), 64 f on 9.5-10.5 GHz, the
    first and last azimuth of the +-3 deg sweep at the full ~2M paths, max 10."""
    sd, _ = airframe(200_000, seed=4)
    s = M.Scene(sd)
    ref_h, port_h = oracle.ref_scene(sd), oracle.port_scene(sd)
    freqs = np.linspace(9.5e9, 10.5e9, 64)
    lam = C0 / freqs[-1]
    for az in (-3.0, 3.0):
        exc = M.monostatic_excitation(90.0, az)
        cfg = M.McConfig(strata_per_wavelength=_spw(s, exc, lam, 2e6), samples_per_stratum=1, max_bounce=10,
                         seed=4)
        r, _, _, _ = _check(sd, s, exc, freqs, cfg, ref_h=ref_h, port_h=port_h)
        assert r.stats.rays_launched > 1_900_000
        assert r.stats.culled_launch_rays > 0  # the coverage bitmap retired provable misses


def _zero_sign_free_records(c):
    """records with -0.0 replaced by +0.0 (the IEEE-equality comparison of
    tests/helpers.py contribs_identical, per record)"""
    c = c.copy()
    for name in c.dtype.names:
        if c.dtype[name].kind == "f" or (c.dtype[name].subdtype and c.dtype[name].subdtype[0].kind == "f"):
            x = c[name]
            x[x == 0] = 0.0
            c[name] = x
    return c


def _accumulate(contribs, exc, freqs):
    """SweepAccumulator::add + finalize (farfield.cpp:106-167) of contribution
    records in numpy -> [4][nf] complex (VV, HH, VH, HV)."""
    ks, rv, rh = (np.asarray(x, float) for x in (exc.k_scatter, exc.rx_v, exc.rx_h))
    k0 = 2 * np.pi * np.asarray(freqs, float) / C0
    out = np.zeros((4, len(k0)), complex)
    for c in contribs:
        aj = c["a_j"][..., 0] + 1j * c["a_j"][..., 1]
        am = c["a_m"][..., 0] + 1j * c["a_m"][..., 1]
        f0 = np.cross(ks, np.cross(ks, aj[0])) + np.cross(ks, am[0])
        f1 = np.cross(ks, np.cross(ks, aj[1])) + np.cross(ks, am[1])
        amp = [f0 @ rv, f1 @ rh, f1 @ rv, f0 @ rh]  # VV, HH, VH, HV
        sp = c["phi_total"] - ks @ c["exit_point"]
        z = np.exp(-1j * k0 * sp)
        for ch in range(4):
            out[ch] += amp[ch] * z
    return out * (1j * k0 / (2 * np.sqrt(np.pi)))


def test_c5_airframe_skin_vs_reference_and_its_bvh_quirk():
    """c5 (lossless twin): 1,000,676 triangles with two nested skins on wings
    and fin, 128 f on 8-12 GHz, azimuth -5 deg, RR q 0.5 from 3, max 24, seed
    5, reduced strata (spw 3).  GPU == oracle bit for bit.  The reference's
    BVH (unpadded fp64 slab test) returns, for a handful of launch rays that
    graze near-coincident skin surfaces, a hit ~1e-14 farther than its own
    brute force (Scene::intersect_brute_force, the ground truth the oracle and
    the GPU follow).  Every path whose contributions differ from the
    reference's must be such a path, and without those paths the sweeps
    agree to 1e-9."""
    sd, _ = airframe(1_000_000, seed=5, dielectric_skin=True)
    sd.eps_imag = None
    s = M.Scene(sd)
    exc = M.monostatic_excitation(90.0, -5.0)
    cfg = M.McConfig(strata_per_wavelength=3, samples_per_stratum=1, max_bounce=24, seed=5,
                     roulette=M.RouletteConfig(enabled=True, q=0.5, min_bounce=3))
    freqs = np.linspace(8e9, 12e9, 128)
    ref_h = oracle.ref_scene(sd)
    r, p, _, gpu_c = _check(sd, s, exc, freqs, cfg, ref_h=None, capacity=1 << 22)
    ref = oracle.ref_estimate(ref_h, exc.to_c(), freqs, cfg.to_c(), CORES, True, 1 << 22)
    rc = sort_contribs(ref["contributions"])
    # paths (cells; spp = 1) whose contribution records differ
    ka = {int(k): i for i, k in enumerate(rc["order_key"])}
    kb = {int(k): i for i, k in enumerate(gpu_c["order_key"])}
    cells = {k >> 8 for k in set(ka) ^ set(kb)}
    rn, gn = _zero_sign_free_records(rc), _zero_sign_free_records(gpu_c)
    cells |= {k >> 8 for k in set(ka) & set(kb) if rn[ka[k]].tobytes() != gn[kb[k]].tobytes()}
    assert len(cells) < 1e-4 * r.stats.rays_launched, len(cells)
    if cells:
        # rebuild the launch rays of those paths (solver_mc.cpp:33-42) and
        # trace them with the reference's BVH and its brute force
        grid, _ = M.launch_plan(s, exc.k_inc, 0.0, cfg.strata_per_wavelength, C0 / freqs[-1], 1)
        L = oracle.port()
        cu = L.orc_counter_uniform
        cu.restype, cu.argtypes = C.c_double, [C.c_uint64] * 5
        rect = grid.rect
        o = []
        for cell in sorted(cells):
            i, j = cell % grid.nu, cell // grid.nu
            su = -1.0 + 2.0 * (i + cu(cfg.seed, cell, 0, 0, 0x101)) / grid.nu
            sv = -1.0 + 2.0 * (j + cu(cfg.seed, cell, 0, 0, 0x102)) / grid.nv
            o.append((np.asarray(rect.center) + np.asarray(rect.u_axis) * (su * rect.half_u))
                     + np.asarray(rect.v_axis) * (sv * rect.half_v))
        o = np.array(o)
        d = np.tile(np.asarray(exc.k_inc, float), (len(o), 1))
        tm = np.zeros(len(o))
        bvh = oracle.intersect("ref", ref_h, o, d, tm, 0)
        brute = oracle.intersect("ref", ref_h, o, d, tm, 1)
        disagree = (bvh[:, 12] != brute[:, 12]) | (bvh[:, 0] != brute[:, 0])
        assert disagree.all(), f"{(~disagree).sum()} differing paths are not reference-BVH quirks"
        # the GPU's first hit of those rays is the brute-force one
        t, ids = s.intersect_batch(o, d, tm)
        assert np.array_equal(ids, brute[:, 12].astype(np.uint32))
    # sweeps without the quirk paths
    sel_r = np.array([(int(k) >> 8) in cells for k in rc["order_key"]], bool)
    sel_g = np.array([(int(k) >> 8) in cells for k in gpu_c["order_key"]], bool)
    vr = ref["values"] - _accumulate(rc[sel_r], exc, freqs)
    vg = r.sweep.values - _accumulate(gpu_c[sel_g], exc, freqs)
    assert np.max(np.abs(vr - vg)) <= 1e-9 * np.max(np.abs(vr))
