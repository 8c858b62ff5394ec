"""CPU: pin the oracle (oracle/mcsbr_oracle.c) to the reference.

Every check is BIT-exact.  The golden vectors in tests/golden/ were produced by
the unmodified reference (tests/golden/make_golden.py over oracle/_ref); the
`ref`-marked tests additionally compare against the live reference library
when it has been built (the build container always has it).
"""
import hashlib
import os

import numpy as np
import pytest

import oracle
import paper_2511_07586_b200 as M
from tests.helpers import det_cases, det_stats_vector, parity_cases, sort_contribs

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
dp = oracle.dp


def load(name):
    return np.load(os.path.join(G, name), allow_pickle=False)


def test_counter_hash_kat(port):
    g = load("rng.npz")
    for k, h, u in zip(g["keys"], g["hash"], g["uniform"]):
        k = [int(x) for x in k]
        assert port.orc_counter_hash(*k) == int(h)
        assert port.orc_counter_uniform(*k) == float(u)


def test_fresnel_golden(port):
    g = load("em.npz")
    out = np.zeros(11)
    for (n1, n2, ci), want in zip(g["fresnel_in"], g["fresnel_out"]):
        assert port.orc_fresnel(n1, n2, ci, dp(out)) == 0
        assert out.tobytes() == want.tobytes()


def test_fresnel_domain_errors(port):
    out = np.zeros(11)
    # em_math.cpp:6-9 (tests/test_em_math.cpp:48-53)
    assert port.orc_fresnel(-1.0, 1.5, 1.0, dp(out)) != 0
    assert port.orc_fresnel(1.0, 0.0, 1.0, dp(out)) != 0
    assert port.orc_fresnel(1.0, 1.5, 0.0, dp(out)) != 0
    assert port.orc_fresnel(1.0, 1.5, 1.5, dp(out)) != 0


def test_sp_basis_golden(port):
    g = load("em.npz")
    out = np.zeros(18)
    for row, want in zip(g["basis_in"], g["basis_out"]):
        d = np.ascontiguousarray(row[0:3])
        n = np.ascontiguousarray(row[3:6])
        assert port.orc_sp_basis(dp(d), dp(n), row[6], row[7], dp(out)) == 0
        assert out.tobytes() == want.tobytes()


def test_interface_transform_golden(port):
    g = load("em.npz")
    out = np.zeros(6)
    for co, e, bas, want in zip(g["transform_coeffs"], g["transform_e"], g["basis_out"],
                                g["transform_out"]):
        for br in (0, 1):
            assert port.orc_interface_transform(dp(np.ascontiguousarray(e)), br,
                                                dp(np.ascontiguousarray(co)),
                                                dp(np.ascontiguousarray(bas)), dp(out)) == 0
            assert out.tobytes() == want[br].tobytes()


def test_branch_outcomes_and_meca_golden(port):
    g = load("em.npz")
    out = np.zeros(63)
    me = np.zeros(12)
    for st, hit, want, wme in zip(g["branch_state"], g["branch_hit"], g["branch_out"], g["meca_out"]):
        st = np.ascontiguousarray(st)
        hit = np.ascontiguousarray(hit)
        assert port.orc_branch_outcomes(dp(st), dp(hit), dp(out)) == 0
        assert out.tobytes() == want.tobytes()
        kind = int(hit[12]) % 3
        for pol in (0, 1):
            e = np.ascontiguousarray(st[6 + 6 * pol:12 + 6 * pol])
            assert port.orc_meca_currents(dp(hit), dp(e), dp(np.ascontiguousarray(st[3:6])), kind,
                                          dp(me)) == 0
            assert me.tobytes() == wme[pol].tobytes()


def test_intersect_golden(port):
    """Closest hit == the reference's Scene::intersect_brute_force bit for bit.

    Half the golden rays are aimed exactly at mesh vertices.  On those the
    reference's own BVH walk (unpadded fp64 slab test, geometry.cpp:48-64)
    misses or mis-breaks ties for hits lying exactly on a box face; the
    golden file records both, and brute force is the ground truth
    (SURVEY.md §7 hard part 1)."""
    g = load("intersect.npz")
    for name, params in [("glass_cube", {}), ("nested", {"subdivisions": 2}),
                         ("sphere", {"subdivisions": 3})]:
        sd = M.make_builtin_scene(name, params)
        ps = oracle.port_scene(sd)
        h = oracle.intersect("port", ps, g[f"{name}_o"], g[f"{name}_d"], g[f"{name}_tmin"], 0)
        assert np.array_equal(h[:, 12].astype(np.uint32), g[f"{name}_id"])
        assert h[:, 0].tobytes() == g[f"{name}_t"].tobytes()
        # where the reference's BVH agrees with its brute force, so do we
        ok = g[f"{name}_bvh_id"] == g[f"{name}_id"]
        assert ok.mean() > 0.85
        assert np.array_equal(h[ok, 12].astype(np.uint32), g[f"{name}_bvh_id"][ok])
        # brute force == BVH (tests/test_geometry.cpp:89-112)
        hb = oracle.intersect("port", ps, g[f"{name}_o"], g[f"{name}_d"], g[f"{name}_tmin"], 1)
        assert hb.tobytes() == h.tobytes()


def _db_close(a, b, tol=1e-6, span=150.0):
    """dB arrays agree wherever the level is within `span` dB of the peak
    (deep nulls are numerically ill-conditioned in dB)."""
    keep = b > b.max() - span
    return np.max(np.abs(a[keep] - b[keep])) <= tol


def test_signal_restatement_against_reference_golden():
    """oracle/signal_ref.py == the reference's range_profile / isar
    (signal_processing.cpp:66-162) on seeded random and point-scatterer sweeps."""
    from oracle import signal_ref as S

    g = load("signal.npz")
    for name in ("rand", "pts"):
        for h in (0, 1):
            r, db, b = S.range_profile(g[f"rp_{name}_{h}_in"], g["rp_freqs"], bool(h), 4)
            assert r.tobytes() == g[f"rp_{name}_{h}_range"].tobytes()
            assert b == g[f"rp_{name}_{h}_bin"][0]
            assert _db_close(db, g[f"rp_{name}_{h}_db"])
    d, c, db, pk = S.isar(g["isar_in"], g["isar_freqs"], g["isar_angles"], True, 4, -40.0)
    assert d.tobytes() == g["isar_down"].tobytes()
    assert np.allclose(c, g["isar_cross"], rtol=1e-14, atol=0)
    assert _db_close(db, g["isar_db"]) and abs(pk - g["isar_peak"][0]) < 1e-9


CASES = parity_cases()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_estimate_golden(case):
    name, sd, exc, freqs, cfg = case
    g = load("estimate.npz")
    r = oracle.port_estimate(oracle.port_scene(sd), exc.to_c(), np.asarray(freqs, float),
                             cfg.to_c(), True, 1 << 21)
    assert r["values"].tobytes() == g[f"{name}_values"].tobytes()
    st = r["stats"]
    got = np.array([st.rays_launched, st.segments_traced, st.contributions, st.grazing_kills,
                    st.cap_kills] + list(st.rays_per_bounce[:32]) + list(st.roulette_candidates[:32])
                   + list(st.roulette_survivors[:32]), dtype=np.uint64)
    assert np.array_equal(got, g[f"{name}_stats"])
    c = sort_contribs(r["contributions"])
    assert hashlib.sha256(c.tobytes()).digest() == g[f"{name}_contrib_sha256"].tobytes()
    assert c[:64].tobytes() == g[f"{name}_contrib_head"].tobytes()


DET = det_cases()


@pytest.mark.parametrize("case", DET, ids=[c[0] for c in DET])
def test_solve_golden(case):
    """C restatement of the deterministic solver == reference solve() bit for bit
    (values, stats incl. the stack accounting, every contribution)."""
    name, sd, exc, freqs, cfg = case
    g = load("det.npz")
    r = oracle.port_solve(oracle.port_scene(sd), exc.to_c(), np.asarray(freqs, float), cfg.to_c(),
                          True, 1 << 21)
    assert r["values"].tobytes() == g[f"{name}_values"].tobytes()
    assert np.array_equal(det_stats_vector(r["stats"]), g[f"{name}_stats"])
    c = sort_contribs(r["contributions"])
    assert hashlib.sha256(c.tobytes()).digest() == g[f"{name}_contrib_sha256"].tobytes()
    assert c[:64].tobytes() == g[f"{name}_contrib_head"].tobytes()


# --------------------------------------------------------------------------
# live reference (skipped when oracle/_ref has not been built)

needs_ref = pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")


@pytest.mark.ref
@needs_ref
def test_oracle_equals_reference_on_fresh_cases():
    """Beyond the goldens: other seeds / angles / strategies, port vs live reference."""
    rng = np.random.default_rng(5)
    scenes = [M.make_builtin_scene("nested", {"subdivisions": 2}),
              M.make_builtin_scene("glass_cube", {"eps_r": 3.1, "size_m": 0.7}),
              M.make_builtin_scene("airplane_stub", {"eps_r": 2.0})]
    for sd in scenes:
        rs, ps = oracle.ref_scene(sd), oracle.port_scene(sd)
        for _ in range(3):
            th, ph = rng.uniform(0, 180), rng.uniform(0, 360)
            exc = M.monostatic_excitation(th, ph) if rng.random() < 0.5 else \
                M.bistatic_excitation(th, ph, rng.uniform(0, 180), rng.uniform(0, 360))
            cfg = M.McConfig(strata_per_wavelength=float(rng.uniform(2, 5)), samples_per_stratum=2,
                             seed=int(rng.integers(1 << 40)), max_bounce=int(rng.integers(2, 12)),
                             branch_strategy=M.BranchStrategy(int(rng.integers(2))),
                             roulette=M.RouletteConfig(enabled=bool(rng.random() < 0.5),
                                                       q=float(rng.uniform(0.2, 0.8)),
                                                       min_bounce=int(rng.integers(1, 4))),
                             block_size=int(rng.integers(50, 5000)))
            freqs = np.linspace(1e9, 3e9, int(rng.integers(1, 6)))
            a = oracle.ref_estimate(rs, exc.to_c(), freqs, cfg.to_c(), 2, True, 1 << 20)
            b = oracle.port_estimate(ps, exc.to_c(), freqs, cfg.to_c(), True, 1 << 20)
            assert a["values"].tobytes() == b["values"].tobytes()
            assert a["contributions"].tobytes() == b["contributions"].tobytes()


@pytest.mark.ref
@needs_ref
def test_solve_oracle_equals_reference_on_fresh_cases():
    rng = np.random.default_rng(11)
    for sd in [M.make_builtin_scene("glass_cube", {"eps_r": 3.1, "size_m": 0.7}),
               M.make_builtin_scene("nested", {"subdivisions": 2})]:
        rs, ps = oracle.ref_scene(sd), oracle.port_scene(sd)
        for _ in range(3):
            exc = M.monostatic_excitation(rng.uniform(0, 180), rng.uniform(0, 360))
            cfg = M.DetConfig(rays_per_wavelength=float(rng.uniform(2, 5)),
                              max_bounce=int(rng.integers(1, 10)),
                              amplitude_cutoff=float(rng.choice([0.0, 0.1, 0.3])),
                              block_size=int(rng.integers(50, 5000)))
            freqs = np.linspace(1e9, 3e9, int(rng.integers(1, 4)))
            a = oracle.ref_solve(rs, exc.to_c(), freqs, cfg.to_c(), 2, True, 1 << 20)
            b = oracle.port_solve(ps, exc.to_c(), freqs, cfg.to_c(), True, 1 << 20)
            assert a["values"].tobytes() == b["values"].tobytes()
            assert a["contributions"].tobytes() == b["contributions"].tobytes()
            assert np.array_equal(det_stats_vector(a["stats"]), det_stats_vector(b["stats"]))


@pytest.mark.ref
@needs_ref
def test_loader_and_builtins_byte_identical_to_reference():
    """paper_2511_07586_b200.geometry == reference load_scene/builtin_scene."""
    import ctypes as C

    from paper_2511_07586_b200 import _abi as A

    L = oracle.ref()
    for name in M.builtin_scene_names():
        params = {"subdivisions": 2.0} if name in ("sphere", "nested") else {}
        if name == "glass_cube_pec_bottom":
            continue  # the reference's own builtin fails its parity walk
        sd = M.make_builtin_scene(name, params)
        keys = (C.c_char_p * len(params))(*[k.encode() for k in params])
        vals = (C.c_double * len(params))(*params.values())
        h = L.ref_scene_builtin(name.encode(), keys, vals, len(params))
        assert h
        nv, nt, nm = C.c_uint32(), C.c_uint32(), C.c_uint32()
        L.ref_scene_sizes(h, C.byref(nv), C.byref(nt), C.byref(nm))
        xyz = np.zeros((nv.value, 3))
        tris = np.zeros(nt.value, dtype=A.TRIANGLE_DTYPE)
        mats = np.zeros(nm.value, dtype=A.MATERIAL_DTYPE)
        b5 = np.zeros(5)
        L.ref_scene_export(h, dp(xyz), tris.ctypes.data, mats.ctypes.data, dp(b5))
        L.ref_scene_free(h)
        assert xyz.tobytes() == sd.vertices.tobytes()
        assert tris.tobytes() == sd.triangles.tobytes()
        assert mats.tobytes() == sd.materials.tobytes()
        assert b5.tobytes() == np.r_[sd.bounding_center, sd.bounding_radius, sd.diameter].tobytes()
    # the config generators load in the reference loader too (parity walk etc.)
    from paper_2511_07586_b200.geometry import airframe, scene_to_text

    small_airframe = scene_to_text(airframe(6_000, seed=5, dielectric_skin=True)[0])
    for obj, mm in [M.dihedral_grid(0.5, 8), M.coated_sphere(subdivisions=2, lossless=True),
                    small_airframe]:
        h = L.ref_scene_load(obj.encode(), mm.encode())
        assert h, L.ref_last_error()
        L.ref_scene_free(h)
