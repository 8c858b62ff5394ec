"""Generate the golden vectors in tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libmcsbr_ref.so, compiled from
/root/reference/proj/src by `make -C oracle ref`):

    python tests/golden/make_golden.py

Outputs (committed; the GPU box and the CPU test suite only read them):
  rng.npz        counter_hash / counter_uniform known answers (rng.hpp:29-44)
  em.npz         fresnel / sp_basis / interface_transform / branch_outcomes /
                 meca_currents on seeded random inputs (em_math.cpp, path_engine.cpp,
                 farfield.cpp)
  intersect.npz  Scene::intersect on seeded random rays, 3 builtin scenes
  estimate.npz   full estimate() sweeps (values, stats, contribution digests)
  det.npz        full solve() (deterministic SBR) sweeps, same fields + stack accounting
                 for the parity cases of tests/helpers.py
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2511_07586_b200 as M  # noqa: E402
from paper_2511_07586_b200 import _abi as A  # noqa: E402

PURPOSES = [0x101, 0x102, 0x201, 0x202]


def rng_kat(L):
    seeds = [0, 1, 2, 99, (1 << 63) + 5]
    strata = [0, 1, 7, 12345, (1 << 32) - 1]
    samples = [0, 1, 15]
    bounces = [0, 1, 2, 8]
    keys, h, u = [], [], []
    for s in seeds:
        for st in strata:
            for sa in samples:
                for b in bounces:
                    for p in PURPOSES:
                        keys.append((s, st, sa, b, p))
                        h.append(L.ref_counter_hash(s, st, sa, b, p))
                        u.append(L.ref_counter_uniform(s, st, sa, b, p))
    return {"keys": np.array(keys, dtype=np.uint64), "hash": np.array(h, dtype=np.uint64),
            "uniform": np.array(u)}


def unit(rng, n):
    v = rng.normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def incidences(rng, n):
    d = unit(rng, n)
    nr = unit(rng, n)
    dn = np.sum(d * nr, axis=1)
    keep = np.abs(dn) > 1e-3
    d, nr, dn = d[keep], nr[keep], dn[keep]
    nr[dn > 0] *= -1
    return d, nr


def em_vectors(L):
    rng = np.random.default_rng(100)
    dp = oracle.dp
    out = {}
    # fresnel: random + TIR + normal incidence + index matched
    n1 = rng.uniform(1.0, 3.0, 500)
    n2 = rng.uniform(1.0, 3.0, 500)
    ci = rng.uniform(0.01, 1.0, 500)
    n1 = np.r_[n1, 1.0, 1.5, 1.4, 1.0, 2.0]
    n2 = np.r_[n2, 1.5, 1.0, 1.4, 1.0, 1.0]
    ci = np.r_[ci, 1.0, 0.5, 0.7, 0.3, 0.999]
    res = np.zeros((len(n1), 11))
    for i in range(len(n1)):
        assert L.ref_fresnel(n1[i], n2[i], ci[i], dp(res[i])) == 0
    out["fresnel_in"] = np.stack([n1, n2, ci], 1)
    out["fresnel_out"] = res
    # sp_basis incl. the normal-incidence fallbacks
    d, nr = incidences(rng, 400)
    d = np.r_[d, [[0, 0, -1.0]], [[1, 0, 0.0]], [[0.0, -1.0, 0.0]]]
    nr = np.r_[nr, [[0, 0, 1.0]], [[-1, 0, 0.0]], [[0.0, 1.0, 0.0]]]
    nn = np.stack([rng.uniform(1, 2.5, len(d)), rng.uniform(1, 2.5, len(d))], 1)
    bas = np.zeros((len(d), 18))
    for i in range(len(d)):
        assert L.ref_sp_basis(dp(np.ascontiguousarray(d[i])), dp(np.ascontiguousarray(nr[i])),
                              nn[i, 0], nn[i, 1], dp(bas[i])) == 0
    out["basis_in"] = np.concatenate([d, nr, nn], 1)
    out["basis_out"] = bas
    # interface_transform of random transverse complex fields, both branches
    co = np.zeros((len(d), 11))
    e6 = np.zeros((len(d), 6))
    tr = np.zeros((len(d), 2, 6))
    for i in range(len(d)):
        cos_i = -float(np.dot(d[i], nr[i]))
        L.ref_fresnel(nn[i, 0], nn[i, 1], cos_i, dp(co[i]))
        s_hat, p_in = bas[i, 0:3], bas[i, 3:6]
        a, b = rng.normal(size=2) + 1j * rng.normal(size=2)
        e = a * s_hat + b * p_in
        e6[i] = np.stack([e.real, e.imag], 1).reshape(-1)
        for br in (0, 1):
            assert L.ref_interface_transform(dp(e6[i]), br, dp(co[i]), dp(bas[i]), dp(tr[i, br])) == 0
    out["transform_coeffs"] = co
    out["transform_e"] = e6
    out["transform_out"] = tr
    # branch_outcomes + meca on random hits (PEC / entering / exiting)
    n = 300
    d, nr = incidences(rng, n)
    st = np.zeros((len(d), 23))
    hit = np.zeros((len(d), 13))
    bo = np.zeros((len(d), 63))
    me = np.zeros((len(d), 2, 12))
    for i in range(len(d)):
        kind = i % 3
        s_hat = np.cross(d[i], [0.3, 0.5, 0.8])
        s_hat /= np.linalg.norm(s_hat)
        p_hat = np.cross(d[i], s_hat)
        ea = (rng.normal() + 1j * rng.normal()) * s_hat + (rng.normal() + 1j * rng.normal()) * p_hat
        eb = (rng.normal() + 1j * rng.normal()) * s_hat + (rng.normal() + 1j * rng.normal()) * p_hat
        n_med = 1.0 if kind != 2 else rng.uniform(1.2, 2.5)
        st[i, 0:3] = rng.normal(size=3)
        st[i, 3:6] = d[i]
        st[i, 6:12] = np.stack([ea.real, ea.imag], 1).reshape(-1)
        st[i, 12:18] = np.stack([eb.real, eb.imag], 1).reshape(-1)
        st[i, 18:23] = [rng.uniform(0, 5), rng.uniform(0.1, 1), rng.uniform(1, 4), n_med, 1 + i % 5]
        hit[i, 0] = rng.uniform(0.1, 2)
        hit[i, 1:4] = rng.normal(size=3)
        hit[i, 4:7] = nr[i]
        hit[i, 7] = n_med
        hit[i, 8] = 0.0 if kind == 0 else (rng.uniform(1.2, 2.5) if kind == 1 else 1.0)
        hit[i, 9] = 1.0 if kind == 0 else 0.0
        hit[i, 10] = 1.0
        hit[i, 11] = 1.0 if kind != 2 else 0.0
        hit[i, 12] = i
        assert L.ref_branch_outcomes(dp(st[i]), dp(hit[i]), dp(bo[i])) == 0
        for pol in (0, 1):
            assert L.ref_meca_currents(dp(hit[i]), dp(st[i, 6 + 6 * pol:12 + 6 * pol]),
                                       dp(np.ascontiguousarray(d[i])), kind, dp(me[i, pol])) == 0
    out["branch_state"] = st
    out["branch_hit"] = hit
    out["branch_out"] = bo
    out["meca_out"] = me
    return out


def intersect_vectors():
    out = {}
    rng = np.random.default_rng(7)
    for name, params in [("glass_cube", {}), ("nested", {"subdivisions": 2}),
                         ("sphere", {"subdivisions": 3})]:
        sd = M.make_builtin_scene(name, params)
        rs = oracle.ref_scene(sd)
        n = 1500
        o = rng.uniform(-4, 4, (n, 3))
        d = unit(rng, n)
        aim = rng.random(n) < 0.5
        d[aim] = sd.vertices[rng.integers(0, len(sd.vertices), aim.sum())] - o[aim]
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        tmin = np.where(rng.random(n) < 0.5, 0.0, sd.self_intersection_epsilon())
        # ground truth: Scene::intersect_brute_force (geometry.cpp:218-240).  The
        # reference's BVH walk (geometry.cpp:177-216) is also recorded: its
        # unpadded fp64 slab test culls hits lying exactly on a box face (rays
        # aimed at vertices), so it can disagree with its own brute force.
        hb = oracle.intersect("ref", rs, o, d, tmin, 1)
        h = oracle.intersect("ref", rs, o, d, tmin, 0)
        out[f"{name}_o"] = o
        out[f"{name}_d"] = d
        out[f"{name}_tmin"] = tmin
        out[f"{name}_t"] = hb[:, 0]
        out[f"{name}_id"] = hb[:, 12].astype(np.uint32)
        out[f"{name}_bvh_t"] = h[:, 0]
        out[f"{name}_bvh_id"] = h[:, 12].astype(np.uint32)
    return out


def estimate_vectors():
    from tests.helpers import parity_cases

    out = {}
    for name, sd, exc, freqs, cfg in parity_cases():
        rs = oracle.ref_scene(sd)
        r = oracle.ref_estimate(rs, exc.to_c(), np.asarray(freqs, float), cfg.to_c(), 1, True,
                                1 << 21)
        c = r["contributions"]
        c = c[np.argsort(c["order_key"], kind="stable")]
        st = r["stats"]
        out[f"{name}_values"] = r["values"]
        out[f"{name}_stats"] = np.array(
            [st.rays_launched, st.segments_traced, st.contributions, st.grazing_kills, st.cap_kills]
            + list(st.rays_per_bounce[:32]) + list(st.roulette_candidates[:32])
            + list(st.roulette_survivors[:32]), dtype=np.uint64)
        out[f"{name}_contrib_sha256"] = np.frombuffer(hashlib.sha256(c.tobytes()).digest(),
                                                      dtype=np.uint8)
        out[f"{name}_contrib_head"] = c[:64]
    return out


def det_vectors():
    """Deterministic solver (solver_det.cpp:30-174) on the reference."""
    from tests.helpers import det_cases, det_stats_vector

    out = {}
    for name, sd, exc, freqs, cfg in det_cases():
        rs = oracle.ref_scene(sd)
        r = oracle.ref_solve(rs, exc.to_c(), np.asarray(freqs, float), cfg.to_c(), 1, True, 1 << 21)
        c = r["contributions"]
        c = c[np.argsort(c["order_key"], kind="stable")]
        out[f"{name}_values"] = r["values"]
        out[f"{name}_stats"] = det_stats_vector(r["stats"])
        out[f"{name}_contrib_sha256"] = np.frombuffer(hashlib.sha256(c.tobytes()).digest(),
                                                      dtype=np.uint8)
        out[f"{name}_contrib_head"] = c[:64]
    return out


def synthetic_sweeps(rng, freqs, angles, n_pts=5):
    """Point-scatterer sweeps values[a][k] = sum_i A_i e^{-j 2 k (x_i cos t + y_i sin t)}."""
    k = 2 * np.pi * np.asarray(freqs) / 299792458.0
    t = np.radians(angles)
    pts = rng.uniform(-2, 2, size=(n_pts, 2))
    amp = rng.normal(size=n_pts) + 1j * rng.normal(size=n_pts)
    proj = np.cos(t)[:, None] * pts[None, :, 0] + np.sin(t)[:, None] * pts[None, :, 1]  # [a][i]
    return np.einsum("i,aik->ak", amp, np.exp(-2j * k[None, None, :] * proj[:, :, None]))


def signal_vectors(L):
    rng = np.random.default_rng(21)
    dp = oracle.dp
    out = {}
    freqs = np.linspace(9.5e9, 10.5e9, 64)
    for name, vals in [("rand", rng.normal(size=64) + 1j * rng.normal(size=64)),
                       ("pts", synthetic_sweeps(rng, freqs, [0.0])[0])]:
        for hann in (0, 1):
            v = np.ascontiguousarray(vals.astype(np.complex128))
            r = np.zeros(256)
            db = np.zeros(256)
            b = np.zeros(1)
            assert L.ref_range_profile(dp(v.view(np.float64)), dp(freqs), 64, hann, 4, dp(r), dp(db), dp(b)) == 0
            out[f"rp_{name}_{hann}_in"] = v
            out[f"rp_{name}_{hann}_range"] = r
            out[f"rp_{name}_{hann}_db"] = db
            out[f"rp_{name}_{hann}_bin"] = b
    out["rp_freqs"] = freqs
    fi = np.linspace(9.5e9, 10.5e9, 32)
    ang = np.linspace(-3.0, 3.0, 16)
    vals = np.ascontiguousarray(synthetic_sweeps(rng, fi, ang, 6).astype(np.complex128))
    down = np.zeros(128)
    cross = np.zeros(64)
    db = np.zeros(128 * 64)
    pk = np.zeros(1)
    assert L.ref_isar(dp(vals.view(np.float64)), dp(fi), 32, dp(ang), 16, 1, 4, -40.0, dp(down), dp(cross),
                      dp(db), dp(pk)) == 0
    out.update({"isar_in": vals, "isar_freqs": fi, "isar_angles": ang, "isar_down": down,
                "isar_cross": cross, "isar_db": db.reshape(128, 64), "isar_peak": pk})
    return out


def main():
    L = oracle.ref()
    np.savez_compressed(os.path.join(HERE, "signal.npz"), **signal_vectors(L))
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **rng_kat(L))
    np.savez_compressed(os.path.join(HERE, "em.npz"), **em_vectors(L))
    np.savez_compressed(os.path.join(HERE, "intersect.npz"), **intersect_vectors())
    np.savez_compressed(os.path.join(HERE, "estimate.npz"), **estimate_vectors())
    np.savez_compressed(os.path.join(HERE, "det.npz"), **det_vectors())
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
