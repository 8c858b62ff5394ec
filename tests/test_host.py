"""CPU: host logic and the C-ABI library (no compute calls without a GPU)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2511_07586_b200 as M
from paper_2511_07586_b200 import _abi as A

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "mcsbr_gpu.h")).read()
    return sorted(set(re.findall(r"MCSBR_API\s+[\w\s\*]+?\b(mcsbr_gpu_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = C.CDLL(A.LIB_PATH)
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    # and the Python binding covers exactly the header
    assert sorted(A.SIGNATURES) == names


def test_library_cpu_entry_points():
    """Host-only entry points work without a device; compute ones fail loudly."""
    L = A.lib()
    assert L.mcsbr_gpu_abi_version() == 3
    det = A.DetConfigC()
    L.mcsbr_gpu_default_det_config(C.byref(det))
    assert (det.rays_per_wavelength, det.max_bounce, det.amplitude_cutoff, det.block_size) == (20.0, 9, 0.0, 8192)
    assert L.mcsbr_gpu_validate_det_config(C.byref(det)) == 0
    det.max_bounce = 0
    assert L.mcsbr_gpu_validate_det_config(C.byref(det)) == A.MCSBR_EINVAL
    assert b"det: max_bounce must be >= 1" in L.mcsbr_gpu_last_error()
    cfg = A.McConfigC()
    L.mcsbr_gpu_default_config(C.byref(cfg))
    assert cfg.strata_per_wavelength == 10.0 and cfg.samples_per_stratum == 16
    assert cfg.max_bounce == 9 and cfg.p_min == 0.05 and cfg.block_size == 8192
    assert L.mcsbr_gpu_validate_config(C.byref(cfg)) == 0
    cfg.max_bounce = 1
    assert L.mcsbr_gpu_validate_config(C.byref(cfg)) == A.MCSBR_EINVAL
    assert b"max_bounce must be >= 2" in L.mcsbr_gpu_last_error()
    # finalize: j k0 / (2 sqrt(pi)) applied, [n][nf][4] -> [n][4][nf]
    raw = np.arange(16, dtype=np.float64)  # n=1, nf=2, 4 ch complex
    f = np.array([1e9, 2e9])
    out = np.zeros(16)
    assert L.mcsbr_gpu_finalize(raw.ctypes.data_as(C.POINTER(C.c_double)), 1,
                                f.ctypes.data_as(C.POINTER(C.c_double)), 2,
                                out.ctypes.data_as(C.POINTER(C.c_double))) == 0
    k0 = 2 * np.pi * f / 299792458.0
    pre = 1j * k0 / (2 * np.sqrt(np.pi))
    sums = (raw[0::2] + 1j * raw[1::2]).reshape(2, 4)  # [nf][ch]
    want = (pre[:, None] * sums).T  # [ch][nf]
    got = (out[0::2] + 1j * out[1::2]).reshape(4, 2)
    assert np.allclose(got, want, rtol=1e-15)


def test_scene_loader_errors():
    """tests/test_geometry.cpp:80-104 error paths."""
    mm = ('{"materials": {"air": {"eps_r": 1.0}, "glass": {"eps_r": 1.5}},'
          ' "regions": {"cube": {"front": "air", "back": "glass"}}}')
    with pytest.raises(M.SceneError):
        M.load_scene("v 0 0 0\nv 1 0 0\nv 0 1 0\ng cube\nf 1 2 3\n",
                     '{"materials": {"air": {"eps_r": 1.0}},'
                     ' "regions": {"cube": {"front": "air", "back": "unobtainium"}}}')
    with pytest.raises(M.SceneError, match="degenerate triangle"):
        M.load_scene("v 0 0 0\nv 1 0 0\nv 2 0 0\ng cube\nf 1 2 3\n", mm)
    with pytest.raises(M.SceneError, match="non-manifold"):
        M.load_scene("v 0 0 0\nv 1 0 0\nv 0 1 0\ng cube\nf 1 2 3\n", mm)
    with pytest.raises(M.SceneError, match="no region entry"):
        M.load_scene("v 0 0 0\nv 1 0 0\nv 0 1 0\ng mystery\nf 1 2 3\n", mm)
    with pytest.raises(M.SceneError, match="scene has no triangles"):
        M.load_scene("v 0 0 0\n", mm)


def test_obj_parser_features():
    """Quads / polygons fan-triangulate, negative and v/vt/vn indices resolve."""
    text = "v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\no sq\nf -4/1/1 -3//2 -2 -1\n"
    mm = M.geometry.materials_json('    "sq": {"front": "air", "back": "metal"}')
    sd = M.load_scene(text, mm)
    assert len(sd.triangles) == 2
    assert list(sd.triangles[1][["v0", "v1", "v2"]]) == [0, 2, 3]
    assert np.allclose(sd.triangles["normal"], [[0, 0, 1], [0, 0, 1]])
    assert sd.triangles["exterior_facing"].all()


def test_material_ids_follow_sorted_keys():
    """nlohmann::json objects iterate sorted: ambient first, then sorted names."""
    sd = M.make_builtin_scene("nested", {"subdivisions": 1})
    assert sd.material_names == ["air", "glass_inner", "glass_outer", "metal"]
    ext = sd.triangles["exterior_facing"].astype(bool)
    assert ext.sum() == 12  # only the outer cube borders air (test_geometry.cpp:72-78)


def test_generators_sizes():
    obj, mm = M.dihedral_grid(0.5, 64)
    sd = M.load_scene(obj, mm)
    assert sd.n_triangles == 2 * 2 * 64 * 64
    # normals point into the opening (+x+y quadrant)
    n = sd.triangles["normal"]
    assert np.all((n[:, 0] > 0.99) | (n[:, 1] > 0.99))
    obj, mm = M.coated_sphere(subdivisions=5, lossless=False)
    sd = M.load_scene(obj, mm)
    assert sd.n_triangles == 3 * 20480
    assert sd.eps_imag is not None and sd.eps_imag.max() == pytest.approx(0.1)


def test_airframe_generator_c4_c5():
    """BASELINE configs 4/5 geometry: triangle budgets, closed consistently
    oriented dielectric skins (the loader's parity walk), outward normals."""
    from paper_2511_07586_b200.geometry import airframe

    sd, info = airframe(200_000, seed=4)
    assert abs(info["triangles"] - 200_000) < 5_000
    assert sd.material_names == ["air", "metal"] and sd.eps_imag is None
    assert 6.0 < sd.bounding_radius < 6.5  # 12 m fuselage dominates
    sd5, info5 = airframe(1_000_000, seed=5, dielectric_skin=True)
    assert abs(info5["triangles"] - 1_000_000) < 25_000
    assert sd5.material_names == ["air", "metal", "skin_in", "skin_out"]
    assert np.allclose(sd5.eps_imag, [0, 0, 1.0, 0.05])
    # deterministic in the seed, different across seeds
    a, _ = airframe(20_000, seed=4)
    b, _ = airframe(20_000, seed=4)
    c, _ = airframe(20_000, seed=5)
    assert a.vertices.tobytes() == b.vertices.tobytes()
    assert a.vertices.tobytes() != c.vertices.tobytes()


def test_scene_text_roundtrip():
    """scene_to_text output reloads through the (reference-compatible) loader
    to the identical scene."""
    from paper_2511_07586_b200.geometry import airframe, scene_to_text

    sd, _ = airframe(6_000, seed=5, dielectric_skin=True)
    obj, mm = scene_to_text(sd)
    sd2 = M.load_scene(obj, mm)
    assert sd2.vertices.tobytes() == sd.vertices.tobytes()
    assert sd2.material_names == sd.material_names
    key = lambda t: np.lexsort((t["v2"], t["v1"], t["v0"]))  # noqa: E731
    t1, t2 = sd.triangles[key(sd.triangles)], sd2.triangles[key(sd2.triangles)]
    assert t1.tobytes() == t2.tobytes()
    assert np.array_equal(sd2.eps_imag, sd.eps_imag)


def test_excitation_bases():
    """solver_common.cpp:15-49: V = theta_hat, H = phi_hat, k_inc = -r_hat."""
    e = M.monostatic_excitation(90.0, 0.0)
    assert np.allclose(e.k_inc, [-1, 0, 0]) and np.allclose(e.k_scatter, [1, 0, 0])
    assert np.allclose(e.pol_v, [0, 0, -1], atol=1e-15) and np.allclose(e.pol_h, [0, 1, 0])
    b = M.bistatic_excitation(90.0, 0.0, 0.0, 0.0)
    assert np.allclose(b.k_scatter, [0, 0, 1])


def _limbs(x: float) -> list:
    """The 192-bit fixed-point pattern (LSB 2^-120) of x as 4 limbs of 48 bits
    (csrc/fixedpoint.cuh), from Python integers."""
    from fractions import Fraction

    v = int(Fraction(x) * (1 << 120))  # exact, truncated toward zero
    v &= (1 << 192) - 1  # two's complement
    return [(v >> (48 * i)) & ((1 << 48) - 1) for i in range(4)]


def test_exact_limbs_finalize_on_host():
    """mcsbr_gpu_finalize_exact: limbs summed over 'ranks' (plain int64 adds,
    as an integer all-reduce does) decode to the exact sum of the terms and
    finalize like mcsbr_gpu_finalize."""
    import ctypes as C

    import numpy as np

    from paper_2511_07586_b200 import _abi as A

    rng = np.random.default_rng(7)
    n, nf = 2, 3
    terms = rng.normal(size=(5, n * nf * 8)) * 10.0 ** rng.integers(-9, 4, size=(5, n * nf * 8))
    terms[0, :4] = [0.0, -0.0, 1.5, -2.75]
    limbs = np.zeros((n * nf * 8, 4), dtype=np.int64)
    for rank in range(5):
        limbs += np.array([_limbs(float(x)) for x in terms[rank]], dtype=np.int64)
    freqs = np.array([1e9, 2e9, 3.5e9])
    got = np.zeros((n, 4, nf, 2))
    L = A.lib()
    A.check(L.mcsbr_gpu_finalize_exact(np.ascontiguousarray(limbs).ctypes.data_as(C.POINTER(C.c_int64)), n,
                                       freqs.ctypes.data_as(C.POINTER(C.c_double)), nf,
                                       got.ctypes.data_as(C.POINTER(C.c_double))))
    raw = np.ascontiguousarray(terms.sum(axis=0))
    want = np.zeros_like(got)
    A.check(L.mcsbr_gpu_finalize(raw.ctypes.data_as(C.POINTER(C.c_double)), n,
                                 freqs.ctypes.data_as(C.POINTER(C.c_double)), nf,
                                 want.ctypes.data_as(C.POINTER(C.c_double))))
    assert np.allclose(got, want, rtol=1e-13, atol=1e-30)
    # a single exact value decodes exactly
    one = np.zeros((n * nf * 8, 4), dtype=np.int64)
    one[0] = _limbs(-2.75)
    out = np.zeros((n, 4, nf, 2))
    A.check(L.mcsbr_gpu_finalize_exact(one.ctypes.data_as(C.POINTER(C.c_int64)), n,
                                       freqs.ctypes.data_as(C.POINTER(C.c_double)), nf,
                                       out.ctypes.data_as(C.POINTER(C.c_double))))
    k0 = 2 * np.pi * freqs[0] / 299792458.0
    assert out[0, 0, 0, 1] == -2.75 * (1.0 * k0 / (2.0 * np.sqrt(np.pi)))
