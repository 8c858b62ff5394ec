"""Runner integration: the reference's own runner,
config parser and artifact writers (proj/src/runner.cpp, config.cpp) linked
with the product's drop-in solver TU (paper_2511_07586_b200/dropin/
solver_b200.cpp) instead of proj/src/solver_mc.cpp + solver_det.cpp, so every
estimate()/solve() runs on the GPU.  Each command is run twice on the same
config -- CPU reference vs drop-in -- and the artifacts are compared:

* byte-identical: every comment/header line, config hash, seed, solver
  names, frequency / angle / range columns, stats.json and manifest.json
  (except wall_ms and the output directory), bench.csv counters and the
  deterministic solver's stack accounting;
* numerically: complex sweep values to 1e-9 of each channel's peak (the GPU
  sums the same contributions in a different order), dB products to 1e-6 dB
  above the -120 dB floor, ISAR PGM pixels within one grey level.
"""
import json
import os
import re

import numpy as np
import pytest

import oracle
from tests.helpers import contribs_identical

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (oracle.have_ref() and oracle.have_dropin()),
                                 reason="oracle/_ref reference + drop-in libraries not built")]

GLASS = {"builtin": "glass_cube", "params": {"eps_r": 2.25, "size_m": 1.0}}


def _cfg(**sections):
    base = {"scene": GLASS, "source": {"theta_deg": 20.0, "phi_deg": 40.0},
            "frequency": {"start_hz": 1e9, "stop_hz": 3e9, "count": 9},
            "solver": {"type": "mc", "mc": {"strata_per_wavelength": 5, "samples_per_stratum": 2,
                                            "roulette": {"enabled": True, "q": 0.4}}},
            "seed": 11}
    base.update(sections)
    return json.dumps(base)


def _run(tmp_path, command, cfg, seed=None):
    a, b = str(tmp_path / "cpu"), str(tmp_path / "gpu")
    assert oracle.ref_run_command(command, cfg, a, 4, seed) == 0
    assert oracle.ref_run_command(command, cfg, b, 4, seed, lib=oracle.dropin()) == 0
    return a, b


def _read(d, name, mode="r"):
    with open(os.path.join(d, name), mode) as f:
        return f.read()


def _split_csv(text):
    head = [l for l in text.splitlines() if l.startswith("#") or not l[:1].isdigit() and l[:1] != "-"]
    rows = [l.split(",") for l in text.splitlines() if l not in head]
    return head, rows


def _compare_values(ra, rb, key_cols, rel=1e-9):
    assert len(ra) == len(rb) and len(ra) > 0
    a = np.array([[float(x) for x in r] for r in ra])
    b = np.array([[float(x) for x in r] for r in rb])
    assert [r[:key_cols] for r in ra] == [r[:key_cols] for r in rb]  # keys byte-identical
    va, vb = a[:, key_cols:], b[:, key_cols:]
    for ch in range(0, va.shape[1], 2):
        scale = max(np.abs(va[:, ch:ch + 2]).max(), 1e-300)
        assert np.abs(va[:, ch:ch + 2] - vb[:, ch:ch + 2]).max() <= rel * scale


def _strip_wall(text, d):
    out = []
    for l in text.splitlines():
        if '"wall_ms"' in l:
            continue
        out.append(l.replace(d, "<out>"))
    return "\n".join(out)


def _compare_json(a, b, name):
    ta, tb = _read(a, name), _read(b, name)
    assert _strip_wall(ta, a) == _strip_wall(tb, b)
    ja, jb = json.loads(ta), json.loads(tb)
    assert ja.keys() == jb.keys()


def test_sweep_command(tmp_path):
    a, b = _run(tmp_path, "sweep", _cfg())
    ha, ra = _split_csv(_read(a, "sweep.csv"))
    hb, rb = _split_csv(_read(b, "sweep.csv"))
    assert ha == hb and "# solver=mc" in ha and "# seed=11" in ha
    _compare_values(ra, rb, 1)
    _compare_json(a, b, "stats.json")
    _compare_json(a, b, "manifest.json")


def test_sweep_deterministic_and_seed_override(tmp_path):
    cfg = _cfg(solver={"type": "deterministic",
                       "deterministic": {"rays_per_wavelength": 6, "max_bounce": 7,
                                         "amplitude_cutoff": 0.05}})
    a, b = _run(tmp_path, "sweep", cfg, seed=5)
    ha, ra = _split_csv(_read(a, "sweep.csv"))
    hb, rb = _split_csv(_read(b, "sweep.csv"))
    assert ha == hb and "# solver=deterministic" in ha
    _compare_values(ra, rb, 1, rel=1e-12)
    _compare_json(a, b, "stats.json")  # incl. peak_live_state_bytes / forced_stack_bytes
    _compare_json(a, b, "manifest.json")


def test_range_profile_command(tmp_path):
    cfg = _cfg(frequency={"start_hz": 8e9, "stop_hz": 12e9, "count": 32},
               scene={"builtin": "dihedral", "params": {}},
               source={"theta_deg": 90.0, "phi_deg": 45.0},
               solver={"type": "mc", "mc": {"strata_per_wavelength": 3, "samples_per_stratum": 1}},
               profile={"window": "hann", "zero_pad": 4})
    a, b = _run(tmp_path, "range-profile", cfg)
    ha, ra = _split_csv(_read(a, "profile.csv"))
    hb, rb = _split_csv(_read(b, "profile.csv"))
    assert ha == hb
    assert [r[0] for r in ra] == [r[0] for r in rb]  # range axis
    da = np.array([float(r[1]) for r in ra])
    db = np.array([float(r[1]) for r in rb])
    keep = da > -120.0
    assert np.abs(da[keep] - db[keep]).max() < 1e-6
    _compare_json(a, b, "manifest.json")


def test_angle_sweep_command(tmp_path):
    cfg = _cfg(angle_sweep={"theta_start_deg": 0.0, "theta_stop_deg": 60.0, "count": 4, "phi_deg": 15.0},
               frequency={"start_hz": 2e9, "stop_hz": 3e9, "count": 3})
    a, b = _run(tmp_path, "angle-sweep", cfg)
    ha, ra = _split_csv(_read(a, "angle_sweep.csv"))
    hb, rb = _split_csv(_read(b, "angle_sweep.csv"))
    assert ha == hb
    _compare_values(ra, rb, 2)
    _compare_json(a, b, "manifest.json")


def test_isar_command(tmp_path):
    cfg = _cfg(scene={"builtin": "airplane_stub", "params": {}},
               frequency={"start_hz": 9.5e9, "stop_hz": 10.5e9, "count": 16},
               solver={"type": "mc", "mc": {"strata_per_wavelength": 1.5, "samples_per_stratum": 1}},
               isar={"theta_deg": 80.0, "azimuth_start_deg": -3.0, "azimuth_stop_deg": 3.0,
                     "angle_count": 8, "zero_pad": 2, "dynamic_floor_db": -40.0})
    a, b = _run(tmp_path, "isar", cfg)
    ta, tb = _read(a, "isar.csv").splitlines(), _read(b, "isar.csv").splitlines()
    assert len(ta) == len(tb)
    assert ta[:2] == tb[:2] and ta[3:5] == tb[3:5]  # kind, hash, column header, cross-range axis
    ga = np.array([[float(x) for x in l.split(",")] for l in ta[5:]])
    gb = np.array([[float(x) for x in l.split(",")] for l in tb[5:]])
    assert np.array_equal(ga[:, 0], gb[:, 0])  # down-range axis
    assert np.abs(ga[:, 1:] - gb[:, 1:]).max() < 1e-6
    pa, pb = _read(a, "isar.pgm", "rb"), _read(b, "isar.pgm", "rb")
    ha, hb = pa.index(b"255\n") + 4, pb.index(b"255\n") + 4
    la, lb = pa[:ha].split(b"\n"), pb[:hb].split(b"\n")
    assert la[-3:] == lb[-3:]  # size + maxval
    # comment lines carry full-precision doubles (dB window, extents): the
    # sums agree to ~1e-15, so their printed digits may differ in the last place
    num = re.compile(rb"-?\d+\.?\d*(?:e[-+]?\d+)?")
    for ca, cb in zip(la[1:-3], lb[1:-3]):
        assert num.sub(b"#", ca) == num.sub(b"#", cb)
        assert np.allclose([float(x) for x in num.findall(ca)], [float(x) for x in num.findall(cb)],
                           rtol=1e-9, atol=1e-9)
    xa = np.frombuffer(pa[ha:], np.uint8).astype(int)
    xb = np.frombuffer(pb[hb:], np.uint8).astype(int)
    assert len(xa) == len(xb)
    assert np.abs(xa - xb).max() <= 1
    _compare_json(a, b, "manifest.json")


def test_convergence_and_bench_commands(tmp_path):
    cfg = _cfg(frequency={"start_hz": 2e9, "stop_hz": 3e9, "count": 3},
               solver={"type": "mc",
                       "mc": {"strata_per_wavelength": 3, "samples_per_stratum": 1},
                       "deterministic": {"rays_per_wavelength": 5, "max_bounce": 6}},
               convergence={"densities": [2.0, 3.0], "samples_per_stratum": [1, 2], "seed_count": 2,
                            "reference_rays_per_wavelength": 6.0},
               bench={"repeats": 1, "warmups": 0})
    a, b = _run(tmp_path, "convergence", cfg)
    ha, ra = _split_csv(_read(a, "convergence.csv"))
    hb, rb = _split_csv(_read(b, "convergence.csv"))
    assert ha == hb
    assert [r[:4] for r in ra] == [r[:4] for r in rb]
    ea = np.array([[float(x) for x in r[4:]] for r in ra])
    eb = np.array([[float(x) for x in r[4:]] for r in rb])
    assert np.abs(ea - eb).max() < 1e-6
    a, b = _run(tmp_path / "bench", "bench", cfg)
    la, lb = _read(a, "bench.csv").splitlines(), _read(b, "bench.csv").splitlines()
    assert la[:4] == lb[:4]
    for x, y in zip(la[4:], lb[4:]):
        fx, fy = x.split(","), y.split(",")
        assert fx[0] == fy[0] and fx[3:] == fy[3:]  # solver, stack MiB, rays, segments, contributions


def test_dropin_contribution_order_matches_reference():
    """estimate()/solve() through the drop-in return the contributions in the
    reference's own emission order (block, wavefront round, entry)."""
    import paper_2511_07586_b200 as M

    sd = M.make_builtin_scene("glass_cube", {"eps_r": 2.25, "size_m": 1.0})
    exc = M.monostatic_excitation(20.0, 40.0).to_c()
    freqs = np.linspace(1e9, 3e9, 4)
    cfg = M.McConfig(strata_per_wavelength=6, samples_per_stratum=2, block_size=700,
                     roulette=M.RouletteConfig(enabled=True)).to_c()
    L = oracle.dropin()
    h = L.ref_scene_from_arrays(oracle.dp(sd.vertices), len(sd.vertices), sd.triangles.ctypes.data,
                                len(sd.triangles), sd.materials.ctypes.data, len(sd.materials))
    dh = oracle._Handle(L, h, L.ref_scene_free)
    got = oracle._estimate(L.ref_estimate, L.ref_last_error, dh.h, exc, freqs, cfg, True, 1 << 20, 4)
    want = oracle.ref_estimate(oracle.ref_scene(sd), exc, freqs, cfg, 4, True, 1 << 20)
    assert contribs_identical(got["contributions"], want["contributions"])
    scale = np.abs(want["values"]).max()
    assert np.abs(got["values"] - want["values"]).max() <= 1e-9 * scale
    dcfg = M.DetConfig(rays_per_wavelength=5, max_bounce=6, amplitude_cutoff=0.05, block_size=500).to_c()
    got = oracle._estimate(L.ref_solve, L.ref_last_error, dh.h, exc, freqs, dcfg, True, 1 << 20, 4)
    want = oracle.ref_solve(oracle.ref_scene(sd), exc, freqs, dcfg, 4, True, 1 << 20)
    assert contribs_identical(got["contributions"], want["contributions"])


@pytest.mark.parametrize("solver", ["mc", "deterministic"])
def test_dropin_artifacts_byte_identical_across_reruns_and_workers(tmp_path, solver):
    """The reference's reproducibility promise (runner.hpp:2-5,
    tests/test_cli_config.cpp:95-123: sweep.csv byte-identical across reruns
    and worker counts) through the drop-in: its solvers sum exactly
    (MCSBR_REDUCE_EXACT), so the GPU artifacts are byte-identical too."""
    cfg = _cfg() if solver == "mc" else _cfg(
        solver={"type": "deterministic", "deterministic": {"rays_per_wavelength": 6, "max_bounce": 7}})
    outs = []
    for k, workers in enumerate((4, 4, 1, 3)):
        d = str(tmp_path / f"run{k}")
        assert oracle.ref_run_command("sweep", cfg, d, workers, None, lib=oracle.dropin()) == 0
        outs.append(_read(d, "sweep.csv", "rb"))
    assert all(o == outs[0] for o in outs[1:])
