"""GPU deterministic SBR solver (solver_det.cpp:30-174)
against the C restatement (oracle/mcsbr_oracle.c orc_solve, pinned bit for bit
to the reference by tests/test_oracle_pins.py::test_solve_golden).

Deterministic, so stricter than the Monte Carlo parity: every contribution
record (currents, optical path, exit point, bounce, cell << 24 | event key)
and every counter, including the reference's stack accounting, is bit-exact;
only the phasor sums differ, by summation order (tolerance 1e-12 of the
largest channel magnitude)."""
import numpy as np
import pytest

import oracle
import paper_2511_07586_b200 as M
from tests.helpers import contribs_identical, det_cases, det_stats_vector, sort_contribs

pytestmark = pytest.mark.gpu

CASES = det_cases()


def _port(sd, exc, freqs, cfg):
    return oracle.port_solve(oracle.port_scene(sd), exc.to_c(), np.asarray(freqs, float), cfg.to_c(),
                             True, 1 << 21)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_solve_matches_oracle(case):
    name, sd, exc, freqs, cfg = case
    want = _port(sd, exc, freqs, cfg)
    col = []
    got = M.solve(M.Scene(sd), exc, freqs, cfg, contributions_out=col)
    assert got.sweep.solver == "deterministic"
    # contributions: bit-exact, same keys (cell << 24 | event_seq)
    a, b = sort_contribs(col[0]), sort_contribs(want["contributions"])
    assert len(a) == len(b) and len(a) > 0
    assert contribs_identical(a, b)
    # counters incl. the stack accounting (max over blocks of sum over rays)
    st = got.stats
    ws = want["stats"]
    assert (st.rays_launched, st.segments_traced, st.contributions, st.grazing_kills, st.cap_kills) == \
        (ws.rays_launched, ws.segments_traced, ws.contributions, ws.grazing_kills, ws.cap_kills)
    assert st.rays_per_bounce == list(ws.rays_per_bounce[:ws.n_rounds])
    assert st.peak_live_state_bytes == ws.peak_live_state_bytes
    assert st.forced_stack_bytes == ws.forced_stack_bytes
    assert st.state_bytes_per_ray == 192 and st.device_stack_bytes > 0
    # phasor sums: summation order only
    scale = np.abs(want["values"]).max()
    assert np.abs(got.sweep.values - want["values"]).max() <= 1e-12 * scale


def test_solve_stats_vector_matches_golden():
    """The GPU's counters equal the reference's own (tests/golden/det.npz)."""
    import os

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "det.npz"))
    from paper_2511_07586_b200 import _abi as A

    for name, sd, exc, freqs, cfg in CASES:
        r = M.solve(M.Scene(sd), exc, freqs, cfg)
        st = A.Stats()
        s = r.stats
        st.rays_launched, st.segments_traced, st.contributions = s.rays_launched, s.segments_traced, s.contributions
        st.grazing_kills, st.cap_kills = s.grazing_kills, s.cap_kills
        st.peak_live_state_bytes, st.forced_stack_bytes = s.peak_live_state_bytes, s.forced_stack_bytes
        st.state_bytes_per_ray, st.n_rounds = s.state_bytes_per_ray, len(s.rays_per_bounce)
        for i, v in enumerate(s.rays_per_bounce):
            st.rays_per_bounce[i] = v
        assert np.array_equal(det_stats_vector(st), g[f"{name}_stats"]), name
        scale = np.abs(g[f"{name}_values"]).max()
        assert np.abs(r.sweep.values - g[f"{name}_values"]).max() <= 1e-12 * scale


def test_det_config_validation_mirrors_reference():
    sd = M.make_builtin_scene("sphere", {"subdivisions": 1})
    s = M.Scene(sd)
    exc = M.monostatic_excitation(0.0, 0.0)
    for cfg, msg in [(M.DetConfig(rays_per_wavelength=0), "rays_per_wavelength must be > 0"),
                     (M.DetConfig(max_bounce=0), "max_bounce must be >= 1"),
                     (M.DetConfig(amplitude_cutoff=-1), "amplitude_cutoff must be >= 0"),
                     (M.DetConfig(block_size=0), "block_size must be >= 1")]:
        with pytest.raises(ValueError, match=msg):
            M.solve(s, exc, [1e9], cfg)
    with pytest.raises(ValueError, match="empty frequency list"):
        M.solve(s, exc, [], M.DetConfig())
    # max_bounce = 1 is valid for the deterministic solver (not for MC)
    r = M.solve(s, exc, [1e9], M.DetConfig(rays_per_wavelength=4, max_bounce=1))
    assert r.stats.cap_kills > 0 and len(r.stats.rays_per_bounce) == 1


def test_det_vs_mc_on_dihedral():
    """Deterministic and Monte Carlo estimates of the same PEC dihedral agree
    (midpoint vs jittered sampling of one aperture): within 0.5 dB."""
    obj, mm = M.dihedral_grid(0.5, 32)
    s = M.Scene(M.load_scene(obj, mm))
    exc = M.monostatic_excitation(90.0, 45.0 + 10.0)
    d = M.solve(s, exc, [10e9], M.DetConfig(rays_per_wavelength=30, max_bounce=4)).sweep.values
    m = M.estimate(s, exc, [10e9], M.McConfig(strata_per_wavelength=20, samples_per_stratum=4,
                                              max_bounce=4, seed=2)).sweep.values
    db = lambda v: 20 * np.log10(np.abs(v[M.VV, 0]))
    assert abs(db(d) - db(m)) < 0.5


def test_det_lossy_zero_loss_equals_lossless():
    """The lossy (complex-index) instantiation with Im(eps) = 0 reproduces the
    lossless deterministic result."""
    obj, mm = M.coated_sphere(subdivisions=2, lossless=True)
    sd = M.load_scene(obj, mm)
    exc = M.monostatic_excitation(90.0, 0.0)
    cfg = M.DetConfig(rays_per_wavelength=5, max_bounce=10, amplitude_cutoff=0.02)
    a = M.solve(M.Scene(sd), exc, [3e9], cfg)
    sd.eps_imag = np.zeros(len(sd.materials))
    b = M.solve(M.Scene(sd), exc, [3e9], cfg)
    assert a.stats.contributions == b.stats.contributions
    assert np.abs(a.sweep.values - b.sweep.values).max() <= 1e-9 * np.abs(a.sweep.values).max()
