"""GPU radar products against the reference's output
(tests/golden/signal.npz) and the numpy restatement (oracle/signal_ref.py)."""
import os

import numpy as np
import pytest

import paper_2511_07586_b200 as M
from paper_2511_07586_b200 import signal as SIG

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "signal.npz")


def _db_close(a, b, tol=1e-6, span=150.0):
    keep = b > b.max() - span
    return np.max(np.abs(a[keep] - b[keep])) <= tol


def _sweep(freqs, vals):
    v = np.zeros((4, len(freqs)), dtype=complex)
    v[M.VV] = vals
    return M.SweepResult(frequencies=np.asarray(freqs), values=v)


def test_range_profile_matches_reference():
    g = np.load(G)
    for name in ("rand", "pts"):
        for h in (0, 1):
            p = SIG.range_profile(_sweep(g["rp_freqs"], g[f"rp_{name}_{h}_in"]), M.VV,
                                  SIG.Window(h), 4)
            assert p.range_m.tobytes() == g[f"rp_{name}_{h}_range"].tobytes()
            assert p.bin_spacing == g[f"rp_{name}_{h}_bin"][0]
            assert _db_close(p.mag_db, g[f"rp_{name}_{h}_db"])


def test_isar_matches_reference():
    g = np.load(G)
    vals = g["isar_in"]
    sweeps = [_sweep(g["isar_freqs"], vals[a]) for a in range(len(vals))]
    img = SIG.isar(sweeps, g["isar_angles"], M.VV, SIG.Window.HANN, 4, -40.0)
    assert img.down_range_m.tobytes() == g["isar_down"].tobytes()
    assert np.allclose(img.cross_range_m, g["isar_cross"], rtol=1e-14, atol=0)
    assert _db_close(img.mag_db, g["isar_db"])
    assert abs(img.peak_db - g["isar_peak"][0]) < 1e-9


def test_signal_errors_mirror_reference():
    f = np.linspace(1e9, 2e9, 8)
    with pytest.raises(SIG.SignalError, match="zero_pad must be >= 1"):
        SIG.range_profile(_sweep(f, np.ones(8)), M.VV, SIG.Window.HANN, 0)
    with pytest.raises(SIG.SignalError, match="grid is not uniform"):
        SIG.range_profile(_sweep(np.array([1e9, 2e9, 4e9]), np.ones(3)), M.VV)
    sw = [_sweep(f, np.ones(8))] * 3
    with pytest.raises(SIG.SignalError, match="small-angle limit"):
        SIG.isar(sw, [0.0, 20.0, 40.0], M.VV)


def test_isar_of_estimator_sweep_locates_dihedral():
    """End to end: a 16-angle x 32-frequency ISAR of the dihedral grid from
    estimate_batch; the brightest pixel is the corner reflector's phase
    centre, which for a dihedral lies on the seam (down range ~0 at the
    origin-referenced phase)."""
    obj, mm = M.dihedral_grid(0.5, 16)
    s = M.Scene(M.load_scene(obj, mm))
    freqs = np.linspace(9.5e9, 10.5e9, 32)
    angles = 45.0 + np.linspace(-3.0, 3.0, 16)
    excs = [M.monostatic_excitation(90.0, float(a)) for a in angles]
    cfg = M.McConfig(strata_per_wavelength=3, samples_per_stratum=1, max_bounce=4, seed=2)
    vals, _ = M.estimate_batch(s, [(e, 0.0) for e in excs], [[e] for e in excs], freqs, cfg)
    img = SIG.isar(vals[:, 0], angles, M.VV, SIG.Window.HANN, 4, -40.0, frequencies=freqs)
    r, c = np.unravel_index(np.argmax(img.mag_db), img.mag_db.shape)
    assert abs(img.down_range_m[r]) <= 0.05 and abs(img.cross_range_m[c]) <= 0.3
