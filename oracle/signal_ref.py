"""TEST INFRASTRUCTURE ONLY: numpy restatement of the reference's radar
products (proj/src/signal_processing.cpp), the checker for the GPU
range-profile / ISAR kernels.  Pinned against the compiled reference's output
(tests/golden/signal.npz, tests/golden/make_golden.py) by
tests/test_oracle_pins.py.  The reference evaluates e^{j 2 pi k m / M} with a
running product; this restatement uses exact integer phase reduction, so the
two agree to ~1e-13 relative (asserted at 1e-9 dB), not bit-for-bit.
"""
from __future__ import annotations

import numpy as np

C0 = 299792458.0


def uniform_step(grid, what):  # :11-19
    g = np.asarray(grid, dtype=np.float64)
    if len(g) < 2:
        raise ValueError(f"{what}: need at least 2 samples")
    step = g[1] - g[0]
    if np.any(np.abs(np.diff(g) - step) > 1e-6 * abs(step)):
        raise ValueError(f"{what}: grid is not uniform")
    return step


def window_coefficients(hann: bool, n: int):  # :21-28
    w = np.ones(n)
    if hann and n > 1:
        k = np.arange(n)
        w = 0.5 - 0.5 * np.cos(2.0 * np.pi * k / (n - 1))
    return w


def padded_idft(x, m, conjugate):  # :31-46 (direct evaluation)
    n = len(x)
    km = (np.arange(n)[:, None] * np.arange(m)[None, :]) % m
    sign = -1.0 if conjugate else 1.0
    e = np.exp(1j * sign * 2.0 * np.pi * km / m)
    return (x[:, None] * e).sum(axis=0) / m


def center_shift(v):  # :49-53
    m = len(v)
    return np.roll(v, -(m - m // 2))


def centered_axis(m, bin_):  # :55-60
    return (np.arange(m) - m // 2) * bin_


def to_db(mag):
    return 20.0 * np.log10(np.maximum(mag, 1e-300))


def range_profile(values, freqs, hann=True, zero_pad=4):  # :66-89
    df = uniform_step(freqs, "range_profile")
    n = len(freqs)
    m = n * zero_pad
    spec = center_shift(padded_idft(np.asarray(values) * window_coefficients(hann, n), m, False))
    bin_ = C0 / (2.0 * df * m)
    return centered_axis(m, bin_), to_db(np.abs(spec)), bin_


def isar(values, freqs, angles, hann=True, zero_pad=4, floor_db=-40.0):  # :91-162
    values = np.asarray(values)
    dtheta_deg = uniform_step(angles, "isar angles")
    df = uniform_step(freqs, "isar frequencies")
    na, nf = values.shape
    mr, mc = nf * zero_pad, na * zero_pad
    data = values * window_coefficients(hann, nf)[None, :] * window_coefficients(hann, na)[:, None]
    cols = np.stack([center_shift(padded_idft(data[a], mr, False)) for a in range(na)])  # [a][r]
    img = np.stack([center_shift(padded_idft(cols[:, r], mc, True)) for r in range(mr)])  # [r][c]
    mags = np.abs(img)
    peak_db = to_db(mags.max())
    mag_db = np.maximum(to_db(mags), peak_db + floor_db)
    f_center = 0.5 * (freqs[0] + freqs[-1])
    dtheta = dtheta_deg * np.pi / 180.0
    down = centered_axis(mr, C0 / (2.0 * df * mr))
    cross = centered_axis(mc, C0 / (2.0 * f_center * dtheta * mc))
    return down, cross, mag_db, peak_db
