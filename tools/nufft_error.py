"""Error of the spreading kernel of csrc/spread.cu, in numpy (design check,
no GPU): for a record at grid offset t + j eta, the NUFFT estimate of
e^{j m (t + j eta) h} for every mode |m| <= F/2 against the exact phasor,
with (a) the exact exponential-of-semicircle kernel, (b) its per-point
polynomials (Chebyshev, 14 coefficients, as the device evaluates them), for
real and complex offsets.

    python tools/nufft_error.py [--nf 128]
"""
import argparse

import numpy as np
from numpy.polynomial import chebyshev as Ch

ap = argparse.ArgumentParser()
ap.add_argument("--nf", type=int, default=128)
ap.add_argument("--trials", type=int, default=200)
a = ap.parse_args()
W, BETA, NPOLY = 16, 2.30 * 16, 14
nf = a.nf
NG, fc = 2 * nf, nf // 2
h = 2 * np.pi / NG
m = np.arange(nf) - fc


def psi(z):
    z = np.asarray(z, dtype=complex)
    v = np.exp(BETA * (np.sqrt(1 - z * z) - 1))
    return np.where(np.abs(z.real) < 1, v, 0)


coef = [Ch.cheb2poly(Ch.chebinterpolate(lambda x, i=i: psi(((x + 1) / 2 + i - 8) / 8).real, NPOLY - 1))
        for i in range(W)]


def horner(c, x):
    r = np.full_like(np.asarray(x, dtype=complex), c[-1])
    for k in range(len(c) - 2, -1, -1):
        r = r * x + c[k]
    return r


g = np.arange(W) - 8
hat = (np.array([horner(coef[i], -1.0).real for i in range(W)])[None, :] * np.cos(np.outer(m, g * h))).sum(1)
rng = np.random.default_rng(5)
print(f"nf {nf}, grid {NG}, kernel width {W}, beta {BETA:.1f}, {NPOLY} coefficients per point")
print("eta (cells)   polynomial   exact kernel   (max relative error over modes and trials)")
for eta in (0.0, 0.001, 0.005, 0.02, 0.05, 0.1, 0.2, 0.41):
    e_poly, e_exact = [], []
    for _ in range(a.trials):
        t = rng.uniform(0, NG)
        g0 = np.ceil(t - 8)
        x = 2 * (g0 - t + 8) - 1
        gi = g0 + np.arange(W)
        E = np.exp(1j * np.outer(m, gi * h))
        ex = np.exp(1j * m * (t + 1j * eta) * h)
        wp = np.array([horner(coef[i], x - 2j * eta) for i in range(W)])
        we = psi((gi - t - 1j * eta) / 8)
        e_poly.append(np.max(np.abs((E * wp[None, :]).sum(1) / hat - ex) / np.abs(ex)))
        e_exact.append(np.max(np.abs((E * we[None, :]).sum(1) / hat - ex) / np.abs(ex)))
    print(f"{eta:10.3f}   {max(e_poly):10.1e}   {max(e_exact):12.1e}")
