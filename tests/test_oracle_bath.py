"""Pins for the oracle's bath quadrature G(tau) and eta classes (CPU only).

G(tau) is the double time integral of alpha (Eq. 4); every eta of
Eqs. 10-16 is a four-corner difference of G over the Strang
windows (reading C.3-1).  The pins are closed forms computed independently
(tests/closed_forms.py) and the constant-/linear-alpha window areas (SPEC's
test hook).
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_1205_6872_b200 import workloads as W
from tests import closed_forms as CF

TAUS = [0.125, 0.5, 1.0, 1.75, 3.75, 4.25]


def prob(**kw):
    w = W.CONFIGS[1]
    d = dict(s=w.s, H=w.H, rho0=w.rho0, kind=w.kind, coupling=w.coupling, omega_c=w.omega_c,
             kT=w.kT, dt=w.dt, n_steps=w.n_steps, L=w.L)
    d.update(kw)
    return O.Problem(**d)


def close(a, b, tol):
    return abs(a - b) <= tol * max(1.0, abs(b))


@pytest.mark.parametrize("tau", TAUS)
@pytest.mark.parametrize("kT", [0.0, 0.2, 1.0])
def test_G_ohmic_closed_form(tau, kT):
    g = O.G(prob(kind=O.J_OHMIC_EXP, kT=kT), tau)
    ex = CF.G_ohmic(0.1, 7.5, kT, tau)
    assert close(g, ex, 3e-15), (g, ex, abs(g - ex))


@pytest.mark.parametrize("tau", TAUS + [0.05])
@pytest.mark.parametrize("kT,wc", [(0.2, 7.5), (1.0, 3.0), (2.0, 1.0)])
def test_G_debye_matsubara(tau, kT, wc):
    """(2.0, 1.0) at tau = 0.05: small wc tau, where the closed-form Debye tail beyond the quadrature
    cutoff needs Omega tau large (the oracle picks Omega >= 400 / tau)."""
    g = O.G(prob(kind=O.J_DEBYE, kT=kT, omega_c=wc), tau)
    ex = CF.G_debye(0.1, wc, kT, tau)
    assert close(g, ex, 3e-15), (g, ex, abs(g - ex))


@pytest.mark.parametrize("tau", [0.05, 0.1, 0.6, 1.2])
@pytest.mark.parametrize("kT", [0.0, 25.0 * W.KB_OVER_HBAR_PS_K])
def test_G_superohmic(tau, kT):
    A = math.pi * 0.027
    g = O.G(prob(kind=O.J_SUPEROHMIC_GAUSS, coupling=A, omega_c=2.2, kT=kT), tau)
    ex = CF.G_superohmic(A, 2.2, kT, tau)
    assert close(g, ex, 3e-15), (g, ex, abs(g - ex))


def test_G_zero_bath_is_exactly_zero():
    for tau in TAUS:
        assert O.G(prob(kind=O.J_ZERO), tau) == 0j


def test_G_symmetries():
    p = prob(kind=O.J_DEBYE)
    # G(-t) = conj G(t)  (alpha(-t) = conj alpha(t), Eq. 4)
    for tau in (0.5, 2.0):
        assert O.G(p, -tau) == O.G(p, tau).conjugate()
    # linear in the coupling (Eq. 3 -> Eq. 4 are linear in J)
    for tau in (0.5, 2.0):
        a = O.G(prob(kind=O.J_OHMIC_EXP, coupling=0.1), tau)
        b = O.G(prob(kind=O.J_OHMIC_EXP, coupling=0.2), tau)
        assert close(b, 2 * a, 1e-15)


def _G_poly(dt, L, a=1.0, b=0.0):
    """alpha(t) = a + b t  =>  G(tau) = a tau^2/2 + b tau^3/6 (G'' = alpha)."""
    taus = 0.5 * dt * np.arange(2 * L + 3)
    return a * taus**2 / 2 + b * taus**3 / 6


def test_eta_constant_alpha_areas():
    """alpha == 1: each eta is the area of its window (pair) -- SPEC S:136-139 values."""
    dt, L = 0.3, 4
    p = prob(L=L, dt=dt, G_in=_G_poly(dt, L).astype(complex))
    d2 = dt * dt
    Nf = 3  # final point of a run of 3 steps, L = 4 > 3 so every class appears
    assert O.eta_pair(p, 1, 1, Nf) == pytest.approx(d2 / 2, abs=1e-15)    # interior self (Eq. 11)
    assert O.eta_pair(p, 0, 0, Nf) == pytest.approx(d2 / 8, abs=1e-15)    # eta_00 (Eq. 13, reading C.3-2)
    assert O.eta_pair(p, 3, 3, Nf) == pytest.approx(d2 / 8, abs=1e-15)    # eta_NN (Eq. 14)
    assert O.eta_pair(p, 2, 1, Nf) == pytest.approx(d2, abs=1e-15)        # interior lag (Eq. 10)
    assert O.eta_pair(p, 3, 0, Nf) == pytest.approx(d2 / 4, abs=1e-15)    # eta_N0 (Eq. 12)
    assert O.eta_pair(p, 2, 0, Nf) == pytest.approx(d2 / 2, abs=1e-15)    # eta_k0 (Eq. 15)
    assert O.eta_pair(p, 3, 1, Nf) == pytest.approx(d2 / 2, abs=1e-15)    # eta_Nk (Eq. 16)


def test_eta_interior_self_is_half_square():
    """Eq. 11: the self term integrates over the triangle t'' < t' of a full window -> dt^2/2."""
    dt, L = 0.3, 4
    p = prob(L=L, dt=dt, G_in=_G_poly(dt, L).astype(complex))
    assert O.eta_pair(p, 2, 2, 5) == pytest.approx(dt * dt / 2, abs=1e-15)


def test_eta_linear_alpha_window_placement():
    """alpha = t: the pair integral is w_a w_b (c_a - c_b) with window centres c.  The Strang
    windows (reading C.3-1) put point k at [k-1/2, k+1/2] (centre k); the printed Eq. 10 would
    put it at [k, k+1] (centre k+1/2)."""
    dt, L = 1.0, 5
    p = prob(L=L, dt=dt, G_in=_G_poly(dt, L, a=0.0, b=1.0).astype(complex))
    # (k=3, k'=0) with final point 6: windows [2.5,3.5] x [0,0.5] -> 1 * 0.5 * (3 - 0.25)
    assert O.eta_pair(p, 3, 0, 6) == pytest.approx(0.5 * 2.75, abs=1e-13)
    # (6, 2) final 6: [5.5,6] x [1.5,2.5] -> 0.5 * 1 * (5.75 - 2)
    assert O.eta_pair(p, 6, 2, 6) == pytest.approx(0.5 * 3.75, abs=1e-13)
    # interior (4,1): 1*1*(4-1)
    assert O.eta_pair(p, 4, 1, 6) == pytest.approx(3.0, abs=1e-13)
    pa = prob(L=L, dt=dt, G_in=_G_poly(dt, L, a=0.0, b=1.0).astype(complex), reading=O.READING_AS_PRINTED)
    assert O.eta_pair(pa, 3, 0, 6) == pytest.approx(0.5 * 3.25, abs=1e-13)


def test_eta_lag_stationary_and_zero_bath():
    p = prob(kind=O.J_DEBYE, L=6)
    # interior pairs depend on the lag only (alpha(t'-t''))
    assert O.eta_pair(p, 5, 2, -1) == O.eta_pair(p, 7, 4, -1)
    z = prob(kind=O.J_ZERO, L=6)
    for (t, tp, kf) in [(3, 3, 5), (5, 0, 5), (4, 1, -1), (2, 0, -1)]:
        assert O.eta_pair(z, t, tp, kf) == 0j


def test_eta_tiling_sums_to_G():
    """Under the Strang tiling the windows of points 0..N partition [0, N dt], so the sum of all
    eta over a run with N <= L equals G(N dt) (reading C.3-1; the printed windows do not tile)."""
    p = prob(kind=O.J_DEBYE, L=6, dt=0.25)
    N = 5
    tot = sum(O.eta_pair(p, t, tp, N) for t in range(N + 1) for tp in range(t + 1))
    assert close(tot, O.G(p, N * 0.25), 1e-14)
    pa = prob(kind=O.J_DEBYE, L=6, dt=0.25, reading=O.READING_AS_PRINTED)
    tota = sum(O.eta_pair(pa, t, tp, N) for t in range(N + 1) for tp in range(t + 1))
    assert abs(tota - O.G(p, N * 0.25)) > 1e-3


def test_pmc_matches_table1():
    """Eqs. 18-19: PMC = 64 M^(2(L+1)) reproduces Table I's column to the printed digits."""
    unit = {"KB": 1e3, "MB": 1e6, "GB": 1e9}
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "table1_pmc.txt")
    rows = [ln.split() for ln in open(path) if ln.strip() and not ln.startswith("#")]
    assert len(rows) == 11
    for dk, val, u in rows:
        pmc = O.pmc_bytes(2, int(dk))
        assert pmc == 64 * 4 ** (int(dk) + 1)
        assert float(f"{pmc / unit[u]:.4g}") == float(val), (dk, pmc, val, u)
