"""Pins for the oracle's propagator, brute-force path sum and iterative engine (CPU only).

What the paper fixes (P:<line> = PAPER.md):
* Eq. 8 is a sum over paths; the tensor propagator is an exact
  reorganisation of the memory-truncated sum -> brute force == iterative.
* trace: at a diagonal final point Delta s = 0 so all its influence factors are 1 and
  unitarity of U collapses the sum -> tr rho(t_k) = tr rho0 for ANY eta table.
* zero coupling (J = 0): rho(t) = e^{-iHt} rho0 e^{iHt} (closed system, checked against scipy expm).
* pure dephasing (H diagonal): only constant paths survive, so rho_ab(t_k) =
  rho0_ab e^{-i(E_a-E_b) t_k} exp(-(s_a-s_b)(s_a S_k - s_b S_k*)) with S_k = G(t_k) for k <= L
  (the exact continuum result -- the Strang windows tile [0, t]) and, for k > L,
  S_k = 2G((L+1/2)dt) - G(L dt) + (k-1-L)[G((L+1)dt) - G(L dt)] (lags > L dropped).
* the paper's §III model at zero coupling: rho_11 = sin^2(Omega t / 2) (Rabi).
"""
import numpy as np
import pytest
import scipy.linalg as sla

import oracle as O
from paper_1205_6872_b200 import workloads as W


def P(w: W.Workload, **kw):
    d = dict(s=w.s, H=w.H, rho0=w.rho0, kind=w.kind, coupling=w.coupling, omega_c=w.omega_c,
             kT=w.kT, dt=w.dt, n_steps=w.n_steps, L=w.L)
    d.update(kw)
    return O.Problem(**d)


# ----------------------------------------------------------------------------- propagator
def test_U_spin_boson_analytic():
    w = W.CONFIGS[1]  # H = -Delta sigma_x, Delta = 1
    U = O.propagator(P(w))
    c, s = np.cos(w.dt), np.sin(w.dt)
    assert np.abs(U - np.array([[c, 1j * s], [1j * s, c]])).max() < 1e-15


def test_U_quantum_dot_analytic():
    w = W.CONFIGS[0]  # H = 1/2 [[0, W],[W, 0]], W = pi/8
    U = O.propagator(P(w))
    a = np.pi / 8 * w.dt / 2
    assert np.abs(U - np.array([[np.cos(a), -1j * np.sin(a)], [-1j * np.sin(a), np.cos(a)]])).max() < 1e-15


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("M", [2, 3, 4, 5])
def test_U_matches_expm_unitary_composes(seed, M):
    rng = np.random.default_rng(seed)
    H = W.random_hermitian(rng, M, 1.3)
    w = W.random_problem(seed, M, 2, 3).with_(H=H, dt=0.37)
    U = O.propagator(P(w))
    assert np.abs(U - sla.expm(-1j * H * 0.37)).max() < 1e-13
    assert np.abs(U.conj().T @ U - np.eye(M)).max() < 1e-14
    U2 = O.propagator(P(w, dt=0.74))
    assert np.abs(U2 - U @ U).max() < 1e-13


def test_U_degenerate_spectrum():
    M = 4
    H = np.diag([0.3, 0.3, -1.0, -1.0]).astype(complex)
    Q = np.linalg.qr(np.random.default_rng(3).standard_normal((M, M)) + 1j)[0]
    H = Q @ H @ Q.conj().T
    H = 0.5 * (H + H.conj().T)
    w = W.random_problem(0, M, 2, 3).with_(H=H, dt=0.5)
    assert np.abs(O.propagator(P(w)) - sla.expm(-0.5j * H)).max() < 1e-13


# ----------------------------------------------------------------------------- brute force == iterative
CASES = [(seed, M, L, Nt, kind)
         for seed in range(20)
         for (M, L, Nt) in [(2, 1, 5), (2, 2, 6), (2, 3, 6), (2, 6, 5), (3, 1, 4), (3, 2, 4), (3, 4, 3)]
         for kind in [(W.J_OHMIC_EXP, W.J_DEBYE, W.J_SUPEROHMIC_GAUSS)[seed % 3]]]


@pytest.mark.parametrize("seed,M,L,Nt,kind", CASES)
def test_brute_force_equals_iterative(seed, M, L, Nt, kind):
    """Master property: truncated and untruncated (Nt <= L) path sums, random H/rho0/s."""
    w = W.random_problem(seed, M, L, Nt, kind=kind, lattice_s=(seed % 2 == 0))
    p = P(w)
    traj = O.run(p)  # every k in 0..Nt
    for k in range(Nt + 1):
        bf = O.brute_force(P(w, n_steps=k))
        assert np.abs(bf - traj[k]).max() < 1e-13, (k, np.abs(bf - traj[k]).max())


def test_k0_is_rho0_exactly():
    w = W.random_problem(1, 3, 2, 0)
    assert np.array_equal(O.brute_force(P(w)), w.rho0)
    assert np.array_equal(O.run(P(w, n_steps=3))[0], w.rho0)


# ----------------------------------------------------------------------------- invariants
@pytest.mark.parametrize("cfg", [0, 1])
def test_trace_and_hermiticity_every_step(cfg):
    w = W.CONFIGS[cfg].with_(n_steps=min(W.CONFIGS[cfg].n_steps, 150), L=min(W.CONFIGS[cfg].L, 6))
    r = O.run(P(w))
    tr = np.einsum("kii->k", r)
    assert np.abs(tr - 1).max() < 1e-12
    assert np.abs(r - r.conj().transpose(0, 2, 1)).max() < 1e-13


@pytest.mark.parametrize("seed", range(6))
def test_trace_any_eta_table(seed):
    """The trace pin holds for ANY eta table, including random complex G (the trace argument
    uses only Delta s = 0 at the final point and unitarity of U)."""
    rng = np.random.default_rng(100 + seed)
    M, L, Nt = (2, 3, 9) if seed % 2 == 0 else (3, 2, 5)
    w = W.random_problem(seed, M, L, Nt)
    G = 0.08 * (rng.standard_normal(2 * L + 3) + 1j * rng.standard_normal(2 * L + 3))
    G[0] = 0
    r = O.run(P(w, G_in=G))
    # exact in exact arithmetic; roundoff scales with the (non-physical, growing) off-diagonals
    scale = max(1.0, np.abs(r).max())
    assert np.abs(np.einsum("kii->k", r) - 1).max() < 1e-13 * scale


@pytest.mark.parametrize("M,L", [(2, 1), (2, 4), (3, 2)])
def test_zero_coupling_is_unitary_evolution(M, L):
    w = W.random_problem(7, M, L, 40, kind=W.J_ZERO)
    r = O.run(P(w))
    for k in range(0, 41, 5):
        Uk = sla.expm(-1j * w.H * w.dt * k)
        assert np.abs(r[k] - Uk @ w.rho0 @ Uk.conj().T).max() < 1e-12


def test_rabi_quantum_dot_zero_bath():
    """§III model with J = 0: rho_11(t) = sin^2(Omega t / 2)."""
    w = W.CONFIGS[0].with_(kind=W.J_ZERO, n_steps=200, L=3)
    r = O.run(P(w))
    t = w.dt * np.arange(201)
    assert np.abs(r[:, 1, 1].real - np.sin(np.pi / 8 * t / 2) ** 2).max() < 1e-12


def _S_closed(G, L, k):
    """S_k in units where G is sampled at half steps: G[m] = G(m dt/2)."""
    if k <= L:
        return G[2 * k]
    return 2 * G[2 * L + 1] - G[2 * L] + (k - 1 - L) * (G[2 * L + 2] - G[2 * L])


@pytest.mark.parametrize("M,L,kind", [(2, 1, W.J_OHMIC_EXP), (2, 3, W.J_DEBYE), (2, 5, W.J_SUPEROHMIC_GAUSS),
                                      (3, 2, W.J_DEBYE), (3, 3, W.J_OHMIC_EXP)])
def test_pure_dephasing_closed_form(M, L, kind):
    rng = np.random.default_rng(M * 10 + L)
    E = rng.uniform(-1, 1, M)
    Nt = 3 * L + 4
    w = W.random_problem(11, M, L, Nt, kind=kind).with_(H=np.diag(E).astype(complex))
    p = P(w)
    r = O.run(p)
    G = O.G_table(p)
    s = w.s
    for k in range(Nt + 1):
        Sk = _S_closed(G, L, k) if k > 0 else 0.0
        ex = np.empty((M, M), dtype=complex)
        for a in range(M):
            for b in range(M):
                ex[a, b] = w.rho0[a, b] * np.exp(-1j * (E[a] - E[b]) * w.dt * k) * np.exp(
                    -(s[a] - s[b]) * (s[a] * Sk - s[b] * np.conj(Sk)))
        assert np.abs(r[k] - ex).max() < 1e-13, (k, np.abs(r[k] - ex).max())


def test_pure_dephasing_rejects_printed_windows():
    """Reading C.3-1: with the windows as printed (point k on [k dt,(k+1) dt]) the exact
    pure-dephasing result is NOT reproduced, with the Strang tiling it is (previous test)."""
    M, L = 2, 4
    w = W.random_problem(11, M, L, 4).with_(H=np.diag([0.3, -0.2]).astype(complex))
    r = O.run(P(w, reading=O.READING_AS_PRINTED))
    G = O.G_table(P(w))
    s, k = w.s, 4
    Sk = G[2 * k]
    ex01 = w.rho0[0, 1] * np.exp(-1j * 0.5 * w.dt * k) * np.exp(-(s[0] - s[1]) * (s[0] * Sk - s[1] * np.conj(Sk)))
    assert abs(r[k][0, 1] - ex01) > 1e-4


# ----------------------------------------------------------------------------- modes / determinism / symmetry
def test_mode_equivalence_bit_identical():
    """justFinalPoint vs allPoints: final rho bit-identical."""
    for seed in range(5):
        w = W.random_problem(seed, 2 if seed % 2 else 3, 3, 12)
        allp = O.run(P(w))
        final = O.run(P(w), out_steps=[12])
        assert np.array_equal(allp[-1], final[0])


def test_thread_count_determinism():
    w = W.CONFIGS[0].with_(n_steps=60, L=6)
    runs = [O.run(P(w), nthreads=t) for t in (1, 2, 8)]
    assert np.array_equal(runs[0], runs[1]) and np.array_equal(runs[0], runs[2])


def test_sigma_x_symmetry_spin_boson():
    """H = -Delta sigma_x, s = +-1: flipping s <-> -s is Q -> -Q (bath statistics unchanged), so
    rho(t; X rho0 X) = X rho(t; rho0) X."""
    w = W.CONFIGS[1].with_(n_steps=30)
    X = np.array([[0, 1], [1, 0]], dtype=complex)
    rho0 = W.random_density_matrix(np.random.default_rng(5), 2)
    a = O.run(P(w, rho0=rho0))
    b = O.run(P(w, rho0=X @ rho0 @ X))
    assert np.abs(b - X @ a @ X).max() < 1e-13


def test_linearity_in_rho0():
    w = W.random_problem(2, 3, 2, 8)
    rng = np.random.default_rng(9)
    r1, r2 = W.random_density_matrix(rng, 3), W.random_density_matrix(rng, 3)
    a = O.run(P(w, rho0=r1))
    b = O.run(P(w, rho0=r2))
    c = O.run(P(w, rho0=0.3 * r1 + 0.7 * r2))
    assert np.abs(c - (0.3 * a + 0.7 * b)).max() < 1e-13


def test_validation_errors():
    w = W.random_problem(2, 2, 2, 3)
    with pytest.raises(O.OracleError, match="trace"):
        O.run(P(w, rho0=0.9 * w.rho0))
    H = w.H.copy()
    H[0, 1] += 0.1
    with pytest.raises(O.OracleError, match="Hermitian"):
        O.run(P(w, H=H))
    with pytest.raises(O.OracleError, match="guard"):
        O.brute_force(P(w, n_steps=12))
