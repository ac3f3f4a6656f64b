"""Oracle pins for the time-dependent (driven) Hamiltonian, SURVEY §8(f1).

The paper's use case is the driven quantum dot of §III, H(t) = (1/2) Omega(t) sigma_x with a pulse
Omega(t), swept over pulse areas.  The oracle takes H_t[k-1] on the interval
(t_{k-1}, t_k] of step k (Eq. 8 with a step-dependent propagator pair K_k).  Pinned against:
the time-independent run (H_t constant), exact unitary evolution at zero coupling (products of
scipy expm), the pulse-area theorem rho_11 = sin^2(A/2), brute-force path sums, the pure-dephasing
closed form with time-dependent energies, and the trace invariant.
"""
import numpy as np
import pytest
import scipy.linalg as sla

import oracle as O
from paper_1205_6872_b200 import workloads as W
from tests.test_oracle_engine import P, _S_closed


def _drive(rng, M, Nt, amp=0.6):
    """A random Hermitian H0 plus f_k H1 with random amplitudes per step."""
    H0 = W.random_hermitian(rng, M)
    H1 = W.random_hermitian(rng, M)
    f = amp * rng.standard_normal(Nt)
    return H0, H1, f, np.stack([H0 + fk * H1 for fk in f]) if Nt else np.zeros((0, M, M), complex)


def test_constant_drive_is_bit_identical_to_static_H():
    w = W.random_problem(3, 2, 4, 17, kind=W.J_DEBYE)
    Ht = np.repeat(w.H[None], w.n_steps, axis=0)
    assert np.array_equal(O.run(P(w, H_t=Ht)), O.run(P(w)))
    assert np.array_equal(O.brute_force(P(w.with_(n_steps=5), H_t=Ht[:5])), O.brute_force(P(w.with_(n_steps=5))))


@pytest.mark.parametrize("M,L", [(2, 1), (2, 4), (3, 2)])
def test_zero_coupling_is_time_ordered_unitary_evolution(M, L):
    rng = np.random.default_rng(40 + M + L)
    Nt = 30
    w = W.random_problem(9, M, L, Nt, kind=W.J_ZERO)
    _, _, _, Ht = _drive(rng, M, Nt)
    r = O.run(P(w, H_t=Ht))
    rho = w.rho0.copy()
    for k in range(1, Nt + 1):
        U = sla.expm(-1j * Ht[k - 1] * w.dt)
        rho = U @ rho @ U.conj().T
        assert np.abs(r[k] - rho).max() < 1e-12, k


def test_pulse_area_theorem():
    """Driven two-level system without bath: H(t) = Omega(t) sigma_x / 2, rho0 = |0><0| gives
    rho_11(T) = sin^2(A / 2), A = sum_k Omega_k dt (the pulse-area dependence of P:420-442)."""
    w0 = W.CONFIGS[0]
    Nt, dt = 120, w0.dt
    t = dt * (np.arange(Nt) + 0.5)
    sx = np.array([[0, 1], [1, 0]], dtype=complex)
    for area in (0.5 * np.pi, np.pi, 1.7 * np.pi, 3 * np.pi):
        env = np.exp(-((t - t.mean()) / (0.2 * t[-1])) ** 2)
        omega = area * env / (env.sum() * dt)
        Ht = np.stack([0.5 * om * sx for om in omega])
        w = w0.with_(kind=W.J_ZERO, n_steps=Nt, L=3)
        r = O.run(P(w, H_t=Ht), out_steps=[Nt])
        assert abs(r[0, 1, 1].real - np.sin(area / 2) ** 2) < 1e-12


CASES = [(seed, M, L, Nt) for seed in range(8) for (M, L, Nt) in [(2, 1, 5), (2, 2, 6), (2, 3, 6), (3, 2, 4)]]


@pytest.mark.parametrize("seed,M,L,Nt", CASES)
def test_brute_force_equals_iterative_with_drive(seed, M, L, Nt):
    """Literal path sum with a different propagator pair on every step vs the iterative engine."""
    rng = np.random.default_rng(200 + seed)
    kind = (W.J_OHMIC_EXP, W.J_DEBYE, W.J_SUPEROHMIC_GAUSS)[seed % 3]
    w = W.random_problem(seed, M, L, Nt, kind=kind)
    _, _, _, Ht = _drive(rng, M, Nt)
    traj = O.run(P(w, H_t=Ht))
    for k in range(Nt + 1):
        bf = O.brute_force(P(w.with_(n_steps=k), H_t=Ht[:k]))
        assert np.abs(bf - traj[k]).max() < 1e-13, (k, np.abs(bf - traj[k]).max())


@pytest.mark.parametrize("M,L", [(2, 3), (3, 2)])
def test_pure_dephasing_with_time_dependent_energies(M, L):
    """Diagonal H_k = diag(E_k): rho_ab(t_k) = rho0_ab exp(-i sum_j (E_a - E_b)_j dt) x the bath
    factor of the static case (the influence functional does not see H)."""
    rng = np.random.default_rng(7 * M + L)
    Nt = 3 * L + 4
    E = rng.uniform(-1, 1, (Nt, M))
    Ht = np.stack([np.diag(e).astype(complex) for e in E])
    w = W.random_problem(13, M, L, Nt, kind=W.J_DEBYE).with_(H=np.diag(E[0]).astype(complex))
    p = P(w, H_t=Ht)
    r = O.run(p)
    G = O.G_table(p)
    s = w.s
    phase = np.vstack([np.zeros(M), np.cumsum(E, axis=0)]) * w.dt
    for k in range(Nt + 1):
        Sk = _S_closed(G, L, k) if k > 0 else 0.0
        ex = np.array([[w.rho0[a, b] * np.exp(-1j * (phase[k, a] - phase[k, b])) *
                        np.exp(-(s[a] - s[b]) * (s[a] * Sk - s[b] * np.conj(Sk))) for b in range(M)] for a in range(M)])
        assert np.abs(r[k] - ex).max() < 1e-13, k


def test_trace_and_hermiticity_with_drive():
    rng = np.random.default_rng(5)
    w = W.random_problem(5, 3, 3, 25, kind=W.J_OHMIC_EXP)
    _, _, _, Ht = _drive(rng, 3, 25)
    r = O.run(P(w, H_t=Ht))
    assert np.abs(np.einsum("kii->k", r) - 1).max() < 1e-12
    assert np.abs(r - r.conj().transpose(0, 2, 1)).max() < 1e-13


def test_drive_validation():
    w = W.random_problem(1, 2, 2, 4)
    Ht = np.repeat(w.H[None], 4, axis=0)
    Ht[2, 0, 1] += 0.1  # not Hermitian
    with pytest.raises(O.OracleError, match="H_t not Hermitian"):
        O.run(P(w, H_t=Ht))
    with pytest.raises(ValueError):
        O.run(P(w, H_t=Ht[:3]))
