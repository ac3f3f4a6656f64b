"""Pins for the oracle's path-filtered mode (reading C.3-15 of DESIGN.md).

The paper cites Sim's on-the-fly filtering of paths as the way to cut the memory of the tensor
propagator, notes that its own program does not do it and invites it
(P:565-566).  Reading C.3-15: after every propagation step k >= 1 the entries of A_k with
|A|^2 < theta^2 are set to 0 (A_0 is never filtered; rho(t_k) is read from the filtered A_{k-1}).
What fixes the mode independently of its own code:
* theta = 0 drops nothing: bit-identical to the plain run;
* pure dephasing (H diagonal): only constant paths carry weight; a population path has |A| = rho0_aa
  at every step and a coherence path |A| <= |rho0_ab|, so a threshold between the two removes the
  coherences after the first step: populations follow the closed form exactly, rho_01(t_1) (read
  from the unfiltered A_0) too, and rho_01(t_k) = 0 exactly for k >= 2; kept counts are 4, then 2;
* a threshold above every entry empties A_1: rho(t_k) = 0 for k >= 2;
* the filtering error vanishes with theta.
"""
import numpy as np
import pytest

import oracle as O
from paper_1205_6872_b200 import workloads as W
from tests.test_oracle_engine import P, _S_closed


@pytest.mark.parametrize("seed,M,L,n", [(0, 2, 3, 12), (1, 2, 5, 14), (2, 3, 3, 9), (3, 2, 4, 4)])
def test_theta_zero_is_bit_identical(seed, M, L, n):
    w = W.random_problem(40 + seed, M, L, n, kind=W.J_DEBYE)
    a = O.run(P(w))
    b = O.run(P(w, filter_theta=0.0))
    assert np.array_equal(a, b)


def test_pure_dephasing_filter_removes_coherence_paths():
    E = np.array([0.3, -0.5])
    rho0 = np.array([[0.6, 1e-3], [1e-3, 0.4]], dtype=complex)
    w = W.CONFIGS[1].with_(H=np.diag(E).astype(complex), rho0=rho0, n_steps=16, L=4)
    kept = np.zeros(w.n_steps + 1, dtype=np.int64)
    r = O.run(P(w, filter_theta=1e-2, kept=kept))
    G = O.G_table(P(w))
    s = w.s
    for k in range(w.n_steps + 1):
        Sk = _S_closed(G, w.L, k) if k > 0 else 0.0
        ex = np.array([[rho0[a, b] * np.exp(-1j * (E[a] - E[b]) * w.dt * k) *
                        np.exp(-(s[a] - s[b]) * (s[a] * Sk - s[b] * np.conj(Sk))) for b in range(2)] for a in range(2)])
        assert abs(r[k][0, 0] - ex[0, 0]) < 1e-14 and abs(r[k][1, 1] - ex[1, 1]) < 1e-14
        if k <= 1:
            assert np.abs(r[k] - ex).max() < 1e-14
        else:
            assert r[k][0, 1] == 0 and r[k][1, 0] == 0
    assert kept[0] == 4 and np.all(kept[1:-1] == 2)  # the last step is read out, not propagated


def test_threshold_above_every_entry_empties_the_tensor():
    w = W.random_problem(7, 2, 3, 8)
    plain = O.run(P(w))
    r = O.run(P(w, filter_theta=10.0))
    assert np.array_equal(r[:2], plain[:2])  # rho(t_0) = rho0, rho(t_1) from the unfiltered A_0
    assert np.all(r[2:] == 0)


def test_filter_error_vanishes_with_theta():
    w = W.random_problem(9, 2, 5, 16, kind=W.J_OHMIC_EXP)
    plain = O.run(P(w))
    errs = []
    for th in (1e-3, 1e-5, 1e-7, 1e-9):
        kept = np.zeros(w.n_steps + 1, dtype=np.int64)
        r = O.run(P(w, filter_theta=th, kept=kept))
        errs.append(np.abs(r - plain).max())
        assert kept.max() <= w.N ** w.L
    assert errs[0] > 0 and errs[-1] < 1e-7
    assert all(errs[i + 1] <= errs[i] for i in range(len(errs) - 1))
