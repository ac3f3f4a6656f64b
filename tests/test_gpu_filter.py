"""GPU parity of the path-filtered mode (reading C.3-15) against the oracle's filtered
mode: rho within 1e-10 and the kept-entry count of every propagated step equal (integer decisions
|A|^2 < theta^2 taken in FP64 without FMA on both sides), for growth and slide steps, M = 2 and 3,
several thresholds; theta = 0 reproduces the dense run; the pure-dephasing coherence removal."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from paper_1205_6872_b200 import quapi as Q  # noqa: E402
from paper_1205_6872_b200 import workloads as W  # noqa: E402
from tests.test_oracle_engine import P  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1205_6872_b200 import build as B
    B.build()


@pytest.mark.parametrize("theta", [1e-3, 1e-5, 1e-8])
@pytest.mark.parametrize("seed,M,L,n", [(0, 2, 5, 24), (1, 2, 7, 30), (2, 3, 4, 14), (3, 2, 9, 26)])
def test_filtered_matches_oracle(theta, seed, M, L, n):
    w = W.random_problem(60 + seed, M, L, n, kind=W.J_DEBYE)
    rg, kg = Q.Plan(w).filter_run(theta)
    kept = np.zeros(n + 1, dtype=np.int64)
    ro = O.run(P(w, filter_theta=theta, kept=kept))
    assert np.abs(rg - ro).max() <= 1e-10
    assert np.array_equal(kg[:n], kept[:n])  # the oracle does not propagate past the last readout
    assert np.abs(np.einsum("kii->k", rg) - np.einsum("kii->k", ro)).max() <= 1e-12


def test_theta_zero_is_the_dense_run():
    w = W.random_problem(70, 2, 6, 22)
    pl = Q.Plan(w)
    a, wk = pl.alloc()
    dense = pl.run(a, wk)
    rg, kg = Q.Plan(w).filter_run(0.0)
    assert np.abs(rg - dense).max() < 1e-13
    assert kg[6] == w.N ** 6  # nothing dropped: the list is the dense ARDM (no exact zeros for random H)


def test_pure_dephasing_coherences_dropped():
    E = np.array([0.3, -0.5])
    rho0 = np.array([[0.6, 1e-3], [1e-3, 0.4]], dtype=complex)
    w = W.CONFIGS[1].with_(H=np.diag(E).astype(complex), rho0=rho0, n_steps=16, L=6)
    rg, kg = Q.Plan(w).filter_run(1e-2)
    ro = O.run(P(w, filter_theta=1e-2))
    assert np.abs(rg - ro).max() < 1e-13
    assert np.all(rg[2:, 0, 1] == 0) and kg[0] == 4 and np.all(kg[1:-1] == 2)


def test_capacity_overflow_is_reported():
    w = W.random_problem(71, 2, 6, 12)
    with pytest.raises(Q.QuapiError) as ei:
        Q.Plan(w).filter_run(1e-12, capacity=100)
    assert ei.value.status == Q.QP_ERR_CAPACITY and "step" in str(ei.value)
