"""Batched sweeps through the C ABI (qp_batch_*) against the oracle.

Every problem b of a batch is compared element by element with the oracle run of the same problem:
the oracle gets H_t[k-1] = H0 + f[b, k-1] H1 (its own Jacobi propagators) and rho0s[b].  Tolerance as
the single-problem path: max |d rho| <= 1e-10, trace within 1e-12.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from paper_1205_6872_b200 import quapi as Q  # noqa: E402
from paper_1205_6872_b200 import workloads as W  # noqa: E402
from tests.test_oracle_engine import P  # noqa: E402

TOL = 1e-10
SX = np.array([[0, 1], [1, 0]], dtype=complex)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1205_6872_b200 import build as B
    B.build()


def batch_run(w, B, **kw):
    bp = Q.BatchPlan(w, B, **kw)
    ardm, work = bp.alloc()
    return bp.run(ardm, work), bp


def oracle_problem(w, b, H1=None, f=None, rho0s=None, out_steps=None):
    Ht = None if f is None else np.stack([w.H + f[b, k] * H1 for k in range(w.n_steps)])
    r0 = w.rho0 if rho0s is None else rho0s[b]
    return O.run(P(w, rho0=r0, H_t=Ht), out_steps=out_steps)


@pytest.mark.parametrize("M,L,n", [(2, 3, 25), (2, 5, 30), (2, 6, 20), (3, 3, 14), (4, 2, 9)])
def test_driven_batch_matches_oracle(M, L, n):
    rng = np.random.default_rng(10 * M + L)
    B = 5
    w = W.random_problem(600 + M + L, M, L, n, kind=W.J_DEBYE)
    H1 = W.random_hermitian(rng, M)
    f = 0.7 * rng.standard_normal((B, n))
    rho0s = np.stack([W.random_density_matrix(rng, M) for _ in range(B)])
    rg, _ = batch_run(w, B, H1=H1, f=f, rho0s=rho0s)
    for b in range(B):
        ro = oracle_problem(w, b, H1, f, rho0s)
        assert np.abs(rg[b] - ro).max() <= TOL, (b, np.abs(rg[b] - ro).max())
        assert np.abs(np.einsum("kii->k", rg[b]) - 1).max() <= 1e-12


def test_static_batch_equals_single_problem_path():
    """No drive: every problem equals the single-problem plan (different kernels, same method)."""
    rng = np.random.default_rng(3)
    w = W.CONFIGS[1].with_(n_steps=40)
    B = 4
    rho0s = np.stack([W.random_density_matrix(rng, 2) for _ in range(B)])
    rg, _ = batch_run(w, B, rho0s=rho0s)
    for b in range(B):
        single = Q.Plan(w.with_(rho0=rho0s[b]))
        a, wk = single.alloc()
        rs = single.run(a, wk)
        assert np.abs(rg[b] - rs).max() < 1e-12
        assert np.abs(rg[b] - O.run(P(w, rho0=rho0s[b]))).max() <= TOL


def test_pulse_area_sweep_zero_bath():
    """The paper's sweep without bath: rho_11(T) = sin^2(A/2) for every pulse area A."""
    w0 = W.CONFIGS[0]
    n = 200
    t = w0.dt * (np.arange(n) + 0.5)
    env = np.exp(-((t - t.mean()) / (0.2 * t[-1])) ** 2)
    areas = np.linspace(0.0, 4 * np.pi, 64)
    f = areas[:, None] * env[None, :] / (env.sum() * w0.dt)
    w = w0.with_(kind=W.J_ZERO, n_steps=n, L=5, H=np.zeros((2, 2), complex))
    rg, _ = batch_run(w, len(areas), H1=0.5 * SX, f=f, out_steps=[n])
    assert np.abs(rg[:, 0, 1, 1].real - np.sin(areas / 2) ** 2).max() < 1e-12


def test_quantum_dot_pulse_sweep_with_bath():
    """Sec. III model (super-Ohmic phonon bath, 25 K) driven by pulses of several areas vs the oracle."""
    w0 = W.CONFIGS[0].with_(L=5, n_steps=60)
    t = w0.dt * (np.arange(w0.n_steps) + 0.5)
    env = np.exp(-((t - 2.5) / 1.0) ** 2)
    areas = np.array([0.5, 1.0, 2.0, 3.0]) * np.pi
    f = areas[:, None] * env[None, :] / (env.sum() * w0.dt)
    w = w0.with_(H=np.zeros((2, 2), complex))
    rg, _ = batch_run(w, len(areas), H1=0.5 * SX, f=f, out_steps=[20, 40, 60])
    for b in range(len(areas)):
        ro = oracle_problem(w, b, 0.5 * SX, f, out_steps=[20, 40, 60])
        assert np.abs(rg[b] - ro).max() <= TOL


def test_batch_determinism_and_edges():
    rng = np.random.default_rng(9)
    w = W.random_problem(9, 2, 4, 17)
    H1 = W.random_hermitian(rng, 2)
    f = rng.standard_normal((3, 17))
    a, _ = batch_run(w, 3, H1=H1, f=f)
    b, _ = batch_run(w, 3, H1=H1, f=f)
    assert np.array_equal(a, b)
    # growth-only run (n < L), output subsets, n_steps = 0
    w2 = W.random_problem(10, 2, 6, 4)
    r2, _ = batch_run(w2, 2, out_steps=[0, 2, 4])
    assert np.abs(r2[1] - O.run(P(w2), out_steps=[0, 2, 4])).max() <= TOL
    r3, _ = batch_run(w2.with_(n_steps=0), 2)
    assert np.array_equal(r3[0, 0], w2.rho0)


@pytest.mark.parametrize("M,L,n", [(2, 4, 24), (2, 6, 18), (3, 3, 12)])
def test_per_problem_baths_match_oracle(M, L, n):
    """Temperature / coupling / spectral-family sweep: problem b has its own bath; its eta
    classes come from the device quadrature (qp_eta_device) and its psi rows from k_psi.  Each problem
    vs the oracle run with that bath (its own adaptive G)."""
    rng = np.random.default_rng(70 + 10 * M + L)
    baths = [(W.J_OHMIC_EXP, 0.1, 7.5, 0.2), (W.J_OHMIC_EXP, 0.3, 2.0, 0.0), (W.J_DEBYE, 0.1, 7.5, 1.0),
             (W.J_DEBYE, 0.2, 3.0, 0.05), (W.J_SUPEROHMIC_GAUSS, 0.05, 2.2, 0.3), (W.J_ZERO, 0.0, 1.0, 0.0)]
    B = len(baths)
    w = W.random_problem(700 + M + L, M, L, n, kind=W.J_ZERO)  # base bath unused
    H1 = W.random_hermitian(rng, M)
    f = 0.5 * rng.standard_normal((B, n))
    rg, _ = batch_run(w, B, H1=H1, f=f, baths=baths)
    for b, (kind, xi, wc, kT) in enumerate(baths):
        wb = w.with_(kind=kind, coupling=xi, omega_c=wc, kT=kT)
        ro = oracle_problem(wb, b, H1, f)
        assert np.abs(rg[b] - ro).max() <= TOL, (b, np.abs(rg[b] - ro).max())
        assert np.abs(np.einsum("kii->k", rg[b]) - 1).max() <= 1e-12


def test_per_problem_baths_equal_shared_bath():
    """baths = B copies of the shared bath reproduces the shared-bath batch (device vs host eta: within
    rounding, so within 1e-13 rather than bit for bit)."""
    w = W.CONFIGS[3].with_(L=5, n_steps=30)
    rng = np.random.default_rng(5)
    rho0s = np.stack([W.random_density_matrix(rng, 2) for _ in range(3)])
    a, _ = batch_run(w, 3, rho0s=rho0s)
    b, _ = batch_run(w, 3, rho0s=rho0s, baths=[Q.bath_of(w)] * 3)
    assert np.abs(a - b).max() < 1e-13
