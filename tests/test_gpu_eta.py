"""Device eta setup (qp_eta_device) against the oracle.

The device integrates each class's window kernel in omega on a fixed composite Gauss-Kronrod rule;
the oracle forms the same classes as four-corner differences of its own adaptively integrated G(tau)
(oracle/oracle.c).  The two formulations share nothing but Eqs. 10-16.  Bars: every class
within 2e-15 * max(1, |G((L+1) dt)|) of the oracle (the host quadrature meets 4e-16), within 2e-15 of
the 30-digit mpmath closed forms / quadratures of G
(tests/closed_forms.py) taken through Eqs. 10-16, and a full run from device-computed eta classes within
the BASELINE tolerance of the oracle's rho(t).
"""
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


def oracle_classes(w):
    """[self_interior, self_end, eta_1..L, E_1..L, TI_1..L] from the oracle's eta_pair (Eqs. 10-16)."""
    p = P(w)
    L = w.L
    v = [O.eta_pair(p, 2, 2, -1), O.eta_pair(p, 0, 0, -1)]
    v += [O.eta_pair(p, j + 1, 1, -1) for j in range(1, L + 1)]
    v += [O.eta_pair(p, j, 0, -1) for j in range(1, L + 1)]
    v += [O.eta_pair(p, j, 0, j) for j in range(1, L + 1)]
    return np.array(v), p


def tol_of(w, p):
    return 2e-15 * max(1.0, abs(O.G(p, (w.L + 1) * w.dt)))


def mp_classes(bath, dt, L):
    """Eqs. 10-16 on the Strang windows (reading C.3-1) from 30-digit G(tau) (G(0) = 0)."""
    from tests import closed_forms as C
    kind, xi, wc, kT = bath
    f = {W.J_OHMIC_EXP: C.G_ohmic, W.J_DEBYE: C.G_debye, W.J_SUPEROHMIC_GAUSS: C.G_superohmic}[kind]
    memo = {}

    def G(x):  # x in units of dt
        if x == 0:
            return 0j
        if x not in memo:
            memo[x] = f(xi, wc, kT, x * dt)
        return memo[x]
    v = [G(1), G(0.5)]
    v += [G(j + 1) + G(j - 1) - 2 * G(j) for j in range(1, L + 1)]
    v += [G(j + 0.5) + G(j - 1) - G(j - 0.5) - G(j) for j in range(1, L + 1)]
    v += [G(j) + G(j - 1) - 2 * G(j - 0.5) for j in range(1, L + 1)]
    return np.array(v), max(1.0, abs(G(L + 1)))


BATHS = [  # (kind, coupling, omega_c, kT): the paper's families over a spread of temperatures
    (W.J_OHMIC_EXP, 0.1, 7.5, 0.2), (W.J_OHMIC_EXP, 0.1, 7.5, 0.0), (W.J_OHMIC_EXP, 0.5, 2.0, 0.05),
    (W.J_OHMIC_EXP, 1.0, 1.0, 5.0), (W.J_DEBYE, 0.1, 7.5, 0.2), (W.J_DEBYE, 0.1, 7.5, 0.0),
    (W.J_DEBYE, 0.3, 1.0, 2.0), (W.J_DEBYE, 0.05, 20.0, 0.5),
    (W.J_SUPEROHMIC_GAUSS, 0.027 * np.pi, 2.2, 25 * W.KB_OVER_HBAR_PS_K), (W.J_SUPEROHMIC_GAUSS, 0.1, 1.0, 0.0),
]


@pytest.mark.parametrize("bath", BATHS, ids=lambda b: f"k{b[0]}_wc{b[2]}_kT{b[3]:.3g}")
@pytest.mark.parametrize("dt,L", [(0.25, 14), (0.1, 6), (0.5, 16)])
def test_eta_device_matches_oracle(bath, dt, L):
    w = W.CONFIGS[1].with_(kind=bath[0], coupling=bath[1], omega_c=bath[2], kT=bath[3], dt=dt, L=L)
    ref, p = oracle_classes(w)
    eta, err = Q.eta_device([bath], dt, L, err=True)
    d = np.abs(eta[0] - ref)
    assert d.max() <= tol_of(w, p), (int(d.argmax()), d.max())
    assert np.all(np.isfinite(err))


@pytest.mark.parametrize("bath", [BATHS[i] for i in (0, 2, 4, 6, 7, 8)], ids=lambda b: f"k{b[0]}_wc{b[2]}_kT{b[3]:.3g}")
@pytest.mark.parametrize("dt", [0.25, 0.1])
def test_eta_device_matches_30_digit_G(bath, dt):
    L = 6
    ref, scale = mp_classes(bath, dt, L)
    eta = Q.eta_device([bath], dt, L)[0]
    d = np.abs(eta - ref)
    assert d.max() <= 2e-15 * scale, (int(d.argmax()), d.max())


def test_eta_device_zero_bath_and_host_agreement():
    w = W.CONFIGS[3]  # cfg3 bath (Debye), L = 14
    eta = Q.eta_device([(0, 0.0, 1.0, 0.0), Q.bath_of(w)], w.dt, w.L)
    assert np.all(eta[0] == 0)
    e = Q.Plan(w, out_steps=[0]).eta()
    host = np.concatenate([[e["self_interior"], e["self_end"]], e["eta"], e["E"], e["TI"]])
    assert np.abs(eta[1] - host).max() <= 2e-15


def test_eta_device_batch_is_per_bath_and_deterministic():
    """A 600-bath temperature/coupling sweep (two launches of <= 512 baths) equals the baths run one
    by one, bit for bit, and repeats bit-identically (fixed-order cluster reductions, no atomics)."""
    rng = np.random.default_rng(7)
    baths = [(int(rng.integers(1, 4)), float(rng.uniform(0.01, 0.5)), float(rng.uniform(1, 10)),
              float(rng.choice([0.0, rng.uniform(0.05, 3)]))) for _ in range(600)]
    a = Q.eta_device(baths, 0.2, 7)
    b = Q.eta_device(baths, 0.2, 7)
    assert np.array_equal(a, b)
    for i in (0, 1, 511, 512, 599):
        assert np.array_equal(Q.eta_device([baths[i]], 0.2, 7)[0], a[i]), i


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
def test_run_from_device_eta_matches_oracle(cfg):
    """End to end: host setup with eta from the device (Plan(eta_setup='device')), propagation on the
    GPU, rho(t) against the oracle to 1e-10 and trace 1e-12."""
    w = W.CONFIGS[cfg].with_(n_steps=60)
    w = w.with_(L=min(w.L, 8))
    plan = Q.Plan(w, eta_setup="device")
    ardm, work = plan.alloc()
    rho = plan.run(ardm, work)
    ref = O.run(P(w))
    assert np.abs(rho - ref).max() <= 1e-10
    assert np.abs(np.einsum("kii->k", rho) - 1).max() <= 1e-12
