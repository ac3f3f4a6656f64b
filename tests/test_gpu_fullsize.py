"""Full-size parity at the BASELINE configs (north_star: rho within 1e-10 of the oracle on all five
configs), in the launch configuration bench.py times.

* cfg3 (L = 14) against the oracle through k = 2L + 3 = 31: every ring slot p0 is contracted at least
  once as the first slot of a fused group, so all four TMA stage views (A: p0 = 1..L-3, B: L-2,
  C: L-1, D: 0) and a full wrap of the ring are compared element by element.
* cfg4 (M = 3, L = 9) against the oracle through k = L + 9.
* cfg5 (L = 16, 4^16 entries = 69 GB) on one B200 against the closed forms that need no oracle
  (SURVEY 8(c) C.4): zero coupling (rho_k = U^k rho0 U^-k, pins K, the contraction and the
  ring-slot 'last' digit) and pure dephasing (pins every eta class, the Strang tiling and the
  truncation hand-off at k = L + 1), 48 steps = three ring wraps.  With >= 150 GB of free host RAM
  cfg5 is also compared with the oracle through k = L + 4 (QUAPI_CFG5_ORACLE=0 skips it).
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from paper_1205_6872_b200 import quapi as Q  # noqa: E402
from paper_1205_6872_b200 import workloads as W  # noqa: E402
from tests.test_oracle_engine import P, _S_closed  # noqa: E402

TOL = 1e-10
TR_TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1205_6872_b200 import build as B
    B.build()


def gpu_rho(w, out_steps=None, **kw):
    plan = Q.Plan(w, out_steps=out_steps, **kw)
    ardm, work = plan.alloc()
    rho = plan.run(ardm, work)
    sz = plan.sizes
    del ardm, work
    torch.cuda.empty_cache()
    return rho, sz


def check(rg, ro):
    err = float(np.abs(rg - ro).max())
    assert err <= TOL, f"max |d rho| = {err:.3e}"
    tr = np.einsum("kii->k", rg)
    assert np.abs(tr - 1).max() <= TR_TOL
    return err


def _need_hbm(gb):
    if torch.cuda.get_device_properties(0).total_memory < gb * 1e9:
        pytest.skip(f"needs > {gb} GB of device memory")


def test_cfg3_full_size_every_view_and_ring_wrap():
    """The bench's launch configuration (four steps per pass, k_fused4) and the three-step kernel with
    its four TMA stage views (k_fused3), both against one oracle run."""
    w = W.CONFIGS[3]
    w = w.with_(n_steps=2 * w.L + 3)
    ro = O.run(P(w))
    rg, sz = gpu_rho(w)
    assert sz.ardm_entries == 4 ** 14 and sz.fuse_steps == 4
    check(rg, ro)
    rg3, sz3 = gpu_rho(w, fuse_steps=3)
    assert sz3.fuse_steps == 3
    check(rg3, ro)


def test_cfg4_full_size_parity():
    w = W.CONFIGS[4]
    w = w.with_(n_steps=w.L + 9)
    rg, sz = gpu_rho(w)
    assert sz.ardm_entries == 9 ** 9
    check(rg, O.run(P(w)))


def test_cfg5_full_size_zero_coupling():
    import scipy.linalg as sla
    _need_hbm(80)
    w = W.CONFIGS[5].with_(kind=W.J_ZERO, n_steps=48)
    rho0 = W.random_density_matrix(np.random.default_rng(16), 2)
    w = w.with_(rho0=rho0)
    rg, sz = gpu_rho(w)
    assert sz.ardm_entries == 4 ** 16
    for k in range(w.n_steps + 1):
        Uk = sla.expm(-1j * w.H * w.dt * k)
        assert np.abs(rg[k] - Uk @ w.rho0 @ Uk.conj().T).max() < 1e-12, k


def test_cfg5_full_size_pure_dephasing():
    _need_hbm(80)
    E = np.array([0.35, -0.45])
    rho0 = W.random_density_matrix(np.random.default_rng(17), 2)
    w = W.CONFIGS[5].with_(H=np.diag(E).astype(complex), rho0=rho0, n_steps=48)
    rg, _ = gpu_rho(w)
    G = O.G_table(P(w))
    s = w.s
    for k in range(w.n_steps + 1):
        Sk = _S_closed(G, w.L, k) if k > 0 else 0.0
        ex = np.array([[rho0[a, b] * np.exp(-1j * (E[a] - E[b]) * w.dt * k) *
                        np.exp(-(s[a] - s[b]) * (s[a] * Sk - s[b] * np.conj(Sk))) for b in range(2)] for a in range(2)])
        assert np.abs(rg[k] - ex).max() < 1e-12, (k, np.abs(rg[k] - ex).max())


def test_cfg5_full_size_sigma_x_symmetry():
    """Metamorphic (C.4): for H = -Delta sigma_x and s = +-1, rho(t; X rho0 X) = X rho(t; rho0) X exactly
    up to rounding -- pins the lag-to-digit mapping with a non-trivial bath at L = 16."""
    _need_hbm(80)
    X = np.array([[0, 1], [1, 0]], dtype=complex)
    rho0 = W.random_density_matrix(np.random.default_rng(18), 2)
    w = W.CONFIGS[5].with_(n_steps=36)
    a, _ = gpu_rho(w.with_(rho0=rho0))
    b, _ = gpu_rho(w.with_(rho0=X @ rho0 @ X))
    assert np.abs(b - X @ a @ X).max() < 1e-12
    assert np.abs(np.einsum("kii->k", a) - 1).max() <= TR_TOL


def _host_ram_free_gb():
    try:
        import psutil
        return psutil.virtual_memory().available / 1e9
    except Exception:
        return 0.0


def test_cfg5_full_size_parity_with_oracle():
    """cfg5 against the oracle (needs 2 x 69 GB of host RAM for the oracle's double buffer)."""
    _need_hbm(80)
    if os.environ.get("QUAPI_CFG5_ORACLE", "1") == "0" or _host_ram_free_gb() < 150:
        pytest.skip(f"oracle at cfg5 needs >= 150 GB of free host RAM (have {_host_ram_free_gb():.0f} GB)")
    w = W.CONFIGS[5]
    w = w.with_(n_steps=w.L + 4)
    rg, _ = gpu_rho(w)
    check(rg, O.run(P(w)))
