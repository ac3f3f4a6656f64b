"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Tolerance (BASELINE north_star): max |rho_gpu - rho_oracle| <= 1e-10 and |tr rho - 1| <= 1e-12 at
every requested step.  Both sides get the same seeded physical inputs (workloads.py) and each
computes its own U and eta (independent quadratures, see test_library_host).
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
TR_TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1205_6872_b200 import build as B
    B.build()


def gpu_run(w, out_steps=None, persist=False, **kw):
    """The per-group launch path by default (QP_FLAG_NO_PERSIST: these tests exercise the fused slide
    kernels at small sizes); persist=True lets the library pick the persistent path
    (tests/test_gpu_persist.py)."""
    if not persist:
        kw["flags"] = kw.get("flags", 0) | Q.QP_FLAG_NO_PERSIST
    plan = Q.Plan(w, out_steps=out_steps, **kw)
    ardm, work = plan.alloc()
    rho = plan.run(ardm, work)
    return rho, plan, ardm


def check(rg, ro, tr_tol=TR_TOL):
    err = np.abs(rg - ro).max()
    assert err <= TOL, f"max |d rho| = {err:.3e}"
    tr = np.einsum("kii->k", rg)
    assert np.abs(tr - np.einsum("kii->k", ro)).max() <= tr_tol
    return err


# ----------------------------------------------------------------------------- small configs, every step
@pytest.mark.parametrize("cfg,L,n", [(1, 5, 100), (0, 6, 200), (2, 10, 60), (4, 5, 40), (3, 8, 50)])
def test_config_trajectory(cfg, L, n):
    w = W.CONFIGS[cfg].with_(L=L, n_steps=n)
    rg, _, _ = gpu_run(w)
    ro = O.run(P(w))
    check(rg, ro)
    assert np.abs(np.einsum("kii->k", rg) - 1).max() <= TR_TOL


RANDOM = [(seed, M, L, n, lat) for seed, (M, L, n, lat) in enumerate(
    [(2, 2, 9, True), (2, 3, 11, True), (2, 4, 13, True), (2, 6, 17, True), (2, 7, 20, True), (2, 9, 14, True),
     (3, 2, 8, True), (3, 3, 9, True), (3, 4, 10, True), (3, 5, 9, True), (3, 3, 8, False), (3, 4, 9, False),
     (4, 2, 6, True), (4, 3, 7, True), (4, 3, 6, False), (2, 5, 3, True), (3, 4, 2, True), (2, 8, 8, True)])]


@pytest.mark.parametrize("seed,M,L,n,lat", RANDOM)
def test_random_problems(seed, M, L, n, lat):
    """Random H, rho0, s (lattice and general), all bath kinds; covers growth-only runs (n < L),
    the first slide (k = L), tile layouts with the contracted digit below / above the tile digits."""
    kind = (W.J_OHMIC_EXP, W.J_DEBYE, W.J_SUPEROHMIC_GAUSS)[seed % 3]
    w = W.random_problem(100 + seed, M, L, n, kind=kind, lattice_s=lat)
    rg, _, _ = gpu_run(w)
    ro = O.run(P(w))
    check(rg, ro, tr_tol=1e-12)


def test_G_table_input_matches_oracle():
    """alpha given directly (kind G_TABLE): identical G to both sides -> kernel-only parity."""
    rng = np.random.default_rng(7)
    w = W.random_problem(7, 3, 4, 14)
    G = 0.05 * (rng.standard_normal(2 * 4 + 3) + 1j * rng.standard_normal(2 * 4 + 3))
    G[0] = 0
    rg, _, _ = gpu_run(w, G_in=G)
    ro = O.run(P(w, G_in=G))
    assert np.abs(rg - ro).max() <= 1e-12 * max(1.0, np.abs(ro).max())


def test_n_steps_zero_and_subsets():
    w = W.CONFIGS[1].with_(n_steps=0)
    rg, _, _ = gpu_run(w)
    assert np.array_equal(rg[0], w.rho0)
    w = W.CONFIGS[1].with_(n_steps=23)
    outs = [0, 3, 4, 5, 6, 17, 23]
    rg, _, _ = gpu_run(w, out_steps=outs)
    check(rg, O.run(P(w), out_steps=outs))


def test_mode_equivalence_and_determinism():
    """justFinalPoint vs allPoints final rho bit-identical; run-to-run bit-identical;
    the final ARDM does not depend on the readout schedule."""
    w = W.CONFIGS[2].with_(n_steps=40)
    ra, _, A1 = gpu_run(w)
    rf, _, A2 = gpu_run(w, out_steps=[40])
    rb, _, A3 = gpu_run(w)
    assert np.array_equal(ra[-1], rf[0])
    assert np.array_equal(ra, rb)
    assert torch.equal(A1, A2) and torch.equal(A1, A3)


def test_step_segments_equal_whole_run():
    """Segment boundaries on fusion-group boundaries (k - L multiple of the fusion depth) give the
    whole run bit for bit; a boundary inside a group splits it into shallower launches, which agree
    to rounding."""
    w = W.CONFIGS[4].with_(L=4, n_steps=19)
    whole, _, _ = gpu_run(w)
    for segs, exact in [([(1, 3), (3, 4), (4, 12), (12, 20)], True), ([(1, 3), (3, 4), (4, 11), (11, 20)], False)]:
        plan = Q.Plan(w, flags=Q.QP_FLAG_NO_PERSIST)
        ardm, work = plan.alloc()
        plan.init(ardm, work)
        for k0, k1 in segs:
            plan.steps(k0, k1, ardm, work)
        if exact:
            assert np.array_equal(plan.read_rho(work), whole)
        else:
            assert np.abs(plan.read_rho(work) - whole).max() < 1e-13
    with pytest.raises(Q.QuapiError, match="order"):
        plan.steps(5, 6, ardm, work)


# ----------------------------------------------------------------------------- full BASELINE sizes
# (oracle parity at full size for cfg3 / cfg4 / cfg5: tests/test_gpu_fullsize.py)
def test_cfg3_full_run_invariants():
    """All 500 steps of config 3: trace and Hermiticity at every step; physical populations."""
    rg, _, _ = gpu_run(W.CONFIGS[3])
    assert np.abs(np.einsum("kii->k", rg) - 1).max() <= TR_TOL
    assert np.abs(rg - rg.conj().transpose(0, 2, 1)).max() <= 1e-13
    pops = np.einsum("kii->ki", rg).real
    assert pops.min() > -1e-9 and pops.max() < 1 + 1e-9


def test_zero_coupling_full_size_is_unitary():
    """J = 0 at config 3's size (L = 14): rho_k = U^k rho0 U^+k exactly (no oracle needed)."""
    import scipy.linalg as sla
    w = W.CONFIGS[3].with_(kind=W.J_ZERO, n_steps=60)
    rg, _, _ = gpu_run(w)
    for k in range(0, 61, 3):
        Uk = sla.expm(-1j * w.H * w.dt * k)
        assert np.abs(rg[k] - Uk @ w.rho0 @ Uk.conj().T).max() < 1e-12


def test_pure_dephasing_full_size_closed_form():
    """Diagonal H at L = 14 (full size): rho_ab(t_k) closed form with S_k from G (see oracle tests)."""
    from tests.test_oracle_engine import _S_closed
    E = np.array([0.4, -0.3])
    rng = np.random.default_rng(4)
    rho0 = W.random_density_matrix(rng, 2)
    w = W.CONFIGS[3].with_(H=np.diag(E).astype(complex), rho0=rho0, n_steps=40)
    rg, _, _ = gpu_run(w)
    G = O.G_table(P(w))
    s = w.s
    for k in range(41):
        Sk = _S_closed(G, w.L, k) if k > 0 else 0.0
        ex = np.array([[rho0[a, b] * np.exp(-1j * (E[a] - E[b]) * w.dt * k) *
                        np.exp(-(s[a] - s[b]) * (s[a] * Sk - s[b] * np.conj(Sk))) for b in range(2)] for a in range(2)])
        assert np.abs(rg[k] - ex).max() < 1e-12, k


def test_sigma_x_symmetry_full_size():
    w = W.CONFIGS[3].with_(n_steps=30)
    X = np.array([[0, 1], [1, 0]], dtype=complex)
    rho0 = W.random_density_matrix(np.random.default_rng(5), 2)
    a, _, _ = gpu_run(w.with_(rho0=rho0))
    b, _, _ = gpu_run(w.with_(rho0=X @ rho0 @ X))
    assert np.abs(b - X @ a @ X).max() < 1e-12


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("fuse", [1, 2, 3, 4])
@pytest.mark.parametrize("M,L,n", [(2, 2, 9), (2, 3, 12), (2, 5, 17), (2, 6, 21), (2, 7, 20), (2, 8, 23), (3, 4, 11), (4, 3, 8)])
def test_fusion_depths(fuse, M, L, n, generic):
    """1 to 4 time steps per HBM pass (qp_problem.fuse_steps caps the depth) against the oracle;
    odd n and L exercise partial groups and super-fibres that wrap around the ring.  For M = 2 with
    s = (+1, -1) the symmetric-moment kernels run unless QP_FLAG_GENERIC_MOMENTS is set."""
    if generic and M != 2:
        pytest.skip("symmetric moments are M = 2 only")
    flags = Q.QP_FLAG_GENERIC_MOMENTS if generic else 0
    for lat in (True, False) if M > 2 else (True,):
        w = W.random_problem(300 + 10 * M + L, M, L, n, kind=W.J_DEBYE, lattice_s=lat)
        rg, plan, _ = gpu_run(w, fuse_steps=fuse, flags=flags)
        assert plan.sizes.fuse_steps == min(fuse, L - 1, (4 if L >= 6 else 3) if M == 2 else (2 if M == 3 else 1))
        check(rg, O.run(P(w)))


def test_fusion_grouping_independent_of_segments():
    """Fusion groups are aligned on k - L, so splitting qp_steps at group boundaries is bit-identical."""
    w = W.CONFIGS[2].with_(L=6, n_steps=31)
    whole, _, _ = gpu_run(w)
    plan = Q.Plan(w, flags=Q.QP_FLAG_NO_PERSIST)
    ardm, work = plan.alloc()
    plan.init(ardm, work)
    f = plan.sizes.fuse_steps
    cuts = [1, 6, 6 + f, 6 + 3 * f, 6 + 5 * f, 32]
    for k0, k1 in zip(cuts[:-1], cuts[1:]):
        plan.steps(k0, k1, ardm, work)
    assert np.array_equal(plan.read_rho(work), whole)


@pytest.mark.parametrize("flags", [0, Q.QP_FLAG_NO_TMA, Q.QP_FLAG_GENERIC_MOMENTS,
                                   Q.QP_FLAG_NO_TMA | Q.QP_FLAG_GENERIC_MOMENTS])
@pytest.mark.parametrize("L,n", [(6, 31), (8, 37), (9, 30)])
def test_fused3_load_paths(flags, L, n):
    """k_fused3's load paths against the oracle: per-warp TMA-staged rounds in all four stage views
    (A: 1 <= p0 <= L-3, B: p0 = L-2, C: p0 = L-1, D: p0 = 0) and plain loads in lane maps 0 and 1
    (QP_FLAG_NO_TMA), 32-byte loads/stores along ring slot 0, symmetric and generic moments;
    L >= 6 so that every start slot p0 occurs."""
    w = W.random_problem(500 + L, 2, L, n, kind=W.J_OHMIC_EXP)
    rg, plan, _ = gpu_run(w, flags=flags, fuse_steps=3)
    assert plan.sizes.fuse_steps == 3
    check(rg, O.run(P(w)))


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("L", [6, 7, 8, 9, 10, 11, 12, 13])
def test_fused4_every_start_slot(L, generic):
    """k_fused4 (four steps per pass, TMA load + store of 8-fibre rounds) against the oracle at every
    start slot p0: odd L visit every residue, so all stage-layout types occur (slot 0 outer: fibres
    as the chunks of a stage row; slot 0 = inner digit 0..3: fibres as row blocks), with run A of one
    digit (p0 = 1, fibre bit 2 in run B) and the readout of every step."""
    n = 2 * L + 4 * L + 3  # >= L start slots of four-step groups after the growth
    w = W.random_problem(700 + L, 2, L, n, kind=W.J_DEBYE)
    flags = Q.QP_FLAG_GENERIC_MOMENTS if generic else 0
    rg, plan, _ = gpu_run(w, flags=flags)
    assert plan.sizes.fuse_steps == 4
    check(rg, O.run(P(w)))


@pytest.mark.parametrize("kind", [W.J_OHMIC_EXP, W.J_DEBYE])
@pytest.mark.parametrize("L", [4, 5, 6, 7])
def test_fused2t_every_start_slot(L, kind):
    """k_fused2t (M = 3, s = (1, 0, -1): two steps per pass, TMA load + store of 27-fibre units,
    conjugate-pair class moments) against the oracle; odd L visit every start slot, so all four TMA
    views occur (p0 = 0, p0 = 1, 2 <= p0 <= L-2, p0 = L-1).  The same run through k_fused2s
    (QP_FLAG_NO_TMA: cp.async staging, nine complex products per moment) agrees to rounding."""
    n = 3 * L + 3
    w = W.random_problem(900 + L, 3, L, n, kind=kind)
    assert tuple(w.s) == (1.0, 0.0, -1.0)
    rg, plan, _ = gpu_run(w)
    assert plan.sizes.fuse_steps == 2 and plan.sizes.block == 576  # the k_fused2t launch configuration
    check(rg, O.run(P(w)))
    rs, plan_s, _ = gpu_run(w, flags=Q.QP_FLAG_NO_TMA)
    assert plan_s.sizes.block == 288
    assert np.abs(rg - rs).max() <= 1e-13
    r2, _, _ = gpu_run(w)  # fixed grid, fixed unit -> CTA assignment and reduction order: bit-identical
    assert np.array_equal(rg, r2)
