"""GPU parity of the persistent path (k_persist_r): a small, L2-resident ARDM runs all
slide steps of one qp_steps call in one cooperative launch, fusion groups of depth <= 2 (M = 2) or 1
separated by a grid-wide barrier.  Checked against the oracle (tolerance of test_gpu_parity), against
the per-group launch path (QP_FLAG_NO_PERSIST, to rounding), for one launch per call, bit-identical
segmentation at group boundaries and run-to-run determinism.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from paper_1205_6872_b200 import quapi as Q  # noqa: E402
from paper_1205_6872_b200 import workloads as W  # noqa: E402
from tests.test_gpu_parity import check, gpu_run  # noqa: E402
from tests.test_oracle_engine import P  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1205_6872_b200 import build as B
    B.build()


CASES = [(2, 3, 17, True, 0), (2, 5, 40, True, 0), (2, 8, 33, True, 0), (2, 9, 21, True, Q.QP_FLAG_GENERIC_MOMENTS),
         (2, 6, 25, False, Q.QP_FLAG_GENERIC_MOMENTS), (3, 3, 12, True, 0), (3, 5, 14, True, 0),
         (3, 4, 11, False, 0), (4, 3, 8, True, 0), (4, 3, 7, False, 0), (2, 2, 9, True, 0)]


@pytest.mark.parametrize("M,L,n,lat,flags", CASES)
def test_persistent_matches_oracle_and_launch_path(M, L, n, lat, flags):
    w = W.random_problem(900 + 10 * M + L, M, L, n, kind=W.J_DEBYE, lattice_s=lat)
    rp, plan, _ = gpu_run(w, persist=True, flags=flags)
    assert plan.sizes.persistent in (1, 2)
    assert plan.sizes.fuse_steps == min(L - 1, 2 if M == 2 else 1)
    check(rp, O.run(P(w)))
    rl, pl, _ = gpu_run(w, flags=flags)
    assert pl.sizes.persistent == 0
    assert np.abs(rp - rl).max() < 1e-13


@pytest.mark.parametrize("cfg,L,n", [(1, 5, 100), (2, 10, 60), (0, 6, 90)])
def test_persistent_configs(cfg, L, n):
    w = W.CONFIGS[cfg].with_(L=L, n_steps=n)
    rp, plan, _ = gpu_run(w, persist=True)
    assert plan.sizes.persistent == (2 if w.N ** L * 16 <= 32 << 10 else 1)
    check(rp, O.run(P(w)))


def test_sparse_readout_slots():
    w = W.CONFIGS[1].with_(L=6, n_steps=41)
    outs = [0, 2, 6, 7, 8, 19, 20, 33, 41]
    rp, plan, _ = gpu_run(w, out_steps=outs, persist=True)
    assert plan.sizes.persistent in (1, 2)
    check(rp, O.run(P(w), out_steps=outs))


@pytest.mark.parametrize("M,L,n", [(2, 4, 30), (2, 5, 27), (3, 3, 15), (4, 2, 9)])
def test_single_cta_path(M, L, n):
    """ARDM + tables in one CTA's shared memory (persistent == 2 after init): oracle parity, agreement
    with the cooperative grid and the per-group launches, one launch per call."""
    w = W.random_problem(950 + 10 * M + L, M, L, n, kind=W.J_OHMIC_EXP)
    rp, plan, _ = gpu_run(w, persist=True)
    assert plan.sizes.persistent == 2 and plan.sizes.grid == 1
    check(rp, O.run(P(w)))
    rl, _, _ = gpu_run(w)
    assert np.abs(rp - rl).max() < 1e-13
    plan = Q.Plan(w)
    ardm, work = plan.alloc()
    plan.init(ardm, work)
    plan.steps(1, L, ardm, work)
    assert plan.steps(L, n + 1, ardm, work) == 1
    assert np.array_equal(plan.read_rho(work), rp)


def test_one_launch_per_call_segments_and_determinism():
    w = W.CONFIGS[2].with_(L=7, n_steps=40)
    whole, _, A1 = gpu_run(w, persist=True)
    again, _, A2 = gpu_run(w, persist=True)
    assert np.array_equal(whole, again) and torch.equal(A1, A2)
    plan = Q.Plan(w)
    assert plan.sizes.persistent == 1 and plan.sizes.fuse_steps == 2
    ardm, work = plan.alloc()
    plan.init(ardm, work)
    assert plan.sizes.persistent == 1  # 4^7 entries: the cooperative grid, not one CTA
    launches = [plan.steps(k0, k1, ardm, work) for k0, k1 in [(1, 7), (7, 9), (9, 25), (25, 41)]]
    assert launches[1:] == [1, 1, 1]  # slide steps: one cooperative launch per call
    assert np.array_equal(plan.read_rho(work), whole)  # cuts on group boundaries (k - L even)
    plan = Q.Plan(w)
    ardm, work = plan.alloc()
    plan.init(ardm, work)
    for k0, k1 in [(1, 7), (7, 10), (10, 41)]:  # a cut inside a group splits it
        plan.steps(k0, k1, ardm, work)
    assert np.abs(plan.read_rho(work) - whole).max() < 1e-13
