"""GPU parity of the persistent path (persist.cu: k_small): a small ARDM
(<= QP_PERSIST_MAX_BYTES) runs all slide steps of one qp_steps call in one single-CTA launch, the ARDM
and every table in shared memory, one step at a time.  Checked against the oracle (tolerance of
test_gpu_parity), against the per-group launch path (QP_FLAG_NO_PERSIST, to rounding), for one
launch per call, bit-identical results under any segmentation, and run-to-run determinism.
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


CASES = [(2, 3, 17, True, 0), (2, 5, 40, True, 0), (2, 6, 33, True, 0), (2, 6, 21, True, Q.QP_FLAG_GENERIC_MOMENTS),
         (2, 4, 25, False, Q.QP_FLAG_GENERIC_MOMENTS), (3, 2, 12, True, 0), (3, 3, 14, True, 0),
         (3, 3, 11, False, 0), (4, 2, 8, True, 0), (4, 2, 7, False, 0), (2, 2, 9, True, 0)]


@pytest.mark.parametrize("M,L,n,lat,flags", CASES)
def test_persistent_matches_oracle_and_launch_path(M, L, n, lat, flags):
    w = W.random_problem(900 + 10 * M + L, M, L, n, kind=W.J_DEBYE, lattice_s=lat)
    rp, plan, _ = gpu_run(w, persist=True, flags=flags)
    sz = plan.sizes
    assert sz.persistent == 1 and sz.fuse_steps == 1 and sz.grid == 1
    check(rp, O.run(P(w)))
    rl, pl, _ = gpu_run(w, flags=flags)
    assert pl.sizes.persistent == 0
    assert np.abs(rp - rl).max() < 1e-13


@pytest.mark.parametrize("cfg,L,n", [(1, 5, 100), (2, 6, 60), (0, 6, 90), (4, 3, 40)])
def test_persistent_configs(cfg, L, n):
    w = W.CONFIGS[cfg].with_(L=L, n_steps=n)
    rp, plan, _ = gpu_run(w, persist=True)
    assert plan.sizes.persistent == 1
    check(rp, O.run(P(w)))


def test_tables_too_large_for_one_cta_fall_back_to_launches():
    """M = 4, L = 3, generic classes: a 64 KB ARDM but 350 KB of factor tables -- qp_init keeps the
    per-step launches (persistent reads 0 after init), same results."""
    w = W.random_problem(977, 4, 3, 7, kind=W.J_DEBYE, lattice_s=False)
    plan = Q.Plan(w)
    assert plan.sizes.persistent == 1  # chosen at plan creation ...
    ardm, work = plan.alloc()
    rho = plan.run(ardm, work)
    assert plan.sizes.persistent == 0  # ... and dropped at qp_init: the tables do not fit
    check(rho, O.run(P(w)))


def test_sparse_readout_slots():
    w = W.CONFIGS[1].with_(L=6, n_steps=41)
    outs = [0, 2, 6, 7, 8, 19, 20, 33, 41]
    rp, plan, _ = gpu_run(w, out_steps=outs, persist=True)
    assert plan.sizes.persistent == 1
    check(rp, O.run(P(w), out_steps=outs))


def test_one_launch_per_call_segments_and_determinism():
    w = W.CONFIGS[2].with_(L=6, n_steps=40)
    whole, _, A1 = gpu_run(w, persist=True)
    again, _, A2 = gpu_run(w, persist=True)
    assert np.array_equal(whole, again) and torch.equal(A1, A2)
    for cuts in ([(1, 6), (6, 9), (9, 25), (25, 41)], [(1, 4), (4, 8), (8, 10), (10, 11), (11, 41)]):
        plan = Q.Plan(w)
        ardm, work = plan.alloc()
        plan.init(ardm, work)
        assert plan.sizes.persistent == 1 and plan.sizes.fuse_steps == 1
        launches = [plan.steps(k0, k1, ardm, work) for k0, k1 in cuts]
        assert all(n == 1 for (k0, k1), n in zip(cuts, launches) if k0 >= 6)  # one launch per call
        assert np.array_equal(plan.read_rho(work), whole)  # one step per group: any cut is exact
