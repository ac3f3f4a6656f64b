"""Sharded multi-GPU path emulated on one GPU: G ranks (plans) in one process, all-to-all by device
copies.  The sharded run must reproduce the single-GPU run (and the oracle) -- same kernels, different
data layout and launch split, so agreement is to rounding (1e-13), not bitwise."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from paper_1205_6872_b200 import quapi as Q  # noqa: E402
from paper_1205_6872_b200 import sharded as SH  # noqa: E402
from paper_1205_6872_b200 import workloads as W  # noqa: E402
from tests.test_oracle_engine import P  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def single(w, out_steps=None):
    pl = Q.Plan(w, out_steps=out_steps)
    a, wk = pl.alloc()
    return pl.run(a, wk)


@pytest.mark.parametrize("G,M,L,n,lat", [(2, 2, 5, 23, True), (4, 2, 6, 30, True), (8, 2, 6, 25, True),
                                          (3, 2, 7, 20, True), (2, 3, 4, 14, True), (3, 3, 5, 12, False),
                                          (2, 2, 4, 3, True), (2, 2, 9, 40, False)])
def test_sharded_matches_single_gpu(G, M, L, n, lat):
    w = W.random_problem(500 + G * 10 + L, M, L, n, kind=W.J_DEBYE, lattice_s=lat)
    ranks = [SH.ShardRank(w, G, r) for r in range(G)]
    parts = SH.run_sharded(ranks, SH.emulated_exchange)
    rho = SH.combine_rho(parts, ranks[0].plan.out_steps, w.L)
    ref = single(w)
    assert np.abs(rho - ref).max() < 1e-13, np.abs(rho - ref).max()
    assert np.abs(rho - O.run(P(w))).max() < 1e-10
    s = ranks[0].sizes
    assert s.segment_steps == L - s.shard_slots
    assert sum(r.sizes.local_entries for r in ranks) == w.N ** L


def test_sharded_full_size_cfg3_two_ranks():
    """Config 3 (4^14) split over 2 emulated ranks for 40 steps (3 re-shards)."""
    w = W.CONFIGS[3].with_(n_steps=W.CONFIGS[3].L + 40)
    outs = list(range(0, w.n_steps + 1, 3))
    ranks = [SH.ShardRank(w, 2, r, out_steps=outs) for r in range(2)]
    parts = SH.run_sharded(ranks, SH.emulated_exchange)
    rho = SH.combine_rho(parts, ranks[0].plan.out_steps, w.L)
    ref = single(w, outs)
    assert np.abs(rho - ref).max() < 1e-13
    assert np.abs(np.einsum("kii->k", rho) - 1).max() < 1e-12
