"""Sharded multi-GPU path on one GPU.

* Emulated: G ranks (plans) in one process, all-to-all by device copies.  The sharded run must
  reproduce the single-GPU run (and the oracle) -- same kernels, different data layout and launch
  split, so agreement is to rounding (1e-13), not bitwise.  Each rank holds two buffers of N^L / G
  entries (+ workspace): no rank ever allocates the N^L ARDM (shard-native growth).
* Distributed: two processes sharing the GPU, torch.distributed over gloo: the real CUDA pack ->
  all_to_all_single -> CUDA unpack path and the all-gather + library sum of rho (the NCCL branch is
  the same code with device tensors).
"""
import os
import socket

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
    from paper_1205_6872_b200 import build as B
    B.build()


def single(w, out_steps=None, **kw):
    pl = Q.Plan(w, out_steps=out_steps, **kw)
    a, wk = pl.alloc()
    return pl.run(a, wk)


@pytest.mark.parametrize("G,M,L,n,lat", [(2, 2, 5, 23, True), (4, 2, 6, 30, True), (8, 2, 6, 25, True),
                                          (3, 2, 7, 20, True), (2, 3, 4, 14, True), (3, 3, 5, 12, False),
                                          (2, 2, 4, 3, True), (2, 2, 9, 40, False), (8, 2, 8, 41, True),
                                          (4, 2, 11, 40, True), (8, 3, 5, 17, True),
                                          # M = 3, s = (1, 0, -1), >= 4 local slots: shard blocks on k_fused2t
                                          (2, 3, 7, 30, True), (3, 3, 6, 26, True)])
def test_sharded_matches_single_gpu(G, M, L, n, lat):
    w = W.random_problem(500 + G * 10 + L, M, L, n, kind=W.J_DEBYE, lattice_s=lat)
    ranks = [SH.ShardRank(w, G, r) for r in range(G)]
    for r in ranks:  # two shard buffers per rank, never the full ARDM
        assert r.local.numel() == 2 * r.sizes.local_entries and r.xbuf.numel() == 2 * r.sizes.xbuf_entries
        assert r.sizes.local_entries < w.N ** L
    assert sum(r.sizes.local_entries for r in ranks) == w.N ** L
    SH.run_sharded(ranks, SH.emulated_exchange)
    rho = SH.emulated_rho(ranks)
    ref = single(w)
    assert np.abs(rho - ref).max() < 1e-13, np.abs(rho - ref).max()
    assert np.abs(rho - O.run(P(w))).max() < 1e-10
    s = ranks[0].sizes
    assert s.segment_steps == L - s.shard_slots


def test_sharded_full_size_cfg3_two_ranks():
    """Config 3 (4^14) split over 2 emulated ranks for 40 slide steps (3 re-shards)."""
    w = W.CONFIGS[3].with_(n_steps=W.CONFIGS[3].L + 40)
    outs = list(range(0, w.n_steps + 1, 3))
    ranks = [SH.ShardRank(w, 2, r, out_steps=outs) for r in range(2)]
    SH.run_sharded(ranks, SH.emulated_exchange)
    rho = SH.emulated_rho(ranks)
    del ranks
    torch.cuda.empty_cache()
    ref = single(w, outs)
    assert np.abs(rho - ref).max() < 1e-13
    assert np.abs(np.einsum("kii->k", rho) - 1).max() < 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dist_worker(rank, world, port, L, n, out_path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        w = W.random_problem(900 + L, 2, L, n, kind=W.J_DEBYE)
        rho = SH.solve_distributed(w)
        if rank == 0:
            np.save(out_path, rho)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,L,n", [(2, 7, 30), (2, 9, 33)])
def test_distributed_two_processes_gloo(world, L, n, tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "rho.npy")
    mp.spawn(_dist_worker, args=(world, _free_port(), L, n, out), nprocs=world, join=True)
    rho = np.load(out)
    w = W.random_problem(900 + L, 2, L, n, kind=W.J_DEBYE)
    assert np.abs(rho - single(w)).max() < 1e-13
    assert np.abs(rho - O.run(P(w))).max() < 1e-10
