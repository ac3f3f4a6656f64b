"""World-size-2 gloo test (CPU) of the sharded path's exchange contract.

Each process configures a sharded plan through the C ABI (host only), takes the per-peer entry
counts from qp_shard_counts, builds its segment-0 shard with an independent numpy derivation of the
layout documented in include/quapi.h / DESIGN §7 (payload = global ARDM index of every entry), packs
it in the documented order, exchanges with torch.distributed.all_to_all_single over gloo, unpacks,
and checks that every rank now holds exactly the entries of its segment-1 shard, each once.
The CUDA pack/unpack kernels implementing the same contract are checked on the GPU
(tests/test_gpu_sharded.py)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layout(L, N, z, G, j):
    """Shard slots of segment j (ascending) and the owned combo ranges."""
    k = L + j * (L - z)
    Z = sorted(((k - 1 - i) % L) for i in range(z))
    NZ = N ** z
    base, extra = divmod(NZ, G)
    n_own = [base + (1 if r < extra else 0) for r in range(G)]
    c_lo = [r * base + min(r, extra) for r in range(G)]
    return Z, c_lo, n_own


def _gidx(L, N, assign):
    return sum(int(assign[q]) * N ** q for q in range(L))


def _combo_digits(c, N, z):
    return [(c // N ** i) % N for i in range(z)]


def _worker(rank, world, port, L, M, out):
    import torch.distributed as dist

    from paper_1205_6872_b200 import quapi as Q
    from paper_1205_6872_b200 import workloads as W
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = M * M
        w = W.random_problem(1, M, L, 3 * L)
        plan = Q.Plan(w)
        sz = plan.shard(world, rank)
        z = sz.shard_slots
        send_c, recv_c = plan.shard_counts()
        Z0, c_lo, n_own = _layout(L, N, z, world, 0)
        Z1, _, _ = _layout(L, N, z, world, 1)
        others = [q for q in range(L) if q not in Z0 and q not in Z1]
        rest = N ** len(others)
        assert sz.segment_steps == L - z and sz.local_entries == n_own[rank] * N ** (L - z)
        assert send_c == [n_own[rank] * n_own[r] * rest for r in range(world)]
        assert recv_c == [n_own[r] * n_own[rank] * rest for r in range(world)]
        # pack (documented order): per destination rank r: [my Z0 combo][r's Z1 combo][others ascending]
        send = []
        for r in range(world):
            for b in range(n_own[rank]):
                c = c_lo[rank] + b
                for b1 in range(n_own[r]):
                    c1 = c_lo[r] + b1
                    for o in range(rest):
                        a = np.zeros(L, dtype=np.int64)
                        for i, q in enumerate(Z0):
                            a[q] = _combo_digits(c, N, z)[i]
                        for i, q in enumerate(Z1):
                            a[q] = _combo_digits(c1, N, z)[i]
                        for t, q in enumerate(others):
                            a[q] = (o // N ** t) % N
                        send.append(_gidx(L, N, a))
        st = torch.tensor(send, dtype=torch.float64)
        rt = torch.empty(sum(recv_c), dtype=torch.float64)
        dist.all_to_all_single(rt, st, output_split_sizes=recv_c, input_split_sizes=send_c)
        got = sorted(int(x) for x in rt.tolist())
        # expected: every entry whose Z1 combo I own
        exp = []
        for b1 in range(n_own[rank]):
            c1 = c_lo[rank] + b1
            for o in range(N ** (L - z)):
                a = np.zeros(L, dtype=np.int64)
                for i, q in enumerate(Z1):
                    a[q] = _combo_digits(c1, N, z)[i]
                for t, q in enumerate([q for q in range(L) if q not in Z1]):
                    a[q] = (o // N ** t) % N
                exp.append(_gidx(L, N, a))
        out[rank] = (got == sorted(exp), len(got), len(set(got)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M,L", [(2, 5), (3, 4)])
def test_exchange_contract_world_size_2(M, L):
    import torch.multiprocessing as mp
    from paper_1205_6872_b200 import build as B
    B.build()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), L, M, out), nprocs=2, join=True)
    for r in range(2):
        ok, n, nuniq = out[r]
        assert ok and n == nuniq, (r, out[r])
