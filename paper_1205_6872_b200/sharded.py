"""Sharded multi-GPU QUAPI propagation: one process per GPU, torch.distributed.

Each rank holds the ARDM entries of its owned value combos of the z shard ring slots; the L - z
steps of a segment run shard-locally in the library's fused kernel; between segments the data is
re-sharded with one all-to-all (`all_to_all_single`, NCCL over NVLink on B200) between the
library's pack and unpack kernels.  Growth steps (k < L) run replicated on the full ARDM, then each
rank extracts its blocks.  rho of slide steps is the sum over ranks of the per-rank partials (fixed
rank order on rank 0); growth-step rho is complete on every rank.

`exchange` is pluggable so the same driver runs with a real process group or with an in-process
emulation of G ranks on one GPU (tests).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import numpy as np

from . import quapi as Q
from . import workloads as W


def segment_bounds(L: int, seg_len: int, n_steps: int):
    """Slide-step segments [k0, k1) (k0 >= L) of a sharded run."""
    out, k = [], L
    while k <= n_steps:
        k1 = min(k + seg_len, n_steps + 1)
        out.append((k, k1))
        k = k1
    return out


class ShardRank:
    """One rank's state of a sharded run (plan, local blocks, exchange buffers)."""

    def __init__(self, w: W.Workload, n_ranks: int, rank: int, out_steps=None, device="cuda", stream=None):
        import torch
        self.w, self.G, self.rank, self.device, self.stream = w, n_ranks, rank, device, stream
        self.plan = Q.Plan(w, out_steps=out_steps)
        self.sizes = self.plan.shard(n_ranks, rank)
        self.send_counts, self.recv_counts = self.plan.shard_counts()
        ps = self.plan.sizes
        self.work = torch.empty((ps.work_bytes + 7) // 8, dtype=torch.float64, device=device)
        self.local = torch.empty(2 * self.sizes.max_local_entries, dtype=torch.float64, device=device)
        self.send = torch.empty(2 * max(1, self.sizes.exchange_entries), dtype=torch.float64, device=device)
        self.recv = torch.empty(2 * max(1, sum(self.recv_counts)), dtype=torch.float64, device=device)
        self.launches = 0

    def growth_and_extract(self):
        """qp_init + replicated growth on a full ARDM, then this rank's segment-0 blocks."""
        import torch
        full = torch.empty(2 * self.plan.sizes.ardm_entries, dtype=torch.float64, device=self.device)
        self.plan.init(full, self.work, self.stream)
        self.launches += self.plan.steps(1, min(self.w.L, self.w.n_steps + 1), full, self.work, self.stream)
        if self.w.n_steps >= self.w.L:
            self.plan.shard_extract(full, self.local, self.stream)
            self.launches += 1
        del full


def advance(ranks: List[ShardRank], k_from: int, k_to: int, exchange: Callable[[List[ShardRank]], None]) -> int:
    """Run slide steps k_from..k_to-1 (k_from >= L) on every local rank, re-sharding (pack ->
    exchange -> unpack) whenever a segment boundary is crossed and further steps follow.
    Returns the number of kernel launches on one rank."""
    L, seg = ranks[0].w.L, ranks[0].sizes.segment_steps
    n = 0
    k = k_from
    while k < k_to:
        seg_end = L + ((k - L) // seg + 1) * seg
        k1 = min(seg_end, k_to)
        for r in ranks:
            n_r = r.plan.shard_steps(k, k1, r.local, r.work, r.stream)
            r.launches += n_r
        n += n_r
        k = k1
        if k == seg_end and k <= ranks[0].w.n_steps:  # boundary reached and the run continues
            for r in ranks:
                r.plan.shard_pack(r.local, r.send, r.stream)
                r.launches += r.G
            exchange(ranks)
            for r in ranks:
                r.plan.shard_unpack(r.recv, r.local, r.stream)
                r.launches += r.G
            n += 2 * ranks[0].G
    return n


def run_sharded(ranks: List[ShardRank], exchange: Callable[[List[ShardRank]], None]) -> List[np.ndarray]:
    """Drive all local ranks (one per process in the distributed case) through the whole run.
    `exchange(ranks)` must fill every rank's `recv` from the ranks' `send` buffers (all-to-all)."""
    w = ranks[0].w
    for r in ranks:
        r.growth_and_extract()
    if w.n_steps >= w.L:
        advance(ranks, w.L, w.n_steps + 1, exchange)
    return [r.plan.read_rho(r.work, r.stream) for r in ranks]


def combine_rho(partials: Sequence[np.ndarray], out_steps: Sequence[int], L: int) -> np.ndarray:
    """Slide-step rho = sum of the rank partials in rank order; growth-step rho from rank 0."""
    out = np.array(partials[0], copy=True)
    slide = np.asarray(out_steps) >= L
    for p in partials[1:]:
        out[slide] = out[slide] + p[slide]
    return out


def emulated_exchange(ranks: List[ShardRank]):
    """All-to-all among ranks living in this process (device copies; tests / single-GPU emulation)."""
    G = len(ranks)
    soff = [np.concatenate([[0], np.cumsum(r.send_counts)]) for r in ranks]
    for dst in range(G):
        off = 0
        for src in range(G):
            n = ranks[src].send_counts[dst]
            a = 2 * int(soff[src][dst])
            ranks[dst].recv[2 * off:2 * (off + n)].copy_(ranks[src].send[a:a + 2 * n])
            off += n


def dist_exchange(group=None):
    """All-to-all through torch.distributed (NCCL over NVLink on the B200 box)."""
    import torch.distributed as dist

    def ex(ranks: List[ShardRank]):
        (r,) = ranks
        recv, send = r.recv[:2 * sum(r.recv_counts)], r.send[:2 * sum(r.send_counts)]
        kw = dict(output_split_sizes=[2 * c for c in r.recv_counts],
                  input_split_sizes=[2 * c for c in r.send_counts], group=group)
        if dist.get_backend(group) == "gloo":  # host-staged (tests on one GPU); NCCL moves device memory
            import torch
            torch.cuda.synchronize()
            rc = recv.cpu()
            dist.all_to_all_single(rc, send.cpu(), **kw)
            recv.copy_(rc)
        else:
            dist.all_to_all_single(recv, send, **kw)
    return ex


def solve_distributed(w: W.Workload, out_steps: Optional[Sequence[int]] = None, group=None):
    """Sharded run on the current process group (one rank per GPU).  Returns rho on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist
    G, rank = dist.get_world_size(group), dist.get_rank(group)
    me = ShardRank(w, G, rank, out_steps=out_steps, device=f"cuda:{torch.cuda.current_device()}")
    (part,) = run_sharded([me], dist_exchange(group))
    t = torch.from_numpy(part.view(np.float64).copy()).to(me.device)
    gathered = [torch.empty_like(t) for _ in range(G)] if rank == 0 else None
    dist.gather(t, gathered, dst=0, group=group)
    if rank != 0:
        return None
    parts = [g.cpu().numpy().view(np.complex128).reshape(part.shape) for g in gathered]
    steps = me.plan.out_steps
    return combine_rho(parts, steps, w.L)
