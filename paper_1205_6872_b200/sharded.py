"""Sharded multi-GPU QUAPI propagation: one process per GPU, torch.distributed.

Argument marshalling and buffer plumbing only (include/quapi.h, sharded execution): each rank holds
two device buffers of its shard (local + exchange) and the workspace -- never the N^L ARDM.  Growth
runs replicated while the tensor is at most one block (N^(L-z) entries) and then produces only the
rank's own combos; the L - z steps of a segment run shard-locally in the library's fused kernels;
between segments the library packs (local -> exchange, send order), the ranks exchange with one
``all_to_all_single`` (NCCL over NVLink on B200), the library unpacks (local -> exchange) and the two
buffers swap roles.  rho: every rank's rho block is gathered in rank order and the library sums it
(``qp_shard_combine``, fixed order on the device).

``exchange`` is pluggable so the same driver runs with a real process group or with an in-process
emulation of G ranks on one GPU (tests).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import numpy as np

from . import quapi as Q
from . import workloads as W


class ShardRank:
    """One rank's state of a sharded run (plan, shard buffers, workspace)."""

    def __init__(self, w: W.Workload, n_ranks: int, rank: int, out_steps=None, device="cuda", stream=None):
        import torch
        self.w, self.G, self.rank, self.device, self.stream = w, n_ranks, rank, device, stream
        self.plan = Q.Plan(w, out_steps=out_steps)
        self.sizes = self.plan.shard(n_ranks, rank)
        self.plan.check()  # two shard buffers + workspace vs the device's free memory
        self.send_counts, self.recv_counts = self.plan.shard_counts()
        ps = self.plan.sizes
        self.work = torch.empty((ps.work_bytes + 7) // 8, dtype=torch.float64, device=device)
        self.local = torch.empty(2 * self.sizes.local_entries, dtype=torch.float64, device=device)
        self.xbuf = torch.empty(2 * self.sizes.xbuf_entries, dtype=torch.float64, device=device)
        self.launches = 0

    def grow(self):
        """qp_init (A_0 into the exchange buffer) + the growth steps 1 .. L-1 (shard-native)."""
        self.plan.init(self.xbuf, self.work, self.stream)
        self.launches += self.plan.shard_steps(1, min(self.w.L, self.w.n_steps + 1), self.local, self.xbuf, self.work,
                                               self.stream)

    def swap(self):
        self.local, self.xbuf = self.xbuf, self.local


def advance(ranks: List[ShardRank], k_from: int, k_to: int, exchange: Callable[[List[ShardRank]], None]) -> int:
    """Slide steps k_from..k_to-1 (k_from >= L) on every local rank, re-sharding (pack -> exchange ->
    unpack -> swap) whenever a segment boundary is crossed and further steps follow.  Returns the
    number of kernel launches on one rank."""
    L, seg = ranks[0].w.L, ranks[0].sizes.segment_steps
    n = 0
    k = k_from
    while k < k_to:
        seg_end = L + ((k - L) // seg + 1) * seg
        k1 = min(seg_end, k_to)
        for r in ranks:
            n_r = r.plan.shard_steps(k, k1, r.local, r.xbuf, r.work, r.stream)
            r.launches += n_r
        n += n_r
        k = k1
        if k == seg_end and k <= ranks[0].w.n_steps:  # boundary reached and the run continues
            for r in ranks:
                r.plan.shard_pack(r.local, r.xbuf, r.stream)
                r.launches += r.G
            exchange(ranks)  # every rank's xbuf (send order) -> every rank's local (receive order)
            for r in ranks:
                r.plan.shard_unpack(r.local, r.xbuf, r.stream)
                r.launches += r.G
                r.swap()
            n += 2 * ranks[0].G
    return n


def run_sharded(ranks: List[ShardRank], exchange: Callable[[List[ShardRank]], None]):
    """Drive all local ranks (one per process in the distributed case) through the whole run."""
    w = ranks[0].w
    for r in ranks:
        r.grow()
    if w.n_steps >= w.L:
        advance(ranks, w.L, w.n_steps + 1, exchange)


def emulated_exchange(ranks: List[ShardRank]):
    """All-to-all among ranks living in this process (device copies; tests / single-GPU emulation):
    rank d's local receives, in source-rank order, every rank's send chunk for d."""
    G = len(ranks)
    soff = [np.concatenate([[0], np.cumsum(r.send_counts)]) for r in ranks]
    for dst in range(G):
        off = 0
        for src in range(G):
            n = ranks[src].send_counts[dst]
            a = 2 * int(soff[src][dst])
            ranks[dst].local[2 * off:2 * (off + n)].copy_(ranks[src].xbuf[a:a + 2 * n])
            off += n


def emulated_rho(ranks: List[ShardRank]) -> np.ndarray:
    """rho of an emulated run: the ranks' rho blocks in rank order, summed by the library."""
    import torch
    parts = torch.stack([r.plan.rho_block(r.work) for r in ranks])
    return ranks[0].plan.shard_combine(parts, ranks[0].work, ranks[0].stream)


def dist_exchange(group=None):
    """All-to-all through torch.distributed (NCCL over NVLink on the B200 box)."""
    import torch.distributed as dist

    def ex(ranks: List[ShardRank]):
        (r,) = ranks
        recv, send = r.local[:2 * sum(r.recv_counts)], r.xbuf[:2 * sum(r.send_counts)]
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


def dist_rho(me: ShardRank, group=None) -> Optional[np.ndarray]:
    """rho of a distributed run on rank 0 (None elsewhere): all-gather of the rho blocks, library sum."""
    import torch
    import torch.distributed as dist
    blk = me.plan.rho_block(me.work).contiguous()
    if dist.get_backend(group) == "gloo":
        torch.cuda.synchronize()
        parts = [torch.empty_like(blk, device="cpu") for _ in range(me.G)]
        dist.all_gather(parts, blk.cpu(), group=group)
        parts = torch.stack(parts).to(blk.device)
    else:
        parts = torch.empty((me.G,) + tuple(blk.shape), dtype=blk.dtype, device=blk.device)
        dist.all_gather_into_tensor(parts, blk, group=group)
    if dist.get_rank(group) != 0:
        return None
    return me.plan.shard_combine(parts, me.work, me.stream)


def solve_distributed(w: W.Workload, out_steps: Optional[Sequence[int]] = None, group=None):
    """Sharded run on the current process group (one rank per GPU).  Returns rho on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist
    G, rank = dist.get_world_size(group), dist.get_rank(group)
    me = ShardRank(w, G, rank, out_steps=out_steps, device=f"cuda:{torch.cuda.current_device()}")
    run_sharded([me], dist_exchange(group))
    return dist_rho(me, group)
