"""Sharded-path data movement on one GPU (emulated ranks): time of a segment's slide steps, of the
re-shard pack and unpack kernels (GB/s against the copy peak), and of the device-copy exchange.
Usage: shard_bench.py [--cfg 3] [--G 2] [--reps 3]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1205_6872_b200 import sharded as SH  # noqa: E402
from paper_1205_6872_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--G", type=int, default=2)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
base = W.CONFIGS[args.cfg]
L = base.L
probe = SH.ShardRank(base.with_(n_steps=L), args.G, 0)
seg = probe.sizes.segment_steps
del probe
torch.cuda.empty_cache()
n = L + seg * (args.reps + 1)
w = base.with_(n_steps=n)
ranks = [SH.ShardRank(w, args.G, r) for r in range(args.G)]
SH.run_sharded  # noqa: B018
for r in ranks:
    r.grow()
st = torch.cuda.current_stream()


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record(st)
    return e


res = {"steps": [], "pack": [], "exchange": [], "unpack": []}
k = L
for rep in range(args.reps):
    e0 = ev()
    for r in ranks:
        r.plan.shard_steps(k, k + seg, r.local, r.xbuf, r.work, st)
    e1 = ev()
    for r in ranks:
        r.plan.shard_pack(r.local, r.xbuf, st)
    e2 = ev()
    SH.emulated_exchange(ranks)
    e3 = ev()
    for r in ranks:
        r.plan.shard_unpack(r.local, r.xbuf, st)
        r.swap()
    e4 = ev()
    k += seg
    torch.cuda.synchronize()
    res["steps"].append(e0.elapsed_time(e1))
    res["pack"].append(e1.elapsed_time(e2))
    res["exchange"].append(e2.elapsed_time(e3))
    res["unpack"].append(e3.elapsed_time(e4))
loc = sum(r.sizes.local_entries for r in ranks)  # all emulated ranks together = N^L entries
med = {key: sorted(v)[len(v) // 2] for key, v in res.items()}
gb = 32 * loc / 1e9  # one read + one write of every entry
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
out = {"cfg": args.cfg, "G": args.G, "segment_steps": seg, "shard_slots": ranks[0].sizes.shard_slots,
       "ms": med, "pack_GBs": gb / med["pack"] * 1e3, "unpack_GBs": gb / med["unpack"] * 1e3,
       "pack_frac": gb / med["pack"] * 1e3 / peak, "unpack_frac": gb / med["unpack"] * 1e3 / peak,
       "segment_steps_per_s": seg / med["steps"] * 1e3, "launches_per_segment": None}
print(json.dumps(out))
