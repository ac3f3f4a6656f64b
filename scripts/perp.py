"""Per-launch-set timing of the fused slide kernel (tuning aid, not product code).

Runs config 3 (or --cfg) through growth, then times each fused group k..k+S-1 separately with
CUDA events on the plan's stream and prints ms per launch and GB/s per launch by start slot p0.
"""
import argparse
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1205_6872_b200 import quapi as Q  # noqa: E402
from paper_1205_6872_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--final-only", action="store_true", help="readout of the last step only (no fused readout)")
ap.add_argument("--so", default=None, help="time another build of libquapi.so (A/B)")
args = ap.parse_args()
if args.so:
    Q.SO_PATH = args.so
w = W.CONFIGS[args.cfg]
L = w.L
n = L + 14 * 3 * (args.reps + 1)
plan = Q.Plan(w.with_(n_steps=n), out_steps=[n] if args.final_only else None)
ardm, work = plan.alloc()
st = torch.cuda.current_stream()
plan.init(ardm, work)
S = plan.sizes.fuse_steps
plan.steps(1, L, ardm, work)
k = L
# first (partial) group: fusion groups are aligned on k - L
res = defaultdict(list)
ev = []
while k + S <= n + 1:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    plan.steps(k, k + S, ardm, work)
    e1.record(st)
    ev.append((k % L, e0, e1))
    k += S
torch.cuda.synchronize()
for p0, e0, e1 in ev[1:]:
    res[p0].append(e0.elapsed_time(e1))
byts = 32 * plan.sizes.ardm_entries
tot = 0.0
for p0 in sorted(res):
    ms = sorted(res[p0])[len(res[p0]) // 2]
    tot += ms
    print(f"p0={p0:2d} {ms:.3f} ms  {byts / ms / 1e6:.0f} GB/s")
print(f"mean {tot / len(res):.3f} ms per launch, {S * len(res) / tot * 1e3:.1f} steps/s")
rho = plan.read_rho(work)
print(f"checksum rho[-1] = {rho[-1].real.sum():.15f} {abs(rho[-1][0, 1]):.15e}")
