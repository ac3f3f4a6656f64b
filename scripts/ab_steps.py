"""A/B timing of the slide path under plan flags (tuning aid, not product code): cfg --cfg, growth,
warm-up, then K steps in one qp_steps call (back-to-back launches) and K steps one fusion group per
call, CUDA events on the plan's stream; prints ms per launch for flags = 0 and each --flags value."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1205_6872_b200 import quapi as Q  # noqa: E402
from paper_1205_6872_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--K", type=int, default=200)
ap.add_argument("--flags", type=int, nargs="*", default=[0, Q.QP_FLAG_NO_TMA])
args = ap.parse_args()
w = W.CONFIGS[args.cfg]
L = w.L
for fl in args.flags:
    n = L + 20 + 2 * args.K + 8
    plan = Q.Plan(w.with_(n_steps=n), flags=fl)
    S = plan.sizes.fuse_steps
    ardm, work = plan.alloc()
    st = torch.cuda.current_stream()
    plan.init(ardm, work)
    plan.steps(1, L + 20, ardm, work)
    torch.cuda.synchronize()
    k = L + 20
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record(st)
    plan.steps(k, k + args.K, ardm, work)
    e[1].record(st)
    k += args.K
    ev = []
    while k + S <= L + 20 + 2 * args.K:
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        plan.steps(k, k + S, ardm, work)
        a1.record(st)
        ev.append((a0, a1))
        k += S
    torch.cuda.synchronize()
    one = e[0].elapsed_time(e[1]) / (args.K / S)
    sep = sorted(a.elapsed_time(b) for a, b in ev)
    print(f"flags={fl}: one call {one:.3f} ms/launch ({args.K / (e[0].elapsed_time(e[1]) / 1e3):.1f} steps/s); "
          f"per-group calls median {sep[len(sep) // 2]:.3f} mean {sum(sep) / len(sep):.3f} ms/launch", flush=True)
    del ardm, work
    torch.cuda.empty_cache()
