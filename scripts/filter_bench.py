"""Path filtering against theta: kept entries (fraction of N^L), filter-buffer bytes vs the
dense ARDM, steps/s of the filtered run (wall time of qp_filter_run, host setup excluded) and max|d rho|
against the dense GPU run.  Usage: filter_bench.py [--cfg 3] [--steps 40] [--L L]"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1205_6872_b200 import quapi as Q  # noqa: E402
from paper_1205_6872_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--L", type=int, default=0)
ap.add_argument("--thetas", default="0,1e-9,1e-7,1e-5,1e-3")
ap.add_argument("--capacity", type=float, default=0, help="list entries (default N^L)")
ap.add_argument("--no-dense", action="store_true")
args = ap.parse_args()
w = W.CONFIGS[args.cfg]
if args.L:
    w = w.with_(L=args.L)
w = w.with_(n_steps=args.steps)
dense = None
if not args.no_dense:
    pl = Q.Plan(w)
    a, wk = pl.alloc()
    dense = pl.run(a, wk)
    del a, wk
    torch.cuda.empty_cache()
for th in [float(t) for t in args.thetas.split(",")]:
    pl = Q.Plan(w)
    cap = int(args.capacity) if args.capacity else pl.sizes.ardm_entries
    Q.Plan(w.with_(L=5, n_steps=8)).filter_run(th)  # warm-up (module load)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rho, kept = pl.filter_run(th, capacity=cap)
    el = time.perf_counter() - t0
    out = {"workload": w.name, "L": w.L, "steps": w.n_steps, "theta": th, "kept_max": int(kept.max()),
           "kept_last": int(kept[-2]), "kept_frac_of_dense": float(kept.max() / w.N ** w.L),
           "filter_buffer_bytes": pl.filter_buffer_bytes, "dense_ardm_bytes": 16 * w.N ** w.L,
           "seconds": el, "steps_per_s": w.n_steps / el,
           "max_abs_drho_vs_dense": None if dense is None else float(np.abs(rho - dense).max()),
           "max_abs_trace_err": float(np.abs(np.einsum("kii->k", rho) - 1).max())}
    print(json.dumps(out), flush=True)
    del pl
    torch.cuda.empty_cache()
