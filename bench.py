#!/usr/bin/env python
"""bench.py -- QUAPI tensor-propagator step on B200 (BASELINE.json metric, config 3 at N=1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--cfg 3]

A "step" is one QUAPI time step k >= L of the BASELINE workload (config 3: spin-boson M=2,
Debye bath, Delta k_max = 14, ARDM of 4^14 complex FP64 entries = 4.3 GB, larger than L2):
the in-place slide of the ARDM with the rho(t_k) readout fused (allPoints mode).  Our arm
times K such steps after W warm-up steps with CUDA events on the launching stream (barrier +
synchronize on both sides, max over ranks).  N > 1 (torchrun): by default one ARDM sharded over the
ranks (strong scaling: shard-native growth, fused slide steps on each rank's shard, NCCL
all_to_all_single re-shard every L - z steps inside the timed region); --mode replica runs
independent replicas (weak scaling).  --cfg 5 is the sharded BASELINE case (L = 16).

--impl reference: the CPU oracle (oracle/liboracle.so) on the host cores, same config/metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QUAPI steps/s & achieved HBM GB/s, spin-boson Δkmax=14 FP64, 1/2/4/8 B200"


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _ncu_traffic(cfg: int):
    """Per-launch DRAM bytes of the slide kernel from the committed ncu --set full summary
    (profiles/ncu_slide_summary.json, captured on config 3); None for other workloads."""
    path = os.path.join(ROOT, "profiles", "ncu_slide_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch") if int(d.get("cfg", 3)) == cfg else None
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        rows = []
        for ln in (self.out or "").strip().splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) >= 9:
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def kernel_name(sz) -> str:
    """The slide kernel the plan runs (include/quapi.h qp_sizes: fuse_steps, persistent)."""
    if sz.persistent:
        return "k_small: every slide step of the call in one single-CTA launch, ARDM + tables in shared memory"
    if sz.M == 3 and sz.fuse_steps == 2:
        if sz.block == 576:  # (qp_sizes.block after qp_init)
            return ("k_fused2t: 2 time steps per HBM pass, TMA load + TMA store of 27-fibre units (5-stage ring, "
                    "load and store warps, 2 x 8 consumer warps, readout sums in TMEM), one CTA per SM")
        return "k_fused2s: 2 time steps per HBM pass, 32-fibre units staged in shared memory (cp.async)"
    return {4: "k_fused4: 4 time steps per HBM pass, TMA load + TMA store of 8-fibre rounds "
               "(6-stage ring, load and store warps, 8 consumer warps, readout sums in TMEM), one CTA per SM",
            3: "k_fused3: 3 time steps per HBM pass, per-warp TMA-staged rounds"}.get(
        sz.fuse_steps, f"k_fused_r: {sz.fuse_steps} time step(s) per HBM pass")


def cpu_baseline(cfg: int, max_slide: int = 3):
    """The oracle as it stands on the host cores, on a bounded sample of the workload:
    init + growth + `max_slide` slide steps with readout; value = slide steps / slide seconds."""
    import numpy as np

    import oracle as O
    from paper_1205_6872_b200 import workloads as W
    w = W.CONFIGS[cfg]
    n = w.L + max_slide  # steps L..L+max_slide contract: >= max_slide timed slide steps whatever the count convention
    p = O.Problem(s=w.s, H=w.H, rho0=w.rho0, kind=w.kind, coupling=w.coupling, omega_c=w.omega_c,
                  kT=w.kT, dt=w.dt, n_steps=n, L=w.L)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    _, tm = O.run(p, out_steps=np.arange(n + 1), nthreads=cores, timings=True)
    wall = time.perf_counter() - t0
    v = tm["n_slide"] / tm["slide_s"] if tm["slide_s"] > 0 else None
    return {"value": v, "unit": "steps/s", "cores": cores, "kind": "oracle", "timed_steps": int(tm["n_slide"]),
            "sample": (f"{w.name}: init + {w.L - 1} growth + {tm['n_slide']} slide steps with readout "
                       f"(allPoints), {cores} OpenMP threads; slide {tm['slide_s']:.2f} s of {wall:.1f} s wall")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cb = cpu_baseline(args.cfg, max_slide=max(1, min(args.steps, 3)))
    from paper_1205_6872_b200 import workloads as W
    w = W.CONFIGS[args.cfg]
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "steps/s",
            "n_gpus": args.gpus, "steps": cb["timed_steps"], "requested_steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 / cb["value"] if cb["value"] else None, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "ardm_entries": w.ardm_entries},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cfg", type=int, default=3)
    ap.add_argument("--fuse-steps", type=int, default=0, help="cap on the steps fused per pass (0: the library's choice)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo stages the all-to-all through host memory; tests only)")
    ap.add_argument("--reps", type=int, default=3,
                    help="timed repetitions of K steps each; value = the median repetition (single GPU)")
    ap.add_argument("--mode", default="shard", choices=["shard", "replica"],
                    help="N > 1: shard one ARDM over the ranks (strong scaling, NCCL all-to-all re-shard) "
                         "or run independent replicas (weak scaling)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1205_6872_b200 import build as B
    from paper_1205_6872_b200 import quapi as Q
    from paper_1205_6872_b200 import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group(args.dist_backend)
    local = local % max(1, torch.cuda.device_count())  # several ranks per GPU only for gloo tests
    torch.cuda.set_device(local)
    B.build()

    base = W.CONFIGS[args.cfg]
    if world > 1 and args.mode == "shard":
        return bench_sharded(args, base, world, rank, local)
    K, Wm, L, R = args.steps, max(args.warmup, 3), base.L, max(1, args.reps)
    fuse = Q.Plan(base.with_(n_steps=L + 4), out_steps=[0], fuse_steps=args.fuse_steps).sizes.fuse_steps
    Wm = -(-Wm // fuse) * fuse  # warm-up rounded up to whole fusion groups: the timed steps start a group
    n_total = L - 1 + Wm + R * K  # growth steps, then W warm-up and R x K timed slide steps
    w = base.with_(n_steps=n_total)
    plan = Q.Plan(w, fuse_steps=args.fuse_steps)  # allPoints readout: every step reduces rho(t_k)
    sz = plan.sizes
    ardm, work = plan.alloc()
    stream = torch.cuda.current_stream()
    plan.init(ardm, work, stream)
    plan.steps(1, L, ardm, work, stream)                 # growth (untimed)
    plan.steps(L, L + Wm, ardm, work, stream)            # warm-up slide steps
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # R repetitions of K steps; inside each, events after every quarter (cuts on fusion-group bounds)
    # give the time-vs-N_t line the paper shows ("the linear scaling" of the propagator)
    q = max(1, K // 4)
    cuts = [0, q, 2 * q, 3 * q, K] if (q % fuse == 0 and K >= 4) else [0, K]
    evs = [[torch.cuda.Event(enable_timing=True) for _ in cuts] for _ in range(R)]
    launches = 0
    with ClockSampler(local) as clk:
        time.sleep(0.3)  # let the sampler start
        for r in range(R):
            k0 = L + Wm + r * K
            evs[r][0].record(stream)
            for i in range(1, len(cuts)):
                launches += plan.steps(k0 + cuts[i - 1], k0 + cuts[i], ardm, work, stream)
                evs[r][i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    rep_ms = [evs[r][0].elapsed_time(evs[r][-1]) for r in range(R)]
    ms = sorted(rep_ms)[R // 2]
    launches //= R
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    nt_fit = None
    if len(cuts) > 2:  # least squares t = a + b N_t over (cut, cumulative ms) of every repetition
        xs = np.array([c for r in range(R) for c in cuts[1:]], dtype=float)
        ys = np.array([evs[r][0].elapsed_time(evs[r][i]) for r in range(R) for i in range(1, len(cuts))])
        b, a = np.polyfit(xs, ys, 1)
        res = ys - (a + b * xs)
        r2 = 1.0 - float(res @ res) / float(((ys - ys.mean()) ** 2).sum())
        nt_fit = {"ms_per_step": float(b), "intercept_ms": float(a), "r2": r2, "points": int(len(xs)),
                  "steps_at": cuts[1:], "note": "wall time linear in the number of time steps (P:455-466)"}
    rho = plan.read_rho(work, stream)
    sz = plan.sizes  # after qp_init: the launch configuration the timed region ran
    tr_err = float(np.abs(np.einsum("kii->k", rho) - 1).max())
    del ardm, work
    torch.cuda.empty_cache()

    # e2e: the whole public-API call from host inputs to host rho (plan setup, H2D tables,
    # growth, all steps of the workload with readout, D2H) for the BASELINE config itself
    e2e = None
    if not args.no_e2e:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pe = Q.Plan(base, eta_setup="device")  # host-setup step a3 on the GPU (qp_eta_device)
        a2, w2 = pe.alloc()
        rho_e = pe.run(a2, w2, stream)
        el = time.perf_counter() - t0
        se = pe.sizes
        h2d = se.init_h2d_bytes  # tables + A_0 + rho(0)
        d2h = se.n_out * se.N * 16
        tt = torch.tensor([el], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": world * base.n_steps / float(tt.item()), "unit": "steps/s",
               "h2d_bytes_per_step": int(h2d // base.n_steps), "d2h_bytes_per_step": int(d2h // base.n_steps),
               "seconds": float(tt.item()), "steps": base.n_steps, "setup_seconds": se.setup_seconds,
               "eta_setup": "device (qp_eta_device)",
               "max_abs_trace_err": float(np.abs(np.einsum("kii->k", rho_e) - 1).max())}
        del a2, w2

    if rank == 0:
        steps_per_s = world * K / (ms_max / 1e3)
        bytes_launch = 32 * sz.ardm_entries                # one read + one write of the ARDM per launch
        per_launch_s = (ms / 1e3) / max(1, launches)       # rank-0 average fused-kernel duration
        achieved = bytes_launch / per_launch_s / 1e9
        peak, peak_kind = _peaks()
        step_equiv = 32 * sz.ardm_entries * (K / (ms / 1e3)) / 1e9  # north_star's 2*16*N^L B per step
        line = {
            "metric": METRIC, "value": steps_per_s, "unit": "steps/s", "n_gpus": world, "steps": K,
            "warmup": Wm, "ms_per_step": ms_max / K, "higher_is_better": True,
            "repetitions": {"count": R, "ms": rep_ms, "reported": "median"},
            "n_t_fit": nt_fit,
            "scaling": "weak" if world > 1 else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": base.name, "ardm_entries": sz.ardm_entries, "ardm_bytes": sz.ardm_bytes,
                       "readout": "every step (allPoints), fused",
                       "l2": (f"inputs larger than L2 ({sz.ardm_bytes / 1e9:.1f} GB ARDM, 126 MB L2)"
                              if sz.ardm_bytes > 2 * 126e6 else
                              f"L2-resident ARDM ({sz.ardm_bytes / 1e6:.1f} MB): not flushed, not a roofline case"),
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "kernel": kernel_name(sz),
                       "steps_per_launch": K / max(1, launches),
                       "timed_steps_aligned_to_fusion_groups": K % fuse == 0, "fuse_steps": fuse},
            "achieved_gbs": achieved,
            "step_equivalent_gbs": step_equiv,
            "frac_of_unfused_roofline": step_equiv / peak,
            "element_updates_per_s": steps_per_s * sz.ardm_entries,
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind, "frac_of_8TBs": achieved / 8000.0,
                         "traffic": _ncu_traffic(args.cfg), "algorithmic_bytes_per_launch": bytes_launch,
                         "steps_per_launch": K / max(1, launches)},
            "clocks": clk.summary(),
            "max_abs_trace_err": tr_err,
            "e2e": e2e,
        }
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(args.cfg)
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def bench_sharded(args, base, world, rank, local):
    """N > 1, one ARDM sharded over the ranks: K slide steps including every re-shard (pack kernel,
    NCCL all_to_all_single over NVLink, unpack kernel) inside the timed region (strong scaling)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1205_6872_b200 import sharded as SH
    K, Wm, L = args.steps, max(args.warmup, 3), base.L
    w = base.with_(n_steps=L - 1 + Wm + K)
    stream = torch.cuda.current_stream()
    me = SH.ShardRank(w, world, rank, device=f"cuda:{local}", stream=stream)
    ex = SH.dist_exchange()
    me.grow()  # shard-native growth: no rank holds the N^L ARDM
    SH.advance([me], L, L + Wm, ex)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        ev0.record(stream)
        launches = SH.advance([me], L + Wm, L + Wm + K, ex)
        ev1.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    rho = SH.dist_rho(me)  # all-gather of the rho blocks, rank-ordered sum in the library (rank 0)
    sz = me.plan.sizes
    ssz = me.sizes
    del me
    torch.cuda.empty_cache()
    e2e = None
    if not args.no_e2e:  # the whole sharded public-API run of the BASELINE config, host in -> host rho
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rho_e = SH.solve_distributed(base)
        el = time.perf_counter() - t0
        tt = torch.tensor([el], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": base.n_steps / float(tt.item()), "unit": "steps/s", "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": int(base.N * 16 * (base.n_steps + 1) * world / base.n_steps),
               "seconds": float(tt.item()), "steps": base.n_steps}
        if rank == 0:
            e2e["max_abs_trace_err"] = float(np.abs(np.einsum("kii->k", rho_e) - 1).max())
    if rank == 0:
        steps_per_s = K / (ms_max / 1e3)
        peak, peak_kind = _peaks()
        passes = K / max(1, sz.fuse_steps)
        agg = 32 * sz.ardm_entries * passes / (ms_max / 1e3) / 1e9  # algorithmic HBM bytes of all ranks
        line = {
            "metric": METRIC, "value": steps_per_s, "unit": "steps/s", "n_gpus": world, "steps": K, "warmup": Wm,
            "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": base.name, "ardm_entries": sz.ardm_entries, "parallelism": f"sharded x{world}",
                       "shard_slots": ssz.shard_slots, "segment_steps": ssz.segment_steps,
                       "local_entries": ssz.local_entries, "exchange_entries_per_rank": ssz.exchange_entries,
                       "readout": "every step (allPoints), fused", "l2": "inputs larger than L2",
                       "collective": "all_to_all_single (NCCL) every segment_steps steps"},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "achieved": agg, "peak": peak * world, "unit": "GB/s",
                         "frac": agg / (peak * world), "peak_kind": peak_kind + " x n_gpus",
                         "traffic": None, "note": "aggregate algorithmic bytes incl. re-shard time"},
            "clocks": clk.summary(),
            "max_abs_trace_err": float(np.abs(np.einsum("kii->k", rho) - 1).max()),
            "e2e": e2e,
        }
        print(json.dumps(line))
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
