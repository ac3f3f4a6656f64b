"""Batched pulse-area sweep benchmark, one JSON line.

The paper's use case: rho_11 of the driven quantum dot (Sec. III model: super-Ohmic
phonon bath at 25 K, H(t) = Omega(t) sigma_x / 2, Delta t = 0.1 ps) at the end of a pulse, swept over
pulse areas.  B problems (one per area) x n_steps, memory length L, rho read out at every step
(allPoints).  Timed on the device with CUDA events around qp_batch_run (tables H2D + one launch),
after warm-up; the CPU oracle runs a bounded sample of the same problems on the host.
"""
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


def sweep_inputs(B, n, L):
    w0 = W.CONFIGS[0].with_(L=L, n_steps=n, H=np.zeros((2, 2), complex))
    t = w0.dt * (np.arange(n) + 0.5)
    t0, width = 0.4 * n * w0.dt, 0.1 * n * w0.dt
    env = np.exp(-((t - t0) / width) ** 2)
    areas = np.linspace(0.0, 6 * np.pi, B)
    f = areas[:, None] * env[None, :] / (env.sum() * w0.dt)
    return w0, f, areas


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--L", type=int, default=7)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--temperature-sweep", action="store_true",
                    help="problem b also gets its own phonon temperature (5..50 K): per-problem baths, "
                         "eta classes on the device inside the timed qp_batch_run (SURVEY 8(f2))")
    a = ap.parse_args()
    w, f, areas = sweep_inputs(a.B, a.steps, a.L)
    H1 = 0.5 * np.array([[0, 1], [1, 0]], dtype=complex)
    baths = None
    if a.temperature_sweep:
        temps = np.linspace(5.0, 50.0, a.B)
        baths = [(w.kind, w.coupling, w.omega_c, float(T) * W.KB_OVER_HBAR_PS_K) for T in temps]
    bp = Q.BatchPlan(w, a.B, H1=H1, f=f, baths=baths)
    ardm, work = bp.alloc()
    st = torch.cuda.current_stream()
    rho = bp.run(ardm, work, st)  # warm-up + result
    torch.cuda.synchronize()
    times = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        bp.run(ardm, work, st, read=False)
        e1.record(st)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    t = float(np.median(times))
    N, L = 4, a.L
    ps = a.B * a.steps / t
    line = {"metric": "batched pulse-area sweep: problem-steps/s (Sec. III dot, allPoints readout)"
                      + (", per-problem temperature 5..50 K" if baths else ""),
            "value": ps, "unit": "problem-steps/s", "n_gpus": 1, "B": a.B, "steps": a.steps, "L": L,
            "seconds": t, "element_updates_per_s": ps * N ** L, "ardm_bytes_total": 16 * a.B * N ** L,
            "launches_per_run": 1, "dtype": "f64", "data": "synthetic (pulse areas 0..6 pi)",
            "rho11_final_min_max": [float(rho[:, -1, 1, 1].real.min()), float(rho[:, -1, 1, 1].real.max())],
            "max_abs_trace_err": float(np.abs(np.einsum("bkii->bk", rho) - 1).max())}
    # roofline of k_batch (one step per pass over each problem's ARDM): FP64 flops per element update
    # counted from the slide step with readout (M = 2, D = 2; per fibre of N = 4 entries: digit-group
    # factor products 24 (G - 1) for G groups of w digits plus the per-step table build
    # 24 (w - 1) tot / N^(L-1), S0 6, beta moments 128, class factors 24, outputs 24, readout 32;
    # w and G as batch.cu batch_bw), bytes 32 per element update when the ARDM streams through HBM
    # (B N^L 16 B > L2), else none (L2 / smem resident)
    nf = N ** (L - 1)
    bw = 1
    for w_ in (4, 3, 2):
        tot_ = sum(N ** min(w_, r) for r in range(L - 1, 0, -w_))
        if 2 * 2 * tot_ * 16 <= 48 * 1024 and 4 * tot_ <= nf:
            bw = w_
            break
    G = -(-(L - 1) // bw)
    tot = sum(N ** min(bw, r) for r in range(L - 1, 0, -bw))
    flops = (24 * (G - 1) + 24 * (bw - 1) * tot / nf + 214) / N
    tflops = ps * N ** L * flops / 1e12
    fp64_peak = 35.1  # measured DFMA rate, scripts/membench.cu (profiles/README.md); no FP64 in MEASURED_PEAKS
    ardm = 16 * a.B * N ** L
    hbm = None
    if ardm > 2 * 126e6:
        pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
        gbs = ps * N ** L * 32 / 1e9
        hbm = {"achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": gbs / pk["hbm_gbs"]}
    alu = {"achieved": tflops, "peak": fp64_peak, "unit": "TFLOP/s", "frac": tflops / fp64_peak,
           "flops_per_element_update": flops, "digit_groups": G, "group_width": bw}
    if hbm and hbm["frac"] > alu["frac"]:
        line["roofline"] = {"bound": "hbm", **hbm, "alu": alu}
    else:
        line["roofline"] = {"bound": "alu", **alu, "hbm": hbm}
    if not a.no_cpu_baseline:
        import oracle as O
        from tests.test_oracle_engine import P
        ncpu = os.cpu_count()
        t0 = time.perf_counter()
        nsample = 0
        while nsample < a.B and time.perf_counter() - t0 < 10.0:
            Ht = np.stack([w.H + f[nsample, k] * H1 for k in range(a.steps)])
            kT = baths[nsample][3] if baths else w.kT
            ro = O.run(P(w, H_t=Ht, kT=kT), nthreads=ncpu)
            assert np.abs(ro - rho[nsample]).max() <= 1e-10
            nsample += 1
        el = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": nsample * a.steps / el, "unit": "problem-steps/s", "cores": ncpu,
                                "kind": "oracle", "sample": f"{nsample} of the {a.B} problems, all {a.steps} steps, "
                                                            "each checked against the GPU result (<= 1e-10)"}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
