"""Setup-step benchmark: eta classes (host-setup step a3) on the device vs the host.

Per workload: the library's host quadrature (qp_plan_create with the bath, threaded adaptive GK21),
the device quadrature (qp_eta_device: kernel time by CUDA events on its stream, and wall time of the
call including the D2H copy), and the oracle's G table (test infrastructure, single thread) for scale.
Sweep: B baths (temperature x coupling grid of the cfg3 Debye bath) in one device call vs the host
quadrature per bath (measured on 8 baths, scaled).  One JSON line per case on stdout.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_1205_6872_b200 import build as B  # noqa: E402
from paper_1205_6872_b200 import quapi as Q  # noqa: E402
from paper_1205_6872_b200 import workloads as W  # noqa: E402
from tests.test_oracle_engine import P  # noqa: E402


def kernel_ms(baths, dt, L, reps=20):
    nc = 3 * L + 2
    out = torch.empty(2 * len(baths) * nc, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(3):
        Q.eta_device(baths, dt, L, stream=s, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        Q.eta_device(baths, dt, L, stream=s, out=out)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def host_ms(w, reps=3):
    ts = []
    for _ in range(reps):
        pl = Q.Plan(w, out_steps=[0])
        ts.append(pl.sizes.setup_seconds * 1e3)
    return min(ts)


def main():
    B.build()
    torch.cuda.set_device(0)
    for cfg in (0, 1, 3, 4, 5):
        w = W.CONFIGS[cfg]
        bath = Q.bath_of(w)
        kms = kernel_ms([bath], w.dt, w.L)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eta = Q.eta_device([bath], w.dt, w.L)
        wall = (time.perf_counter() - t0) * 1e3
        e = Q.Plan(w, out_steps=[0]).eta()
        host = np.concatenate([[e["self_interior"], e["self_end"]], e["eta"], e["E"], e["TI"]])
        t0 = time.perf_counter()
        O.G_table(P(w))
        ora = (time.perf_counter() - t0) * 1e3
        print(json.dumps({"case": w.name, "L": w.L, "classes": 3 * w.L + 2, "device_kernel_ms": kms,
                          "device_call_wall_ms": wall, "host_plan_setup_ms": host_ms(w),
                          "oracle_G_table_ms_1thread": ora,
                          "max_abs_device_minus_host": float(np.abs(eta[0] - host).max())}), flush=True)
    w = W.CONFIGS[3]
    temps = np.linspace(0.05, 2.0, 32)
    couplings = np.linspace(0.02, 0.5, 32)
    baths = [(W.J_DEBYE, float(c), w.omega_c, float(t)) for t in temps for c in couplings]
    kms = kernel_ms(baths, w.dt, w.L, reps=5)
    hs = [host_ms(w.with_(coupling=b[1], kT=b[3]), reps=1) for b in baths[::128]]
    print(json.dumps({"case": f"sweep: {len(baths)} Debye baths (32 kT x 32 coupling), L={w.L}",
                      "device_kernel_ms": kms, "device_ms_per_bath": kms / len(baths),
                      "host_ms_per_bath": float(np.mean(hs)), "host_baths_measured": len(hs),
                      "host_total_ms_scaled": float(np.mean(hs)) * len(baths)}), flush=True)


if __name__ == "__main__":
    main()
