"""Small runs of every kernel path for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1205_6872_b200 import quapi as Q  # noqa: E402
from paper_1205_6872_b200 import sharded as SH  # noqa: E402
from paper_1205_6872_b200 import workloads as W  # noqa: E402

for kind in ("reg", "warp", "async", "split"):
    os.environ["QUAPI_FUSED_KIND"] = kind
    for w in (W.CONFIGS[1].with_(n_steps=14), W.random_problem(3, 3, 4, 9), W.random_problem(4, 4, 3, 7),
              W.random_problem(5, 2, 7, 15, lattice_s=False)):
        pl = Q.Plan(w)
        a, wk = pl.alloc()
        r = pl.run(a, wk)
        assert np.isfinite(r).all()
os.environ["QUAPI_FUSED_KIND"] = "3"
for env in ({}, {"QUAPI_NO_TMA": "1"}, {"QUAPI_F3TMAP": "1"}, {"QUAPI_NO_VIEWB": "1", "QUAPI_NO_VIEWC": "1", "QUAPI_NO_VIEWD": "1"}, {"QUAPI_NO_TMA": "1", "QUAPI_F3MAP": "1"}, {"QUAPI_CA": "1"}):
    os.environ.update(env)
    w = W.random_problem(7, 2, 8, 20)  # L = 8: TMA-staged, plain-load and 32-B-load ring slots all occur
    pl = Q.Plan(w)
    a, wk = pl.alloc()
    assert np.isfinite(pl.run(a, wk)).all()
    for k in env:
        del os.environ[k]
for env in ({"QUAPI_VIEWD64": "1", "QUAPI_VIEWC_OLD": "1"},):
    os.environ.update(env)
    w = W.random_problem(7, 2, 8, 20)
    pl = Q.Plan(w)
    a, wk = pl.alloc()
    assert np.isfinite(pl.run(a, wk)).all()
    for k in env:
        del os.environ[k]
# device eta setup (k_eta: 8-CTA clusters, DSMEM reduction) and a plan built from it
eta = Q.eta_device([(1, 0.1, 7.5, 0.2), (2, 0.1, 7.5, 0.0), (3, 0.08, 2.2, 0.3), (0, 0.0, 1.0, 0.0)], 0.25, 6)
assert np.isfinite(eta).all()
pl = Q.Plan(W.CONFIGS[1].with_(n_steps=12), eta_setup="device")
a, wk = pl.alloc()
assert np.isfinite(pl.run(a, wk)).all()
# batched sweeps: shared-memory ARDM (L = 4), global ARDM (QUAPI_BATCH_GLOBAL), per-problem baths (k_psi)
wb = W.random_problem(8, 2, 4, 12)
H1 = np.array([[0, 1], [1, 0]], dtype=complex)
f = np.random.default_rng(1).standard_normal((3, 12))
for env in ({}, {"QUAPI_BATCH_GLOBAL": "1"}):
    os.environ.update(env)
    bp = Q.BatchPlan(wb, 3, H1=H1, f=f, baths=[(1, 0.1, 7.5, 0.2), (2, 0.2, 3.0, 1.0), (3, 0.05, 2.2, 0.3)])
    a, wk = bp.alloc()
    assert np.isfinite(bp.run(a, wk)).all()
    for k in env:
        del os.environ[k]
bp = Q.BatchPlan(W.random_problem(9, 3, 3, 8), 2)
a, wk = bp.alloc()
assert np.isfinite(bp.run(a, wk)).all()
os.environ["QUAPI_FUSED_KIND"] = "reg"
w = W.random_problem(6, 2, 6, 20)
ranks = [SH.ShardRank(w, 2, i) for i in range(2)]
SH.run_sharded(ranks, SH.emulated_exchange)
print("sanitize run ok")
