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
os.environ["QUAPI_FUSED_KIND"] = "reg"
w = W.random_problem(6, 2, 6, 20)
ranks = [SH.ShardRank(w, 2, i) for i in range(2)]
SH.run_sharded(ranks, SH.emulated_exchange)
print("sanitize run ok")
