"""Small runs of every kernel path for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1205_6872_b200 import quapi as Q  # noqa: E402
from paper_1205_6872_b200 import sharded as SH  # noqa: E402
from paper_1205_6872_b200 import workloads as W  # noqa: E402


def run(w, **kw):
    pl = Q.Plan(w, **kw)
    a, wk = pl.alloc()
    r = pl.run(a, wk)
    assert np.isfinite(r).all()


NP = Q.QP_FLAG_NO_PERSIST  # the per-group launch kernels (small problems otherwise take k_small)
# k_fused_r (S = 1, 2; M = 2, 3, 4; lattice and general s), k_fused2s (M = 3, S = 2) and k_grow
for fuse in (1, 2):
    for w in (W.CONFIGS[1].with_(n_steps=14), W.random_problem(3, 3, 4, 9), W.random_problem(4, 4, 3, 7),
              W.random_problem(5, 2, 7, 15, lattice_s=False), W.random_problem(6, 3, 4, 9, lattice_s=False)):
        run(w, fuse_steps=fuse, flags=NP)
# k_fused3: TMA-staged rounds (all four views at L = 8), plain loads (lane maps 0 and 1), generic moments
for flags in (0, Q.QP_FLAG_NO_TMA, Q.QP_FLAG_GENERIC_MOMENTS):
    run(W.random_problem(7, 2, 8, 20), fuse_steps=3, flags=flags | NP)
# k_fused4: TMA load + store rounds, every start slot at L = 8 and L = 9, symmetric and generic moments
for flags in (0, Q.QP_FLAG_GENERIC_MOMENTS):
    for L in (8, 9):
        run(W.random_problem(7, 2, L, 2 * L + 6), flags=flags)
# k_fused2t (M = 3, s = (1, 0, -1): TMA units, all four views at L = 5) and the same through k_fused2s
for flags in (0, Q.QP_FLAG_NO_TMA):
    run(W.random_problem(9, 3, 5, 18), flags=flags | NP)
# k_small: one CTA, ARDM and tables in shared memory (M = 2, 3, 4)
for w in (W.CONFIGS[1].with_(n_steps=14), W.random_problem(3, 3, 3, 9), W.random_problem(4, 4, 2, 7),
          W.random_problem(5, 2, 6, 15, lattice_s=False)):
    run(w)
# OFPF path filtering (k_ofpf_count / scan / scatter)
rf, kept = Q.Plan(W.random_problem(11, 2, 6, 18)).filter_run(1e-3)
assert np.isfinite(rf).all()
# device eta setup (k_eta: 8-CTA clusters, DSMEM reduction) and a plan built from it
eta = Q.eta_device([(1, 0.1, 7.5, 0.2), (2, 0.1, 7.5, 0.0), (3, 0.08, 2.2, 0.3), (0, 0.0, 1.0, 0.0)], 0.25, 6)
assert np.isfinite(eta).all()
run(W.CONFIGS[1].with_(n_steps=12), eta_setup="device")
# batched sweeps: shared-memory ARDM (L = 4), global ARDM (L = 7), per-problem baths (k_psi)
H1 = np.array([[0, 1], [1, 0]], dtype=complex)
for L in (4, 7):
    wb = W.random_problem(8, 2, L, 12)
    f = np.random.default_rng(1).standard_normal((3, 12))
    bp = Q.BatchPlan(wb, 3, H1=H1, f=f, baths=[(1, 0.1, 7.5, 0.2), (2, 0.2, 3.0, 1.0), (3, 0.05, 2.2, 0.3)])
    a, wk = bp.alloc()
    assert np.isfinite(bp.run(a, wk)).all()
bp = Q.BatchPlan(W.random_problem(9, 3, 3, 8), 2)
a, wk = bp.alloc()
assert np.isfinite(bp.run(a, wk)).all()
# sharded path (emulated ranks): shard launch sets, pack / unpack
w = W.random_problem(6, 2, 6, 20)
ranks = [SH.ShardRank(w, 2, i) for i in range(2)]
SH.run_sharded(ranks, SH.emulated_exchange)
print("sanitize run ok")
