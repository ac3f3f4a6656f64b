import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import oracle as O
from paper_1205_6872_b200 import quapi as Q, workloads as W
from tests.test_oracle_engine import P
for fuse in ['1','2']:
    os.environ['QUAPI_FUSE_S'] = fuse
    for w in [W.CONFIGS[1].with_(n_steps=12), W.random_problem(3, 2, 3, 9)]:
        pl = Q.Plan(w); a, wk = pl.alloc(); r = pl.run(a, wk)
        ro = O.run(P(w))
        err = np.abs(r - ro).max(axis=(1,2))
        print(fuse, w.L, pl.sizes.fuse_steps, ["%.1e" % e for e in err])
