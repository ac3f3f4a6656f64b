"""Debug: k_fused4 against the oracle for several L (correctness of every stage layout type)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import oracle as O
from paper_1205_6872_b200 import quapi as Q, workloads as W
from tests.test_oracle_engine import P
for L in [int(x) for x in sys.argv[1:]] or [6]:
    w = W.random_problem(700 + L, 2, L, 6 * L + 3, kind=W.J_DEBYE)
    p = Q.Plan(w)
    a, wk = p.alloc()
    r = p.run(a, wk)
    ro = O.run(P(w))
    print(L, p.sizes.fuse_steps, "max|drho| %.3e" % np.abs(r - ro).max(), flush=True)
