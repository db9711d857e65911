import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_gpu_decomp import _run_single, _run_group
from cgks_inputs import random_smooth
case = random_smooth((16, 12, 20), seed=9, jump=0.0)
rng = np.random.default_rng(5)
L = case.G[np.array([1, 2, 1, 2, 2, 0, 2, 0, 0, 1, 0, 1])] + 0.01 * rng.standard_normal((12, 5) + tuple(case.n[::-1]))
kw = dict(mu=1e-3, Pr=0.72, lines=1)
for steps in (0, 1, 2):
    Q1, G1, t1, L1 = _run_single(case, 1, 0, steps, L=L, **kw)
    Qp, Gp, tp, Lp = _run_group(case, 1, 0, steps, 4, L=L, **kw)
    print("steps", steps, "t", t1 == tp, t1, tp)
    for nm, a, b, ax in (("Q", Q1, Qp, 1), ("G", G1, Gp, 2), ("L", L1, Lp, 2)):
        d = np.abs(a - b)
        dz = d.max(axis=tuple(i for i in range(d.ndim) if i != ax))
        print(nm, d.max(), "z planes with diff:", np.nonzero(dz)[0].tolist())
