import sys, math, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle
from cgks_inputs import gl_average, line_derivatives, stretched_nodes
from paper_2508_19911_b200 import Solver
from parity_util import rel_linf, worst
n = (20, 12, 10)
lo, hi = (0.0, 0.0, 0.0), (2 * math.pi,) * 3
def prim(x, y, z):
    return (1.0 + 0.2 * np.sin(x) * np.cos(2 * y) + 0.1 * np.cos(z), 0.3 * np.sin(y + z),
            -0.2 * np.cos(x) * np.sin(z), 0.25 * np.sin(x + 2 * y), 1.0 + 0.1 * np.cos(x + y) * np.sin(z))
for stretched in (0, 1):
    nodes = (stretched_nodes(20, 0.0, 2 * math.pi, 2.0, "tanh"), stretched_nodes(12, 0.0, 2 * math.pi, 0.25), None) if stretched else None
    mn = (nodes[0], nodes[1], np.linspace(0.0, 2 * math.pi, 11)) if stretched else None
    Q, G = gl_average(prim, n, lo, hi, 1.4, nq=4, mesh_nodes=mn)
    L = line_derivatives(prim, n, lo, hi, 1.4, mesh_nodes=mn)
    for nl in (0, 1):
        for bc in (((2, 2), (0, 0), (0, 0)), ((1, 1), (0, 0), (0, 0)), ((0, 0), (2, 2), (0, 0))):
            kw = dict(mu=2e-3, Pr=0.72, nonlinear=nl, cfl=0.3, bc=bc, lines=1, fixed_dt=0.01)
            p = oracle.Problem(n=n, lo=lo, hi=hi, scheme=1, time_scheme=2, nodes=nodes, **kw)
            Qo, Go, Lo, to, _, rc = oracle.run_lines(p, Q, G, L, 1)
            S = Solver(n=n, lo=lo, hi=hi, scheme=1, time_scheme=2, nodes=nodes, **kw)
            S.set_state(Q, G); S.set_lines(L); S.step(1)
            Qg, Gg = S.get_state(); Lg = S.get_lines(); S.close()
            dq = np.abs(Qg - Qo).max(axis=(0,))
            where = np.argwhere(dq > 1e-12)
            print("str", stretched, "nl", nl, "bc", bc, "rc", rc, worst(rel_linf(Qg, Qo, Gg, Go, L=2 * math.pi)),
                  "L", np.abs(Lg - Lo).max(), "bad cells (z,y,x) sample", where[:4].tolist(), len(where))
