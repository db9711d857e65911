import os, sys, math
sys.path.insert(0, ".")
import torch
from cgks_inputs import tgv_supersonic
from paper_2508_19911_b200 import CGKS_CGKS5, Solver, CgksError
case = tgv_supersonic(116)
S = Solver.from_case(case, scheme=CGKS_CGKS5, nonlinear=1, tau_C=0.0)
S.set_state(case.Q, case.G)
S.step(460)
print("at", S.get_time(), flush=True)
for s in range(40):
    try:
        S.step(1)
    except CgksError as e:
        print("step", 460 + s + 1, "error", e, flush=True)
        break
try:
    print("time after", S.get_time(), flush=True)
    S.step(1)
except CgksError as e:
    print("next step call:", e, flush=True)
try:
    Q, G = S.get_state()
    print("get_state ok", float(Q[0].min()), flush=True)
except CgksError as e:
    print("get_state:", e, flush=True)
