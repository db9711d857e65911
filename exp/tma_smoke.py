import sys; sys.path.insert(0,'.')
import numpy as np
from cgks_inputs import random_smooth
from paper_2508_19911_b200 import Solver
c = random_smooth((20, 12, 16), seed=8)
S = Solver.from_case(c, scheme=1, mu=1e-3, Pr=0.72)
S.set_state(c.Q, c.G)
S.step(1)
print("ok")
