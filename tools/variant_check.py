"""Bitwise comparison of two builds of libcgks.so on several small cases (TMA and cp.async tiles, GENO, box
BCs, line DOFs, 2-D), 5 steps each.  Used for the schedule-perturbation race check (DESIGN 10a):

  CGKS_LIB=libcgks_jz.so  CHECK_REF=jz python tools/variant_check.py jz    # -DCGKS_JITTER -DCGKS_JITTER_ZERO
  CGKS_LIB=libcgks_jit.so CHECK_REF=jz python tools/variant_check.py jit   # -DCGKS_JITTER (0-4 us per warp)

and for experiment variants against the default build (CHECK_REF=base).  States go to /tmp/var_states."""
import sys, os, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from cgks_inputs import cases
from paper_2508_19911_b200 import Solver
v = sys.argv[1]
out = {}
runs = (("tgv", cases.tgv(40), dict(nonlinear=0)),
        ("hit", cases.hit(24), dict(nonlinear=1)),
        ("rs", cases.random_smooth((36, 20, 18), seed=3, mu=1e-3, jump=0.3), dict(nonlinear=1)),
        ("rsl", cases.random_smooth((20, 18, 16), seed=5, mu=1e-3), dict(nonlinear=1, lines=1)),
        ("sv", cases.shock_vortex(64, 32), dict(nonlinear=1)))
for name, case, kw in runs:
    S = Solver.from_case(case, scheme=1, **kw)
    S.set_state(case.Q, case.G)
    S.step(5)
    Q, G = S.get_state()
    S.close()
    out[name + "_Q"] = Q
    out[name + "_G"] = G
os.makedirs("/tmp/var_states", exist_ok=True)
np.savez(f"/tmp/var_states/state_{v}.npz", **out)
REF = os.environ.get("CHECK_REF", "base")
if v != REF and os.path.exists(f"/tmp/var_states/state_{REF}.npz"):
    b = np.load(f"/tmp/var_states/state_{REF}.npz")
    worst = 0.0
    for k in out:
        e = np.abs(out[k] - b[k]).max() / np.abs(b[k]).max()
        worst = max(worst, e)
    for k in out:
        if not np.array_equal(out[k], b[k]):
            d = np.abs(out[k] - b[k]); print("  ", k, "diff %.2e at" % (d.max() / np.abs(b[k]).max()), np.unravel_index(d.argmax(), d.shape), "n_diff", int((d > 0).sum()), "of", d.size)
    print(v, "max rel diff vs base %.2e" % worst, "bitwise" if all(np.array_equal(out[k], b[k]) for k in out) else "NOT bitwise")
