#!/usr/bin/env python
"""Time histories of the Taylor-Green diagnostics and the cost to reach a given time (SURVEY 8(f)
NEXT-3: the paper's equal-resolution methodology, at user-chosen sizes).

  python tools/tgv_history.py --case tgv_ss --n 116 --scheme cgks5 --t-end 1.0 --every 10
  python tools/tgv_history.py --case tgv_ss --n 384 --scheme gks2 --t-end 1.0 --every 10

Prints one JSON line per diagnostic sample (t, E_k, eps_S, eps_D, eps_T normalised by
rho0 U0^2 |Omega|, as P:474-479) and a final line with the device time spent stepping (CUDA events
around the steps, diagnostics excluded).  Runs on one GPU through the public Python API.
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="tgv_ss", choices=["tgv", "tgv_ss"])
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--scheme", default="cgks5", choices=["cgks5", "gks2"])
    ap.add_argument("--nonlinear", type=int, default=None)
    ap.add_argument("--t-end", type=float, default=1.0)
    ap.add_argument("--every", type=int, default=10)
    ap.add_argument("--lines", type=int, default=0, help="CGKS-5th with line-averaged derivative DOFs (NEXT-1)")
    ap.add_argument("--chi-c", type=float, default=None, help="GENO chi constant (reading R8; default 0.01)")
    ap.add_argument("--param", action="append", default=[], help="scheme parameter override k=v (tau_C, relax_C, ...)")
    args = ap.parse_args()
    import torch
    from cgks_inputs import tgv, tgv_supersonic
    from paper_2508_19911_b200 import CGKS_CGKS5, CGKS_GKS2, Solver
    if args.case == "tgv_ss":
        case = tgv_supersonic(args.n)
        U0 = math.sqrt(case.gamma) * 2.0
    else:
        case = tgv(args.n)
        U0 = 1.0
    norm = 1.0 * U0 * U0 * (2 * math.pi) ** 3  # rho0 U0^2 |Omega|
    scheme = CGKS_CGKS5 if args.scheme == "cgks5" else CGKS_GKS2
    nl = case.nonlinear if args.nonlinear is None else args.nonlinear
    stream = torch.cuda.current_stream()
    kw = {} if args.chi_c is None else {"chi_c": args.chi_c}
    for kv in args.param:
        k, v = kv.split("=", 1)
        kw[k] = float(v)
    S = Solver.from_case(case, scheme=scheme, nonlinear=nl, stream=stream.cuda_stream, lines=args.lines, **kw)
    S.set_state(case.Q, case.G if scheme == CGKS_CGKS5 else None)
    ms = 0.0
    t = 0.0
    while True:
        d = S.diagnostics()
        t, steps, _ = S.get_time()
        print(json.dumps({"t": t, "steps": steps, "E_k": d[0] / norm, "eps_S": d[1] / norm, "eps_D": d[2] / norm,
                          "eps_T": (d[1] + d[2]) / norm}), flush=True)
        if t >= args.t_end:
            break
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        S.step(args.every)
        e1.record(stream)
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1)
    print(json.dumps({"case": case.name, "n": args.n, "scheme": args.scheme, "nonlinear": nl, "lines": args.lines,
                      "chi_c": args.chi_c, "params": args.param, "t_end": t,
                      "steps": steps, "device_seconds_stepping": ms * 1e-3}), flush=True)
    S.close()


if __name__ == "__main__":
    main()
