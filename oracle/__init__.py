"""CPU oracle of the CGKS-5th / GKS-2nd time step (arXiv 2508.19911).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import this
package.  The product path (``paper_2508_19911_b200``) never imports it and
shares no code with it; see ``cgks_oracle.cpp`` for the algorithm and its
citations (PAPER.md line numbers "P:n", readings "R<k>" of DESIGN.md section 3).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cgks_oracle.cpp")
_LIB = os.path.join(_HERE, "libcgks_oracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle shared library (plain g++, OpenMP, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
               "-o", _LIB, _SRC]
        subprocess.run(cmd, check=True)
    return _LIB


class OrcParams(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int * 3),
        ("lo", ctypes.c_double * 3),
        ("hi", ctypes.c_double * 3),
        ("bc", (ctypes.c_int * 2) * 3),
        ("bc_state", ((ctypes.c_double * 5) * 2) * 3),
        ("gamma", ctypes.c_double),
        ("mu", ctypes.c_double),
        ("Pr", ctypes.c_double),
        ("scheme", ctypes.c_int),
        ("nonlinear", ctypes.c_int),
        ("time_scheme", ctypes.c_int),
        ("cfl", ctypes.c_double),
        ("fixed_dt", ctypes.c_double),
        ("tau_eps", ctypes.c_double),
        ("tau_C", ctypes.c_double),
        ("relax_C", ctypes.c_double),
        ("k_venkat", ctypes.c_double),
        ("chi_c", ctypes.c_double),
        ("sutherland_S", ctypes.c_double),
        ("lines", ctypes.c_int),
        ("nodes", ctypes.POINTER(ctypes.c_double) * 3),
        ("chi_scale", ctypes.c_double),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int)
        pp = ctypes.POINTER(OrcParams)
        L.orc_run.argtypes = [pp, dp, dp, ctypes.c_int, ctypes.c_int, dp]
        L.orc_run.restype = ctypes.c_int
        L.orc_dt.argtypes = [pp, dp, dp]
        L.orc_dt.restype = ctypes.c_double
        L.orc_moments_1d.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int, dp]
        L.orc_micro_slope.argtypes = [dp, ctypes.c_double, dp, dp]
        L.orc_time_integrals.argtypes = [ctypes.c_double, ctypes.c_double, dp]
        L.orc_flux_point.argtypes = [dp, dp, dp, dp, ctypes.c_double, dp, dp, dp]
        L.orc_flux_point.restype = ctypes.c_int
        L.orc_recon5_matrix.argtypes = [ctypes.c_int, ip, dp, ip, ip, dp]
        L.orc_recon5_matrix.restype = ctypes.c_int
        L.orc_recon_eval.argtypes = [pp, dp, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp]
        L.orc_recon_eval.restype = ctypes.c_int
        L.orc_geno_cell.argtypes = [pp, dp, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp]
        L.orc_geno_cell.restype = ctypes.c_int
        L.orc_stage_residual.argtypes = [pp, dp, dp, ctypes.c_double, dp, dp, dp, dp]
        L.orc_stage_residual.restype = ctypes.c_int
        L.orc_recon_eval_l.argtypes = [pp, dp, dp, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp,
                                       dp]
        L.orc_recon_eval_l.restype = ctypes.c_int
        L.orc_run_l.argtypes = [pp, dp, dp, dp, ctypes.c_int, ctypes.c_int, dp]
        L.orc_run_l.restype = ctypes.c_int
        L.orc_nlines.argtypes = [ctypes.c_int]
        L.orc_nlines.restype = ctypes.c_int
        L.orc_diagnostics.argtypes = [pp, dp, dp, dp]
        L.orc_diagnostics.restype = ctypes.c_int
        L.orc_qcriterion.argtypes = [pp, dp, dp, dp]
        L.orc_qcriterion.restype = ctypes.c_int
        L.orc_diagnostics_l.argtypes = [pp, dp, dp, dp, dp]
        L.orc_diagnostics_l.restype = ctypes.c_int
        L.orc_qcriterion_l.argtypes = [pp, dp, dp, dp, dp]
        L.orc_qcriterion_l.restype = ctypes.c_int
        L.orc_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


@dataclass
class Problem:
    """Problem description shared by the oracle wrapper (plain data, no arithmetic)."""
    n: tuple
    lo: tuple
    hi: tuple
    gamma: float = 1.4
    mu: float = 0.0
    Pr: float = 1.0
    scheme: int = 1            # 0 GKS-2nd, 1 CGKS-5th
    nonlinear: int = 0
    time_scheme: int = 2       # 1 S1O2, 2 S2O4
    cfl: float = 0.5
    fixed_dt: float = 0.0
    tau_eps: float = 0.05
    tau_C: float = 10.0
    relax_C: float = 10.0
    k_venkat: float = 0.3
    chi_c: float = 0.01
    chi_scale: float = 1.0     # GENO: zeta (R8) divided by chi_scale
    sutherland_S: float = 0.0  # 0: constant mu; 0.4042: the paper's Sutherland law
    lines: int = 0             # CGKS-5th: 1 = line-averaged derivatives as the own-cell data (NEXT-1)
    nodes: tuple = None        # stretched tensor-product mesh (NEXT-4): per-axis node coordinates (n_a + 1) or None
    bc: tuple = ((0, 0), (0, 0), (0, 0))
    bc_state: np.ndarray = field(default_factory=lambda: np.zeros((3, 2, 5)))

    def to_c(self) -> OrcParams:
        p = OrcParams()
        for a in range(3):
            p.n[a] = int(self.n[a])
            p.lo[a] = float(self.lo[a])
            p.hi[a] = float(self.hi[a])
            for s in range(2):
                p.bc[a][s] = int(self.bc[a][s])
                for v in range(5):
                    p.bc_state[a][s][v] = float(np.asarray(self.bc_state)[a, s, v])
        p.gamma, p.mu, p.Pr = self.gamma, self.mu, self.Pr
        p.scheme, p.nonlinear, p.time_scheme = self.scheme, self.nonlinear, self.time_scheme
        p.cfl, p.fixed_dt = self.cfl, self.fixed_dt
        p.tau_eps, p.tau_C, p.relax_C = self.tau_eps, self.tau_C, self.relax_C
        p.k_venkat, p.chi_c = self.k_venkat, self.chi_c
        p.chi_scale = float(self.chi_scale)
        p.sutherland_S = self.sutherland_S
        p.lines = int(self.lines)
        self._keep = []
        for a in range(3):
            if self.nodes is not None and self.nodes[a] is not None:
                arr = np.ascontiguousarray(self.nodes[a], dtype=np.float64)
                assert arr.shape == (self.n[a] + 1,)
                self._keep.append(arr)
                p.nodes[a] = arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        return p


def run(prob: Problem, Q: np.ndarray, G: np.ndarray | None, nsteps: int, nthreads: int = 0):
    """Advance (Q, G) by nsteps; returns (Q, G, t, last_dt, rc). Arrays are copied."""
    Q = np.ascontiguousarray(Q, dtype=np.float64).copy()
    Gc = None if G is None else np.ascontiguousarray(G, dtype=np.float64).copy()
    if Gc is None and prob.scheme == 1:
        Gc = np.zeros((3,) + Q.shape, dtype=np.float64)
    tout = np.zeros(3)
    p = prob.to_c()
    rc = lib().orc_run(ctypes.byref(p), _ptr(Q), _ptr(Gc), int(nsteps), int(nthreads), _ptr(tout))
    return Q, Gc, float(tout[0]), float(tout[1]), int(rc)


def nlines(dim: int) -> int:
    return int(lib().orc_nlines(int(dim)))


def run_lines(prob: Problem, Q: np.ndarray, G: np.ndarray, L: np.ndarray, nsteps: int, nthreads: int = 0):
    """Line-DOF variant (prob.lines = 1): advance (Q, G, L) by nsteps; L = [nlines][5][nz][ny][nx].
    Returns (Q, G, L, t, last_dt, rc).  Arrays are copied."""
    Q = np.ascontiguousarray(Q, dtype=np.float64).copy()
    Gc = np.ascontiguousarray(G, dtype=np.float64).copy()
    Lc = np.ascontiguousarray(L, dtype=np.float64).copy()
    tout = np.zeros(3)
    p = prob.to_c()
    rc = lib().orc_run_l(ctypes.byref(p), _ptr(Q), _ptr(Gc), _ptr(Lc), int(nsteps), int(nthreads), _ptr(tout))
    return Q, Gc, Lc, float(tout[0]), float(tout[1]), int(rc)


def dt(prob: Problem, Q: np.ndarray) -> float:
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    p = prob.to_c()
    return float(lib().orc_dt(ctypes.byref(p), _ptr(Q), None))


def moments_1d(U: float, lam: float, side: int) -> np.ndarray:
    out = np.zeros(9)
    lib().orc_moments_1d(U, lam, side, _ptr(out))
    return out


def micro_slope(prim, gamma: float, b) -> np.ndarray:
    prim = np.ascontiguousarray(prim, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    a = np.zeros(5)
    lib().orc_micro_slope(_ptr(prim), gamma, _ptr(b), _ptr(a))
    return a


def time_integrals(T: float, tau: float) -> np.ndarray:
    C = np.zeros(6)
    lib().orc_time_integrals(T, tau, _ptr(C))
    return C


def flux_point(WL, dWL, WR, dWR, gamma, dt, mu=0.0, Pr=1.0, tau_eps=0.05, tau_C=10.0, relax_C=10.0,
               compact=1, sutherland_S=0.0):
    """Interface flux at one Gauss point (normal frame). Returns a dict of outputs."""
    WL = np.ascontiguousarray(WL, dtype=np.float64)
    WR = np.ascontiguousarray(WR, dtype=np.float64)
    dWL = np.ascontiguousarray(dWL, dtype=np.float64).reshape(15)
    dWR = np.ascontiguousarray(dWR, dtype=np.float64).reshape(15)
    fpar = np.array([dt, mu, Pr, tau_eps, tau_C, relax_C, compact, sutherland_S], dtype=np.float64)
    out = np.zeros(64)
    sl = np.zeros(60)
    rc = lib().orc_flux_point(_ptr(WL), _ptr(dWL), _ptr(WR), _ptr(dWR), gamma, _ptr(fpar), _ptr(out), _ptr(sl))
    if rc:
        raise ValueError(f"oracle flux failed rc={rc}")
    names = ["Fn", "Ft", "Qn", "Qt", "QLn", "QLt", "QRn", "QRt", "Fbar_dt", "Fbar_half"]
    d = {nm: out[5 * i:5 * i + 5].copy() for i, nm in enumerate(names)}
    d["tau"], d["tau0"] = out[50], out[51]
    d["W0"] = out[52:57].copy()
    d["aL"] = sl[0:15].reshape(3, 5).copy()
    d["aR"] = sl[15:30].reshape(3, 5).copy()
    d["abar"] = sl[30:45].reshape(3, 5).copy()
    d["AL"], d["AR"], d["Abar"] = sl[45:50].copy(), sl[50:55].copy(), sl[55:60].copy()
    return d


def recon5_matrix(dim: int):
    sizes = (ctypes.c_int * 3)()
    L = lib()
    L.orc_recon5_matrix(dim, sizes, None, None, None, None)
    nb, nc, nd = sizes[0], sizes[1], sizes[2]
    R = np.zeros((nb, nd))
    B = np.zeros((nb, 3), dtype=np.int32)
    N = np.zeros((nc, 3), dtype=np.int32)
    LS = np.zeros((nd - nc, 4))
    ok = L.orc_recon5_matrix(dim, sizes, _ptr(R), B.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                             N.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), _ptr(LS))
    return dict(R=R, basis=B, nbrs=N, ls=LS, rank_ok=bool(ok), nb=nb, nc=nc, nd=nd)


def recon_eval_lines(prob: Problem, Q, G, L, ijk, x):
    """recon_eval with the line-averaged derivatives L ([nlines][5][nz][ny][nx]) of the line-DOF variant."""
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    G = np.ascontiguousarray(G, dtype=np.float64)
    L = np.ascontiguousarray(L, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 3)
    out = np.zeros((x.shape[0], 20))
    chi = np.zeros(5)
    p = prob.to_c()
    rc = lib().orc_recon_eval_l(ctypes.byref(p), _ptr(Q), _ptr(G), _ptr(L), int(ijk[0]), int(ijk[1]), int(ijk[2]),
                                x.shape[0], _ptr(x), _ptr(out), _ptr(chi))
    if rc:
        raise ValueError(f"recon_eval rc={rc}")
    return out[:, :5], out[:, 5:].reshape(-1, 3, 5), chi


def geno_cell(prob: Problem, Q, G, ijk):
    """GENO internals of cell ijk (CGKS-5th, nonlinear): IS (6,5), omega (6,5), bsub (6,3,5), chi (5,);
    sub-stencil m = 2 axis + side (0 minus, 1 plus); only the first 2*dim rows are meaningful."""
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    G = np.ascontiguousarray(G, dtype=np.float64)
    IS, om, bs, chi = np.zeros((6, 5)), np.zeros((6, 5)), np.zeros((6, 3, 5)), np.zeros(5)
    p = prob.to_c()
    rc = lib().orc_geno_cell(ctypes.byref(p), _ptr(Q), _ptr(G), int(ijk[0]), int(ijk[1]), int(ijk[2]),
                             _ptr(IS), _ptr(om), _ptr(bs), _ptr(chi))
    if rc:
        raise ValueError(f"geno_cell rc={rc}")
    return IS, om, bs, chi


def recon_eval(prob: Problem, Q, G, ijk, x):
    """Reconstruct cell ijk and evaluate at reference points x (npts,3). Returns (W (npts,5), dW (npts,3,5), chi/phi)."""
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    G = None if G is None else np.ascontiguousarray(G, dtype=np.float64)
    if G is None:
        G = np.zeros((3,) + Q.shape)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 3)
    out = np.zeros((x.shape[0], 20))
    chi = np.zeros(5)
    p = prob.to_c()
    rc = lib().orc_recon_eval(ctypes.byref(p), _ptr(Q), _ptr(G), int(ijk[0]), int(ijk[1]), int(ijk[2]),
                              x.shape[0], _ptr(x), _ptr(out), _ptr(chi))
    if rc:
        raise ValueError(f"recon_eval rc={rc}")
    return out[:, :5], out[:, 5:].reshape(-1, 3, 5), chi


def diagnostics(prob: Problem, Q, G=None, L=None):
    """Quadrature of the reconstructed state (orc_diagnostics): returns
    (int 1/2 rho|U|^2 dV, int mu|curl U|^2 dV, int 4/3 mu (div U)^2 dV, int rho dV).  L: line DOFs."""
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    G = np.zeros((3,) + Q.shape) if G is None else np.ascontiguousarray(G, dtype=np.float64)
    out = np.zeros(4)
    p = prob.to_c()
    if L is not None:
        L = np.ascontiguousarray(L, dtype=np.float64)
        rc = lib().orc_diagnostics_l(ctypes.byref(p), _ptr(Q), _ptr(G), _ptr(L), _ptr(out))
    else:
        rc = lib().orc_diagnostics(ctypes.byref(p), _ptr(Q), _ptr(G), _ptr(out))
    if rc:
        raise ValueError(f"oracle diagnostics failed rc={rc}")
    return out


def qcriterion(prob: Problem, Q, G=None, L=None):
    """Q-criterion at every cell centroid from the cell's reconstruction (orc_qcriterion): [nz][ny][nx]."""
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    G = np.zeros((3,) + Q.shape) if G is None else np.ascontiguousarray(G, dtype=np.float64)
    out = np.zeros(Q.shape[1:])
    p = prob.to_c()
    if L is not None:
        L = np.ascontiguousarray(L, dtype=np.float64)
        rc = lib().orc_qcriterion_l(ctypes.byref(p), _ptr(Q), _ptr(G), _ptr(L), _ptr(out))
    else:
        rc = lib().orc_qcriterion(ctypes.byref(p), _ptr(Q), _ptr(G), _ptr(out))
    if rc:
        raise ValueError(f"oracle qcriterion failed rc={rc}")
    return out


def stage_residual(prob: Problem, Q, G, dt: float):
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    G = np.zeros((3,) + Q.shape) if G is None else np.ascontiguousarray(G, dtype=np.float64)
    L = np.zeros_like(Q)
    Lt = np.zeros_like(Q)
    Gn = np.zeros((3,) + Q.shape)
    Gt = np.zeros((3,) + Q.shape)
    p = prob.to_c()
    rc = lib().orc_stage_residual(ctypes.byref(p), _ptr(Q), _ptr(G), dt, _ptr(L), _ptr(Lt), _ptr(Gn), _ptr(Gt))
    if rc:
        raise ValueError(f"stage_residual rc={rc}")
    return L, Lt, Gn, Gt


def max_threads() -> int:
    return int(lib().orc_max_threads())
