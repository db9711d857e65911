"""Thin ctypes binding of the C ABI in include/cgks.h (argument marshalling only).

Every step of the path runs in libcgks.so (sm_100a CUDA).  There is no CPU
fallback: if the library is missing or cannot be loaded this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CGKS_LIB", os.path.join(_HERE, "libcgks.so"))  # override for experiments only

CGKS_OK, CGKS_ERR_CONFIG, CGKS_ERR_POSITIVITY, CGKS_ERR_NUMERICAL, CGKS_ERR_CUDA, CGKS_ERR_COMM = 0, 2, 3, 4, 5, 6
CGKS_BC_PERIODIC, CGKS_BC_INFLOW, CGKS_BC_OUTFLOW = 0, 1, 2
CGKS_GKS2, CGKS_CGKS5 = 0, 1
CGKS_TIME_DEFAULT, CGKS_TIME_S1O2, CGKS_TIME_S2O4 = 0, 1, 2


class cgks_grid(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64 * 3),
        ("lo", ctypes.c_double * 3),
        ("hi", ctypes.c_double * 3),
        ("bc", (ctypes.c_int * 2) * 3),
        ("bc_state", ((ctypes.c_double * 5) * 2) * 3),
        ("nproc", ctypes.c_int * 3),
        ("rank", ctypes.c_int),
        ("nccl_id", ctypes.c_void_p),
        ("stream", ctypes.c_void_p),
        ("nodes", ctypes.POINTER(ctypes.c_double) * 3),
    ]


class cgks_scheme(ctypes.Structure):
    _fields_ = [
        ("id", ctypes.c_int),
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
        ("chi_scale", ctypes.c_double),
    ]


class CgksError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"cgks error {code}: {msg}")
        self.code = code


_lib = None

EXPORTS = ["cgks_scheme_defaults", "cgks_create", "cgks_local_extent", "cgks_set_state", "cgks_step",
           "cgks_get_state", "cgks_get_time", "cgks_last_error", "cgks_launches_per_step", "cgks_profile",
           "cgks_algorithmic_flops", "cgks_fp64_peak", "cgks_decompose", "cgks_decompose_pencil", "cgks_nccl_unique_id", "cgks_step_group", "cgks_comm_info",
           "cgks_z_chunk",
           "cgks_set_state_async", "cgks_step_async", "cgks_get_state_async", "cgks_sync", "cgks_destroy"]


def load(path: str = LIB_PATH):
    """Load libcgks.so (raises if missing: the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(path)
    vp, dp = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)
    L.cgks_scheme_defaults.argtypes = [ctypes.c_int, ctypes.POINTER(cgks_scheme)]
    L.cgks_create.argtypes = [ctypes.POINTER(cgks_grid), ctypes.c_double, ctypes.c_double, ctypes.c_double,
                              ctypes.POINTER(cgks_scheme), ctypes.POINTER(vp)]
    L.cgks_create.restype = ctypes.c_int
    L.cgks_local_extent.argtypes = [vp, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    L.cgks_set_state.argtypes = [vp, vp, vp]
    L.cgks_step.argtypes = [vp, ctypes.c_int]
    L.cgks_get_state.argtypes = [vp, vp, vp]
    L.cgks_set_state_async.argtypes = [vp, vp, vp]
    L.cgks_step_async.argtypes = [vp, ctypes.c_int]
    L.cgks_get_state_async.argtypes = [vp, vp, vp]
    L.cgks_sync.argtypes = [vp]
    L.cgks_get_time.argtypes = [vp, dp, ctypes.POINTER(ctypes.c_int64), dp]
    L.cgks_diagnostics.argtypes = [vp, dp]
    L.cgks_set_lines.argtypes = [vp, vp]
    L.cgks_get_lines.argtypes = [vp, vp]
    L.cgks_qcriterion.argtypes = [vp, dp]
    L.cgks_last_error.argtypes = [vp]
    L.cgks_last_error.restype = ctypes.c_char_p
    L.cgks_launches_per_step.argtypes = [vp]
    L.cgks_profile.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_char_p, dp,
                               ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)]
    L.cgks_algorithmic_flops.argtypes = [vp, ctypes.c_int, ctypes.c_char_p, dp, dp, ctypes.POINTER(ctypes.c_int)]
    L.cgks_fp64_peak.argtypes = [dp, dp]
    i64p = ctypes.POINTER(ctypes.c_int64)
    L.cgks_decompose.argtypes = [i64p, ctypes.POINTER(ctypes.c_int), ctypes.c_int, i64p, i64p,
                                 ctypes.POINTER(ctypes.c_int)]
    L.cgks_decompose_pencil.argtypes = [i64p, ctypes.POINTER(ctypes.c_int), ctypes.c_int, i64p, i64p,
                                        ctypes.POINTER(ctypes.c_int)]
    L.cgks_nccl_unique_id.argtypes = [ctypes.c_void_p]
    L.cgks_step_group.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int]
    ip = ctypes.POINTER(ctypes.c_int)
    L.cgks_comm_info.argtypes = [vp, ip, ip, ip]
    L.cgks_z_chunk.argtypes = [vp]
    L.cgks_destroy.argtypes = [vp]
    L.cgks_destroy.restype = None
    _lib = L
    return L


def fp64_peak():
    """Measured FP64 FMA throughput of the current device: (TFLOP/s, ms)."""
    t = ctypes.c_double()
    m = ctypes.c_double()
    rc = load().cgks_fp64_peak(ctypes.byref(t), ctypes.byref(m))
    if rc:
        raise CgksError(rc, "fp64 probe failed")
    return t.value, m.value


def decompose(n, nproc, rank):
    """Host-only z-slab decomposition of the library: (offset, local size, (lower, upper) neighbours)."""
    nn = (ctypes.c_int64 * 3)(*[int(x) for x in n])
    npr = (ctypes.c_int * 3)(*[int(x) for x in nproc])
    off = (ctypes.c_int64 * 3)()
    nl = (ctypes.c_int64 * 3)()
    nb = (ctypes.c_int * 2)()
    rc = load().cgks_decompose(nn, npr, int(rank), off, nl, nb)
    if rc:
        raise CgksError(rc, "unsupported decomposition")
    return tuple(off), tuple(nl), (nb[0], nb[1])


def decompose_pencil(n, nproc, rank):
    """Host-only pencil / y-slab decomposition nproc = (1, Py, Pz), rank = ry + Py rz:
    (offset, local size, (y lower, y upper, z lower, z upper) neighbours)."""
    nn = (ctypes.c_int64 * 3)(*[int(x) for x in n])
    npr = (ctypes.c_int * 3)(*[int(x) for x in nproc])
    off = (ctypes.c_int64 * 3)()
    nl = (ctypes.c_int64 * 3)()
    nb = (ctypes.c_int * 4)()
    rc = load().cgks_decompose_pencil(nn, npr, int(rank), off, nl, nb)
    if rc:
        raise CgksError(rc, "unsupported decomposition")
    return tuple(off), tuple(nl), tuple(nb)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = load().cgks_nccl_unique_id(buf)
    if rc:
        raise CgksError(rc, "cannot create an ncclUniqueId (libnccl.so.2 not loadable)")
    return buf.raw


def step_group(solvers, nsteps):
    """Advance the in-process slab contexts (ranks 0..n-1, nccl_id=None) in lock-step."""
    arr = (ctypes.c_void_p * len(solvers))(*[s.ctx.value for s in solvers])
    rc = load().cgks_step_group(arr, len(solvers), int(nsteps))
    if rc:
        raise CgksError(rc, solvers[0].last_error())


def scheme_defaults(scheme_id: int) -> cgks_scheme:
    s = cgks_scheme()
    load().cgks_scheme_defaults(scheme_id, ctypes.byref(s))
    return s


def _ptr(a):
    """Device pointer of a torch CUDA tensor, or host pointer of a contiguous float64 numpy array."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(a.data_ptr())
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]):
        raise ValueError("expected a C-contiguous float64 numpy array")
    return ctypes.c_void_p(a.ctypes.data)


class Solver:
    """One context of the C ABI: cgks_create / set_state / step / get_state / destroy."""

    def __init__(self, n, lo, hi, gamma=1.4, mu=0.0, Pr=1.0, scheme=CGKS_CGKS5, nonlinear=0,
                 time_scheme=CGKS_TIME_DEFAULT, cfl=None, fixed_dt=0.0, tau_eps=0.05, tau_C=10.0, relax_C=10.0,
                 k_venkat=0.3, chi_c=0.01, sutherland_S=0.0, lines=0, chi_scale=1.0, bc=((0, 0), (0, 0), (0, 0)), bc_state=None,
                 stream=None, nodes=None,
                 nproc=(1, 1, 1), rank=0, nccl_id=None):
        L = load()
        g = cgks_grid()
        for a in range(3):
            g.n[a] = int(n[a])
            g.lo[a] = float(lo[a])
            g.hi[a] = float(hi[a])
            g.nproc[a] = int(nproc[a])
            for s in range(2):
                g.bc[a][s] = int(bc[a][s])
                if bc_state is not None:
                    for v in range(5):
                        g.bc_state[a][s][v] = float(np.asarray(bc_state)[a, s, v])
        g.rank = int(rank)
        self._nodes = []
        if nodes is not None:
            for a in range(3):
                if nodes[a] is not None:
                    arr = np.ascontiguousarray(nodes[a], dtype=np.float64)
                    if arr.shape != (int(n[a]) + 1,):
                        raise ValueError(f"nodes[{a}] must hold n[{a}]+1 coordinates")
                    self._nodes.append(arr)
                    g.nodes[a] = arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        self._nccl_id = nccl_id
        self._nccl_buf = None if nccl_id is None else ctypes.create_string_buffer(bytes(nccl_id), 128)
        g.nccl_id = None if nccl_id is None else ctypes.cast(self._nccl_buf, ctypes.c_void_p)
        g.stream = None if stream is None else ctypes.c_void_p(int(stream))
        sc = scheme_defaults(scheme)
        sc.nonlinear = int(nonlinear)
        sc.time_scheme = int(time_scheme)
        if cfl is not None:
            sc.cfl = float(cfl)
        sc.fixed_dt = float(fixed_dt)
        sc.tau_eps, sc.tau_C, sc.relax_C = float(tau_eps), float(tau_C), float(relax_C)
        sc.k_venkat, sc.chi_c = float(k_venkat), float(chi_c)
        sc.sutherland_S = float(sutherland_S)
        sc.lines = int(lines)
        sc.chi_scale = float(chi_scale)
        ctx = ctypes.c_void_p()
        rc = L.cgks_create(ctypes.byref(g), float(gamma), float(mu), float(Pr), ctypes.byref(sc), ctypes.byref(ctx))
        if rc != CGKS_OK:
            raise CgksError(rc, "cgks_create failed (see stderr)")
        self._L = L
        self.ctx = ctx
        self._async_refs = []
        self.n = tuple(int(x) for x in n)
        self.scheme = scheme

    def _check(self, rc):
        if rc != CGKS_OK:
            raise CgksError(rc, self._L.cgks_last_error(self.ctx).decode())

    @property
    def local_shape(self):
        off = (ctypes.c_int64 * 3)()
        nn = (ctypes.c_int64 * 3)()
        self._check(self._L.cgks_local_extent(self.ctx, off, nn))
        return tuple(off), tuple(nn)

    def set_state(self, Q, G=None):
        self._check(self._L.cgks_set_state(self.ctx, _ptr(Q), _ptr(G)))

    def step(self, nsteps=1):
        rc = self._L.cgks_step(self.ctx, int(nsteps))
        self._check(rc)

    def step_rc(self, nsteps=1):
        """cgks_step returning the status code instead of raising."""
        return self._L.cgks_step(self.ctx, int(nsteps))

    def get_state(self, Q=None, G=None, with_grad=True):
        off, nn = self.local_shape
        shp = (nn[2], nn[1], nn[0])
        if Q is None:
            Q = np.zeros((5,) + shp)
        if G is None and with_grad:
            G = np.zeros((3, 5) + shp)
        self._check(self._L.cgks_get_state(self.ctx, _ptr(Q), _ptr(G)))
        return Q, G

    # -- asynchronous host I/O (cgks_*_async, cgks_sync): the arrays are kept alive until sync()
    def set_state_async(self, Q, G=None):
        self._async_refs.append((Q, G))
        self._check(self._L.cgks_set_state_async(self.ctx, _ptr(Q), _ptr(G)))

    def step_async(self, nsteps=1):
        self._check(self._L.cgks_step_async(self.ctx, int(nsteps)))

    def get_state_async(self, Q, G=None):
        """Enqueue the copy-out into the caller's buffers (valid after sync())."""
        self._async_refs.append((Q, G))
        self._check(self._L.cgks_get_state_async(self.ctx, _ptr(Q), _ptr(G)))

    def sync(self):
        rc = self._L.cgks_sync(self.ctx)
        self._async_refs.clear()
        self._check(rc)

    def get_time(self):
        t = ctypes.c_double()
        s = ctypes.c_int64()
        d = ctypes.c_double()
        self._check(self._L.cgks_get_time(self.ctx, ctypes.byref(t), ctypes.byref(s), ctypes.byref(d)))
        return t.value, s.value, d.value

    def set_lines(self, L):
        """cgks_set_lines: line-averaged derivatives [nl][5][nz][ny][nx] (line-DOF contexts)."""
        L = np.ascontiguousarray(L, dtype=np.float64)
        self._check(self._L.cgks_set_lines(self.ctx, _ptr(L)))

    def get_lines(self):
        """cgks_get_lines: [nl][5][nz][ny][nx] of this rank's cells, nl = 12 / 4 / 1 for 3-D / 2-D / 1-D."""
        dim = 3 if self.n[2] > 1 else (2 if self.n[1] > 1 else 1)
        nl = {3: 12, 2: 4, 1: 1}[dim]
        _, nn = self.local_shape
        out = np.zeros((nl, 5, nn[2], nn[1], nn[0]))
        self._check(self._L.cgks_get_lines(self.ctx, ctypes.c_void_p(out.ctypes.data)))
        return out

    def diagnostics(self):
        """cgks_diagnostics: (int 1/2 rho|U|^2 dV, int mu|curl U|^2 dV, int 4/3 mu (div U)^2 dV,
        int rho dV) of the current state, by quadrature of the reconstruction (unnormalised)."""
        out = np.zeros(4)
        self._check(self._L.cgks_diagnostics(self.ctx, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def qcriterion(self):
        """cgks_qcriterion: Q-criterion at every cell centroid, [nz][ny][nx] (rank-local)."""
        out = np.zeros(self.n[::-1])
        self._check(self._L.cgks_qcriterion(self.ctx, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def comm_info(self):
        """cgks_comm_info: (rank, nranks, backend) as the live communicator reports them (backend 0 single,
        1 NCCL, 2 in-process group)."""
        r, n, b = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        self._check(self._L.cgks_comm_info(self.ctx, ctypes.byref(r), ctypes.byref(n), ctypes.byref(b)))
        return r.value, n.value, b.value

    def z_chunk(self):
        """cgks_z_chunk: planes per z-chunk of the stages (0 = the whole grid per pass)."""
        return int(self._L.cgks_z_chunk(self.ctx))

    def last_error(self):
        return self._L.cgks_last_error(self.ctx).decode()

    def launches_per_step(self):
        return int(self._L.cgks_launches_per_step(self.ctx))

    def profile(self, nsteps):
        """Per-kernel CUDA-event timing over nsteps: {name: (total_ms, launches)}."""
        mx = 32
        names = ctypes.create_string_buffer(64 * mx)
        tot = (ctypes.c_double * mx)()
        cnt = (ctypes.c_int64 * mx)()
        nout = ctypes.c_int()
        self._check(self._L.cgks_profile(self.ctx, int(nsteps), mx, names, tot, cnt, ctypes.byref(nout)))
        out = {}
        for i in range(nout.value):
            nm = names.raw[64 * i:64 * (i + 1)].split(b"\0")[0].decode()
            out[nm] = (tot[i], cnt[i])
        return out

    def algorithmic_flops(self):
        """({kernel: FP64 flops per launch}, flops per cell-update) of this formulation."""
        mx = 16
        names = ctypes.create_string_buffer(64 * mx)
        fl = (ctypes.c_double * mx)()
        per = ctypes.c_double()
        nout = ctypes.c_int()
        self._check(self._L.cgks_algorithmic_flops(self.ctx, mx, names, fl, ctypes.byref(per), ctypes.byref(nout)))
        out = {}
        for i in range(nout.value):
            out[names.raw[64 * i:64 * (i + 1)].split(b"\0")[0].decode()] = fl[i]
        return out, per.value

    def close(self):
        if getattr(self, "ctx", None):
            self._L.cgks_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @classmethod
    def from_case(cls, case, scheme=CGKS_CGKS5, **kw):
        d = dict(gamma=case.gamma, mu=case.mu, Pr=case.Pr, nonlinear=case.nonlinear, cfl=case.cfl,
                 tau_eps=case.tau_eps, tau_C=case.tau_C, relax_C=case.relax_C, bc=case.bc,
                 bc_state=case.bc_state, sutherland_S=getattr(case, "sutherland_S", 0.0))
        d.update(kw)
        return cls(case.n, case.lo, case.hi, scheme=scheme, **d)
