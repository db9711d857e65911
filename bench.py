#!/usr/bin/env python
"""Benchmark of the CGKS-5th hot path on B200 (BASELINE.json metric: CGKS-5th FP64
cell-updates/s and the fraction of the FP64/HBM roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload tgv<N>|hit<N>|tgv_ss<N>|tgv512slab|shock_vortex|vortex40] [--scheme cgks5|gks2]

Multi-GPU (one process per GPU, NCCL): `python bench.py --gpus N` starts the N ranks itself
(torch.distributed.run, 127.0.0.1) unless it already runs under a launcher (WORLD_SIZE set), and
refuses a WORLD_SIZE that differs from --gpus.  Default workloads: N = 1 the 128^3 TGV (the
north_star roofline case); N > 1 the north_star weak-scaling run, a 512 x 512 x 64 block of the
512^3 TGV per GPU (BASELINE configs[4]: N = 8 is the 512^3 run); --strong --workload tgv<n> splits
a global n^3 grid instead.  Every rank prints one line on stderr with its communicator's own rank
and rank count (cgks_comm_info: ncclCommUserRank / ncclCommCount).

A step is one full S2O4 time step of CGKS-5th (dt min-reduction + two stages of
reconstruction, fluxes and update) over the whole grid.  Default workload: the
128^3 Taylor-Green vortex (BASELINE configs[1], the north_star's roofline case),
linear CGKS-5th as in the paper's subsonic TGV.  Inputs are synthetic (the
analytic TGV initial condition) and resident in HBM; the state (335 MB) is larger
than L2 (126 MB), so no flush is needed between steps.

--impl reference times the CPU oracle (oracle/, test infrastructure) on the host
cores on a bounded sample of the same workload (the paper's code is not available;
this tier's reference arm is the oracle).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "CGKS-5th FP64 cell-updates/sec at 1/2/4/8 B200; % of HBM/FP64 roofline"


def slab512(ws, rank):
    """BASELINE configs[4] per-GPU block: 512 x 512 x 64 planes of the 512^3 TGV,
    z-planes [64 rank, 64 rank + 64); N ranks hold a 512 x 512 x 64N grid (N = 8: the 512^3 run)."""
    from cgks_inputs import tgv
    c = tgv(512, z0=64 * rank, nzb=64)
    c.n = (512, 512, 64 * ws)
    c.hi = (c.hi[0], c.hi[1], c.lo[2] + 2 * math.pi * 64 * ws / 512)
    return c


def pencil_block(nb, py, pz, rank):
    """Rank ry + py rz's block of the global nb^3 TGV split into py x pz pencils (cgks_decompose_pencil's layout):
    rows [ry nb/py, (ry+1) nb/py) of the planes [rz nb/pz, (rz+1) nb/pz); case.n stays the global grid."""
    from cgks_inputs import tgv
    ry, rz = rank % py, rank // py
    case = tgv(nb, z0=rz * (nb // pz), nzb=nb // pz)  # the rank's z-slab, then its rows
    ysl = slice(ry * (nb // py), (ry + 1) * (nb // py))
    case.Q = np.ascontiguousarray(case.Q[:, :, ysl])
    case.G = np.ascontiguousarray(case.G[:, :, :, ysl])
    return case


def make_case(name):
    """tgv<N> (TGV, BASELINE configs[1]), tgv_ss<N> (high-speed TGV with Sutherland viscosity, nonlinear,
    P:455-474, NEXT-2: the paper's meshes are 116^3 and 384^3), hit<N>, shock_vortex, vortex40."""
    import re
    from cgks_inputs import hit, shock_vortex, tgv, tgv_supersonic, vortex
    m = re.fullmatch(r"(tgv_ss|tgv|hit)(\d+)", name)
    if m:
        n = int(m.group(2))
        return {"tgv_ss": tgv_supersonic, "tgv": tgv, "hit": hit}[m.group(1)](n)
    if name == "shock_vortex":
        return shock_vortex()
    if name == "vortex40":
        return vortex(40)
    raise ValueError(name)


def workload_desc(name, ws):
    """(config name, global cells, nonlinear) of a workload without building its initial state"""
    import re
    if name == "tgv512slab":
        return f"tgv 512x512x{64 * ws}", 512 * 512 * 64 * ws, 0
    m = re.fullmatch(r"(tgv_ss|tgv|hit)(\d+)", name)
    if m:
        n = int(m.group(2))
        return f"{m.group(1)} {n}x{n}x{n}", n ** 3, 0 if m.group(1) == "tgv" else 1
    c = make_case(name)
    return f"{c.name} {c.n[0]}x{c.n[1]}x{c.n[2]}", c.ncell, c.nonlinear


class ClockSampler:
    """SM clocks, power and throttle reasons sampled during the timed region (NVML in-process; nvidia-smi as the fallback)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.source = "nvml"
        self._stop = threading.Event()
        self._t = None

    def _nvml_handle(self):
        """NVML handle of this rank's GPU (by the CUDA device's UUID; by index when the UUID is unavailable)."""
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(torch.cuda.current_device()).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid) if not uuid.startswith("GPU-") else uuid)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _run_nvml(self):
        """In-process NVML sampling every 10 ms (a 20-step region of 0.2 s yields ~20 samples; an nvidia-smi
        process per sample yields one or two).  Rows in the nvidia-smi column order."""
        nv, h = self._nvml_handle()
        bits = [(0x8, 3), (0x40, 4), (0x20, 5), (0x4, 6)]  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            try:
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
            except Exception:
                pw = float("nan")
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            row = [str(sm), str(mx), f"{pw:.1f}", "", "", "", ""]
            for bit, col in bits:
                row[col] = "Active" if (r & bit) else "Not Active"
            self.rows.append(row)
            self._stop.wait(0.01)

    def _run(self):
        try:
            self._run_nvml()
            return
        except Exception:
            self.source = "nvidia-smi"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": self.source,
                "sm_mhz_min": min(sm) if sm else None, "power_w_max": max(pw) if pw else None}


def dist_init():
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.is_available():
        torch.cuda.set_device(lr)
    if ws > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        dist.init_process_group(backend=backend)
    return rank, ws, lr


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_baseline(case_name, scheme, budget_s=20.0):
    """The oracle as it stands, on the host cores, on a bounded sample of the same workload:
    the same flow at 32^3 (the per-cell work of a step does not depend on the grid size)."""
    import oracle
    from cgks_inputs import tgv
    oracle.build()
    if case_name.startswith("tgv_ss"):
        from cgks_inputs import tgv_supersonic
        c = tgv_supersonic(32)
    else:
        c = tgv(32) if case_name.startswith("tgv") else make_case(case_name)
    if case_name.startswith("hit"):
        from cgks_inputs import hit
        c = hit(32)
    prob = oracle.Problem(**c.problem_kwargs(), scheme=1 if scheme == "cgks5" else 0,
                          time_scheme=2 if scheme == "cgks5" else 1)
    Q, G = c.Q, c.G
    steps, t_used = 0, 0.0
    while t_used < budget_s * 0.5 or steps == 0:
        t0 = time.perf_counter()
        Q, G, _, _, rc = oracle.run(prob, Q, G, 1)
        t_used += time.perf_counter() - t0
        steps += 1
        if rc or t_used > budget_s:
            break
    cores = oracle.max_threads()
    # one thread: the same flow at 16^3, one step (~5 s)
    from cgks_inputs import hit, tgv_supersonic
    c1 = tgv_supersonic(16) if case_name.startswith("tgv_ss") else (hit(16) if case_name.startswith("hit") else tgv(16))
    p1 = oracle.Problem(**c1.problem_kwargs(), scheme=1 if scheme == "cgks5" else 0,
                        time_scheme=2 if scheme == "cgks5" else 1)
    t0 = time.perf_counter()
    oracle.run(p1, c1.Q, c1.G, 1, nthreads=1)
    t1 = time.perf_counter() - t0
    return {"value": c.ncell * steps / t_used, "unit": "cell-updates/s", "cores": cores, "kind": "oracle",
            "sample": f"{c.name} {c.n[0]}x{c.n[1]}x{c.n[2]}, {steps} step(s), {t_used:.1f} s, "
                      f"OpenMP threads={cores}",
            "value_1thread": c1.ncell / t1,
            "sample_1thread": f"{c1.name} {c1.n[0]}x{c1.n[1]}x{c1.n[2]}, 1 step, {t1:.1f} s, 1 thread"}


def run_reference(args, rank, ws):
    """The reference arm: the oracle as it stands, W untimed + K timed steps of a bounded sample
    (the same flow at 24^3) of our arm's workload, on the host cores; the line carries our arm's
    config (metric, unit and workload), the sample is named in cpu_baseline."""
    if rank != 0:
        return 0
    import oracle
    from cgks_inputs import hit, tgv, tgv_supersonic
    oracle.build()
    full_name, full_cells, full_nl = workload_desc(args.workload, ws)
    if args.workload.startswith("tgv_ss"):
        c = tgv_supersonic(24)
    elif args.workload.startswith("tgv"):
        c = tgv(24)
    elif args.workload.startswith("hit"):
        c = hit(24)
    else:
        c = make_case(args.workload)
    prob = oracle.Problem(**c.problem_kwargs(), scheme=1 if args.scheme == "cgks5" else 0,
                          time_scheme=2 if args.scheme == "cgks5" else 1)
    Q, G = c.Q, c.G
    # all host cores (a launcher such as torch.distributed.run sets OMP_NUM_THREADS=1 per rank)
    nth = os.cpu_count() or 1
    for _ in range(args.warmup):
        Q, G, _, _, _ = oracle.run(prob, Q, G, 1, nthreads=nth)
    t0 = time.perf_counter()
    Q, G, _, _, _ = oracle.run(prob, Q, G, args.steps, nthreads=nth)
    dt = time.perf_counter() - t0
    value = c.ncell * args.steps / dt
    cores = oracle.max_threads()
    line = {"metric": METRIC, "value": value, "unit": "cell-updates/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": full_name,
                       "scheme": args.scheme + ("-geno" if full_nl else "-linear"),
                       "time_scheme": "S2O4" if args.scheme == "cgks5" else "S1O2", "global_cells": full_cells,
                       "parallelism": "host cores (CPU oracle)"},
            "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": cores, "kind": "oracle",
                             "sample": f"{c.name} {c.n[0]}x{c.n[1]}x{c.n[2]} (bounded sample of the workload), "
                                       f"{args.warmup} untimed + {args.steps} timed steps, OpenMP threads={cores}"},
            "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, rank, ws, lr):
    import torch

    from paper_2508_19911_b200 import Solver
    from paper_2508_19911_b200.binding import fp64_peak

    scheme_id = 1 if args.scheme == "cgks5" else 0
    stream = torch.cuda.current_stream()
    if ws > 1:
        # weak scaling (BASELINE configs[4] strategy): each GPU owns a 128^3 z-slab of the TGV on
        # [-pi,pi]^2 x [-pi, -pi + 2 pi N]; halo exchange and dt allreduce over NCCL inside cgks_step
        if not args.workload.startswith("tgv") or args.workload.startswith("tgv_ss"):
            raise SystemExit("multi-GPU runs use the TGV workload")
        import torch.distributed as dist

        from cgks_inputs import tgv
        from paper_2508_19911_b200 import nccl_unique_id
        nproc = (1, 1, ws)
        if args.pencil:
            py, pz = (int(x) for x in args.pencil.lower().split("x"))
            if py * pz != ws or not args.strong:
                raise SystemExit("--pencil PyxPz needs Py * Pz = N ranks and --strong --workload tgv<n>")
            nproc = (1, py, pz)
        if args.workload == "tgv512slab":
            case = slab512(ws, rank)
        elif args.strong and args.pencil:  # strong scaling over Py x Pz pencils (rank = ry + Py rz)
            nb = int(args.workload[3:])
            py, pz = nproc[1], nproc[2]
            if nb % py or nb % pz or nb // py < 4 or nb // pz < 4:
                raise SystemExit(f"pencils need n divisible by Py and Pz with >= 4 rows / planes per rank ({nb}, {py}x{pz})")
            case = pencil_block(nb, py, pz, rank)
        elif args.strong:  # strong scaling: the global n^3 TGV split into N z-slabs
            nb = int(args.workload[3:])
            if nb % ws or nb // ws < 4:
                raise SystemExit(f"strong scaling needs n divisible by N with >= 4 planes per rank ({nb}, {ws})")
            case = tgv(nb, z0=rank * (nb // ws), nzb=nb // ws)
        else:
            nb = int(args.workload[3:])
            case = tgv(nb, zrep=ws, z0=rank * nb, nzb=nb)
        if args.nonlinear is not None:
            case.nonlinear = args.nonlinear
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        S = Solver.from_case(case, scheme=scheme_id, stream=stream.cuda_stream, nproc=nproc, rank=rank,
                             nccl_id=obj[0])
        cr, cn, cb = S.comm_info()
        print(json.dumps({"bench_rank": rank, "world_size": ws, "comm_rank": cr, "comm_nranks": cn,
                          "backend": "nccl" if cb == 1 else cb, "device": torch.cuda.current_device()}),
              file=sys.stderr, flush=True)
        if (cr, cn) != (rank, ws):
            raise SystemExit(f"communicator reports rank {cr} of {cn}, expected {rank} of {ws}")
    else:
        if args.workload == "tgv512slab":  # the block of one rank of the 512^3 run, with the periodic self halo
            case = slab512(1, 0)
            args.nccl_self = True
        else:
            case = make_case(args.workload)
        if args.nonlinear is not None:
            case.nonlinear = args.nonlinear
        nodes = None
        if args.stretch:  # sine-stretched tensor-product mesh (NEXT-4); the state is the workload's own IC
            from cgks_inputs import stretched_nodes
            nodes = tuple(stretched_nodes(case.n[a], case.lo[a], case.hi[a], args.stretch) if case.n[a] > 1 else None
                          for a in range(3))
        nid = None
        if args.nccl_self:  # the slab path on one GPU: NCCL halo exchange with itself (overlapped)
            from paper_2508_19911_b200 import nccl_unique_id
            nid = nccl_unique_id()
        S = Solver.from_case(case, scheme=scheme_id, stream=stream.cuda_stream, lines=args.lines, nodes=nodes,
                             nccl_id=nid)
    NV = 20 if scheme_id == 1 else 5
    if case.ncell > (1 << 25):  # large grids: from host memory (the library stages one field at a time)
        S.set_state(np.ascontiguousarray(case.Q), np.ascontiguousarray(case.G) if scheme_id == 1 else None)
    else:
        Qd = torch.from_numpy(np.ascontiguousarray(case.Q)).cuda()
        Gd = torch.from_numpy(np.ascontiguousarray(case.G)).cuda()
        S.set_state(Qd, Gd if scheme_id == 1 else None)
        del Qd, Gd  # the library holds the state
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    z_chunk = S.z_chunk()
    free_b, total_b = torch.cuda.mem_get_info()
    hbm_used_gb = (total_b - free_b) / 1e9
    for _ in range(args.warmup):
        S.step(1)
    torch.cuda.synchronize()
    barrier(ws)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(lr) as clk:
        torch.cuda.synchronize()
        barrier(ws)
        e0.record(stream)
        S.step(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
    ms = e0.elapsed_time(e1)
    ms = max_over_ranks(ms, ws)
    cells = case.ncell  # global cells (case.n is the global grid)
    value = cells * args.steps / (ms * 1e-3)

    # e2e through the C ABI with host buffers: H2D of the inputs + steps + D2H of the result per step
    Qh = np.ascontiguousarray(case.Q)
    Gh = np.ascontiguousarray(case.G)
    Qo = np.empty_like(Qh)
    Go = np.empty_like(Gh) if scheme_id == 1 else None
    Qh_pin = torch.from_numpy(Qh).pin_memory()
    Gh_pin = torch.from_numpy(Gh).pin_memory()
    Qo_pin = torch.empty(Qh.shape, dtype=torch.float64).pin_memory()
    Go_pin = torch.empty(Gh.shape, dtype=torch.float64).pin_memory()
    # (a) the pipelined public calls: set_state_async / step_async / get_state_async, one cgks_sync at
    # the end; every step still copies its whole input in and its whole result out, the copies run
    # on the library's copy streams and overlap the neighbouring steps
    e2e_steps = max(1, args.steps)
    e2e_mode = "pipelined (cgks_set_state_async / cgks_step_async / cgks_get_state_async, copy streams)"
    try:  # W untimed warm-up iterations of the same calls (allocates the library's staging buffers)
        for _ in range(max(1, args.warmup)):
            S.set_state_async(Qh_pin, Gh_pin if scheme_id == 1 else None)
            S.step_async(1)
            S.get_state_async(Qo_pin, Go_pin if scheme_id == 1 else None)
        S.sync()
    except Exception:
        S.sync()
    torch.cuda.synchronize()
    barrier(ws)
    t0 = time.perf_counter()
    try:
        for _ in range(e2e_steps):
            S.set_state_async(Qh_pin, Gh_pin if scheme_id == 1 else None)
            S.step_async(1)
            S.get_state_async(Qo_pin, Go_pin if scheme_id == 1 else None)
        S.sync()
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - t0, ws)
    except Exception as ex:  # staging buffers do not fit next to a very large state: serial calls only
        e2e_s, e2e_mode = None, f"serial only ({ex})"
        S.sync()
    # (b) the synchronous calls, one after the other (no overlap)
    ser_steps = max(1, min(args.steps, 5))
    torch.cuda.synchronize()
    barrier(ws)
    t0 = time.perf_counter()
    for _ in range(ser_steps):
        S.set_state(Qh_pin.numpy(), Gh_pin.numpy() if scheme_id == 1 else None)
        S.step(1)
        S.get_state(Qo_pin.numpy(), Go_pin.numpy() if scheme_id == 1 else None, with_grad=scheme_id == 1)
    torch.cuda.synchronize()
    ser_s = max_over_ranks(time.perf_counter() - t0, ws)
    ser_val = cells * ser_steps / ser_s
    e2e_val = cells * e2e_steps / e2e_s if e2e_s else ser_val
    nbytes = Qh.nbytes + (Gh.nbytes if scheme_id == 1 else 0)

    # roofline of the dominant kernel: per-kernel CUDA-event durations on the library stream
    S.set_state(Qh, Gh if scheme_id == 1 else None)
    prof = S.profile(max(2, min(args.steps, 4)))
    flops, per_cell = S.algorithmic_flops()
    dom = max(prof, key=lambda k: prof[k][0])
    dom_ms = prof[dom][0] / prof[dom][1]
    total_prof = sum(v[0] for v in prof.values())
    peak64, _ = fp64_peak()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    achieved = flops.get(dom, 0.0) / (dom_ms * 1e-3) / 1e12
    # measured DRAM traffic per launch of the dominant kernel from the committed ncu --set full
    # capture of this workload (tools/ncu_summary.py traffic), else null
    traffic, traffic_src = None, None
    wl = f"{case.name} {case.n[0]}x{case.n[1]}x{case.n[2]} {args.scheme}" + ("-geno" if case.nonlinear else "-linear")
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        if tj.get("workload") == wl and ws == 1:
            traffic = tj["per_launch_bytes"].get(dom)
            traffic_src = "profiles/ncu_traffic.json (" + tj.get("source", "?") + ")"
    except Exception:
        pass
    roof = {"bound": "alu", "achieved": achieved, "peak": peak64, "unit": "TFLOP/s",
            "frac": achieved / peak64 if peak64 else None, "traffic": traffic, "traffic_unit": "bytes/launch",
            "traffic_source": traffic_src,
            "kernel": dom, "kernel_ms": dom_ms, "kernel_share": prof[dom][0] / total_prof,
            "algorithmic_flops_per_launch": flops.get(dom, 0.0),
            "peak_source": "measured FP64 DFMA probe (cgks_fp64_peak) in this run; MEASURED_PEAKS.json has no FP64",
            "step_frac": (per_cell * cells / ws) / (ms / args.steps * 1e-3) / 1e12 / peak64 if peak64 else None,
            "hbm_gbs_peak": peaks.get("hbm_gbs")}
    per_kernel = {k: {"ms_per_launch": v[0] / v[1], "launches": v[1],
                      "tflops": (flops.get(k, 0.0) / (v[0] / v[1] * 1e-3) / 1e12) if k in flops else None}
                  for k, v in prof.items()}
    S.close()

    if rank != 0:
        return 0
    line = {"metric": METRIC, "value": value, "unit": "cell-updates/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.strong and ws > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{case.name} {case.n[0]}x{case.n[1]}x{case.n[2]}"
                                   + (("" if args.strong else f" ({case.n[0]}^2 x {len(case.Q[0])} per GPU)") if ws > 1 else ""),
                       "scheme": args.scheme + ("-geno" if case.nonlinear else "-linear")
                       + ("-lines" if args.lines else "") + (f"-stretched{args.stretch:g}" if args.stretch else ""),
                       "time_scheme": "S2O4" if scheme_id == 1 else "S1O2", "global_cells": cells,
                       "parallelism": (f"pencil{args.pencil} (NCCL y + z halos, allreduce-min)" if args.pencil else
                                       f"zslab{ws} (NCCL halo + allreduce-min)") if ws > 1 else (
                           "zslab1 (NCCL self halo, overlapped)" if args.nccl_self else "1gpu"),
                       "l2": "state larger than L2 (no flush)",
                       "hbm_used_gb": round(hbm_used_gb, 1),
                       "z_chunk_planes": z_chunk},
            "roofline": roof,
            "algorithmic_flops_per_cell_update": per_cell,
            "per_kernel": per_kernel,
            "clocks": clk.summary(),
            "e2e": {"value": e2e_val, "unit": "cell-updates/s", "h2d_bytes_per_step": nbytes,
                    "d2h_bytes_per_step": nbytes, "steps": e2e_steps, "mode": e2e_mode,
                    "serial_value": ser_val, "serial_steps": ser_steps,
                    "host_buffers": "pinned (torch pin_memory)"},
            "gpu_launches": S.launches_per_step() * args.steps if S.ctx else None}
    line["gpu_launches"] = int(sum(v[1] for v in prof.values()) / max(2, min(args.steps, 4)) * args.steps)
    if not args.no_cpu_baseline and ws == 1:
        line["cpu_baseline"] = cpu_baseline(args.workload, args.scheme)
    print(json.dumps(line), flush=True)
    return 0


def launch_plan(gpus, env):
    """("run", None) under a launcher or for one GPU, ("exec", argv) to start the ranks with
    torch.distributed.run, ("refuse", msg) if WORLD_SIZE contradicts --gpus."""
    ws = env.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != gpus:
            return "refuse", f"WORLD_SIZE={ws} but --gpus {gpus}: refusing to run a different rank count"
        return "run", None
    if gpus <= 1:
        return "run", None
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    return "exec", [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
                    "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None,
                    help="default: tgv128 on 1 GPU, tgv512slab (512 x 512 x 64 per GPU) on N > 1")
    ap.add_argument("--scheme", default="cgks5", choices=["cgks5", "gks2"])
    ap.add_argument("--nonlinear", type=int, default=None)
    ap.add_argument("--lines", type=int, default=0, help="CGKS-5th with line-averaged derivative DOFs (NEXT-1)")
    ap.add_argument("--stretch", type=float, default=0.0,
                    help="sine-stretched tensor-product mesh with this amplitude (NEXT-4; timing only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pencil", default=None,
                    help="N > 1 with --strong: Py x Pz pencils (e.g. 2x4) instead of N z-slabs")
    ap.add_argument("--strong", action="store_true",
                    help="N > 1: split the global tgv<n> grid over the ranks (strong scaling) instead of n^3 per GPU")
    ap.add_argument("--nccl-self", action="store_true",
                    help="1 GPU through the z-slab path: ghost planes + NCCL halo exchange with itself")
    args = ap.parse_args()
    what, info = launch_plan(args.gpus, os.environ)
    if what == "refuse":
        print(info, file=sys.stderr)
        return 2
    if what == "exec":
        return subprocess.call(info + sys.argv[1:])
    rank, ws, lr = dist_init()
    if args.workload is None:
        args.workload = "tgv512slab" if ws > 1 and not args.strong else ("tgv512" if args.strong else "tgv128")
    if args.impl == "reference":
        return run_reference(args, rank, ws)
    return run_ours(args, rank, ws, lr)


if __name__ == "__main__":
    sys.exit(main())
