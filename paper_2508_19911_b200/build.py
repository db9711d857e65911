"""Build the sm_100a shared library libcgks.so in-tree (explicit nvcc; no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcgks.so")
SOURCES = ["cgks_api.cu", "cls_build.cpp", "stage_d1.cu", "stage_d2.cu", "stage_d3.cu"]
HEADERS = ["kernels.cuh", "flux1.cuh", "gks_flux.cuh", "cls_build.h", "flop_count.h", "recon_gen.cuh", "types.h", "driver.h",
           "stage_impl.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

# --register-usage-level=3 (ptxas default 5: "lower values inhibit optimizations that aggressively increase
# register usage"): the flux kernels sit at their 168-register cap, and at levels 0-3 ptxas schedules the stage-2
# (time-derivative-only) sweeps 2.4 / 4.5 / 5.3 % faster (x / y / z: 1.357 / 1.362 / 1.360 -> 1.325 / 1.300 /
# 1.288 ms, 8 instead of 32-48 bytes of spills), the full sweeps unchanged, k_recon5 +1 %: TGV 128^3 10.47 ->
# 10.29 ms/step (A/B on one box, levels 0-3 alike, 4 and 8 like the default); results bitwise equal
# Only the 3-D translation unit takes it: the 2-D kernels lose 1-3 % (flux) and 10 % (recon2) with it; within the
# 3-D unit GKS-2nd's recon2 is 15 % slower and its update 4 % faster (+0.7 % per GKS-2nd step)
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
FLAGS_PER_SOURCE = {"stage_d3.cu": ["-Xptxas", "--register-usage-level=3"]}
# experiment knobs (defaults are the tuned values): extra -D flags, alternate output name
EXTRA = os.environ.get("CGKS_NVCC_DEFS", "").split()
BUILD = os.path.join(HERE, "build")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "cgks.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None) -> str:
    sys.path.insert(0, HERE)
    import gen_recon
    gen_recon.emit()
    if not force and not needs_build():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    log = os.path.join(HERE, "build.log")
    procs, objs = [], []
    for s in SOURCES:  # one process per translation unit, in parallel
        obj = os.path.join(BUILD, s + ".o")
        cmd = [NVCC] + FLAGS + FLAGS_PER_SOURCE.get(s, []) + EXTRA + ["-c", os.path.join(CSRC, s), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    text, failed = "", False
    for cmd, p in procs:
        so, se = p.communicate()
        text += " ".join(cmd) + "\n" + so + se
        failed |= p.returncode != 0
    if not failed:
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out or LIB] + objs + ["-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        text += " ".join(cmd) + "\n" + r.stdout + r.stderr
        failed = r.returncode != 0
    with open(log, "w") as f:
        f.write(text)
    if failed:
        sys.stderr.write(text[-8000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stdout.write(text)
    return out or LIB


if __name__ == "__main__":
    o = None
    for a in sys.argv[1:]:
        if a.startswith("--out="):
            o = a.split("=", 1)[1]
    print(build(force=True, verbose="-v" in sys.argv, out=o))
