"""B200-native (sm_100a, FP64) hot path of CGKS-5th / GKS-2nd (arXiv 2508.19911).

The compute path is libcgks.so (csrc/, C ABI in include/cgks.h); this package only
builds it and marshals arguments.  See DESIGN.md.
"""
from .binding import (CGKS_CGKS5, CGKS_GKS2, CGKS_TIME_DEFAULT, CGKS_TIME_S1O2, CGKS_TIME_S2O4, CgksError, Solver,
                      decompose, decompose_pencil, load, nccl_unique_id, scheme_defaults, step_group)

__all__ = ["Solver", "CgksError", "load", "scheme_defaults", "decompose", "decompose_pencil", "nccl_unique_id", "step_group", "CGKS_CGKS5", "CGKS_GKS2", "CGKS_TIME_DEFAULT",
           "CGKS_TIME_S1O2", "CGKS_TIME_S2O4"]
