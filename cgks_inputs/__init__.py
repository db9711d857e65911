"""Seeded synthetic inputs (initial conditions) shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic: it only builds initial cell
averages Q and exact cell-averaged gradients grad Q of analytic or seeded random
fields (R26 of DESIGN.md), in the user-facing layout
``Q[5][nz][ny][nx]`` and ``G[3][5][nz][ny][nx]`` (x fastest).
"""
from .cases import (Case, tgv, tgv_supersonic, vortex, vortex_exact, random_smooth, uniform, double_sod,
                    shock_vortex, hit, CASES, make_case, line_derivatives, line_points,
                    stretched_nodes, jet_inflow, gl_average)

__all__ = ["Case", "tgv", "tgv_supersonic", "vortex", "vortex_exact", "random_smooth", "uniform", "double_sod", "shock_vortex",
           "hit", "CASES", "make_case", "line_derivatives", "line_points",
           "stretched_nodes", "jet_inflow", "gl_average"]
