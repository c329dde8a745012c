"""paper_1906_10811_b200 -- B200-native acoustic-wave hot path (arXiv 1906.10811).

Explicit leapfrog time stepping of  m u_tt - Lap(u) + eta u_t = q  on 2D/3D
grids: space-order-k star Laplacian, damped update, sparse Ricker injection
and receiver interpolation, all in hand-written sm_100a CUDA kernels behind
the C ABI of include/aw.h (libaw.so).  This package is the thin Python
binding (ctypes marshalling) plus the multi-process team bootstrap.
"""
from ._binding import *  # noqa: F401,F403
from ._binding import Grid, AwError, critical_dt, team_connect_local, team_run, EXPORTED, LIB_PATH  # noqa: F401

__all__ = ["Grid", "AwError", "critical_dt", "team_connect_local", "team_run", "EXPORTED", "LIB_PATH"]
