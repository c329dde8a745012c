"""paper_1906_10811_b200 -- B200-native acoustic-wave hot path (arXiv 1906.10811).

Explicit leapfrog time stepping of  m u_tt - Lap(u) + eta u_t = q  on 2D/3D
grids: space-order-k star Laplacian, damped update, sparse Ricker injection
and receiver interpolation, all in hand-written sm_100a CUDA kernels behind
the C ABI of include/aw.h (libaw.so).  This package is the thin Python
binding (ctypes marshalling) plus the multi-process team bootstrap.

The binding is loaded lazily so that ``paper_1906_10811_b200.build`` can be
imported (and run) before libaw.so exists; any other attribute access loads
libaw.so and raises ImportError if it has not been built (no CPU fallback).
"""
import importlib as _importlib

_SUBMODULES = ("_binding", "build", "team")


def __getattr__(name):
    if name.startswith("__") or name in _SUBMODULES:
        raise AttributeError(name)
    binding = _importlib.import_module(__name__ + "._binding")
    try:
        return getattr(binding, name)
    except AttributeError:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}") from None
