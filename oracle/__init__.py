"""CPU oracle for the acoustic-wave hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_1906_10811_b200`` never imports it and shares no code
with it.  The arithmetic lives in ``aw_oracle.c`` (plain C,
``-ffp-contract=off``); this module is ctypes marshalling only.

Modes:
  FP32CANON  the parity target (exact fp32 op sequence)
  FP64CANON  same sequence in fp64 with the same fp32 coefficients
  FP64EXACT  textbook fp64 formula with fp64 coefficients
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

FP32CANON, FP64CANON, FP64EXACT = 0, 1, 2
MAXR = 8

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "aw_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile aw_oracle.c -> liboracle.so (gcc, OpenMP, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
               "-fno-fast-math", "-Wall", "-o", tmp, _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i64p = ctypes.POINTER(ctypes.c_int64)
            L.oracle_fd_weights.argtypes = [ctypes.c_int, i64p, i64p]
            L.oracle_fd_weights_f64.argtypes = [ctypes.c_int, P]
            L.oracle_axis_coeffs.argtypes = [ctypes.c_int, P, P, ctypes.c_int, P, P, P, P]
            L.oracle_sparse.argtypes = [ctypes.c_int, P, P, P, ctypes.c_int, P, P, P]
            L.oracle_run.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, ctypes.c_int, P, P,
                                     ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, P, P, ctypes.c_int, P, P, P, P, ctypes.c_int]
            L.oracle_point_coeffs.argtypes = [ctypes.c_int64, P, P, ctypes.c_double, P, P]
            L.oracle_point_coeffs.restype = None
            L.oracle_source_scales.argtypes = [ctypes.c_int, P, P, P, P, P, ctypes.c_double,
                                               ctypes.c_int, P, P, P]
            _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check(st, what):
    if st != 0:
        raise ValueError(f"oracle {what} failed with status {st}")


def fd_weights(space_order: int):
    """Exact reduced rationals (num, den) for c_0..c_{k/2}."""
    num = (ctypes.c_int64 * (MAXR + 1))()
    den = (ctypes.c_int64 * (MAXR + 1))()
    _check(lib().oracle_fd_weights(space_order, num, den), "fd_weights")
    R = space_order // 2
    return [(num[j], den[j]) for j in range(R + 1)]


def fd_weights_f64(space_order: int) -> np.ndarray:
    c = np.zeros(MAXR + 1)
    _check(lib().oracle_fd_weights_f64(space_order, _p(c)), "fd_weights_f64")
    return c[: space_order // 2 + 1]


def axis_coeffs(shape, extent, space_order):
    """Returns (C [ndim][MAXR+1] fp32, C0 fp32, C64, C064)."""
    ndim = len(shape)
    sh = np.asarray(shape, dtype=np.int64)
    ex = np.asarray(extent, dtype=np.float64)
    C = np.zeros((ndim, MAXR + 1), np.float32)
    C64 = np.zeros((ndim, MAXR + 1), np.float64)
    C0 = np.zeros(1, np.float32)
    C064 = np.zeros(1, np.float64)
    _check(lib().oracle_axis_coeffs(ndim, _p(sh), _p(ex), space_order, _p(C), _p(C0), _p(C64), _p(C064)),
           "axis_coeffs")
    return C, C0[0], C64, C064[0]


def sparse(shape, extent, origin, coords):
    """(corner int64 [n][2^ndim] (-1 = skipped), w64 [n][2^ndim])."""
    ndim = len(shape)
    sh = np.asarray(shape, dtype=np.int64)
    ex = np.asarray(extent, dtype=np.float64)
    org = None if origin is None else np.asarray(origin, dtype=np.float64)
    co = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, ndim)
    n = co.shape[0]
    corner = np.zeros((n, 1 << ndim), np.int64)
    w = np.zeros((n, 1 << ndim), np.float64)
    _check(lib().oracle_sparse(ndim, _p(sh), _p(ex), _p(org), n, _p(co), _p(corner), _p(w)), "sparse")
    return corner, w


def point_coeffs(m, damp, dt):
    m = np.ascontiguousarray(m, np.float32).ravel()
    d = None if damp is None else np.ascontiguousarray(damp, np.float32).ravel()
    b = np.zeros_like(m)
    a = np.zeros_like(m)
    lib().oracle_point_coeffs(m.size, _p(m), _p(d), dt, _p(b), _p(a))
    return b, a


def source_scales(shape, extent, origin, m, damp, dt, coords):
    ndim = len(shape)
    sh = np.asarray(shape, dtype=np.int64)
    ex = np.asarray(extent, dtype=np.float64)
    org = None if origin is None else np.asarray(origin, dtype=np.float64)
    co = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, ndim)
    m = np.ascontiguousarray(m, np.float32)
    d = None if damp is None else np.ascontiguousarray(damp, np.float32)
    n = co.shape[0]
    corner = np.zeros((n, 1 << ndim), np.int64)
    s = np.zeros((n, 1 << ndim), np.float32)
    _check(lib().oracle_source_scales(ndim, _p(sh), _p(ex), _p(org), _p(m), _p(d), dt, n, _p(co),
                                      _p(corner), _p(s)), "source_scales")
    return corner, s


def run(mode, shape, extent, space_order, m, dt, nt, *, damp=None, origin=None,
        src_coords=None, wavelet=None, rec_coords=None, u_cur=None, u_prev=None, n0=0,
        nthreads=0):
    """Advance nt steps.  Returns (u_cur, u_prev, rec[nt][nr]) in fp32 (mode 0) or fp64.

    u_cur / u_prev are the levels n0 and n0-1 (zeros if None); the returned
    ones are levels n0+nt and n0+nt-1.  wavelet is [rows >= n0+nt][ns] fp32.
    """
    ndim = len(shape)
    shape = tuple(int(s) for s in shape)
    dtype = np.float32 if mode == FP32CANON else np.float64
    sh = np.asarray(shape, dtype=np.int64)
    ex = np.asarray(extent, dtype=np.float64)
    org = None if origin is None else np.asarray(origin, dtype=np.float64)
    m = np.ascontiguousarray(m, np.float32).reshape(shape)
    d = None if damp is None else np.ascontiguousarray(damp, np.float32).reshape(shape)
    uc = np.zeros(shape, dtype) if u_cur is None else np.array(u_cur, dtype=dtype, copy=True).reshape(shape)
    up = np.zeros(shape, dtype) if u_prev is None else np.array(u_prev, dtype=dtype, copy=True).reshape(shape)
    if src_coords is None:
        ns, sc, wv = 0, None, None
    else:
        sc = np.ascontiguousarray(src_coords, np.float64).reshape(-1, ndim)
        ns = sc.shape[0]
        wv = np.ascontiguousarray(wavelet, np.float32).reshape(-1, ns)
        if wv.shape[0] < n0 + nt:
            raise ValueError("wavelet shorter than n0+nt")
    if rec_coords is None:
        nr, rc = 0, None
    else:
        rc = np.ascontiguousarray(rec_coords, np.float64).reshape(-1, ndim)
        nr = rc.shape[0]
    rec = np.zeros((nt, max(nr, 0)), dtype)
    _check(lib().oracle_run(mode, ndim, _p(sh), _p(ex), _p(org), space_order, _p(m), _p(d), float(dt),
                            int(n0), int(nt), ns, _p(sc), _p(wv), nr, _p(rc), _p(rec) if nr else None,
                            _p(uc), _p(up), int(nthreads)), "run")
    return uc, up, rec


def fwi_gradient(mode, shape, extent, space_order, m, dt, nt, d_obs, *, damp=None, origin=None,
                 src_coords=None, wavelet=None, rec_coords=None, nthreads=0):
    """NEXT-3: adjoint-state gradient of J = 1/2 sum (rec - d_obs)^2 w.r.t. m (see aw_oracle.c).

    Returns (grad [shape], residual [nt][nr], J); fp32 arrays for mode 0, else fp64.
    """
    L = lib()
    if not hasattr(L, "_fwi_sig"):
        P = ctypes.c_void_p
        L.oracle_fwi_gradient.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, ctypes.c_int, P, P, ctypes.c_double,
                                          ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int, P, P, P, P, P,
                                          ctypes.c_int]
        L._fwi_sig = True
    ndim = len(shape)
    shape = tuple(int(s) for s in shape)
    dtype = np.float32 if mode == FP32CANON else np.float64
    sh = np.asarray(shape, dtype=np.int64)
    ex = np.asarray(extent, dtype=np.float64)
    org = None if origin is None else np.asarray(origin, dtype=np.float64)
    m = np.ascontiguousarray(m, np.float32).reshape(shape)
    d = None if damp is None else np.ascontiguousarray(damp, np.float32).reshape(shape)
    if src_coords is None:
        ns, sc, wv = 0, None, None
    else:
        sc = np.ascontiguousarray(src_coords, np.float64).reshape(-1, ndim)
        ns = sc.shape[0]
        wv = np.ascontiguousarray(wavelet, np.float32).reshape(-1, ns)
        if wv.shape[0] < nt:
            raise ValueError("wavelet shorter than nt")
    rc = np.ascontiguousarray(rec_coords, np.float64).reshape(-1, ndim)
    nr = rc.shape[0]
    dobs = np.ascontiguousarray(d_obs, np.float32).reshape(nt, nr)
    grad = np.zeros(shape, dtype)
    res = np.zeros((nt, nr), dtype)
    J = ctypes.c_double(0.0)
    _check(L.oracle_fwi_gradient(mode, ndim, _p(sh), _p(ex), _p(org), space_order, _p(m), _p(d), float(dt),
                                 int(nt), ns, _p(sc), _p(wv), nr, _p(rc), _p(dobs), _p(grad), _p(res),
                                 ctypes.byref(J), int(nthreads)), "fwi_gradient")
    return grad, res, J.value


def run_slabs(world, shape, extent, space_order, m, dt, nt, *, damp=None, origin=None, src_coords=None,
              wavelet=None, rec_coords=None, u_cur=None, u_prev=None):
    """FP32CANON run decomposed into `world` virtual slabs of axis 0 with explicit halo exchange
    (SURVEY §8(c) P12, §8(e)); returns (u_cur, u_prev, rec) gathered like run()."""
    L = lib()
    if not hasattr(L, "_slab_sig"):
        P = ctypes.c_void_p
        L.oracle_run_slabs.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, ctypes.c_int, P, P, ctypes.c_double,
                                       ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int, P, P, P, P]
        L._slab_sig = True
    ndim = len(shape)
    shape = tuple(int(s) for s in shape)
    sh = np.asarray(shape, dtype=np.int64)
    ex = np.asarray(extent, dtype=np.float64)
    org = None if origin is None else np.asarray(origin, dtype=np.float64)
    m = np.ascontiguousarray(m, np.float32).reshape(shape)
    d = None if damp is None else np.ascontiguousarray(damp, np.float32).reshape(shape)
    uc = np.zeros(shape, np.float32) if u_cur is None else np.array(u_cur, dtype=np.float32, copy=True).reshape(shape)
    up = np.zeros(shape, np.float32) if u_prev is None else np.array(u_prev, dtype=np.float32, copy=True).reshape(shape)
    if src_coords is None:
        ns, sc, wv = 0, None, None
    else:
        sc = np.ascontiguousarray(src_coords, np.float64).reshape(-1, ndim)
        ns = sc.shape[0]
        wv = np.ascontiguousarray(wavelet, np.float32).reshape(-1, ns)
    if rec_coords is None:
        nr, rc = 0, None
    else:
        rc = np.ascontiguousarray(rec_coords, np.float64).reshape(-1, ndim)
        nr = rc.shape[0]
    rec = np.zeros((nt, max(nr, 0)), np.float32)
    _check(L.oracle_run_slabs(int(world), ndim, _p(sh), _p(ex), _p(org), space_order, _p(m), _p(d), float(dt),
                              int(nt), ns, _p(sc), _p(wv), nr, _p(rc), _p(rec) if nr else None, _p(uc), _p(up)),
           "run_slabs")
    return uc, up, rec


def diffusion_run(mode, shape, extent, space_order, nu, dt, nt, u0, nthreads=0):
    """NEXT-2: forward-Euler diffusion; returns u^nt (fp32 for mode 0, else fp64)."""
    L = lib()
    if not hasattr(L, "_diff_sig"):
        L.oracle_diffusion_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_void_p,
                                           ctypes.c_int]
        L._diff_sig = True
    shape = tuple(int(s) for s in shape)
    dtype = np.float32 if mode == FP32CANON else np.float64
    sh = np.asarray(shape, dtype=np.int64)
    ex = np.asarray(extent, dtype=np.float64)
    u = np.array(u0, dtype=dtype, copy=True).reshape(shape)
    _check(L.oracle_diffusion_run(mode, len(shape), _p(sh), _p(ex), space_order, float(nu), float(dt), int(nt),
                                  _p(u), int(nthreads)), "diffusion_run")
    return u
