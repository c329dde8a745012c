"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no FD weights, no update,
no interpolation).  It only manufactures the *inputs* of the problem -- the
velocity model m = 1/v^2, the damping profile eta, the Ricker wavelet, and the
source / receiver coordinates -- following the recipe of SURVEY.md §8(d)
(readings Q13-Q15, all [proposed]/[external] since the paper never ran the
acoustic operator).  The same recipe feeds the parity tests,
smoke() and bench.py, so both sides see identical arrays.

Units (Q15): velocity km/s, spacing m, time ms, f0 kHz; h = 10 m everywhere.
dt values are the survey's 0.9*dt_c literals; the tests
check them against the CFL bound computed from the oracle's weights.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

H = 10.0  # grid spacing in metres on every axis


@dataclasses.dataclass
class Workload:
    name: str
    shape: tuple
    space_order: int
    nt: int
    dt: float
    m: np.ndarray                 # fp32 slowness^2, shape `shape`
    damp: Optional[np.ndarray]    # fp32 eta >= 0 or None
    src_coords: np.ndarray        # [ns][ndim] fp64
    wavelet: np.ndarray           # [nt][ns] fp32
    rec_coords: np.ndarray        # [nr][ndim] fp64
    extent: tuple = None
    origin: tuple = None
    f0: float = 0.0
    nbl: int = 0

    def __post_init__(self):
        if self.extent is None:
            self.extent = tuple(H * (n - 1) for n in self.shape)
        if self.origin is None:
            self.origin = tuple(0.0 for _ in self.shape)

    @property
    def ndim(self):
        return len(self.shape)

    @property
    def npoints(self):
        return int(np.prod(self.shape))


# --------------------------------------------------------------------------
# Ricker wavelet (Q13): r(t) = (1 - 2 pi^2 f0^2 (t-t0)^2) exp(-pi^2 f0^2 (t-t0)^2),
# t0 = 1/f0, sampled at t_n = n dt in fp64 and rounded once to fp32.
# --------------------------------------------------------------------------
def ricker(nt: int, dt: float, f0: float, ns: int = 1, t0: Optional[float] = None) -> np.ndarray:
    t0 = 1.0 / f0 if t0 is None else t0
    t = np.arange(nt, dtype=np.float64) * dt
    a = (math.pi * f0 * (t - t0)) ** 2
    r = (1.0 - 2.0 * a) * np.exp(-a)
    return np.repeat(r.astype(np.float32)[:, None], ns, axis=1).copy()


# --------------------------------------------------------------------------
# Damping profile (Q14): in layers of nbl cells on each face,
# eta = sum_d (1.5 ln(1000)/nbl) (p - sin(2 pi p)/(2 pi)) / h_d,
# p = (nbl - distance)/nbl in (0, 1].  Computed in fp64, rounded once.
# --------------------------------------------------------------------------
def damping_profile(shape, nbl: int, spacing=None, z0: int = 0, nz: Optional[int] = None) -> np.ndarray:
    """eta for the planes [z0, z0+nz) of axis 0 (whole grid by default)."""
    ndim = len(shape)
    spacing = spacing or [H] * ndim
    nz = shape[0] - z0 if nz is None else nz
    coef = 1.5 * math.log(1000.0) / nbl
    eta = np.zeros((nz,) + tuple(shape[1:]), np.float64)
    for d in range(ndim):
        n = shape[d]
        idx = np.arange(z0, z0 + nz) if d == 0 else np.arange(n)
        dist = np.minimum(idx, n - 1 - idx).astype(np.float64)
        p = (nbl - dist) / nbl
        prof = np.where(dist < nbl, coef * (p - np.sin(2 * math.pi * p) / (2 * math.pi)) / spacing[d], 0.0)
        bshape = [1] * ndim
        bshape[d] = -1
        eta = eta + prof.reshape(bshape)
    return eta.astype(np.float32)


# --------------------------------------------------------------------------
# Random smooth model: rng = default_rng(1906), 16 modes;
# kappa_i = 2 pi j_i / (512 h), j_i uniform in {-4..4}^ndim \ {0},
# phi_i ~ U[0, 2pi), a_i ~ U[0.5, 1]/16;  s(x) = sum_i a_i cos(kappa_i . x + phi_i),
# v = 3 + 1.5 tanh(2 s),  m = fl32(1/v^2) in fp64.  Element-wise, so any slab
# can be generated alone and equals the global generation.
# --------------------------------------------------------------------------
def random_smooth_modes(ndim: int, seed: int = 1906, nmodes: int = 16):
    rng = np.random.default_rng(seed)
    modes = []
    while len(modes) < nmodes:
        j = rng.integers(-4, 5, size=ndim)
        if not np.any(j):
            continue
        phi = rng.uniform(0.0, 2 * math.pi)
        amp = rng.uniform(0.5, 1.0) / nmodes
        modes.append((2 * math.pi * j / (512 * H), phi, amp))
    return modes


def random_smooth_m(shape, z0: int = 0, nz: Optional[int] = None, device: str = "cpu", seed: int = 1906):
    """m = 1/v^2 (fp32) for planes [z0, z0+nz).  Uses torch (fp64) so the bench can
    build 1024^3 models on the GPU; tests build them on the CPU."""
    import torch

    ndim = len(shape)
    nz = shape[0] - z0 if nz is None else nz
    modes = random_smooth_modes(ndim, seed)
    dev = torch.device(device)
    axes = [torch.arange(z0, z0 + nz, dtype=torch.float64, device=dev) * H]
    axes += [torch.arange(n, dtype=torch.float64, device=dev) * H for n in shape[1:]]
    out = torch.empty((nz,) + tuple(shape[1:]), dtype=torch.float32, device=dev)
    # plane-chunked evaluation to bound memory (cos of a sum = Re of a product of exponentials)
    chunk = max(1, (1 << 24) // max(1, int(np.prod(shape[1:]))))
    for c0 in range(0, nz, chunk):
        c1 = min(nz, c0 + chunk)
        s = None
        for kap, phi, amp in modes:
            arg = None
            for d in range(ndim):
                ax = axes[d][c0:c1] if d == 0 else axes[d]
                v = kap[d] * ax
                bshape = [1] * ndim
                bshape[d] = -1
                v = v.reshape(bshape)
                arg = v if arg is None else arg + v
            term = amp * torch.cos(arg + phi)
            s = term if s is None else s + term
        v = 3.0 + 1.5 * torch.tanh(2.0 * s)
        out[c0:c1] = (1.0 / (v * v)).to(torch.float32)
    return out if device != "cpu" else out.numpy()


def two_layer_m(shape, v_top=1.5, v_bot=2.5, split=None):
    split = shape[0] // 2 if split is None else split
    v = np.full(shape, v_top, np.float64)
    v[split:] = v_bot
    return (1.0 / (v * v)).astype(np.float32)


def constant_m(shape, v=1.5):
    return np.full(shape, np.float32(1.0 / (v * v)), np.float32)


# --------------------------------------------------------------------------
# The BASELINE.json configs C1..C5
# --------------------------------------------------------------------------
def c1():
    shape, nt, dt, f0 = (101, 101), 100, 4.2426, 0.010
    src = np.array([[500.0, 500.0]])
    rec = np.array([[203.7, 10.0 * r] for r in range(101)])
    return Workload("C1", shape, 2, nt, dt, constant_m(shape, 1.5), None, src,
                    ricker(nt, dt, f0), rec, f0=f0)


def c2(nt: int = 500):
    shape, dt, f0, nbl = (128, 128, 128), 1.8000, 0.015, 16
    src = np.array([[200.3, 635.7, 641.1]])
    rec = np.array([[400.5, 640.0, 10.0 * r] for r in range(128)])
    return Workload("C2", shape, 4, nt, dt, two_layer_m(shape), damping_profile(shape, nbl), src,
                    ricker(nt, dt, f0), rec, f0=f0, nbl=nbl)


def c3(nt: int = 1000, device: str = "cpu", with_arrays: bool = True):
    shape, dt, f0, nbl = (512, 512, 512), 0.9057, 0.015, 32
    src = np.array([[2555.3, 2555.7, 2556.1]])
    rec = np.array([[400.5, 2555.0, 10.0 * r] for r in range(512)])
    m = random_smooth_m(shape, device=device) if with_arrays else None
    damp = damping_profile(shape, nbl) if with_arrays else None
    return Workload("C3", shape, 8, nt, dt, m, damp, src, ricker(nt, dt, f0), rec, f0=f0, nbl=nbl)


def c4_sparse(n=1024):
    src = np.array([[5115.3, 5115.7, 5116.1]])
    rec = [[400.5, 5115.0, 10.0 * r] for r in range(n)] + [[10.0 * r, 5115.3, 5114.7] for r in range(n)]
    return src, np.array(rec)


def c4(nt: int = 1000, device: str = "cpu", with_arrays: bool = True):
    shape, dt, f0, nbl = (1024, 1024, 1024), 0.8684, 0.015, 32
    src, rec = c4_sparse()
    m = random_smooth_m(shape, device=device) if with_arrays else None
    damp = damping_profile(shape, nbl) if with_arrays else None
    return Workload("C4", shape, 12, nt, dt, m, damp, src, ricker(nt, dt, f0), rec, f0=f0, nbl=nbl)


def c5_sparse(N: int):
    n0 = 512 * N
    src = np.array([[10.0 * (512 * i + 255) + 3.3, 2555.3, 2555.7] for i in range(N)])
    rec = [[400.5, 2555.0, 10.0 * r] for r in range(512)] + [[10.0 * r, 2555.3, 2554.7] for r in range(n0)]
    return src, np.array(rec)


def c5(N: int = 1, nt: int = 1000, device: str = "cpu", with_arrays: bool = True):
    shape, dt, f0, nbl = (512 * N, 512, 512), 0.8474, 0.015, 32
    src, rec = c5_sparse(N)
    m = random_smooth_m(shape, device=device) if with_arrays else None
    damp = damping_profile(shape, nbl) if with_arrays else None
    return Workload("C5", shape, 16, nt, dt, m, damp, src, ricker(nt, dt, f0, ns=N), rec, f0=f0, nbl=nbl)


# --------------------------------------------------------------------------
# Small parity cases: random smooth models, off-node sparse points, ragged
# shapes (not multiples of any tile), damping on every face.
# --------------------------------------------------------------------------
def small_case(shape, space_order, nt, *, seed=10811, nbl=None, ns=2, nr=7, v=None, f0=0.02,
               courant=0.8):
    rng = np.random.default_rng(seed)
    ndim = len(shape)
    if v is None:
        # smooth random velocity in (1.5, 4.5)
        grids = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij")
        s = sum(0.25 * np.cos(2 * math.pi * g / max(8.0, n / 1.7) + rng.uniform(0, 6.28)) for g, n in zip(grids, shape))
        vel = 3.0 + 1.5 * np.tanh(s)
    else:
        vel = np.full(shape, float(v))
    m = (1.0 / (vel * vel)).astype(np.float32)
    damp = damping_profile(shape, nbl) if nbl else None
    # dt: courant * 2 / (vmax sqrt(ndim * S / h^2)) with S <= 8 (bound on sum|c| for k<=16)
    vmax = float(vel.max())
    dt = courant * 2.0 * H / (vmax * math.sqrt(ndim * 7.5))
    ext = [H * (n - 1) for n in shape]
    src = np.stack([rng.uniform(0.2 * e, 0.8 * e, size=ns) for e in ext], axis=1)
    rec = np.stack([rng.uniform(0.0, e, size=nr) for e in ext], axis=1)
    wav = ricker(nt, dt, f0, ns=ns) * rng.uniform(0.5, 2.0, size=ns).astype(np.float32)
    return Workload(f"small{shape}so{space_order}", tuple(shape), space_order, nt, dt, m, damp, src,
                    wav.astype(np.float32), rec, f0=f0, nbl=nbl or 0)
