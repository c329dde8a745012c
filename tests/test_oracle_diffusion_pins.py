"""Pins for the oracle's NEXT-2 operator: forward-Euler diffusion u_t = nu (u_xx + u_yy)
(PAPER.md:732-744), checked against the SPEC.md:599 worked example, the exact
discrete eigenmode decay, dense brute force, polynomial exactness and the
explicit stability limit."""
import math
import os

import numpy as np
import pytest

import oracle
from tests import _indep

HERE = os.path.dirname(os.path.abspath(__file__))


def test_d1_spec_worked_example_3x3():
    want = np.zeros((3, 3))
    with open(os.path.join(HERE, "golden", "diffusion_3x3.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if line:
                r, c, v = line.split()
                want[int(r), int(c)] = float(v)
    u = np.zeros((3, 3))
    u[1, 1] = 1.0
    got = oracle.diffusion_run(oracle.FP64EXACT, (3, 3), (2.0, 2.0), 2, 0.5, 0.1, 1, u)
    assert np.abs(got - want).max() <= 1e-15
    # fp32 canonical: centre fma(D, C0, 1), neighbours fl32(D*C) with D = fl32(nu dt), C from the exact weights
    got32 = oracle.diffusion_run(oracle.FP32CANON, (3, 3), (2.0, 2.0), 2, 0.5, 0.1, 1, u.astype(np.float32))
    c = _indep.vandermonde_weights(2)
    D = np.float32(0.5 * 0.1)
    C0 = np.float32(2 * float(c[0]))
    C1 = np.float32(float(c[1]))
    assert got32[1, 1] == np.float32(np.float64(D) * np.float64(C0) + 1.0)
    for rc in ((0, 1), (1, 0), (1, 2), (2, 1)):
        assert got32[rc] == np.float32(np.float64(D) * np.float64(C1))
    assert got32[0, 0] == 0 and got32[2, 2] == 0


def test_d2_dirichlet_eigenmode_decay_k2():
    """k=2 with zero ghosts == Dirichlet: S = prod sin(pi q (i+1)/(n+1)) is an exact eigenvector,
    u^n = S (1 - nu dt lambda_h)^n on the whole grid."""
    shape = (33, 29)
    extent = (1.0, 1.0)
    h = [e / (n - 1) for e, n in zip(extent, shape)]
    nu = 0.5
    lam = 0.0
    S = np.ones(shape)
    q = (2, 3)
    for d in range(2):
        i = np.arange(shape[d])
        kap = math.pi * q[d] / ((shape[d] + 1) * h[d])
        S = S * np.sin(kap * (i + 1) * h[d]).reshape([-1 if e == d else 1 for e in range(2)])
        lam += _indep.symbol(2, kap, h[d])
    dt = 0.9 * min(h) ** 2 / (4 * nu)
    nt = 50
    got = oracle.diffusion_run(oracle.FP64EXACT, shape, extent, 2, nu, dt, nt, S)
    want = S * (1 - nu * dt * lam) ** nt
    assert np.abs(got - want).max() <= 1e-13


@pytest.mark.parametrize("shape,k", [((7, 9), 2), ((9, 8), 4), ((12, 11), 8), ((14, 13), 12), ((5, 4, 6), 4)])
def test_d3_brute_force_dense(shape, k):
    rng = np.random.default_rng(13)
    ndim = len(shape)
    extent = [1.0, 0.7, 1.3][:ndim]
    h = [extent[d] / (shape[d] - 1) for d in range(ndim)]
    nu = 0.5
    S = sum(abs(float(c)) for c in _indep.vandermonde_weights(k)) * 2 - abs(float(_indep.vandermonde_weights(k)[0]))
    dt = 0.8 * 2 / (nu * sum(S / hh ** 2 for hh in h))
    u0 = rng.standard_normal(shape)
    nt = 15
    got = oracle.diffusion_run(oracle.FP64EXACT, shape, extent, k, nu, dt, nt, u0)
    Lap = _indep.laplacian_matrix(shape, h, k)
    u = u0.ravel().copy()
    for _ in range(nt):
        u = u + nu * dt * (Lap @ u)
    assert np.abs(got.ravel() - u).max() <= 1e-12 * max(1.0, np.abs(u).max())
    got32 = oracle.diffusion_run(oracle.FP32CANON, shape, extent, k, nu, dt, nt, u0.astype(np.float32))
    assert np.linalg.norm(got32.ravel() - u) <= 1e-5 * np.linalg.norm(u)


@pytest.mark.parametrize("k", (2, 8, 12))
def test_d4_polynomial_step_exact(k):
    """One step on u = x^a y^b (a, b <= k+1): u + nu dt (u_xx + u_yy) exactly in the core."""
    R = k // 2
    shape = (2 * R + 7, 2 * R + 8)
    x = [np.arange(n) - (n - 1) / 2.0 for n in shape]
    X, Y = np.meshgrid(x[0], x[1], indexing="ij")
    a, b = min(k + 1, 5), 2
    u = X ** a * Y ** b
    lap = a * (a - 1) * X ** (a - 2) * Y ** b + b * (b - 1) * X ** a * Y ** (b - 2)
    nu, dt = 0.5, 0.01
    got = oracle.diffusion_run(oracle.FP64EXACT, shape, [n - 1.0 for n in shape], k, nu, dt, 1, u)
    core = (slice(R, -R), slice(R, -R))
    assert np.abs(got[core] - (u + nu * dt * lap)[core]).max() <= 1e-12 * np.abs(u).max()


def test_d5_stability_limit_and_max_principle():
    rng = np.random.default_rng(5)
    shape = (40, 40)
    extent = (1.0, 1.0)
    h = 1.0 / 39
    nu = 0.5
    lim = h * h / (4 * nu)  # SPEC.md:640, so=2 in 2-D
    u0 = np.abs(rng.standard_normal(shape))
    u = u0
    mx = [np.abs(u).max()]
    for _ in range(10):
        u = oracle.diffusion_run(oracle.FP64EXACT, shape, extent, 2, nu, 0.999 * lim, 20, u)
        mx.append(np.abs(u).max())
    assert all(b <= a * (1 + 1e-14) for a, b in zip(mx, mx[1:]))
    for k in (2, 8):
        S = 2 * sum(abs(float(c)) for c in _indep.vandermonde_weights(k)[1:]) + abs(float(_indep.vandermonde_weights(k)[0]))
        dtc = 2 / (nu * 2 * S / h ** 2)
        stable = oracle.diffusion_run(oracle.FP64EXACT, shape, extent, k, nu, 0.99 * dtc, 400, rng.standard_normal(shape))
        assert np.abs(stable).max() < 10
        unstable = oracle.diffusion_run(oracle.FP64EXACT, shape, extent, k, nu, 1.05 * dtc, 400, rng.standard_normal(shape))
        assert np.abs(unstable).max() > 1e3
