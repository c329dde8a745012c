"""Independent test-side mathematics used to PIN the oracle.

Nothing here is copied from oracle/aw_oracle.c: the FD weights come from a
Vandermonde (moment-condition) solve in exact rationals (the method SPEC.md:130-138
names), the discrete Laplacian is a dense matrix built from those weights, and
multilinear interpolation weights are written as the textbook tensor product.
"""
from __future__ import annotations

import itertools
import math
from fractions import Fraction

import numpy as np


def vandermonde_weights(space_order: int):
    """Second-derivative weights c_0..c_m on offsets -m..m (symmetric), exact.

    Moment conditions: sum_{j=-m}^{m} c_|j| j^(2q) = 2 * [q == 1], q = 0..m
    (d^2/dx^2 of x^(2q) at 0 is 2 for q = 1 and 0 otherwise; odd moments vanish
    by symmetry).  Solved by Gaussian elimination over Fractions.
    """
    m = space_order // 2
    n = m + 1
    A = [[Fraction(0)] * n for _ in range(n)]
    rhs = [Fraction(2 if q == 1 else 0) for q in range(n)]
    for q in range(n):
        A[q][0] = Fraction(1 if q == 0 else 0)
        for j in range(1, n):
            A[q][j] = Fraction(2 * j ** (2 * q))
    # Gauss-Jordan
    for col in range(n):
        piv = next(r for r in range(col, n) if A[r][col] != 0)
        A[col], A[piv] = A[piv], A[col]
        rhs[col], rhs[piv] = rhs[piv], rhs[col]
        for r in range(n):
            if r != col and A[r][col] != 0:
                f = A[r][col] / A[col][col]
                A[r] = [a - f * b for a, b in zip(A[r], A[col])]
                rhs[r] -= f * rhs[col]
    return [rhs[i] / A[i][i] for i in range(n)]


def weights_f64(space_order):
    return np.array([float(c) for c in vandermonde_weights(space_order)])


def laplacian_1d_matrix(n: int, h: float, space_order: int) -> np.ndarray:
    """Dense 1-D second-difference matrix with zero ghosts outside [0, n)."""
    c = weights_f64(space_order)
    m = space_order // 2
    D = np.zeros((n, n))
    for i in range(n):
        for j in range(-m, m + 1):
            if 0 <= i + j < n:
                D[i, i + j] += c[abs(j)] / (h * h)
    return D


def laplacian_matrix(shape, spacing, space_order) -> np.ndarray:
    """Dense N-D Laplacian = sum_d I x .. x D_d x .. x I (row-major, axis 0 slowest)."""
    mats = [np.eye(n) for n in shape]
    N = int(np.prod(shape))
    L = np.zeros((N, N))
    for d, n in enumerate(shape):
        ops = list(mats)
        ops[d] = laplacian_1d_matrix(n, spacing[d], space_order)
        K = ops[0]
        for o in ops[1:]:
            K = np.kron(K, o)
        L += K
    return L


def apply_laplacian(u: np.ndarray, spacing, space_order) -> np.ndarray:
    """Matrix-free version (zero-padded shifts) for larger fields."""
    c = weights_f64(space_order)
    m = space_order // 2
    out = np.zeros_like(u, dtype=np.float64)
    pad = np.pad(u.astype(np.float64), m)
    core = tuple(slice(m, m + n) for n in u.shape)
    for d in range(u.ndim):
        for j in range(-m, m + 1):
            sl = list(core)
            sl[d] = slice(m + j, m + j + u.shape[d])
            out += c[abs(j)] / (spacing[d] ** 2) * pad[tuple(sl)]
    return out


def interp_matrix(shape, spacing, origin, coords) -> np.ndarray:
    """Dense multilinear interpolation matrix [npts][N] (textbook tensor product)."""
    ndim = len(shape)
    N = int(np.prod(shape))
    P = np.zeros((len(coords), N))
    for s, x in enumerate(coords):
        base, frac = [], []
        for d in range(ndim):
            p = (x[d] - origin[d]) / spacing[d]
            i = min(int(math.floor(p)), shape[d] - 1)
            base.append(i)
            frac.append(p - i)
        for corner in itertools.product((0, 1), repeat=ndim):
            idx = [base[d] + corner[d] for d in range(ndim)]
            if any(idx[d] >= shape[d] for d in range(ndim)):
                continue
            w = 1.0
            for d in range(ndim):
                w *= frac[d] if corner[d] else 1.0 - frac[d]
            P[s, np.ravel_multi_index(idx, shape)] += w
    return P


def critical_dt(space_order, spacing, vmax):
    """Leapfrog stability limit 2 / (v sqrt(sum_d sum_j |c_j| / h_d^2)) (Nyquist eigenvalue)."""
    c = vandermonde_weights(space_order)
    S = float(abs(c[0]) + 2 * sum(abs(x) for x in c[1:]))
    return 2.0 / (vmax * math.sqrt(sum(S / (h * h) for h in spacing)))


def symbol(space_order, kappa, h):
    """lambda_h(kappa) = (-c0 - 2 sum_j c_j cos(j kappa h)) / h^2 (1-D)."""
    c = weights_f64(space_order)
    return (-c[0] - 2 * sum(c[j] * math.cos(j * kappa * h) for j in range(1, len(c)))) / (h * h)
