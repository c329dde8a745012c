"""Pins for the CPU oracle -- run on CPU (-m "not gpu").

Every check compares the oracle against something OTHER than its own formulas:
exact Vandermonde weights, printed paper values, closed-form discrete
solutions, conservation laws, adjointness, reciprocity, brute force with dense
matrices, symmetry/linearity, and restart bit-exactness.  A dropped term, a
wrong sign, a wrong index or a transposed operand in aw_oracle.c fails one.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads
from tests import _indep

HERE = os.path.dirname(os.path.abspath(__file__))
ORDERS = (2, 4, 8, 12, 16)


def _golden_weights():
    out = {}
    with open(os.path.join(HERE, "golden", "fd_weights.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if not line:
                continue
            k, *cs = line.split()
            out[int(k)] = [Fraction(c) for c in cs]
    return out


# ---------------------------------------------------------------- P1 weights
@pytest.mark.parametrize("k", ORDERS)
def test_p1_fd_weights_equal_vandermonde_solve(k):
    got = [Fraction(n, d) for n, d in oracle.fd_weights(k)]
    assert got == _indep.vandermonde_weights(k)
    # fp64 values are the correctly rounded rationals
    f64 = oracle.fd_weights_f64(k)
    assert [float(g) for g in got] == list(f64)


def test_p1_fd_weights_golden():
    gold = _golden_weights()
    for k, cs in gold.items():
        assert [Fraction(n, d) for n, d in oracle.fd_weights(k)] == cs, k


def test_p1_paper_listing_so2():
    """so=2 diffusion kernel: centre -1.0F = -2*nu, neighbour 5.0e-1F = 1*nu (nu=0.5)."""
    vals = {}
    with open(os.path.join(HERE, "golden", "paper_listing_so2.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if line:
                k, v = line.split()
                vals[k] = float(v)
    nu = 0.5
    c = oracle.fd_weights_f64(2)
    assert c[0] * nu == vals["centre_coeff"]
    assert c[1] * nu == vals["neighbour_coeff"]


def test_p1_bad_orders_rejected():
    for k in (0, 1, 3, 18):
        with pytest.raises(ValueError):
            oracle.fd_weights(k)


# ----------------------------------------------- helpers: one-step Laplacian
def oracle_laplacian(mode, u, spacing, k):
    """One oracle step with m=1, dt=1, eta=0 and u_prev = 2u gives u_next = L(u) exactly."""
    shape = u.shape
    extent = [spacing[d] * (shape[d] - 1) for d in range(u.ndim)]
    m = np.ones(shape, np.float32)
    uc, _, _ = oracle.run(mode, shape, extent, k, m, 1.0, 1, u_cur=u, u_prev=2 * u)
    return uc


# ------------------------------------------- P2 polynomial exactness, order k
@pytest.mark.parametrize("k", ORDERS)
@pytest.mark.parametrize("axis", [0, 1])
def test_p2_polynomial_exactness(k, axis):
    R = k // 2
    shape = (2 * R + 9, 2 * R + 7)
    x = np.arange(shape[axis], dtype=np.float64) - (shape[axis] - 1) / 2.0  # h = 1, centred
    core = tuple(slice(R, n - R) for n in shape)
    for p in range(0, k + 2):
        prof = x ** p
        u = np.broadcast_to(prof.reshape([-1 if d == axis else 1 for d in range(2)]), shape).copy()
        exact1 = p * (p - 1) * x ** (p - 2) if p >= 2 else np.zeros_like(x)
        exact = np.broadcast_to(exact1.reshape([-1 if d == axis else 1 for d in range(2)]), shape)
        L = oracle_laplacian(oracle.FP64EXACT, u, (1.0, 1.0), k)
        scale = np.abs(u).max() * 8
        assert np.abs(L[core] - exact[core]).max() <= 1e-13 * scale, (k, p)
    # degree k+2 is NOT reproduced (the order is exactly k)
    p = k + 2
    u = np.broadcast_to((x ** p).reshape([-1 if d == axis else 1 for d in range(2)]), shape).copy()
    exact = np.broadcast_to((p * (p - 1) * x ** (p - 2)).reshape([-1 if d == axis else 1 for d in range(2)]), shape)
    L = oracle_laplacian(oracle.FP64EXACT, u, (1.0, 1.0), k)
    assert np.abs(L[core] - exact[core]).max() > 1e-6 * np.abs(exact[core]).max()


@pytest.mark.parametrize("k", (2, 8, 16))
def test_p2_mixed_3d_polynomial_all_modes(k):
    """x^a y^b z^c with a,b,c <= k+1 on anisotropic spacing, all three modes."""
    R = k // 2
    shape = (2 * R + 5, 2 * R + 4, 2 * R + 6)
    h = (1.0, 0.5, 2.0)
    g = np.meshgrid(*[(np.arange(n) - (n - 1) / 2.0) * h[d] for d, n in enumerate(shape)], indexing="ij")
    a, b, c = min(3, k + 1), 2, min(k + 1, 5)
    u = g[0] ** a * g[1] ** b * g[2] ** c
    exact = (a * (a - 1) * g[0] ** (a - 2) * g[1] ** b * g[2] ** c
             + b * (b - 1) * g[0] ** a * g[1] ** (b - 2) * g[2] ** c
             + c * (c - 1) * g[0] ** a * g[1] ** b * g[2] ** (c - 2))
    core = tuple(slice(R, n - R) for n in shape)
    L = oracle_laplacian(oracle.FP64EXACT, u, h, k)
    assert np.abs(L[core] - exact[core]).max() <= 1e-12 * np.abs(u).max() * 10
    L = oracle_laplacian(oracle.FP64CANON, u, h, k)  # fp32-rounded coefficients
    assert np.abs(L[core] - exact[core]).max() <= 3e-6 * np.abs(u).max() * 10
    L = oracle_laplacian(oracle.FP32CANON, u.astype(np.float32), h, k)
    assert np.abs(L[core] - exact[core]).max() <= 3e-5 * np.abs(u).max() * 10


# ----------------------------------------------------------- P3 symbol order
@pytest.mark.parametrize("k", ORDERS)
def test_p3_symbol_order(k):
    """Order of the oracle's exact weights from the symbol, in 60-digit arithmetic."""
    import mpmath
    mpmath.mp.dps = 60
    w = [mpmath.mpf(n) / d for n, d in oracle.fd_weights(k)]
    kappa = 2 * mpmath.pi / 200

    def err(h):
        lam = (-w[0] - 2 * sum(w[j] * mpmath.cos(j * kappa * h) for j in range(1, len(w)))) / h ** 2
        return abs(lam - kappa ** 2)

    order = float(mpmath.log(err(mpmath.mpf(4)) / err(mpmath.mpf(2)), 2))
    assert abs(order - k) < 0.1, (k, order)


# ------------------------------------------- P4 fully discrete standing wave
def _standing_wave_run(mode, shape, k, h, courant, nt, kappas, phis, v=2.0):
    """u^0 = S, u^{-1} = S cos(theta), cos(theta) = 1 - v^2 dt^2 lambda_h / 2 => u^n = S cos(n theta)."""
    ndim = len(shape)
    spacing = [h] * ndim
    m32 = np.float32(1.0 / (v * v))
    v2 = 1.0 / float(m32)
    dt = courant * _indep.critical_dt(k, spacing, math.sqrt(v2))
    g = np.meshgrid(*[np.arange(n) * h for n in shape], indexing="ij")
    S = np.ones(shape)
    lam = 0.0
    for d in range(ndim):
        S = S * np.sin(kappas[d] * g[d] + phis[d])
        lam += _indep.symbol(k, kappas[d], h)
    cos_t = 1.0 - v2 * dt * dt * lam / 2.0
    theta = math.acos(cos_t)
    extent = [h * (n - 1) for n in shape]
    m = np.full(shape, m32, np.float32)
    uc, _, _ = oracle.run(mode, shape, extent, k, m, dt, nt, u_cur=S, u_prev=S * cos_t)
    return uc, S * math.cos(nt * theta), S


@pytest.mark.parametrize("shape,k", [((61, 57), 4), ((61, 61), 8), ((33, 31, 35), 4), ((45, 43, 41), 2)])
def test_p4_standing_wave_core_exact(shape, k):
    R = k // 2
    nt = 6
    got, want, S = _standing_wave_run(oracle.FP64EXACT, shape, k, 10.0, 0.8, nt,
                                      [0.021 * (d + 1) for d in range(len(shape))],
                                      [0.3 + d for d in range(len(shape))])
    margin = nt * R + 1
    core = tuple(slice(margin, n - margin) for n in shape)
    assert np.abs(got[core] - want[core]).max() <= 1e-13
    # and near the edge the zero-ghost boundary does differ (the check has teeth)
    assert np.abs(got - want).max() > 1e-6


def test_p4_dirichlet_mode_exact_everywhere_k2():
    """k = 2: zero ghosts == Dirichlet at the ghost nodes, so sin(pi q (i+1)/(n+1)) is an
    exact eigenvector of the discrete Laplacian on the whole grid."""
    shape = (37, 29)
    h = 10.0
    q = (3, 2)
    nt = 40
    ndim = 2
    v = 1.7
    m32 = np.float32(1.0 / (v * v))
    v2 = 1.0 / float(m32)
    dt = 0.9 * _indep.critical_dt(2, [h, h], math.sqrt(v2))
    S = np.ones(shape)
    lam = 0.0
    for d in range(ndim):
        i = np.arange(shape[d])
        kap = math.pi * q[d] / ((shape[d] + 1) * h)
        prof = np.sin(kap * (i + 1) * h)
        S = S * prof.reshape([-1 if e == d else 1 for e in range(ndim)])
        lam += _indep.symbol(2, kap, h)
    cos_t = 1.0 - v2 * dt * dt * lam / 2.0
    m = np.full(shape, m32, np.float32)
    uc, _, _ = oracle.run(oracle.FP64EXACT, shape, [h * (n - 1) for n in shape], 2, m, dt, nt,
                          u_cur=S, u_prev=S * cos_t)
    want = S * math.cos(nt * math.acos(cos_t))
    assert np.abs(uc - want).max() <= 1e-12
    # fp32 canonical mode stays within fp32 noise of the closed form
    uc32, _, _ = oracle.run(oracle.FP32CANON, shape, [h * (n - 1) for n in shape], 2, m, dt, nt,
                            u_cur=S.astype(np.float32), u_prev=(S * cos_t).astype(np.float32))
    assert np.abs(uc32 - want).max() <= 2e-5


# ---------------------------------------------- P5 convergence order (k = 2)
def test_p5_convergence_order_continuous():
    """Dirichlet eigenmode vs continuous S(x) cos(v |kappa| t) at fixed Courant: order 2."""
    errs = []
    v = 1.5
    m32 = np.float32(1.0 / (v * v))
    v2 = 1.0 / float(m32)
    Lx = 1000.0
    T = 300.0
    for n in (21, 41, 81):
        h = Lx / (n + 1)
        shape = (n, n)
        kap = math.pi / Lx * 2
        dt0 = 0.5 * _indep.critical_dt(2, [h, h], math.sqrt(v2))
        nt = int(math.ceil(T / dt0))
        dt = T / nt
        g = np.meshgrid(*[(np.arange(nn) + 1) * h for nn in shape], indexing="ij")
        S = np.sin(kap * g[0]) * np.sin(kap * g[1])
        w = math.sqrt(v2) * kap * math.sqrt(2)
        m = np.full(shape, m32, np.float32)
        uc, _, _ = oracle.run(oracle.FP64EXACT, shape, [h * (nn - 1) for nn in shape], 2, m, dt, nt,
                              u_cur=S, u_prev=S * math.cos(w * dt))
        errs.append(np.abs(uc - S * math.cos(w * T)).max())
    o1 = math.log(errs[0] / errs[1], 2)
    o2 = math.log(errs[1] / errs[2], 2)
    assert 1.8 < o1 < 2.3 and 1.8 < o2 < 2.3, (errs, o1, o2)


# ------------------------------------------------------ P7 energy and CFL
def _energy(m, dt, u_next, u, spacing, k):
    lap = _indep.apply_laplacian(u, spacing, k)
    return float(np.sum(m * (u_next - u) ** 2) / dt ** 2 - np.sum(u_next * lap))


@pytest.mark.parametrize("k", (2, 8))
def test_p7_energy_conserved_and_damped(k):
    rng = np.random.default_rng(7)
    shape = (30, 26)
    h = 10.0
    spacing = [h, h]
    extent = [h * (n - 1) for n in shape]
    vel = 1.5 + rng.uniform(0, 1.0, shape)
    m = (1.0 / vel ** 2).astype(np.float32)
    dt = 0.9 * _indep.critical_dt(k, spacing, vel.max())
    u0 = rng.standard_normal(shape)
    u1 = u0 + 0.01 * rng.standard_normal(shape)
    E = []
    uc, up = u1, u0
    for _ in range(20):
        uc2, up2, _ = oracle.run(oracle.FP64EXACT, shape, extent, k, m, dt, 10, u_cur=uc, u_prev=up)
        # E^{n+1/2} from (u^{n}, u^{n+1}) = (up2, uc2)
        E.append(_energy(m.astype(np.float64), dt, uc2, up2, spacing, k))
        uc, up = uc2, up2
    E = np.array(E)
    assert np.abs(E - E[0]).max() <= 1e-11 * abs(E[0])
    # damping: energy is non-increasing
    damp = workloads.damping_profile(shape, 6)
    uc, up = u1, u0
    E = []
    for _ in range(20):
        uc2, up2, _ = oracle.run(oracle.FP64EXACT, shape, extent, k, m, dt, 10, u_cur=uc, u_prev=up, damp=damp)
        E.append(_energy(m.astype(np.float64), dt, uc2, up2, spacing, k))
        uc, up = uc2, up2
    E = np.array(E)
    assert np.all(np.diff(E) <= 1e-12 * abs(E[0]))
    assert E[-1] < 0.9 * E[0]


@pytest.mark.parametrize("k", (2, 8, 16))
def test_p7_cfl_bound(k):
    rng = np.random.default_rng(3)
    shape = (32, 32)
    h = 10.0
    v = 2.0
    m = np.full(shape, np.float32(1 / v ** 2), np.float32)
    vtrue = math.sqrt(1.0 / float(m[0, 0]))
    dtc = _indep.critical_dt(k, [h, h], vtrue)
    u0 = rng.standard_normal(shape)
    extent = [h * 31, h * 31]
    stable, _, _ = oracle.run(oracle.FP64EXACT, shape, extent, k, m, 0.99 * dtc, 2000, u_cur=u0, u_prev=u0)
    assert np.abs(stable).max() < 1e3
    unstable, _, _ = oracle.run(oracle.FP64EXACT, shape, extent, k, m, 1.01 * dtc, 600, u_cur=u0, u_prev=u0)
    assert not np.isfinite(unstable).all() or np.abs(unstable).max() > 1e6


def test_workload_dt_below_cfl():
    """The configs' dt literals are 0.9 dt_c of their v_max."""
    for k, nd, vmax, dt in ((2, 2, 1.5, 4.2426), (4, 3, 2.5, 1.8000), (8, 3, 4.5, 0.9057),
                            (12, 3, 4.5, 0.8684), (16, 3, 4.5, 0.8474)):
        dtc = _indep.critical_dt(k, [10.0] * nd, vmax)
        assert dt <= 0.9001 * dtc and dt >= 0.899 * dtc, (k, dt, dtc)


# -------------------------------------------- P8 injection is the adjoint
@pytest.mark.parametrize("shape", [(13, 11), (7, 9, 8)])
def test_p8_adjoint_and_linear_exactness(shape):
    rng = np.random.default_rng(8)
    ndim = len(shape)
    h = 10.0
    extent = [h * (n - 1) for n in shape]
    npts = 6
    coords = np.stack([rng.uniform(0, e, npts) for e in extent], axis=1)
    coords[0] = extent  # the upper corner node (skipped corners)
    coords[1] = [h * 3] * ndim  # exactly on a node
    m = np.ones(shape, np.float32)
    q = rng.standard_normal(npts).astype(np.float32)
    # I_s^T q: one step from rest with m = 1, dt = 1 -> u^1 = sum_s w * q_s
    inj, _, _ = oracle.run(oracle.FP64EXACT, shape, extent, 2, m, 1.0, 1,
                           src_coords=coords, wavelet=q.reshape(1, -1))
    vfield = rng.standard_normal(shape)
    _, _, rec = oracle.run(oracle.FP64EXACT, shape, extent, 2, m, 1.0, 1, rec_coords=coords,
                           u_cur=vfield, u_prev=vfield)
    lhs = float(np.sum(inj * vfield))
    rhs = float(np.sum(q.astype(np.float64) * rec[0]))
    assert abs(lhs - rhs) <= 1e-13 * max(1.0, abs(lhs))
    # equals the textbook interpolation matrix
    P = _indep.interp_matrix(shape, [h] * ndim, [0.0] * ndim, coords)
    assert np.abs(rec[0] - P @ vfield.ravel()).max() <= 1e-13
    # a linear field is interpolated exactly
    g = np.meshgrid(*[np.arange(n) * h for n in shape], indexing="ij")
    beta = rng.standard_normal(ndim)
    lin = 0.7 + sum(beta[d] * g[d] for d in range(ndim))
    _, _, rec = oracle.run(oracle.FP64EXACT, shape, extent, 2, m, 1.0, 1, rec_coords=coords,
                           u_cur=lin, u_prev=lin)
    want = 0.7 + coords @ beta
    assert np.abs(rec[0] - want).max() <= 1e-11


def test_p8_sparse_rejects_outside_points():
    with pytest.raises(ValueError):
        oracle.sparse((10, 10), (90.0, 90.0), None, np.array([[-1e-9, 5.0]]))
    with pytest.raises(ValueError):
        oracle.sparse((10, 10), (90.0, 90.0), None, np.array([[5.0, 90.0000001]]))
    c, w = oracle.sparse((10, 10), (90.0, 90.0), None, np.array([[90.0, 0.0]]))
    # bit d of the corner id <-> +1 on axis d; (10, *) is outside and skipped
    assert list(c[0]) == [90, -1, 91, -1] and list(w[0]) == [1.0, 0.0, 0.0, 0.0]


# ------------------------------------------------------- P9 reciprocity
def test_p9_reciprocity_damped():
    rng = np.random.default_rng(9)
    shape = (40, 48)
    k = 8
    h = 10.0
    extent = [h * (n - 1) for n in shape]
    vel = 2.0 + rng.uniform(0, 1.5, shape)
    m = (1.0 / vel ** 2).astype(np.float32)
    damp = workloads.damping_profile(shape, 8)
    dt = 0.8 * _indep.critical_dt(k, [h, h], vel.max())
    A = np.array([[35.3, 41.7]])    # inside the damping layer
    B = np.array([[250.1, 300.9]])
    nt = 300
    wav = workloads.ricker(nt, dt, 0.02)
    _, _, ab = oracle.run(oracle.FP64EXACT, shape, extent, k, m, dt, nt, damp=damp,
                          src_coords=A, wavelet=wav, rec_coords=B)
    _, _, ba = oracle.run(oracle.FP64EXACT, shape, extent, k, m, dt, nt, damp=damp,
                          src_coords=B, wavelet=wav, rec_coords=A)
    assert np.abs(ab - ba).max() <= 1e-13 * np.abs(ab).max()
    assert np.abs(ab).max() > 0


# ------------------------------------------------------ P10 brute force
@pytest.mark.parametrize("shape,k", [((8, 7), 2), ((8, 7), 4), ((9, 10), 8), ((5, 4, 4), 2), ((6, 5, 7), 4)])
def test_p10_brute_force_dense(shape, k):
    rng = np.random.default_rng(10)
    ndim = len(shape)
    h = [10.0, 7.0, 12.0][:ndim]
    extent = [h[d] * (shape[d] - 1) for d in range(ndim)]
    vel = 1.5 + rng.uniform(0, 2.0, shape)
    m = (1.0 / vel ** 2).astype(np.float32)
    damp = rng.uniform(0, 0.05, shape).astype(np.float32)
    dt = 0.8 * _indep.critical_dt(k, h, vel.max())
    ns, nr, nt = 2, 3, 25
    src = np.stack([rng.uniform(0, e, ns) for e in extent], axis=1)
    rec = np.stack([rng.uniform(0, e, nr) for e in extent], axis=1)
    wav = rng.standard_normal((nt, ns)).astype(np.float32)
    u0 = rng.standard_normal(shape)
    um = rng.standard_normal(shape)
    got, _, grec = oracle.run(oracle.FP64EXACT, shape, extent, k, m, dt, nt, damp=damp,
                              src_coords=src, wavelet=wav, rec_coords=rec, u_cur=u0, u_prev=um)
    # dense brute force: (M + D) u+ = dt^2 (Lap u + P^T q) + M (2u - u-) + D u-
    Lap = _indep.laplacian_matrix(shape, h, k)
    M = m.astype(np.float64).ravel()
    D = damp.astype(np.float64).ravel() * dt / 2
    Ps = _indep.interp_matrix(shape, h, [0.0] * ndim, src)
    Pr = _indep.interp_matrix(shape, h, [0.0] * ndim, rec)
    u, uprev = u0.ravel().copy(), um.ravel().copy()
    recs = []
    for n in range(nt):
        recs.append(Pr @ u)
        rhs = dt * dt * (Lap @ u + Ps.T @ wav[n].astype(np.float64)) + M * (2 * u - uprev) + D * uprev
        u, uprev = rhs / (M + D), u
    scale = max(1.0, np.abs(u).max())
    assert np.abs(got.ravel() - u).max() <= 1e-12 * scale
    assert np.abs(grec - np.array(recs)).max() <= 1e-12 * scale
    # fp32 canonical mode within fp32 noise of the brute force
    got32, _, grec32 = oracle.run(oracle.FP32CANON, shape, extent, k, m, dt, nt, damp=damp,
                                  src_coords=src, wavelet=wav, rec_coords=rec,
                                  u_cur=u0.astype(np.float32), u_prev=um.astype(np.float32))
    assert np.linalg.norm(got32.ravel() - u) <= 1e-5 * np.linalg.norm(u)


# --------------------------------------------------- P11 symmetry, linearity
def test_p11_mirror_symmetry_and_linearity_fp32():
    n = 41
    shape = (n, n)
    k = 8
    h = 10.0
    extent = [h * (n - 1)] * 2
    m = workloads.constant_m(shape, 2.0)
    damp = workloads.damping_profile(shape, 6)
    dt = 0.8 * _indep.critical_dt(k, [h, h], 2.0)
    nt = 60
    wav = workloads.ricker(nt, dt, 0.02)
    src = np.array([[h * (n // 2), h * (n // 2)]])
    u, up, _ = oracle.run(oracle.FP32CANON, shape, extent, k, m, dt, nt, damp=damp, src_coords=src, wavelet=wav)
    assert np.abs(u).max() > 0
    assert np.array_equal(u, u[::-1, :]) and np.array_equal(u, u[:, ::-1])
    u2, _, _ = oracle.run(oracle.FP32CANON, shape, extent, k, m, dt, nt, damp=damp, src_coords=src, wavelet=2 * wav)
    assert np.array_equal(u2, 2 * u)
    u0, _, _ = oracle.run(oracle.FP32CANON, shape, extent, k, m, dt, nt, damp=damp, src_coords=src, wavelet=0 * wav)
    assert not np.any(u0)


# ------------------------------------------------- P6 impulse response fp32
@pytest.mark.parametrize("k", ORDERS)
def test_p6_impulse_response_fp32(k):
    """u^0 = delta_p, u^-1 = 0, eta = 0, one fp32 step (SPEC.md:599 pattern):
    u_p = fma(b, C0, 2), u_{p +- j e_d} = fl32(b C[d][j]), 0 elsewhere; the weights come
    from the exact Vandermonde rationals and h_d, not from the oracle."""
    R = k // 2
    shape = (2 * R + 3, 2 * R + 5, 2 * R + 4)
    h = (10.0, 7.5, 12.5)
    extent = [h[d] * (shape[d] - 1) for d in range(3)]
    v = 2.5
    m = np.full(shape, np.float32(1 / v ** 2), np.float32)
    dt = 1.3
    p = (R + 1, R + 2, R + 1)
    u0 = np.zeros(shape, np.float32)
    u0[p] = 1.0
    u1, _, _ = oracle.run(oracle.FP32CANON, shape, extent, k, m, dt, 1, u_cur=u0)
    cw = _indep.vandermonde_weights(k)
    b = np.float32(dt * dt / float(m[0, 0, 0]))
    C0 = np.float32(sum(float(cw[0]) / (hh * hh) for hh in h))
    want = np.zeros(shape, np.float32)
    want[p] = np.float32(np.float64(b) * np.float64(C0) + 2.0)  # fma is exact-then-round
    for d in range(3):
        Cd = [np.float32(float(cw[j]) / (h[d] * h[d])) for j in range(R + 1)]
        for j in range(1, R + 1):
            for s in (-1, 1):
                q = list(p)
                q[d] += s * j
                if 0 <= q[d] < shape[d]:
                    want[tuple(q)] = np.float32(np.float64(b) * np.float64(Cd[j]))
    assert np.array_equal(u1, want)


# ------------------------------------------------- P12 restart, rotation
def test_p12_restart_bit_exact():
    w = workloads.small_case((23, 19, 21), 4, 30, nbl=4, ns=2, nr=5)
    args = dict(damp=w.damp, src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    full, fullp, frec = oracle.run(oracle.FP32CANON, w.shape, w.extent, 4, w.m, w.dt, 30, **args)
    a, ap, arec = oracle.run(oracle.FP32CANON, w.shape, w.extent, 4, w.m, w.dt, 13, **args)
    b, bp, brec = oracle.run(oracle.FP32CANON, w.shape, w.extent, 4, w.m, w.dt, 17, n0=13, u_cur=a, u_prev=ap, **args)
    assert np.array_equal(b, full) and np.array_equal(bp, fullp)
    assert np.array_equal(np.concatenate([arec, brec]), frec)


def test_p12_three_slot_rotation_matches_full_history():
    """PAPER.md:443 rotation vs a full-history run built from single steps."""
    w = workloads.small_case((17, 15), 8, 12, nbl=3, ns=1, nr=3)
    args = dict(damp=w.damp, src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    full, _, frec = oracle.run(oracle.FP32CANON, w.shape, w.extent, 8, w.m, w.dt, 12, **args)
    hist = [np.zeros(w.shape, np.float32), np.zeros(w.shape, np.float32)]  # levels -1, 0
    recs = []
    for n in range(12):
        un, _, r = oracle.run(oracle.FP32CANON, w.shape, w.extent, 8, w.m, w.dt, 1, n0=n,
                              u_cur=hist[-1], u_prev=hist[-2], **args)
        hist.append(un)
        recs.append(r[0])
    assert np.array_equal(hist[-1], full)
    assert np.array_equal(np.array(recs), frec)


# ---------------------------------------------------- P12 virtual slabs
@pytest.mark.parametrize("shape,so,world", [((23, 30), 4, 2), ((23, 30), 4, 5), ((17, 12, 14), 8, 2),
                                             ((26, 9, 11), 4, 3), ((40, 10, 11), 16, 5)])
def test_p12_virtual_slabs_equal_single_domain(shape, so, world):
    """decomposing axis 0 into slabs with an R-plane halo exchange, owner-
    computes receivers (base corner) and owner-injection changes no arithmetic: bit-exact with one
    domain, including sources and receivers on slab-boundary planes and the +1 corner in a halo."""
    w = workloads.small_case(shape, so, 14, nbl=3, ns=3, nr=6, seed=world + so)
    n0 = shape[0]
    base, rem = divmod(n0, world)
    bounds = [r * base + min(r, rem) for r in range(1, world)]
    h = workloads.H
    # put sources and receivers right at / between the slab boundary planes
    extra_src = [[h * (z - 0.5)] + [h * (n - 1) * 0.37 for n in shape[1:]] for z in bounds[:2]]
    extra_rec = [[h * (z - 1 + 0.25)] + [h * (n - 1) * 0.61 for n in shape[1:]] for z in bounds] + \
                [[h * z] + [h * (n - 1) * 0.5 for n in shape[1:]] for z in bounds]
    src = np.concatenate([w.src_coords, np.array(extra_src).reshape(-1, len(shape))])
    rec = np.concatenate([w.rec_coords, np.array(extra_rec).reshape(-1, len(shape))])
    wav = workloads.ricker(w.nt, w.dt, 0.02, ns=src.shape[0])
    rng = np.random.default_rng(1)
    u0 = rng.standard_normal(shape).astype(np.float32) * 1e-3
    u1 = rng.standard_normal(shape).astype(np.float32) * 1e-3
    kw = dict(damp=w.damp, src_coords=src, wavelet=wav, rec_coords=rec, u_cur=u0, u_prev=u1)
    ou, oup, orec = oracle.run(oracle.FP32CANON, w.shape, w.extent, so, w.m, w.dt, w.nt, **kw)
    su, sup, srec = oracle.run_slabs(world, w.shape, w.extent, so, w.m, w.dt, w.nt, **kw)
    assert np.array_equal(su, ou) and np.array_equal(sup, oup)
    assert np.array_equal(srec, orec)


def test_p12_virtual_slabs_detect_a_missing_halo():
    """The check above can fail: a slab thinner than R (no full halo from one neighbour) is rejected,
    and a one-plane-narrower halo (exchange of R-1 planes, emulated with so-2 weights on one side)
    would differ -- here: slabs vs one domain at different space orders must differ."""
    w = workloads.small_case((20, 16), 8, 6, nbl=2, ns=1, nr=2)
    with pytest.raises(ValueError):
        oracle.run_slabs(6, w.shape, w.extent, 8, w.m, w.dt, w.nt)  # 20/6 = 3 planes < R = 4
    a, _, _ = oracle.run_slabs(2, w.shape, w.extent, 8, w.m, w.dt, w.nt, src_coords=w.src_coords,
                               wavelet=w.wavelet)
    b, _, _ = oracle.run(oracle.FP32CANON, w.shape, w.extent, 6, w.m, w.dt, w.nt, src_coords=w.src_coords,
                         wavelet=w.wavelet)
    assert not np.array_equal(a, b)
