"""Pins for the NEXT-3 oracle (adjoint-state FWI gradient, oracle_fwi_gradient) -- CPU.

The gradient formula (time-reversed adjoint run + imaging condition, DESIGN.md
§3 Q23-Q26) is checked against things that do not share it:
  G1  directional central finite differences of J computed with oracle.run only
      (second-order convergence in eps, 2D and 3D, damping + several sources);
  G2  pointwise finite differences at a damping-layer point, a source corner,
      a receiver corner and an interior point;
  G3  zero residual -> J = 0 and gradient exactly 0 (fp32 parity mode);
  G4  the fp32 and fp64-canonical modes agree with the fp64 textbook mode;
  G5  affine in the observed data; nt = 1 gives a zero gradient (psi^0 = 0);
  G6  J and the residual equal their definitions from oracle.run traces.
A dropped damping term, a wrong time index (psi^{k+1} instead of psi^k), a sign,
the dt^2 scale or a receiver/source mix-up fails G1/G2.
"""
import numpy as np
import pytest

import oracle
import workloads


def _case(shape, so, nt, seed=3):
    w = workloads.small_case(shape, so, nt, nbl=3, ns=2, nr=5, seed=seed)
    rng = np.random.default_rng(seed + 100)
    m_true = (w.m * (1.0 + 0.05 * rng.standard_normal(w.m.shape))).astype(np.float32)
    _, _, d64 = oracle.run(oracle.FP64EXACT, w.shape, w.extent, so, m_true, w.dt, nt, damp=w.damp,
                           src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    return w, d64.astype(np.float32)


def _J(w, m, dobs, mode=oracle.FP64EXACT):
    _, _, rec = oracle.run(mode, w.shape, w.extent, w.space_order, m, w.dt, w.nt, damp=w.damp,
                           src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    r = rec.astype(np.float64) - dobs.astype(np.float64)
    return 0.5 * float(np.sum(r * r))


def _grad(w, dobs, mode=oracle.FP64EXACT, m=None):
    return oracle.fwi_gradient(mode, w.shape, w.extent, w.space_order, w.m if m is None else m, w.dt, w.nt, dobs,
                               damp=w.damp, src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)


def _fd(w, dobs, dm, eps):
    """central difference along dm, with the perturbation actually representable in fp32 m."""
    mp = (w.m.astype(np.float64) + eps * dm).astype(np.float32)
    mm = (w.m.astype(np.float64) - eps * dm).astype(np.float32)
    return _J(w, mp, dobs) - _J(w, mm, dobs), mp.astype(np.float64) - mm.astype(np.float64)


@pytest.mark.parametrize("shape,so,nt", [((24, 30), 4, 60), ((12, 14, 16), 8, 40)])
def test_g1_directional_fd_second_order(shape, so, nt):
    w, dobs = _case(shape, so, nt)
    g, _, J = _grad(w, dobs)
    assert J > 0
    dm = np.random.default_rng(7).standard_normal(w.m.shape)
    errs = []
    for eps in (1e-3, 1e-4, 1e-5):
        dJ, delta = _fd(w, dobs, dm, eps)
        pred = float(np.sum(g * delta))
        errs.append(abs(dJ - pred) / abs(dJ))
    # O(eps^2) convergence: each decade of eps removes ~2 decades of error
    assert errs[1] < errs[0] / 30 and errs[2] < errs[1] / 30, errs
    assert errs[2] < 1e-5, errs


def test_g2_pointwise_fd():
    w, dobs = _case((20, 26), 4, 50, seed=5)
    g, _, _ = _grad(w, dobs)
    sc, _ = oracle.sparse(w.shape, w.extent, None, w.src_coords)
    rc, _ = oracle.sparse(w.shape, w.extent, None, w.rec_coords)
    pts = {
        "damping layer": np.ravel_multi_index((1, 13), w.shape),
        "source corner": int(sc[0][sc[0] >= 0][0]),
        "receiver corner": int(rc[1][rc[1] >= 0][-1]),
        "interior": np.ravel_multi_index((10, 12), w.shape),
    }
    assert w.damp.ravel()[pts["damping layer"]] > 0
    for name, p in pts.items():
        dm = np.zeros(w.m.size)
        dm[p] = 1.0
        dm = dm.reshape(w.m.shape)
        dJ, delta = _fd(w, dobs, dm, 1e-4)
        pred = g.ravel()[p] * delta.ravel()[p]
        assert abs(dJ - pred) <= 1e-5 * abs(dJ) + 1e-14, (name, dJ, pred)


def test_g3_zero_residual_zero_gradient():
    w, _ = _case((18, 22), 2, 30)
    _, _, rec32 = oracle.run(oracle.FP32CANON, w.shape, w.extent, w.space_order, w.m, w.dt, w.nt, damp=w.damp,
                             src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    g, res, J = _grad(w, rec32, mode=oracle.FP32CANON)
    assert J == 0.0 and not res.any() and not g.any()


@pytest.mark.parametrize("shape,so", [((22, 25), 8), ((10, 12, 14), 4)])
def test_g4_modes_agree(shape, so):
    w, dobs = _case(shape, so, 40)
    g64, r64, J64 = _grad(w, dobs)
    g32, r32, J32 = _grad(w, dobs, mode=oracle.FP32CANON)
    gc, rc, Jc = _grad(w, dobs, mode=oracle.FP64CANON)
    rel = lambda a, b: np.linalg.norm(a.astype(np.float64) - b) / np.linalg.norm(b)
    # fp32-rounded coefficients (b, a, C: 6e-8 each) move the traces by ~1e-5 relative; the residual is
    # a difference of nearly equal traces, so its (and the gradient's) relative change is ~20x larger
    assert rel(rc, r64) < 1e-3 and rel(gc, g64) < 1e-3
    assert rel(g32, gc) < 2e-4      # fp32 arithmetic over 2 x 40 steps, same coefficients
    assert abs(J32 - J64) <= 1e-3 * J64 and abs(Jc - J64) <= 1e-3 * J64
    assert g32.dtype == np.float32 and r32.dtype == np.float32


def test_g5_affine_in_data_and_nt1():
    """g(d) = A (rec - d) is affine in the observed data: the second difference along an exactly
    representable data direction vanishes; nt = 1 gives a zero gradient (only psi^0 = 0 is imaged)."""
    w, dobs = _case((16, 20), 4, 30)
    rng = np.random.default_rng(11)
    q = np.round(dobs.astype(np.float64) * 2.0**20) / 2.0**20           # exact in fp32 (|d| < 16)
    delta = rng.integers(-4096, 4096, size=q.shape) / 2.0**20
    ds = [(q + i * delta).astype(np.float32) for i in range(3)]
    assert all(np.array_equal(d.astype(np.float64), q + i * delta) for i, d in enumerate(ds))
    g0, g1, g2 = (_grad(w, d)[0] for d in ds)
    assert np.linalg.norm(g0 - 2 * g1 + g2) <= 1e-9 * np.linalg.norm(g0 - g1)
    assert np.linalg.norm(g0 - g1) > 0
    w1 = workloads.small_case((16, 20), 4, 1, nbl=3, ns=2, nr=5)
    g, _, _ = oracle.fwi_gradient(oracle.FP64EXACT, w1.shape, w1.extent, 4, w1.m, w1.dt, 1, np.ones((1, 5), np.float32),
                                  damp=w1.damp, src_coords=w1.src_coords, wavelet=w1.wavelet,
                                  rec_coords=w1.rec_coords)
    assert not g.any()


def test_g6_residual_and_misfit_definitions():
    w, dobs = _case((18, 21), 4, 25)
    for mode in (oracle.FP32CANON, oracle.FP64EXACT):
        _, _, rec = oracle.run(mode, w.shape, w.extent, w.space_order, w.m, w.dt, w.nt, damp=w.damp,
                               src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
        _, res, J = _grad(w, dobs, mode=mode)
        want = rec - (dobs if mode == oracle.FP32CANON else dobs.astype(np.float64))
        assert np.array_equal(res, want)
        assert J == pytest.approx(0.5 * float(np.sum(want.astype(np.float64) ** 2)), rel=1e-14)
