"""GPU parity of NEXT-3, the adjoint-state FWI gradient (aw_fwi_gradient), vs the fp32 oracle.

The oracle (oracle_fwi_gradient, pinned by finite differences in
tests/test_oracle_fwi_pins.py) keeps the whole forward history; the CUDA path
replays it from checkpoints (segments of K steps) and images in reversed time.
Recomputation is deterministic, so the gradient and the residual are
value-identical for every K (asserted, with the relL2 <= 1e-5 contract);
J is a fp64 reduction in another order (rel 1e-12).
"""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def aw():
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    return aw


def _case(shape, so, nt, seed=3, nbl=3, ns=2, nr=6):
    w = workloads.small_case(shape, so, nt, nbl=nbl, ns=ns, nr=nr, seed=seed)
    rng = np.random.default_rng(seed + 100)
    m_true = (w.m * (1.0 + 0.05 * rng.standard_normal(w.m.shape))).astype(np.float32)
    _, _, d = oracle.run(oracle.FP32CANON, w.shape, w.extent, so, m_true, w.dt, nt, damp=w.damp,
                         src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    return w, d


def _want(w, dobs):
    return oracle.fwi_gradient(oracle.FP32CANON, w.shape, w.extent, w.space_order, w.m, w.dt, w.nt, dobs,
                               damp=w.damp, src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)


def _grid(aw, w, kernel=None, ckpt=None):
    g = aw.Grid(w.shape, w.extent, w.space_order, w.origin)
    if kernel is not None:
        g.set_option(aw.AW_OPT_KERNEL, kernel)
    if ckpt is not None:
        g.set_option(aw.AW_OPT_CHECKPOINT_STEPS, ckpt)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.nt)
    return g


def _assert_identical(got, want, what):
    got = np.asarray(got)
    den = max(np.linalg.norm(want.astype(np.float64)), 1e-300)
    err = np.linalg.norm(got.astype(np.float64) - want) / den
    assert err <= TOL, f"{what}: relL2 {err:.3e}"
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{what}: {len(bad)} values differ (relL2 {err:.2e}), first at {bad[0].tolist()}"


CASES = [
    ((37, 45), 4, 40, None),           # 2D: v1 kernel + sparse kernel
    ((20, 34, 70), 8, 30, None),       # 3D: streaming kernel, ragged tiles
    ((20, 34, 70), 8, 30, 1),          # 3D: reference-grade v1 kernel
    ((18, 40, 33), 16, 24, None),      # 3D so=16 (R=8 streaming configuration)
]


@pytest.mark.parametrize("shape,so,nt,kernel", CASES)
@pytest.mark.parametrize("ckpt", [0, 7, 1])
def test_fwi_gradient_value_identical(aw, shape, so, nt, kernel, ckpt):
    w, dobs = _case(shape, so, nt)
    g_want, r_want, J_want = _want(w, dobs)
    with _grid(aw, w, kernel=kernel, ckpt=ckpt) as g:
        grad, res, J = g.fwi_gradient(nt, w.dt, dobs)
        st = g.stats()
        K = st["fwi_checkpoint"]
        assert K == (nt if ckpt == 0 else ckpt)
        # forward nt + replay (every segment but the last, which is a full K) + adjoint nt-1 steps
        assert st["fwi_steps"] == nt + (nt - min(K, nt)) + (nt - 1)
        _assert_identical(res, r_want, "residual")
        _assert_identical(grad, g_want, "gradient")
        assert J == pytest.approx(J_want, rel=1e-12)
        # the forward traces stay readable; the wavefield is not a forward state
        _, _, rec = oracle.run(oracle.FP32CANON, w.shape, w.extent, so, w.m, w.dt, nt, damp=w.damp,
                               src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
        _assert_identical(g.read_receivers(), rec, "forward traces")
        with pytest.raises(aw.AwError) as e:
            g.run(1, w.dt)
        assert e.value.status == aw.AW_ESTATE
        with pytest.raises(aw.AwError):
            g.read_wavefield(0)


def test_fwi_repeat_reset_and_forward(aw):
    """Second call (pool reuse), a call with another dt, then aw_reset and an ordinary forward run."""
    w, dobs = _case((16, 30, 40), 4, 20)
    with _grid(aw, w, ckpt=6) as g:
        a = g.fwi_gradient(w.nt, w.dt, dobs)
        b = g.fwi_gradient(w.nt, w.dt, dobs)
        assert np.array_equal(a[0], b[0]) and a[2] == b[2]
        dt2 = 0.9 * w.dt
        w2 = workloads.Workload(w.name, w.shape, w.space_order, w.nt, dt2, w.m, w.damp, w.src_coords,
                                w.wavelet, w.rec_coords)
        g2, _, _ = g.fwi_gradient(w.nt, dt2, dobs)
        want2, _, _ = _want(w2, dobs)
        _assert_identical(g2, want2, "gradient at another dt")
        g.reset()
        g.run(w.nt, w.dt)
        u, _, _ = oracle.run(oracle.FP32CANON, w.shape, w.extent, 4, w.m, w.dt, w.nt, damp=w.damp,
                             src_coords=w.src_coords, wavelet=w.wavelet)
        _assert_identical(g.read_wavefield(0), u, "forward after gradient + reset")


def test_fwi_device_pointers(aw):
    import torch
    w, dobs = _case((14, 26, 36), 8, 18)
    want, rwant, _ = _want(w, dobs)
    with _grid(aw, w, ckpt=5) as g:
        d = torch.from_numpy(dobs).cuda()
        grad = torch.zeros(w.shape, dtype=torch.float32, device="cuda")
        res = torch.zeros((w.nt, w.rec_coords.shape[0]), dtype=torch.float32, device="cuda")
        g.fwi_gradient(w.nt, w.dt, d, grad=grad, residual=res)
        torch.cuda.synchronize()
        _assert_identical(grad.cpu().numpy(), want, "gradient (device out)")
        _assert_identical(res.cpu().numpy(), rwant, "residual (device out)")


def test_fwi_zero_residual(aw):
    w, _ = _case((16, 22, 36), 4, 16)
    _, _, rec = oracle.run(oracle.FP32CANON, w.shape, w.extent, 4, w.m, w.dt, w.nt, damp=w.damp,
                           src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    with _grid(aw, w) as g:
        grad, res, J = g.fwi_gradient(w.nt, w.dt, rec)
        assert J == 0.0 and not res.any() and not grad.any()


def test_fwi_errors(aw):
    w, dobs = _case((16, 22), 2, 10)
    g = aw.Grid(w.shape, w.extent, 2)
    with pytest.raises(aw.AwError) as e:
        g.fwi_gradient(w.nt, w.dt, dobs)
    assert e.value.status == aw.AW_ESTATE  # no model
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    with pytest.raises(aw.AwError) as e:
        g.fwi_gradient(w.nt, w.dt, dobs)
    assert e.value.status == aw.AW_EINVAL  # no receivers
    g.add_receivers(w.rec_coords, w.nt)
    for nt, dt in ((w.nt + 1, w.dt), (0, w.dt), (w.nt, -1.0)):
        with pytest.raises(aw.AwError) as e:
            g.fwi_gradient(max(nt, 1) if nt else 0, dt, np.zeros((max(nt, 1), 6), np.float32))
        assert e.value.status == aw.AW_EINVAL
    g.close()
    t = aw.Grid(w.shape, w.extent, 2, rank=0, world=2)
    t.set_model(w.m, w.damp)
    t.add_receivers(w.rec_coords, w.nt)
    with pytest.raises(aw.AwError) as e:
        t.fwi_gradient(w.nt, w.dt, dobs)
    assert e.value.status == aw.AW_EUNSUPPORTED
    t.close()


def test_fwi_c2_size(aw):
    """Config C2's grid and model (128^3, so 4, two layers, damping nbl 16) for 120 steps with K = 16."""
    nt = 120
    w = workloads.c2(nt)
    rng = np.random.default_rng(5)
    m_true = (w.m * (1.0 + 0.02 * rng.standard_normal(w.m.shape))).astype(np.float32)
    _, _, dobs = oracle.run(oracle.FP32CANON, w.shape, w.extent, 4, m_true, w.dt, nt, damp=w.damp,
                            src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    want, rwant, J_want = oracle.fwi_gradient(oracle.FP32CANON, w.shape, w.extent, 4, w.m, w.dt, nt, dobs,
                                              damp=w.damp, src_coords=w.src_coords, wavelet=w.wavelet,
                                              rec_coords=w.rec_coords)
    g = aw.Grid(w.shape, w.extent, 4, w.origin)
    g.set_option(aw.AW_OPT_CHECKPOINT_STEPS, 16)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, nt)
    grad, res, J = g.fwi_gradient(nt, w.dt, dobs)
    g.close()
    _assert_identical(res, rwant, "C2 residual")
    _assert_identical(grad, want, "C2 gradient")
    assert J == pytest.approx(J_want, rel=1e-12)
