"""GPU: NEXT-4 multi-shot forward runs and the summed FWI gradient of several shots.

On one rank the library sums the per-shot gradients in shot order (fp32 adds, AW_OPT_FWI_ACCUMULATE),
so the result is value-identical to the fp32 sum, in the same order, of the oracle's per-shot
gradients; the misfit is the sum of the per-shot misfits."""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aw():
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    return aw


def _shots(w, nshots, seed=21):
    rng = np.random.default_rng(seed)
    ext = w.extent
    out = []
    for s in range(nshots):
        src = np.array([[rng.uniform(0.2, 0.8) * e for e in ext]])
        wav = workloads.ricker(w.nt, w.dt, 0.02) * np.float32(rng.uniform(0.5, 2.0))
        out.append((src, wav.astype(np.float32)))
    return out


@pytest.mark.parametrize("shape,so", [((24, 30, 66), 8), ((40, 52), 4)])
def test_multishot_gradient_sum(aw, shape, so):
    from paper_1906_10811_b200 import shots as S
    w = workloads.small_case(shape, so, 24, nbl=3, ns=1, nr=7, seed=4)
    rng = np.random.default_rng(9)
    m_true = (w.m * (1.0 + 0.05 * rng.standard_normal(w.m.shape))).astype(np.float32)
    shot_list, want_sum, J_sum = [], None, 0.0
    for src, wav in _shots(w, 3):
        _, _, d = oracle.run(oracle.FP32CANON, w.shape, w.extent, so, m_true, w.dt, w.nt, damp=w.damp,
                             src_coords=src, wavelet=wav, rec_coords=w.rec_coords)
        gk, _, Jk = oracle.fwi_gradient(oracle.FP32CANON, w.shape, w.extent, so, w.m, w.dt, w.nt, d, damp=w.damp,
                                        src_coords=src, wavelet=wav, rec_coords=w.rec_coords)
        want_sum = gk if want_sum is None else (want_sum + gk).astype(np.float32)  # fp32, shot order
        J_sum += Jk
        shot_list.append(S.Shot(src, wav, d))
    g = aw.Grid(w.shape, w.extent, so, w.origin)
    g.set_option(aw.AW_OPT_CHECKPOINT_STEPS, 5)
    g.set_model(w.m, w.damp)
    g.add_receivers(w.rec_coords, w.nt)
    grad, J = S.fwi_gradient(g, shot_list, S.assign(3, 1, 0), w.nt, w.dt)
    assert np.array_equal(grad, want_sum), np.abs(grad - want_sum).max()
    assert J == pytest.approx(J_sum, rel=1e-12)
    # the accumulator is disarmed afterwards: a plain call returns one shot's gradient
    g.add_sources(shot_list[0].src_coords, shot_list[0].wavelet)
    one, _, _ = g.fwi_gradient(w.nt, w.dt, shot_list[0].d_obs)
    g0, _, _ = oracle.fwi_gradient(oracle.FP32CANON, w.shape, w.extent, so, w.m, w.dt, w.nt, shot_list[0].d_obs,
                                   damp=w.damp, src_coords=shot_list[0].src_coords, wavelet=shot_list[0].wavelet,
                                   rec_coords=w.rec_coords)
    assert np.array_equal(one, g0)
    # forward runs of the shots
    g.reset()
    traces = S.forward(g, shot_list, [2, 0], w.nt, w.dt)
    for k, i in enumerate([2, 0]):
        _, _, rec = oracle.run(oracle.FP32CANON, w.shape, w.extent, so, w.m, w.dt, w.nt, damp=w.damp,
                               src_coords=shot_list[i].src_coords, wavelet=shot_list[i].wavelet,
                               rec_coords=w.rec_coords)
        assert np.array_equal(traces[k], rec)
    g.close()
