"""GPU parity of the 2D hot path: the TMA-tiled kernel (AW_KERNEL_TILE2D, chosen by AUTO in 2D)
and the reference-grade v1 kernel vs the fp32 oracle, every space order, ragged tiles (shapes not
multiples of 64 x 32, odd widths for the column-pair stores), damping, several sources/receivers."""
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


def _run(aw, w, kernel):
    g = aw.Grid(w.shape, w.extent, w.space_order, w.origin)
    g.set_option(aw.AW_OPT_KERNEL, kernel)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.nt)
    g.run(w.nt, w.dt)
    out = g.read_wavefield(0), g.read_wavefield(1), g.read_receivers(), g.stats()["kernel"]
    g.close()
    return out


@pytest.mark.parametrize("so", [2, 4, 6, 8, 10, 12, 14, 16])
@pytest.mark.parametrize("shape", [(101, 101), (67, 131), (40, 64)])
def test_tile2d_equals_oracle_and_v1(aw, so, shape):
    w = workloads.small_case(shape, so, 30, nbl=6, ns=2, nr=9, seed=so + shape[1])
    ou, oup, orec = oracle.run(oracle.FP32CANON, w.shape, w.extent, so, w.m, w.dt, w.nt, damp=w.damp,
                               src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    for kernel, want_kernel in ((aw.AW_KERNEL_AUTO, aw.AW_KERNEL_TILE2D), (aw.AW_KERNEL_V1, aw.AW_KERNEL_V1)):
        u, up, rec, used = _run(aw, w, kernel)
        assert used == want_kernel
        for got, want, what in ((u, ou, "u^n"), (up, oup, "u^{n-1}"), (rec, orec, "traces")):
            err = np.linalg.norm((got - want).astype(np.float64)) / max(np.linalg.norm(want.astype(np.float64)), 1e-30)
            assert err <= 1e-5, (kernel, what, err)
            assert np.array_equal(got, want), (kernel, what, err)


def test_tile2d_c1(aw):
    w = workloads.c1()
    ou, oup, orec = oracle.run(oracle.FP32CANON, w.shape, w.extent, 2, w.m, w.dt, w.nt, damp=w.damp,
                               src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    u, up, rec, used = _run(aw, w, aw.AW_KERNEL_AUTO)
    assert used == aw.AW_KERNEL_TILE2D
    assert np.array_equal(u, ou) and np.array_equal(up, oup) and np.array_equal(rec, orec)
