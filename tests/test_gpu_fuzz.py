"""Seeded random sweep of the CUDA path vs the fp32 oracle (value-identical): random ragged 2D/3D
shapes (not multiples of any tile, down to k/2+1 points per axis), space orders 2..16, damping
widths, source/receiver counts and positions (including exact nodes and domain faces), step counts,
kernel choice (auto / v1) and temporal blocking (0/1).  Catches geometry corner cases the hand-made
cases miss (tile and z-chunk edges, one-tile grids, thin axes)."""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

N_CASES = 64


@pytest.fixture(scope="module")
def aw():
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    return aw


def _case(i):
    rng = np.random.default_rng(20261017 + i)
    ndim = 3 if i % 3 else 2
    so = int(rng.choice([2, 4, 6, 8, 10, 12, 14, 16]))
    R = so // 2
    if ndim == 3:
        shape = tuple(int(rng.integers(R + 1, hi)) for hi in (70, 50, 140))
    else:
        shape = tuple(int(rng.integers(R + 1, hi)) for hi in (150, 300))
    nt = int(rng.integers(1, 8))
    nbl = int(rng.integers(0, max(1, min(shape) // 3)))
    w = workloads.small_case(shape, so, nt, nbl=nbl or None, ns=int(rng.integers(0, 4)) or 1,
                             nr=int(rng.integers(1, 9)), seed=int(rng.integers(1 << 30)))
    ext = np.array(w.extent)
    # a few sparse points on exact nodes / faces / the far corner
    extra = [ext * rng.integers(0, 2, size=ndim), np.round(rng.uniform(0, 1, ndim) * (np.array(shape) - 1)) * 10.0]
    w.rec_coords = np.concatenate([w.rec_coords, np.array(extra)])
    kernel = int(rng.choice([0, 0, 1]))
    temporal = int(rng.integers(0, 2))
    return w, kernel, temporal


@pytest.mark.parametrize("i", range(N_CASES))
def test_fuzz_equals_oracle(aw, i):
    w, kernel, temporal = _case(i)
    g = aw.Grid(w.shape, w.extent, w.space_order)
    g.set_option(aw.AW_OPT_KERNEL, kernel)
    g.set_option(aw.AW_OPT_TEMPORAL, temporal)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.nt)
    g.run(w.nt, w.dt)
    u, up, rec = g.read_wavefield(0), g.read_wavefield(1), g.read_receivers()
    g.close()
    ou, oup, orec = oracle.run(oracle.FP32CANON, w.shape, w.extent, w.space_order, w.m, w.dt, w.nt, damp=w.damp,
                               src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords)
    for got, want, what in ((u, ou, "u^n"), (up, oup, "u^{n-1}"), (rec, orec, "traces")):
        assert np.array_equal(got, want), (i, w.shape, w.space_order, kernel, temporal, what)
